// Drop-in replacement for pkifmm::evaluate (include/pkifmm/fmm.hpp:141,
// src/fmm.cpp:690-742) and pkifmm::solve_m2l (include/pkifmm/periodize.hpp:42-46,
// src/periodize.cpp:113-158) that run on the B200 through the C ABI in include/pkgpu.h.
//
// Compiled against the reference's own headers; linking this object ahead of the
// reference's fmm.o (whose evaluate symbol is weakened) makes every existing caller —
// tools/pkifmm.cpp cmd_eval, src/experiments.cpp — run the GPU path unchanged.
// Exceptions are rethrown with the reference's classes and messages.
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "pkgpu.h"
#include "pkifmm/fmm.hpp"
#include "pkifmm/periodize.hpp"

namespace {

pkgpu_context *context() {
    static std::once_flag once;
    static pkgpu_context *ctx = nullptr;
    std::call_once(once, [] {
        char err[512];
        int dev = 0;
        if (const char *e = std::getenv("PKGPU_DEVICE")) dev = std::atoi(e);
        if (pkgpu_context_create(dev, &ctx, err, sizeof err) != PKGPU_OK)
            throw std::runtime_error(std::string("pkgpu: ") + err);
    });
    return ctx;
}

pkgpu_setup to_setup(const pkifmm::PeriodicSetup &s) {
    pkgpu_setup o{};
    o.periodicity = static_cast<int>(s.periodicity);
    for (int a = 0; a < 3; a++) o.axes[a] = s.axes[a] ? 1 : 0;
    o.box_length = s.box_length;
    o.ell = s.ell;
    return o;
}

[[noreturn]] void rethrow(pkgpu_status st, const char *msg) {
    switch (st) {
    case PKGPU_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PKGPU_CONFIG_ERROR: throw pkifmm::ConfigError(msg);
    default: throw std::runtime_error(msg);
    }
}

} // namespace

namespace pkifmm {

EvalResult evaluate(const EvalRequest &request) {
    static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be 3 packed doubles");
    const KernelSpec &kernel = request.kernel;
    char err[2048] = {0};
    pkgpu_operator *op = nullptr;
    if (request.op) {
        const PeriodizingOperator &p = *request.op;
        const pkgpu_setup s = to_setup(p.setup);
        const pkgpu_status st = pkgpu_operator_create(static_cast<int>(p.kernel.type), &s, p.p, p.matrix.data.data(),
                                                      p.matrix.rows, &op, err, sizeof err);
        if (st != PKGPU_OK) rethrow(st, err);
    }
    struct OpGuard {
        pkgpu_operator *p;
        ~OpGuard() { pkgpu_operator_free(p); }
    } guard{op};

    pkgpu_request r{};
    r.kernel = static_cast<int>(kernel.type);
    r.n_sources = static_cast<int64_t>(request.sources.size());
    r.sources = request.sources.empty() ? nullptr : request.sources.data()->data();
    r.n_strengths = static_cast<int64_t>(request.strengths.size());
    r.strengths = request.strengths.data();
    r.n_targets = static_cast<int64_t>(request.targets.size());
    r.targets = request.targets.empty() ? nullptr : request.targets.data()->data();
    r.setup = to_setup(request.setup);
    r.p = request.p;
    r.op = op;
    r.mode = request.mode == EvalMode::direct ? PKGPU_MODE_DIRECT : PKGPU_MODE_FMM;
    r.leaf_capacity = request.leaf_capacity;
    r.force = request.force ? 1 : 0;
    r.device_pointers = 0;

    EvalResult result;
    result.potentials.assign(static_cast<size_t>(kernel.kt) * request.targets.size(), 0.0);
    pkgpu_timings tm{};
    pkgpu_compat cp{};
    const pkgpu_status st = pkgpu_evaluate(context(), &r, result.potentials.data(), &tm, &cp, err, sizeof err);
    if (st != PKGPU_OK) rethrow(st, err);
    result.timings.tree = tm.tree;
    result.timings.near = tm.near;
    result.timings.m2l_apply = tm.m2l_apply;
    result.timings.far = tm.far;
    result.compat.ok = cp.ok != 0;
    result.compat.residual = cp.residual;
    result.compat.violated = cp.violated;
    return result;
}

// solve_m2l on the GPU (pkgpu_operator_solve): K^{P,F} by per-pair Ewald / image sums,
// T = pinv(a_dn) K^{P,F} with the device's own downward factors (cuSOLVER; equivalent to
// the caller's up to rounding), the same 1e-11 residual gate and messages.
namespace {
PeriodizingOperator solve_on_gpu(const PeriodicKernelSpec &spec, int p) {
    validate_method(spec);
    const pkgpu_setup s = to_setup(spec.setup);
    const pkgpu_ewald e{spec.params.xi, spec.params.real_shells, spec.params.wave_cutoff, spec.params.n_images};
    pkgpu_operator *op = nullptr;
    char err[2048] = {0};
    const pkgpu_status st =
        pkgpu_operator_solve(context(), static_cast<int>(spec.kernel.type), &s, p, &e, 1, &op, err, sizeof err);
    if (st != PKGPU_OK) rethrow(st, err);
    int64_t dim = 0;
    double residual = 0.0;
    pkgpu_operator_info(op, nullptr, nullptr, nullptr, &dim, &residual);
    PeriodizingOperator out;
    out.matrix = DenseMatrix(static_cast<int>(dim), static_cast<int>(dim));
    pkgpu_operator_matrix(op, out.matrix.data.data());
    pkgpu_operator_free(op);
    out.kernel = spec.kernel;
    out.setup = spec.setup;
    out.p = p;
    out.method = spec.method;
    out.params = spec.params;
    out.residual_max = residual;
    return out;
}
} // namespace

PeriodizingOperator solve_m2l(const PeriodicKernelSpec &spec, int p, const SvdFactors &) {
    return solve_on_gpu(spec, p);
}

PeriodizingOperator solve_m2l(const PeriodicKernelSpec &spec, int p) { return solve_on_gpu(spec, p); }

} // namespace pkifmm
