// extern "C" boundary of libpkgpu (include/pkgpu.h). Translates C++ exceptions into
// status codes + messages, owns the PKM2L operator reader, and hosts the synthetic
// workload generator.
#include <array>
#include <memory>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <random>
#include <sstream>

#include "context.h"
#include "gemm.h"
#include "periodize.h"
#include "tuning.h"

using namespace pkgpu;

namespace {

void set_err(char *err, size_t errlen, const std::string &msg) {
    if (err && errlen) {
        std::strncpy(err, msg.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
}

template <class F> pkgpu_status guarded(char *err, size_t errlen, F &&f) {
    try {
        f();
        return PKGPU_OK;
    } catch (const InvalidArgument &e) {
        set_err(err, errlen, e.what());
        return PKGPU_INVALID_ARGUMENT;
    } catch (const ConfigError &e) {
        set_err(err, errlen, e.what());
        return PKGPU_CONFIG_ERROR;
    } catch (const CudaError &e) {
        set_err(err, errlen, e.what());
        return PKGPU_CUDA_ERROR;
    } catch (const std::invalid_argument &e) {
        set_err(err, errlen, e.what());
        return PKGPU_INVALID_ARGUMENT;
    } catch (const std::exception &e) {
        set_err(err, errlen, e.what());
        return PKGPU_RUNTIME_ERROR;
    }
}

// ---------------------------------------------------------------------------
// minimal JSON reader for the PKM2L header (flat object + one nested "params")
struct JVal {
    enum Kind { Null, Num, Str, Obj, Bool } kind = Null;
    std::string text; // numbers kept verbatim (payload_crc64 is a full uint64)
    std::map<std::string, JVal> obj;
    bool b = false;
};

struct JParser {
    const std::string &s;
    size_t i = 0;
    explicit JParser(const std::string &str) : s(str) {}
    [[noreturn]] void fail() { throw RuntimeError("load_operator: malformed JSON header"); }
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) i++;
    }
    std::string str() {
        if (s[i] != '"') fail();
        i++;
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                i++;
                if (i >= s.size()) fail();
                const char c = s[i];
                out += c == 'n' ? '\n' : c == 't' ? '\t' : c;
            } else {
                out += s[i];
            }
            i++;
        }
        if (i >= s.size()) fail();
        i++;
        return out;
    }
    JVal value() {
        ws();
        if (i >= s.size()) fail();
        JVal v;
        if (s[i] == '{') {
            v.kind = JVal::Obj;
            i++;
            ws();
            if (s[i] == '}') {
                i++;
                return v;
            }
            for (;;) {
                ws();
                const std::string k = str();
                ws();
                if (s[i] != ':') fail();
                i++;
                v.obj[k] = value();
                ws();
                if (s[i] == ',') {
                    i++;
                    continue;
                }
                if (s[i] == '}') {
                    i++;
                    break;
                }
                fail();
            }
        } else if (s[i] == '"') {
            v.kind = JVal::Str;
            v.text = str();
        } else if (s.compare(i, 4, "true") == 0) {
            v.kind = JVal::Bool, v.b = true, i += 4;
        } else if (s.compare(i, 5, "false") == 0) {
            v.kind = JVal::Bool, i += 5;
        } else if (s.compare(i, 4, "null") == 0) {
            i += 4;
        } else {
            v.kind = JVal::Num;
            const size_t b = i;
            while (i < s.size() && (std::isdigit((unsigned char)s[i]) || s[i] == '-' || s[i] == '+' || s[i] == '.' ||
                                    s[i] == 'e' || s[i] == 'E'))
                i++;
            if (i == b) fail();
            v.text = s.substr(b, i - b);
        }
        return v;
    }
};

const JVal &at(const JVal &o, const std::string &k) {
    auto it = o.obj.find(k);
    if (it == o.obj.end()) throw RuntimeError("load_operator: header key '" + k + "' missing");
    return it->second;
}

uint64_t crc64_xz(const void *data, size_t len) {
    // CRC-64/XZ: ECMA-182 polynomial, reflected (src/periodize.cpp:40-55)
    struct Table {
        uint64_t t[256];
        Table() {
            for (uint64_t i = 0; i < 256; i++) {
                uint64_t c = i;
                for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ 0xC96C5795D7870F42ull : c >> 1;
                t[i] = c;
            }
        }
    };
    static const Table tab; // thread-safe one-time initialisation
    const uint64_t *table = tab.t;
    uint64_t crc = ~0ull;
    const auto *p = static_cast<const unsigned char *>(data);
    for (size_t i = 0; i < len; i++) crc = table[(crc ^ p[i]) & 0xff] ^ (crc >> 8);
    return ~crc;
}

int periodicity_from(const std::string &n) {
    if (n == "none") return PKGPU_NONE;
    if (n == "sp") return PKGPU_SP;
    if (n == "dp") return PKGPU_DP;
    if (n == "tp") return PKGPU_TP;
    throw InvalidArgument("unknown periodicity: " + n);
}

int kernel_from(const std::string &n) {
    if (n == "laplace") return PKGPU_LAPLACE;
    if (n == "stokeslet" || n == "stokes") return PKGPU_STOKESLET;
    throw InvalidArgument("unknown kernel name: " + n);
}

int method_from(const std::string &n) {
    if (n == "direct_sp") return PKGPU_DIRECT_SP;
    if (n == "ewald_laplace_dp") return PKGPU_EWALD_LAPLACE_DP;
    if (n == "ewald_laplace_tp") return PKGPU_EWALD_LAPLACE_TP;
    if (n == "ewald_stokes_tp_hasimoto") return PKGPU_EWALD_STOKES_TP;
    throw InvalidArgument("unknown periodic method: " + n);
}

// load_operator, src/periodize.cpp:231-278 (same checks, same messages)
pkgpu_operator *load_pkm2l(const std::string &path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw RuntimeError("load_operator: cannot open " + path);
    char magic[6];
    f.read(magic, 6);
    static const char kMagic[6] = {'P', 'K', 'M', '2', 'L', '\x01'};
    if (!f || std::memcmp(magic, kMagic, 6) != 0) throw RuntimeError("load_operator: bad magic in " + path);
    unsigned char lenbuf[8];
    f.read(reinterpret_cast<char *>(lenbuf), 8);
    uint64_t hlen = 0;
    for (int i = 0; i < 8; i++) hlen |= static_cast<uint64_t>(lenbuf[i]) << (8 * i);
    if (!f || hlen > (1ull << 20)) throw RuntimeError("load_operator: bad header length in " + path);
    std::string hs(hlen, '\0');
    f.read(hs.data(), static_cast<std::streamsize>(hlen));
    if (!f) throw RuntimeError("load_operator: truncated header in " + path);
    JParser jp(hs);
    const JVal h = jp.value();
    auto op = std::make_unique<pkgpu_operator>();
    op->kernel = kernel_from(at(h, "kernel").text);
    op->setup.periodicity = periodicity_from(at(h, "periodicity").text);
    const std::string axes = at(h, "periodic_axes").text;
    op->setup.axes[0] = axes.find('x') != std::string::npos;
    op->setup.axes[1] = axes.find('y') != std::string::npos;
    op->setup.axes[2] = axes.find('z') != std::string::npos;
    op->setup.box_length = 1.0; // not serialised by the reference (PeriodicSetup default)
    op->setup.ell = std::stoi(at(h, "ell").text);
    op->p = std::stoi(at(h, "p").text);
    op->method = method_from(at(h, "method").text);
    op->residual_max = std::stod(at(h, "residual_max").text);
    if (h.obj.count("params")) {
        const JVal &pa = at(h, "params");
        if (pa.obj.count("xi")) op->xi = std::stod(at(pa, "xi").text);
        if (pa.obj.count("real_shells")) op->real_shells = std::stoi(at(pa, "real_shells").text);
        if (pa.obj.count("wave_cutoff")) op->wave_cutoff = std::stoi(at(pa, "wave_cutoff").text);
        if (pa.obj.count("n_images")) op->n_images = std::stoll(at(pa, "n_images").text);
    }
    if (h.obj.count("created")) op->created = at(h, "created").text;
    const int rows = std::stoi(at(h, "rows").text), cols = std::stoi(at(h, "cols").text);
    const int ks = op->kernel == PKGPU_LAPLACE ? 1 : 3;
    const int n = surface_point_count(op->p);
    if (rows != ks * n || cols != ks * n || std::stoi(at(h, "n").text) != n)
        throw RuntimeError("load_operator: inconsistent dimensions in " + path);
    op->dim = rows;
    op->matrix.resize(static_cast<size_t>(rows) * cols);
    f.read(reinterpret_cast<char *>(op->matrix.data()),
           static_cast<std::streamsize>(op->matrix.size() * sizeof(double)));
    if (!f) throw RuntimeError("load_operator: truncated payload in " + path);
    op->crc = crc64_xz(op->matrix.data(), op->matrix.size() * sizeof(double));
    if (op->crc != std::stoull(at(h, "payload_crc64").text))
        throw RuntimeError("load_operator: payload CRC mismatch in " + path);
    return op.release();
}

} // namespace

pkgpu_operator::~pkgpu_operator() {
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : d_matrix) {
        cudaSetDevice(kv.first);
        cudaFree(kv.second);
    }
    cudaSetDevice(cur);
}

// one device copy per device, uploaded on first use and kept until the operator is
// destroyed (contexts on other devices never free a copy another one may be using)
const double *pkgpu_operator::device_matrix(int device, cudaStream_t st) const {
    std::lock_guard<std::mutex> lock(mtx);
    auto it = d_matrix.find(device);
    if (it != d_matrix.end()) return it->second;
    double *d = nullptr;
    PK_CUDA(cudaMalloc(&d, matrix.size() * sizeof(double)));
    PK_CUDA(cudaMemcpyAsync(d, matrix.data(), matrix.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaStreamSynchronize(st));
    d_matrix.emplace(device, d);
    return d;
}

extern "C" {

pkgpu_status pkgpu_context_create(int device, pkgpu_context **ctx, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        int ndev = 0;
        PK_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw InvalidArgument("pkgpu_context_create: no CUDA device " + std::to_string(device));
        PK_CUDA(cudaSetDevice(device));
        auto c = std::make_unique<pkgpu_context>();
        c->device = device;
        PK_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        // the work stream and the list stream run at the highest priority, the stream of the
        // overlapped lattice M2L at the lowest: its big grids fill the SMs the latency-bound
        // chain leaves idle and yield to the chain's CTAs as soon as those are launched
        int prio_least = 0, prio_greatest = 0;
        PK_CUDA(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
        PK_CUDA(cudaStreamCreateWithPriority(&c->own_stream, cudaStreamNonBlocking, prio_greatest));
        c->stream = c->own_stream;
        for (auto &e : c->ev) PK_CUDA(cudaEventCreate(&e));
        PK_CUDA(cudaStreamCreateWithPriority(&c->aux_stream, cudaStreamNonBlocking, prio_greatest));
        PK_CUDA(cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming));
        PK_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        PK_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        PK_CUDA(cudaStreamCreateWithPriority(&c->aux2_stream, cudaStreamNonBlocking, prio_least));
        PK_CUDA(cudaStreamCreateWithPriority(&c->aux3_stream, cudaStreamNonBlocking, (prio_least + prio_greatest) / 2));
        for (auto &e : c->ev_lat_fork) PK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto &e : c->ev_lat_join) PK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        *ctx = c.release();
    });
}

void pkgpu_context_destroy(pkgpu_context *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto &e : ctx->ev) cudaEventDestroy(e);
    cudaStreamDestroy(ctx->own_stream);
    if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->ev_user) cudaEventDestroy(ctx->ev_user);
    if (ctx->h_layout) cudaFreeHost(ctx->h_layout);
    if (ctx->aux2_stream) cudaStreamDestroy(ctx->aux2_stream);
    if (ctx->aux3_stream) cudaStreamDestroy(ctx->aux3_stream);
    for (auto e : ctx->ev_lat_fork)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_lat_join)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->evpool) cudaEventDestroy(e);
    delete ctx;
}

pkgpu_status pkgpu_context_set_stream(pkgpu_context *ctx, void *stream) {
    std::lock_guard<std::mutex> lock(ctx->mtx);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return PKGPU_OK;
}

void *pkgpu_context_stream(pkgpu_context *ctx) { return ctx->stream; }

int64_t pkgpu_context_launch_count(pkgpu_context *ctx) { return ctx->launches; }

pkgpu_status pkgpu_context_set_profiling(pkgpu_context *ctx, int on) {
    std::lock_guard<std::mutex> lock(ctx->mtx);
    ctx->profiling = on != 0;
    return PKGPU_OK;
}

pkgpu_status pkgpu_context_set_m2l(pkgpu_context *ctx, int path, int64_t min_boxes, int nmod, int beta_a,
                                   int beta_b) {
    if (path < 0 || path > 4 || (nmod > 0 && (nmod < 14 || nmod > kI8MaxModuli))) return PKGPU_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lock(ctx->mtx);
    I8Settings &s = ctx->i8;
    s.enabled = path == 0 || path == 2 || path == 4;
    s.trans = path == 2;
    s.fft = path == 3;
    s.lattice = (path == 0 || path == 2 || path == 3) && tuning().m2l_lattice;
    if (min_boxes > 0) s.min_boxes = min_boxes;
    if (nmod > 0) s.nmod = nmod;
    if (beta_a > 0) s.beta_a = beta_a;
    if (beta_b > 0) s.beta_b = beta_b;
    double logm = 0;
    for (int t = 0; t < s.nmod; t++) logm += std::log2((double)i8_moduli()[t]);
    if (s.beta_a + s.beta_b + 20 >= logm) {
        s = i8_settings();
        return PKGPU_INVALID_ARGUMENT;
    }
    return PKGPU_OK;
}

pkgpu_status pkgpu_context_reset_stats(pkgpu_context *ctx) {
    std::lock_guard<std::mutex> lock(ctx->mtx);
    ctx->stats.clear();
    return PKGPU_OK;
}

pkgpu_status pkgpu_context_stage_stats(pkgpu_context *ctx, const char *stage, double *seconds, double *units,
                                       double *flops, int64_t *launches) {
    std::lock_guard<std::mutex> lock(ctx->mtx);
    auto it = ctx->stats.find(stage ? stage : "");
    const pkgpu_context::StageStat s = it == ctx->stats.end() ? pkgpu_context::StageStat{} : it->second;
    if (seconds) *seconds = s.seconds;
    if (units) *units = s.units;
    if (flops) *flops = s.flops;
    if (launches) *launches = s.launches;
    return it == ctx->stats.end() ? PKGPU_INVALID_ARGUMENT : PKGPU_OK;
}

pkgpu_status pkgpu_evaluate(pkgpu_context *ctx, const pkgpu_request *req, double *out, pkgpu_timings *timings,
                            pkgpu_compat *compat, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        evaluate(*ctx, *req, out, timings, compat);
    });
}

pkgpu_status pkgpu_evaluate_partitioned(pkgpu_context *ctx, const pkgpu_request *req, const pkgpu_partition *part,
                                        double *out, pkgpu_timings *timings, pkgpu_compat *compat, char *err,
                                        size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        evaluate(*ctx, *req, out, timings, compat, part);
    });
}

pkgpu_status pkgpu_operator_load(const char *path, pkgpu_operator **op, char *err, size_t errlen) {
    return guarded(err, errlen, [&] { *op = load_pkm2l(path); });
}

pkgpu_status pkgpu_operator_create(int kernel, const pkgpu_setup *setup, int p, const double *matrix, int64_t dim,
                                   pkgpu_operator **op, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const int ks = kernel == PKGPU_LAPLACE ? 1 : 3;
        if (p < 2) throw InvalidArgument("surface grid requires p >= 2");
        if (dim != (int64_t)ks * surface_point_count(p))
            throw InvalidArgument("apply_m2l: density length does not match operator dimension");
        auto o = std::make_unique<pkgpu_operator>();
        o->kernel = kernel;
        o->setup = *setup;
        o->p = p;
        o->dim = dim;
        o->matrix.assign(matrix, matrix + dim * dim);
        o->crc = crc64_xz(o->matrix.data(), o->matrix.size() * sizeof(double));
        *op = o.release();
    });
}

void pkgpu_operator_free(pkgpu_operator *op) { delete op; }

pkgpu_status pkgpu_operator_info(const pkgpu_operator *op, int *kernel, pkgpu_setup *setup, int *p, int64_t *dim,
                                 double *residual_max) {
    if (!op) return PKGPU_INVALID_ARGUMENT;
    if (kernel) *kernel = op->kernel;
    if (setup) *setup = op->setup;
    if (p) *p = op->p;
    if (dim) *dim = op->dim;
    if (residual_max) *residual_max = op->residual_max;
    return PKGPU_OK;
}

pkgpu_status pkgpu_operator_relabel(pkgpu_operator *op, int kernel, const pkgpu_setup *setup) {
    if (!op || !setup) return PKGPU_INVALID_ARGUMENT;
    const int ks = kernel == PKGPU_LAPLACE ? 1 : 3;
    if (op->dim != (int64_t)ks * surface_point_count(op->p)) return PKGPU_INVALID_ARGUMENT;
    op->kernel = kernel;
    op->setup = *setup;
    return PKGPU_OK;
}

pkgpu_status pkgpu_operator_matrix(const pkgpu_operator *op, double *out) {
    if (!op) return PKGPU_INVALID_ARGUMENT;
    std::memcpy(out, op->matrix.data(), op->matrix.size() * sizeof(double));
    return PKGPU_OK;
}

uint64_t pkgpu_crc64(const void *data, size_t len) { return crc64_xz(data, len); }

namespace {

EwaldSettings ewald_from(const pkgpu_ewald *e) {
    EwaldSettings s;
    if (e) {
        s.xi = e->xi;
        s.real_shells = e->real_shells;
        s.wave_cutoff = e->wave_cutoff;
        s.n_images = e->n_images;
    }
    if (!(s.xi > 0.0) || s.real_shells < 0 || s.wave_cutoff < 1 || s.n_images < 1)
        throw InvalidArgument("EwaldParams: xi > 0, real_shells >= 0, wave_cutoff >= 1, n_images >= 1 required");
    return s;
}

// shortest round-trip decimal, with a ".0" on integral values (nlohmann's number format)
std::string json_double(double v) {
    char buf[40];
    for (int prec = 1; prec <= 17; prec++) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string json_str(const std::string &v) { return "\"" + v + "\""; }

const char *kernel_label(int k) { return k == PKGPU_LAPLACE ? "laplace" : "stokeslet"; }
const char *periodicity_label(int p) {
    switch (p) {
    case PKGPU_SP: return "sp";
    case PKGPU_DP: return "dp";
    case PKGPU_TP: return "tp";
    }
    return "none";
}

} // namespace

pkgpu_status pkgpu_operator_solve(pkgpu_context *ctx, int kernel, const pkgpu_setup *setup, int p,
                                  const pkgpu_ewald *params, int gated, pkgpu_operator **op, char *err,
                                  size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        if (kernel != PKGPU_LAPLACE && kernel != PKGPU_STOKESLET) throw InvalidArgument("unknown kernel");
        if (p < 2) throw InvalidArgument("surface grid requires p >= 2");
        const EwaldSettings e = ewald_from(params);
        pkgpu_setup s = *setup;
        // singly periodic along x: build along z (the reference's SP sum) and permute the
        // surface indices by the axis rotation (x, y, z) -> (y, z, x) (cfg 1)
        const bool spx = s.periodicity == PKGPU_SP && s.axes[0] && !s.axes[1] && !s.axes[2];
        if (s.periodicity == PKGPU_SP && !spx && !(s.axes[2] && !s.axes[0] && !s.axes[1]))
            throw InvalidArgument("solve_m2l: singly periodic operators are built along z or x");
        if (spx) {
            if (kernel != PKGPU_LAPLACE) throw InvalidArgument("spx permutation implemented for scalar kernels only");
            s.axes[0] = 0, s.axes[2] = 1;
        }
        PeriodicSolve r = solve_periodizing_operator(*ctx, kernel, s, p, e, gated != 0);
        auto o = std::make_unique<pkgpu_operator>();
        o->kernel = kernel;
        o->setup = *setup;
        o->p = p;
        o->dim = r.dim;
        if (spx) {
            const auto g = surface_grid(p);
            const int n = (int)g.size() / 3;
            std::map<std::array<int, 3>, int> at;
            for (int i = 0; i < n; i++) at[{g[3 * i], g[3 * i + 1], g[3 * i + 2]}] = i;
            std::vector<int> pi(n);
            for (int i = 0; i < n; i++) pi[i] = at.at({g[3 * i + 1], g[3 * i + 2], g[3 * i]});
            o->matrix.resize(r.matrix.size());
            for (int i = 0; i < n; i++)
                for (int j = 0; j < n; j++) o->matrix[(size_t)i * n + j] = r.matrix[(size_t)pi[i] * n + pi[j]];
        } else {
            o->matrix = std::move(r.matrix);
        }
        o->method = r.method;
        o->residual_max = r.residual_max;
        o->xi = e.xi;
        o->real_shells = e.real_shells;
        o->wave_cutoff = e.wave_cutoff;
        o->n_images = e.n_images;
        o->created = iso_now();
        o->crc = crc64_xz(o->matrix.data(), o->matrix.size() * sizeof(double));
        *op = o.release();
    });
}

pkgpu_status pkgpu_operator_save(const pkgpu_operator *op, const char *path, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!op) throw InvalidArgument("save_operator: null operator");
        const int ks = op->kernel == PKGPU_LAPLACE ? 1 : 3;
        std::string axes;
        for (int a = 0; a < 3; a++)
            if (op->setup.axes[a]) axes += "xyz"[a];
        const uint64_t crc = crc64_xz(op->matrix.data(), op->matrix.size() * sizeof(double));
        // keys in the order the reference's (sorted) JSON object writes them
        std::ostringstream h;
        h << "{\"cols\":" << op->dim << ",\"created\":" << json_str(op->created) << ",\"ell\":" << op->setup.ell
          << ",\"format\":\"pkm2l\",\"inner_scale\":" << json_double(1.05) << ",\"kernel\":"
          << json_str(kernel_label(op->kernel)) << ",\"ks\":" << ks << ",\"kt\":" << ks
          << ",\"method\":" << json_str(method_label(op->method)) << ",\"n\":" << surface_point_count(op->p)
          << ",\"outer_scale\":" << json_double(2.95) << ",\"p\":" << op->p << ",\"params\":{\"n_images\":"
          << op->n_images << ",\"real_shells\":" << op->real_shells << ",\"wave_cutoff\":" << op->wave_cutoff
          << ",\"xi\":" << json_double(op->xi) << "},\"payload_crc64\":" << crc
          << ",\"periodic_axes\":" << json_str(axes) << ",\"periodicity\":"
          << json_str(periodicity_label(op->setup.periodicity)) << ",\"residual_max\":"
          << json_double(op->residual_max) << ",\"rows\":" << op->dim << ",\"version\":1}";
        const std::string hs = h.str();
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) throw RuntimeError(std::string("save_operator: cannot open ") + path);
        static const char kMagic[6] = {'P', 'K', 'M', '2', 'L', '\x01'};
        f.write(kMagic, 6);
        char lenbuf[8];
        for (int i = 0; i < 8; i++) lenbuf[i] = static_cast<char>((hs.size() >> (8 * i)) & 0xff);
        f.write(lenbuf, 8);
        f.write(hs.data(), static_cast<std::streamsize>(hs.size()));
        f.write(reinterpret_cast<const char *>(op->matrix.data()),
                static_cast<std::streamsize>(op->matrix.size() * sizeof(double)));
        if (!f) throw RuntimeError(std::string("save_operator: write failed for ") + path);
    });
}

pkgpu_status pkgpu_periodic_block(pkgpu_context *ctx, int kernel, const pkgpu_setup *setup, const pkgpu_ewald *params,
                                  int far_only, const double *targets, int64_t nt, const double *sources, int64_t ns,
                                  double *out, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        const EwaldSettings e = ewald_from(params);
        const int k = kernel == PKGPU_LAPLACE ? 1 : 3;
        cudaStream_t st = ctx->stream;
        double *t = ctx->ws.get<double>("pb_t", 3 * nt + 1), *s = ctx->ws.get<double>("pb_s", 3 * ns + 1);
        double *o = ctx->ws.get<double>("pb_o", (size_t)k * nt * k * ns + 1);
        PK_CUDA(cudaMemcpyAsync(t, targets, 3 * nt * sizeof(double), cudaMemcpyHostToDevice, st));
        PK_CUDA(cudaMemcpyAsync(s, sources, 3 * ns * sizeof(double), cudaMemcpyHostToDevice, st));
        periodic_block_device(kernel, *setup, e, far_only != 0, t, (int)nt, s, (int)ns, o, k * ns, st);
        PK_CUDA(cudaMemcpyAsync(out, o, (size_t)k * nt * k * ns * sizeof(double), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        ctx->launches += 1;
    });
}

pkgpu_status pkgpu_oracle_system_eval(pkgpu_context *ctx, int kernel, const pkgpu_setup *setup,
                                      const pkgpu_ewald *params, const double *sources, int64_t ns,
                                      const double *strengths, const double *targets, int64_t nt, double *out,
                                      char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        const EwaldSettings e = ewald_from(params);
        periodic_method(kernel, *setup); // ConfigError for unsupported combinations first
        const int k = kernel == PKGPU_LAPLACE ? 1 : 3;
        // check_compatibility (src/refsum.cpp:733-756)
        if (!(kernel == PKGPU_STOKESLET && setup->periodicity == PKGPU_TP)) {
            double abs_total = 0.0, worst = 0.0;
            for (int64_t i = 0; i < k * ns; i++) abs_total += std::fabs(strengths[i]);
            for (int a = 0; a < k; a++) {
                double sum = 0.0;
                for (int64_t i = 0; i < ns; i++) sum += strengths[i * k + a];
                worst = std::max(worst, std::fabs(sum));
            }
            if (worst > 1e-12 * abs_total) {
                char msg[256];
                std::snprintf(msg, sizeof msg, "oracle_system_eval: compatibility violation (%s, residual=%f)",
                              kernel == PKGPU_LAPLACE ? "neutrality: net charge must vanish"
                                                      : "neutrality: net force must vanish",
                              worst);
                throw ConfigError(msg);
            }
        }
        cudaStream_t st = ctx->stream;
        double *s = ctx->ws.get<double>("os_s", 3 * ns + 1), *q = ctx->ws.get<double>("os_q", k * ns + 1);
        PK_CUDA(cudaMemcpyAsync(s, sources, 3 * ns * sizeof(double), cudaMemcpyHostToDevice, st));
        PK_CUDA(cudaMemcpyAsync(q, strengths, k * ns * sizeof(double), cudaMemcpyHostToDevice, st));
        // targets in chunks: K^P block (chunk x ns) then a gemv
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)(1 << 27) / (k * k * ns + 1)));
        double *t = ctx->ws.get<double>("os_t", 3 * chunk + 1), *B = ctx->ws.get<double>("os_B", k * chunk * k * ns + 1);
        double *y = ctx->ws.get<double>("os_y", k * chunk + 1);
        for (int64_t t0 = 0; t0 < nt; t0 += chunk) {
            const int64_t m = std::min(chunk, nt - t0);
            PK_CUDA(cudaMemcpyAsync(t, targets + 3 * t0, 3 * m * sizeof(double), cudaMemcpyHostToDevice, st));
            periodic_block_device(kernel, *setup, e, false, t, (int)m, s, (int)ns, B, k * ns, st);
            gemv(B, (int)(k * m), (int)(k * ns), (int)(k * ns), q, y, 1.0, 0.0, nullptr, 0.0, st);
            PK_CUDA(cudaMemcpyAsync(out + k * t0, y, k * m * sizeof(double), cudaMemcpyDeviceToHost, st));
            ctx->launches += 2;
        }
        PK_CUDA(cudaStreamSynchronize(st));
    });
}

pkgpu_status pkgpu_set_kifmm_factors(pkgpu_context *ctx, int kernel, int p, const double *u_up, const double *s_up,
                                     const double *vt_up, const double *u_dn, const double *s_dn,
                                     const double *vt_dn, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        const size_t K = (size_t)(kernel == PKGPU_LAPLACE ? 1 : 3) * surface_point_count(p);
        HostFactors up, dn;
        up.u.assign(u_up, u_up + K * K);
        up.sigma.assign(s_up, s_up + K);
        up.vt.assign(vt_up, vt_up + K * K);
        dn.u.assign(u_dn, u_dn + K * K);
        dn.sigma.assign(s_dn, s_dn + K);
        dn.vt.assign(vt_dn, vt_dn + K * K);
        ctx->ops.inject(kernel, p, up, dn, ctx->stream, &ctx->launches);
    });
}

pkgpu_status pkgpu_get_kifmm_factors(pkgpu_context *ctx, int kernel, int p, double *u_up, double *s_up,
                                     double *vt_up, double *u_dn, double *s_dn, double *vt_dn, char *err,
                                     size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        KifmmOps &ops = ctx->ops.get(kernel, p, ctx->stream, &ctx->launches);
        auto cp = [](const std::vector<double> &v, double *o) {
            if (o) std::memcpy(o, v.data(), v.size() * sizeof(double));
        };
        cp(ops.up.u, u_up);
        cp(ops.up.sigma, s_up);
        cp(ops.up.vt, vt_up);
        cp(ops.dn.u, u_dn);
        cp(ops.dn.sigma, s_dn);
        cp(ops.dn.vt, vt_dn);
    });
}

pkgpu_status pkgpu_kifmm_matrix(pkgpu_context *ctx, int kernel, int p, int which, int i0, int i1, int i2,
                                double *out, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        const auto m = ctx->ops.matrix(kernel, p, which, i0, i1, i2, ctx->stream, &ctx->launches);
        std::memcpy(out, m.data(), m.size() * sizeof(double));
    });
}

pkgpu_status pkgpu_kernel_block_apply(pkgpu_context *ctx, int kernel, const double *targets, int64_t nt,
                                      const double *sources, int64_t ns, const double *shift,
                                      const double *density, double *out, int skip_coincident, char *err,
                                      size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        kernel_block_apply_device(*ctx, kernel, targets, nt, sources, ns, shift, density, out, skip_coincident);
    });
}

pkgpu_status pkgpu_i8_gather_gemm(pkgpu_context *ctx, const int8_t *A, int nmat, const int8_t *B, int rows_per_mod,
                                  int zero_row, int Ki, int nmod, const int32_t *src, int64_t ld_src, int64_t box0,
                                  int nslots, int ncols, int32_t *R, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        ctx->launches += i8_gather_gemm(A, nmat, B, rows_per_mod, zero_row, Ki, nmod, src, ld_src, box0, nslots,
                                        ncols, R, ctx->ws, ctx->stream);
        PK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int pkgpu_i8_moduli(int32_t *out, int n) {
    const int *m = i8_moduli();
    for (int i = 0; i < n && i < kI8MaxModuli; i++) out[i] = m[i];
    return kI8MaxModuli;
}

pkgpu_status pkgpu_surface_points(int p, const double *center, double edge, double *out) {
    if (p < 2) return PKGPU_INVALID_ARGUMENT;
    const auto pts = surface_points(p, center, edge);
    std::memcpy(out, pts.data(), pts.size() * sizeof(double));
    return PKGPU_OK;
}

pkgpu_status pkgpu_tree_build(pkgpu_context *ctx, const double *sources, int64_t ns, const double *targets,
                              int64_t nt, int leaf_capacity, pkgpu_tree **tree, char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        auto t = std::make_unique<pkgpu_tree>();
        t->ctx = ctx;
        cudaStream_t st = ctx->stream;
        double *s = t->tree.ws.get<double>("host_src", 3 * ns + 1), *g = t->tree.ws.get<double>("host_trg", 3 * nt + 1);
        if (ns) PK_CUDA(cudaMemcpyAsync(s, sources, 3 * ns * sizeof(double), cudaMemcpyHostToDevice, st));
        if (nt) PK_CUDA(cudaMemcpyAsync(g, targets, 3 * nt * sizeof(double), cudaMemcpyHostToDevice, st));
        build_tree(t->tree, s, ns, g, nt, leaf_capacity, st, &ctx->launches);
        *tree = t.release();
    });
}

void pkgpu_tree_free(pkgpu_tree *tree) { delete tree; }

static void ensure_export(pkgpu_tree *t) {
    if (t->exported) return;
    export_tree(t->tree, t->table, t->srcidx, t->trgidx, t->hash);
    t->exported = true;
}

pkgpu_status pkgpu_tree_info(pkgpu_tree *tree, int64_t *nboxes, int64_t *nleaves, int *depth, uint64_t *hash) {
    char e[8];
    return guarded(e, sizeof e, [&] {
        if (hash) ensure_export(tree);
        if (nboxes) *nboxes = tree->tree.nboxes;
        if (nleaves) *nleaves = tree->tree.nleaves;
        if (depth) *depth = tree->tree.depth;
        if (hash) *hash = tree->hash;
    });
}

pkgpu_status pkgpu_tree_boxes(pkgpu_tree *tree, int32_t *table, int32_t *srcidx, int32_t *trgidx) {
    char e[8];
    return guarded(e, sizeof e, [&] {
        ensure_export(tree);
        if (table) std::memcpy(table, tree->table.data(), tree->table.size() * sizeof(int32_t));
        if (srcidx) std::memcpy(srcidx, tree->srcidx.data(), tree->srcidx.size() * sizeof(int32_t));
        if (trgidx) std::memcpy(trgidx, tree->trgidx.data(), tree->trgidx.size() * sizeof(int32_t));
    });
}

pkgpu_status pkgpu_tree_lists(pkgpu_tree *tree, const pkgpu_setup *setup, int which, int64_t *off, int32_t *ent,
                              char *err, size_t errlen) {
    return guarded(err, errlen, [&] {
        pkgpu_context *ctx = tree->ctx;
        std::lock_guard<std::mutex> lock(ctx->mtx);
        PK_CUDA(cudaSetDevice(ctx->device));
        ListSetup ls{};
        if (setup && setup->periodicity != PKGPU_NONE && setup->ell >= 1)
            for (int a = 0; a < 3; a++) ls.periodic[a] = setup->axes[a] != 0;
        DeviceLists L;
        build_lists_csr(tree->tree, ls, L, ctx->stream, &ctx->launches);
        const CsrList *c = which == 'u' ? &L.u : which == 'v' ? &L.v : which == 'w' ? &L.w : which == 'x' ? &L.x : nullptr;
        if (!c) throw InvalidArgument("pkgpu_tree_lists: which must be one of u, v, w, x");
        const int64_t nb = tree->tree.nboxes;
        std::vector<int64_t> hoff(nb + 1);
        PK_CUDA(cudaMemcpy(hoff.data(), c->off, (nb + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
        if (off) std::memcpy(off, hoff.data(), hoff.size() * sizeof(int64_t));
        if (!ent) return;
        std::vector<int2> h(c->count);
        if (c->count) PK_CUDA(cudaMemcpy(h.data(), c->ent, c->count * sizeof(int2), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < c->count; i++) {
            ent[4 * i] = h[i].x;
            int a, b, d;
            if (which == 'v') {
                a = h[i].y / 49 - 3, b = (h[i].y / 7) % 7 - 3, d = h[i].y % 7 - 3;
            } else {
                shift_decode(h[i].y, a, b, d);
            }
            ent[4 * i + 1] = a, ent[4 * i + 2] = b, ent[4 * i + 3] = d;
        }
    });
}

} // extern "C"
