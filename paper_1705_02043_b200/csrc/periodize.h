// Periodizing-operator precompute and the periodic reference kernel on the device
// (csrc/periodize.cu). Replaces solve_m2l (include/pkifmm/periodize.hpp:42-46),
// periodic_block / kpf_block (include/pkifmm/refsum.hpp:68-72) and oracle_system_eval
// (include/pkifmm/refsum.hpp:88).
#pragma once

#include <string>
#include <vector>

#include "common.h"
#include "pkgpu.h"

struct pkgpu_context;

namespace pkgpu {

struct EwaldSettings { // EwaldParams (include/pkifmm/refsum.hpp:21-27)
    double xi = 8.0;
    int real_shells = 2;
    int wave_cutoff = 64;
    long long n_images = 1000000;
};

struct PeriodicSolve {
    std::vector<double> matrix; // dim x dim row-major
    int64_t dim = 0;
    int method = 0;
    double residual_max = 0.0;  // -1 when ungated (as refdump --ungated)
};

const char *method_label(int method);
// make_periodic_spec's method choice with its ConfigErrors
int periodic_method(int kernel, const pkgpu_setup &setup);
// out[(kt i + a) ld + ks j + b] = K^P(t_i, s_j) (far_only: K^{P,F}); device pointers
void periodic_block_device(int kernel, const pkgpu_setup &setup, const EwaldSettings &e, bool far_only,
                           const double *d_trg, int nt, const double *d_src, int ns, double *d_out, int64_t ld,
                           cudaStream_t st);
// solve_m2l with the context's KIFMM factors; gated: throw past the 1e-11 residual gate
PeriodicSolve solve_periodizing_operator(pkgpu_context &ctx, int kernel, const pkgpu_setup &setup, int p,
                                         const EwaldSettings &e, bool gated);
std::string iso_now();

} // namespace pkgpu
