// Device-resident KIFMM translation operators per (kernel, p): the replacement for
// KifmmOperators / build_operators / operators_registry (src/fmm.cpp:55-259) and
// root_image_operator (src/fmm.cpp:262-283).
#pragma once

#include <array>
#include <map>
#include <memory>
#include <vector>

#include "common.h"
#include "m2l_fft.h"
#include "m2l_i8.h"

namespace pkgpu {

struct HostFactors {           // SvdFactors layout (include/pkifmm/linalg.hpp:45-53)
    std::vector<double> u;     // K x K row-major
    std::vector<double> sigma; // K
    std::vector<double> vt;    // K x K row-major
    double eps = 0.0;          // eps_svd = DBL_EPSILON * sigma_max (src/linalg.cpp:64-66)
};

struct KifmmOps {
    int kernel = 0, p = 0, n = 0, ks = 1, kt = 1, K = 0, Kp = 0;
    std::vector<double> tmpl;               // n x 3 template t = fma(g, 2/(p-1), -1)
    std::vector<double> inner, outer;       // root surfaces (edges 1.05 / 2.95)
    HostFactors up, dn;                     // a_up = K(outer, inner), a_dn = K(inner, outer)
    bool injected = false;
    Workspace ws;
    double *d_tmpl = nullptr;               // n x 3
    double *Ut_up = nullptr, *V_up = nullptr, *s_up = nullptr; // Kp x Kp, Kp x Kp, Kp
    double *Ut_dn = nullptr, *V_dn = nullptr, *s_dn = nullptr;
    double *m2l = nullptr;                  // 316 x Kp x Kp, per offset slot
    double *m2m = nullptr, *l2l = nullptr;  // 8 x Kp x Kp
    int *slot_of_code = nullptr;            // device [343]
    std::vector<int> h_slot_of_code, h_code_of_slot;
    std::map<std::pair<int, int>, double *> img; // (axes mask, ell) -> M_img Kp x Kp
    I8Operators i8;                         // M2L residues for the int8 tensor pipe (lazy)
    I8Operators i8_m2m, i8_l2l;             // M2M / L2L residues (lazy, i8_translate)
    I8Operators i8_ut_up, i8_v_up, i8_ut_dn, i8_v_dn; // pseudo-inverse factors (reset on upload)
    FftOps fft;                             // M2L kernel spectra (lazy, the FFT M2L path)
    bool factors_ready = false, translations_ready = false;
};

class OperatorCache {
  public:
    // Operators with factors + translation matrices ready (builds lazily).
    KifmmOps &get(int kernel, int p, cudaStream_t st, int64_t *launches);
    void inject(int kernel, int p, const HostFactors &up, const HostFactors &dn, cudaStream_t st, int64_t *launches);
    // M_img for image layers 2..ell on the given periodic axes (src/fmm.cpp:262-283)
    const double *image_operator(KifmmOps &ops, const int axes[3], int ell, cudaStream_t st, int64_t *launches);
    // dense matrices for parity checks (pkgpu_kifmm_matrix)
    std::vector<double> matrix(int kernel, int p, int which, int i0, int i1, int i2, cudaStream_t st,
                               int64_t *launches);

  private:
    KifmmOps &base(int kernel, int p, cudaStream_t st);
    void ensure_factors(KifmmOps &ops, cudaStream_t st, int64_t *launches);
    void upload_factors(KifmmOps &ops, cudaStream_t st);
    void ensure_translations(KifmmOps &ops, cudaStream_t st, int64_t *launches);
    std::map<std::pair<int, int>, std::unique_ptr<KifmmOps>> cache_;
    void *solver_ = nullptr; // cusolverDnHandle_t
  public:
    ~OperatorCache();
};

// host helpers (bit-exact geometry, src/geometry.cpp:41-87)
std::vector<int> surface_grid(int p); // n x 3
std::vector<double> surface_template(int p);
std::vector<double> surface_points(int p, const double center[3], double edge);
std::vector<std::array<int, 3>> image_offsets(const int axes[3], int min_norm, int max_norm);

// device dense kernel block: out[(kt i + a) * ld + ks j + b] = K(t_i, s_j)
void kernel_block_device(int kernel, const double *d_trg, int nt, const double *d_src, int ns, double *d_out,
                         int64_t ld, cudaStream_t st);

} // namespace pkgpu
