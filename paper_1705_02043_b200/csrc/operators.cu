// KIFMM operators on the device (replaces build_operators, src/fmm.cpp:180-236).
//
//  * surfaces are generated on the host with std::fma exactly as the compiled
//    reference evaluates surface_points (src/geometry.cpp:60-71, FMA-contracted);
//  * dense kernel blocks are assembled on the device bit-exactly (kernels.cuh);
//  * a_up / a_dn are factorised with cuSOLVER gesvd (or injected, parity mode);
//  * M2L: the reference stores 16 octahedral class matrices K(inner, inner + c) and
//    applies the signed permutation at run time (src/fmm.cpp:111-175). Here the class
//    matrices are expanded once into one matrix per offset slot (316 of them) by that
//    same exact permutation, so the GEMM streams plain row-major tiles. The expanded
//    entries equal the reference's effective operator bit for bit.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cusolverDn.h>
#include <limits>

#include "kernels.cuh"
#include "operators.h"

namespace pkgpu {

// ---------------------------------------------------------------------------
// host geometry

std::vector<int> surface_grid(int p) {
    // fixed ordering of src/geometry.cpp:43-58: origin corner, faces x=0, y=0, z=0,
    // then the point reflection of that first half
    std::vector<int> g{0, 0, 0};
    for (int i = 0; i < p - 1; i++)
        for (int j = 0; j < p - 1; j++) g.insert(g.end(), {0, i + 1, j});
    for (int i = 0; i < p - 1; i++)
        for (int j = 0; j < p - 1; j++) g.insert(g.end(), {i, 0, j + 1});
    for (int i = 0; i < p - 1; i++)
        for (int j = 0; j < p - 1; j++) g.insert(g.end(), {i + 1, j, 0});
    const size_t half = g.size();
    for (size_t i = 0; i < half; i += 3) g.insert(g.end(), {p - 1 - g[i], p - 1 - g[i + 1], p - 1 - g[i + 2]});
    return g;
}

std::vector<double> surface_template(int p) {
    const auto g = surface_grid(p);
    std::vector<double> t(g.size());
    const double scale = 2.0 / (p - 1);
    for (size_t i = 0; i < g.size(); i++) t[i] = std::fma(static_cast<double>(g[i]), scale, -1.0);
    return t;
}

std::vector<double> surface_points(int p, const double center[3], double edge) {
    const auto t = surface_template(p);
    const double half = 0.5 * edge;
    std::vector<double> pts(t.size());
    for (size_t i = 0; i < t.size(); i++) pts[i] = std::fma(half, t[i], center[i % 3]);
    return pts;
}

std::vector<std::array<int, 3>> image_offsets(const int axes[3], int min_norm, int max_norm) {
    std::vector<std::array<int, 3>> out;
    const int lx = axes[0] ? max_norm : 0, ly = axes[1] ? max_norm : 0, lz = axes[2] ? max_norm : 0;
    for (int ox = -lx; ox <= lx; ox++)
        for (int oy = -ly; oy <= ly; oy++)
            for (int oz = -lz; oz <= lz; oz++) {
                const int nrm = std::max({std::abs(ox), std::abs(oy), std::abs(oz)});
                if (nrm < min_norm || nrm > max_norm) continue;
                out.push_back({ox, oy, oz});
            }
    return out;
}

namespace {

// signed permutation g: (g v)_o = sign[o] * v[perm[o]]
struct SPerm {
    int perm[3], sign[3];
};

std::vector<SPerm> octahedral_group() {
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    std::vector<SPerm> g;
    for (const auto &pm : perms)
        for (int s = 0; s < 8; s++) {
            SPerm e{};
            for (int o = 0; o < 3; o++) {
                e.perm[o] = pm[o];
                e.sign[o] = ((s >> o) & 1) ? -1 : 1;
            }
            g.push_back(e);
        }
    return g;
}

SPerm inverse(const SPerm &g) {
    SPerm r{};
    for (int o = 0; o < 3; o++) {
        r.perm[g.perm[o]] = o;
        r.sign[g.perm[o]] = g.sign[o];
    }
    return r;
}

// ---------------------------------------------------------------------------
// device kernels

template <int KERNEL>
__global__ void kblock_kernel(const double *__restrict__ trg, int nt, const double *__restrict__ src, int ns,
                              double *__restrict__ out, int64_t ld) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nt * ns) return;
    const int i = (int)(idx / ns), j = (int)(idx % ns);
    double blk[9];
    kernel_entry_exact<KERNEL>(trg[3 * i], trg[3 * i + 1], trg[3 * i + 2], src[3 * j], src[3 * j + 1], src[3 * j + 2],
                               blk);
    constexpr int k = KERNEL == 0 ? 1 : 3;
#pragma unroll
    for (int a = 0; a < k; a++)
#pragma unroll
        for (int b = 0; b < k; b++) out[(int64_t)(k * i + a) * ld + k * j + b] = blk[a * k + b];
}

// M_img = sum_d K(inner, inner + d), summed entry-wise in image_offsets order
template <int KERNEL>
__global__ void image_sum_kernel(const double *__restrict__ pts, int n, const int *__restrict__ offs, int noff,
                                 double *__restrict__ out, int64_t ld) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * n) return;
    const int i = (int)(idx / n), j = (int)(idx % n);
    constexpr int k = KERNEL == 0 ? 1 : 3;
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < noff; q++) {
        double blk[9];
        kernel_entry_exact<KERNEL>(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2],
                                   __dadd_rn(pts[3 * j], (double)offs[3 * q]),
                                   __dadd_rn(pts[3 * j + 1], (double)offs[3 * q + 1]),
                                   __dadd_rn(pts[3 * j + 2], (double)offs[3 * q + 2]), blk);
#pragma unroll
        for (int a = 0; a < k * k; a++) acc[a] = __dadd_rn(acc[a], blk[a]);
    }
#pragma unroll
    for (int a = 0; a < k; a++)
#pragma unroll
        for (int b = 0; b < k; b++) out[(int64_t)(k * i + a) * ld + k * j + b] = acc[a * k + b];
}

// expand class matrices into per-slot matrices:
//   M_d[kt i + o][ks j + o'] = sign[o] sign[o'] M_cls[ks sigma(i) + perm[o]][ks sigma(j) + perm[o']]
__global__ void expand_m2l_kernel(const double *__restrict__ cls, const int *__restrict__ slot_cls,
                                  const int *__restrict__ slot_g, const int *__restrict__ sigma,
                                  const int *__restrict__ gperm, const int *__restrict__ gsign, int n, int k, int Kp,
                                  double *__restrict__ out) {
    const int slot = blockIdx.y;
    const int64_t KK = (int64_t)(k * n) * (k * n);
    const int c = slot_cls[slot], g = slot_g[slot];
    const double *M = cls + (int64_t)c * Kp * Kp;
    const int *sg = sigma + (int64_t)g * n;
    double *D = out + (int64_t)slot * Kp * Kp;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < KK; idx += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(idx / (k * n)), cidx = (int)(idx % (k * n));
        const int i = r / k, o = r % k, j = cidx / k, o2 = cidx % k;
        double v;
        if (k == 1) {
            v = M[(int64_t)sg[i] * Kp + sg[j]];
        } else {
            const int rr = 3 * sg[i] + gperm[3 * g + o], cc = 3 * sg[j] + gperm[3 * g + o2];
            v = (double)(gsign[3 * g + o] * gsign[3 * g + o2]) * M[(int64_t)rr * Kp + cc];
        }
        D[(int64_t)r * Kp + cidx] = v;
    }
}

void upload(Workspace &ws, const std::string &name, const std::vector<double> &h, double *&d, cudaStream_t st) {
    d = ws.get<double>(name, h.size());
    PK_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, st));
}

#define PK_SOLVER(x)                                                                                                \
    do {                                                                                                            \
        cusolverStatus_t s_ = (x);                                                                                  \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                          \
            throw RuntimeError("cuSOLVER error " + std::to_string((int)s_) + " at " + __FILE__ + ":" +             \
                               std::to_string(__LINE__));                                                           \
    } while (0)

} // namespace

void kernel_block_device(int kernel, const double *d_trg, int nt, const double *d_src, int ns, double *d_out,
                         int64_t ld, cudaStream_t st) {
    const int64_t tot = (int64_t)nt * ns;
    if (tot == 0) return;
    if (kernel == 0)
        kblock_kernel<0><<<blocks_for(tot, 256), 256, 0, st>>>(d_trg, nt, d_src, ns, d_out, ld);
    else
        kblock_kernel<1><<<blocks_for(tot, 256), 256, 0, st>>>(d_trg, nt, d_src, ns, d_out, ld);
    PK_CUDA(cudaGetLastError());
}

OperatorCache::~OperatorCache() {
    if (solver_) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(solver_));
}

KifmmOps &OperatorCache::base(int kernel, int p, cudaStream_t st) {
    if (p < 2) throw InvalidArgument("surface grid requires p >= 2");
    auto &slot = cache_[{kernel, p}];
    if (slot) return *slot;
    auto ops = std::make_unique<KifmmOps>();
    ops->kernel = kernel;
    ops->p = p;
    ops->n = surface_point_count(p);
    ops->ks = ops->kt = kernel == 0 ? 1 : 3;
    ops->K = ops->ks * ops->n;
    ops->Kp = round_up(ops->K, 64);
    ops->tmpl = surface_template(p);
    const double c[3] = {0.5, 0.5, 0.5};
    ops->inner = surface_points(p, c, kInner);
    ops->outer = surface_points(p, c, kOuter);
    upload(ops->ws, "tmpl", ops->tmpl, ops->d_tmpl, st);
    slot = std::move(ops);
    return *slot;
}

void OperatorCache::upload_factors(KifmmOps &ops, cudaStream_t st) {
    const int K = ops.K, Kp = ops.Kp;
    auto build = [&](const HostFactors &f, const char *tag, double *&Ut, double *&V, double *&s) {
        std::vector<double> ut((size_t)Kp * Kp, 0.0), v((size_t)Kp * Kp, 0.0), sg(Kp, 0.0);
        for (int i = 0; i < K; i++)
            for (int j = 0; j < K; j++) {
                ut[(size_t)i * Kp + j] = f.u[(size_t)j * K + i];  // (U^T)[i][j] = U[j][i]
                v[(size_t)i * Kp + j] = f.vt[(size_t)j * K + i];  // V[i][j] = Vt[j][i]
            }
        for (int i = 0; i < K; i++) sg[i] = f.sigma[i];
        upload(ops.ws, std::string("Ut_") + tag, ut, Ut, st);
        upload(ops.ws, std::string("V_") + tag, v, V, st);
        upload(ops.ws, std::string("s_") + tag, sg, s, st);
        PK_CUDA(cudaStreamSynchronize(st));
    };
    build(ops.up, "up", ops.Ut_up, ops.V_up, ops.s_up);
    build(ops.dn, "dn", ops.Ut_dn, ops.V_dn, ops.s_dn);
    // int8 residues of the factors are rebuilt from the new matrices on next use
    ops.i8_ut_up.res = ops.i8_v_up.res = ops.i8_ut_dn.res = ops.i8_v_dn.res = nullptr;
    ops.factors_ready = true;
}

void OperatorCache::ensure_factors(KifmmOps &ops, cudaStream_t st, int64_t *launches) {
    if (ops.factors_ready) return;
    const int n = ops.n, K = ops.K;
    double *d_in = ops.ws.get<double>("surf_in", 3 * n), *d_out = ops.ws.get<double>("surf_out", 3 * n);
    PK_CUDA(cudaMemcpyAsync(d_in, ops.inner.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(d_out, ops.outer.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (!solver_) {
        cusolverDnHandle_t h;
        PK_SOLVER(cusolverDnCreate(&h));
        solver_ = h;
    }
    auto h = static_cast<cusolverDnHandle_t>(solver_);
    PK_SOLVER(cusolverDnSetStream(h, st));
    double *A = ops.ws.get<double>("svd_a", (size_t)K * K);
    double *S = ops.ws.get<double>("svd_s", K);
    double *U = ops.ws.get<double>("svd_u", (size_t)K * K);
    double *VT = ops.ws.get<double>("svd_vt", (size_t)K * K);
    int *info = ops.ws.get<int>("svd_info", 1);
    int lwork = 0;
    PK_SOLVER(cusolverDnDgesvd_bufferSize(h, K, K, &lwork));
    double *work = ops.ws.get<double>("svd_work", lwork);
    double *rwork = ops.ws.get<double>("svd_rwork", K);
    for (int which = 0; which < 2; which++) {
        // a_up = K(outer, inner), a_dn = K(inner, outer), row-major K x K
        kernel_block_device(ops.kernel, which == 0 ? d_out : d_in, n, which == 0 ? d_in : d_out, n, A, K, st);
        // row-major A is column-major A^T = U' S V'^T  =>  A = V' S U'^T:
        // u_A (row-major) = buffer of V'^T, vt_A (row-major) = buffer of U'
        PK_SOLVER(cusolverDnDgesvd(h, 'A', 'A', K, K, A, K, S, U, K, VT, K, work, lwork, rwork, info));
        HostFactors &f = which == 0 ? ops.up : ops.dn;
        f.u.resize((size_t)K * K);
        f.vt.resize((size_t)K * K);
        f.sigma.resize(K);
        int hinfo = 0;
        PK_CUDA(cudaMemcpyAsync(f.u.data(), VT, (size_t)K * K * sizeof(double), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaMemcpyAsync(f.vt.data(), U, (size_t)K * K * sizeof(double), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaMemcpyAsync(f.sigma.data(), S, K * sizeof(double), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        if (hinfo != 0) throw RuntimeError("svd: LAPACK did not converge (info=" + std::to_string(hinfo) + ")");
        f.eps = std::numeric_limits<double>::epsilon() * (K ? f.sigma[0] : 0.0);
        *launches += 2;
    }
    upload_factors(ops, st);
}

void OperatorCache::inject(int kernel, int p, const HostFactors &up, const HostFactors &dn, cudaStream_t st,
                           int64_t *) {
    KifmmOps &ops = base(kernel, p, st);
    const size_t K = ops.K;
    if (up.u.size() != K * K || up.vt.size() != K * K || up.sigma.size() != K || dn.u.size() != K * K ||
        dn.vt.size() != K * K || dn.sigma.size() != K)
        throw InvalidArgument("set_kifmm_factors: factor dimensions do not match K");
    ops.up = up;
    ops.dn = dn;
    ops.up.eps = std::numeric_limits<double>::epsilon() * up.sigma[0];
    ops.dn.eps = std::numeric_limits<double>::epsilon() * dn.sigma[0];
    ops.injected = true;
    upload_factors(ops, st);
}

void OperatorCache::ensure_translations(KifmmOps &ops, cudaStream_t st, int64_t *launches) {
    if (ops.translations_ready) return;
    const int n = ops.n, Kp = ops.Kp, k = ops.ks;
    const int p = ops.p;
    // --- octahedral group, sigma maps and class table (mirrors src/fmm.cpp:189-233) ---
    const auto group = octahedral_group();
    const auto grid = surface_grid(p);
    std::vector<int> lookup((size_t)p * p * p, -1);
    for (int i = 0; i < n; i++) lookup[(grid[3 * i] * p + grid[3 * i + 1]) * p + grid[3 * i + 2]] = i;
    std::vector<int> sigma(48 * (size_t)n), gperm(48 * 3), gsign(48 * 3);
    for (int e = 0; e < 48; e++) {
        const SPerm inv = inverse(group[e]);
        for (int o = 0; o < 3; o++) {
            gperm[3 * e + o] = group[e].perm[o];
            gsign[3 * e + o] = group[e].sign[o];
        }
        for (int i = 0; i < n; i++) {
            int t[3];
            for (int o = 0; o < 3; o++) {
                const int v = grid[3 * i + inv.perm[o]];
                t[o] = inv.sign[o] > 0 ? v : p - 1 - v;
            }
            sigma[(size_t)e * n + i] = lookup[(t[0] * p + t[1]) * p + t[2]];
        }
    }
    std::vector<std::array<int, 3>> class_repr;
    std::vector<int> code_cls(343, -1), code_g(343, -1);
    for (int dx = -3; dx <= 3; dx++)
        for (int dy = -3; dy <= 3; dy++)
            for (int dz = -3; dz <= 3; dz++) {
                if (std::max({std::abs(dx), std::abs(dy), std::abs(dz)}) < 2) continue;
                std::array<int, 3> c{std::abs(dx), std::abs(dy), std::abs(dz)};
                std::sort(c.begin(), c.end(), std::greater<int>());
                int cls = -1;
                for (size_t q = 0; q < class_repr.size(); q++)
                    if (class_repr[q] == c) cls = (int)q;
                if (cls < 0) {
                    cls = (int)class_repr.size();
                    class_repr.push_back(c);
                }
                int ge = -1;
                for (int e = 0; e < 48 && ge < 0; e++) {
                    const SPerm &g = group[e];
                    const int v0 = g.sign[0] * c[g.perm[0]], v1 = g.sign[1] * c[g.perm[1]],
                              v2 = g.sign[2] * c[g.perm[2]];
                    if (v0 == dx && v1 == dy && v2 == dz) ge = e;
                }
                const int code = offset_code(dx, dy, dz);
                code_cls[code] = cls;
                code_g[code] = ge;
            }
    ops.h_slot_of_code.assign(343, -1);
    ops.h_code_of_slot.clear();
    std::vector<int> slot_cls, slot_g;
    for (int code = 0; code < 343; code++) {
        if (code_cls[code] < 0) continue;
        ops.h_slot_of_code[code] = (int)ops.h_code_of_slot.size();
        ops.h_code_of_slot.push_back(code);
        slot_cls.push_back(code_cls[code]);
        slot_g.push_back(code_g[code]);
    }
    if ((int)ops.h_code_of_slot.size() != kNumM2L) throw RuntimeError("M2L slot table size mismatch");
    // --- class matrices K(inner, inner + c), exact ---
    const int ncls = (int)class_repr.size();
    double *cls = ops.ws.get<double>("m2l_cls", (size_t)ncls * Kp * Kp);
    PK_CUDA(cudaMemsetAsync(cls, 0, (size_t)ncls * Kp * Kp * sizeof(double), st));
    double *d_in = ops.ws.get<double>("surf_in", 3 * n);
    PK_CUDA(cudaMemcpyAsync(d_in, ops.inner.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    std::vector<double> shifted_all((size_t)ncls * 3 * n);
    for (int c = 0; c < ncls; c++)
        for (int i = 0; i < n; i++)
            for (int o = 0; o < 3; o++)
                shifted_all[(size_t)c * 3 * n + 3 * i + o] = ops.inner[3 * i + o] + (double)class_repr[c][o];
    double *d_sh = nullptr;
    upload(ops.ws, "m2l_shifted", shifted_all, d_sh, st);
    for (int c = 0; c < ncls; c++)
        kernel_block_device(ops.kernel, d_in, n, d_sh + (size_t)c * 3 * n, n, cls + (size_t)c * Kp * Kp, Kp, st);
    *launches += ncls;
    // --- expand to 316 per-offset matrices ---
    ops.m2l = ops.ws.get<double>("m2l", (size_t)kNumM2L * Kp * Kp);
    PK_CUDA(cudaMemsetAsync(ops.m2l, 0, (size_t)kNumM2L * Kp * Kp * sizeof(double), st));
    int *d_slot_cls = ops.ws.get<int>("slot_cls", kNumM2L), *d_slot_g = ops.ws.get<int>("slot_g", kNumM2L);
    int *d_sigma = ops.ws.get<int>("sigma", sigma.size()), *d_gperm = ops.ws.get<int>("gperm", 144),
        *d_gsign = ops.ws.get<int>("gsign", 144);
    ops.slot_of_code = ops.ws.get<int>("slot_of_code", 343);
    PK_CUDA(cudaMemcpyAsync(d_slot_cls, slot_cls.data(), kNumM2L * sizeof(int), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(d_slot_g, slot_g.data(), kNumM2L * sizeof(int), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(d_sigma, sigma.data(), sigma.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(d_gperm, gperm.data(), 144 * sizeof(int), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(d_gsign, gsign.data(), 144 * sizeof(int), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(ops.slot_of_code, ops.h_slot_of_code.data(), 343 * sizeof(int), cudaMemcpyHostToDevice,
                            st));
    expand_m2l_kernel<<<dim3(64, kNumM2L), 256, 0, st>>>(cls, d_slot_cls, d_slot_g, d_sigma, d_gperm, d_gsign, n, k,
                                                         Kp, ops.m2l);
    PK_CUDA(cudaGetLastError());
    *launches += 1;
    // --- M2M_o = K(outer, child-inner(o)), L2L_o = K(child-inner(o), outer) ---
    ops.m2m = ops.ws.get<double>("m2m", (size_t)8 * Kp * Kp);
    ops.l2l = ops.ws.get<double>("l2l", (size_t)8 * Kp * Kp);
    PK_CUDA(cudaMemsetAsync(ops.m2m, 0, (size_t)8 * Kp * Kp * sizeof(double), st));
    PK_CUDA(cudaMemsetAsync(ops.l2l, 0, (size_t)8 * Kp * Kp * sizeof(double), st));
    double *d_out = ops.ws.get<double>("surf_out", 3 * n);
    PK_CUDA(cudaMemcpyAsync(d_out, ops.outer.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    std::vector<double> child_all((size_t)8 * 3 * n);
    for (int o = 0; o < 8; o++) {
        const double c[3] = {0.5 + ((o & 1) ? 0.25 : -0.25), 0.5 + ((o & 2) ? 0.25 : -0.25),
                             0.5 + ((o & 4) ? 0.25 : -0.25)};
        const auto pts = surface_points(p, c, 0.5 * kInner);
        std::copy(pts.begin(), pts.end(), child_all.begin() + (size_t)o * 3 * n);
    }
    double *d_child = nullptr;
    upload(ops.ws, "child_inner", child_all, d_child, st);
    for (int o = 0; o < 8; o++) {
        kernel_block_device(ops.kernel, d_out, n, d_child + (size_t)o * 3 * n, n, ops.m2m + (size_t)o * Kp * Kp, Kp,
                            st);
        kernel_block_device(ops.kernel, d_child + (size_t)o * 3 * n, n, d_out, n, ops.l2l + (size_t)o * Kp * Kp, Kp,
                            st);
    }
    *launches += 16;
    PK_CUDA(cudaStreamSynchronize(st));
    ops.translations_ready = true;
}

KifmmOps &OperatorCache::get(int kernel, int p, cudaStream_t st, int64_t *launches) {
    KifmmOps &ops = base(kernel, p, st);
    ensure_factors(ops, st, launches);
    ensure_translations(ops, st, launches);
    return ops;
}

const double *OperatorCache::image_operator(KifmmOps &ops, const int axes[3], int ell, cudaStream_t st,
                                            int64_t *launches) {
    const int mask = (axes[0] ? 1 : 0) | (axes[1] ? 2 : 0) | (axes[2] ? 4 : 0);
    auto it = ops.img.find({mask, ell});
    if (it != ops.img.end()) return it->second;
    const auto offs = image_offsets(axes, 2, ell);
    std::vector<int> flat;
    for (const auto &d : offs) flat.insert(flat.end(), d.begin(), d.end());
    const int n = ops.n, Kp = ops.Kp;
    double *m = ops.ws.get<double>("img_" + std::to_string(mask) + "_" + std::to_string(ell), (size_t)Kp * Kp);
    PK_CUDA(cudaMemsetAsync(m, 0, (size_t)Kp * Kp * sizeof(double), st));
    if (!offs.empty()) {
        int *d_offs = ops.ws.get<int>("img_offs_tmp", flat.size());
        PK_CUDA(cudaMemcpyAsync(d_offs, flat.data(), flat.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        double *d_in = ops.ws.get<double>("surf_in", 3 * n);
        PK_CUDA(cudaMemcpyAsync(d_in, ops.inner.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
        const int64_t tot = (int64_t)n * n;
        if (ops.kernel == 0)
            image_sum_kernel<0><<<blocks_for(tot, 128), 128, 0, st>>>(d_in, n, d_offs, (int)offs.size(), m, Kp);
        else
            image_sum_kernel<1><<<blocks_for(tot, 128), 128, 0, st>>>(d_in, n, d_offs, (int)offs.size(), m, Kp);
        PK_CUDA(cudaGetLastError());
        PK_CUDA(cudaStreamSynchronize(st));
        *launches += 1;
    }
    ops.img[{mask, ell}] = m;
    return m;
}

std::vector<double> OperatorCache::matrix(int kernel, int p, int which, int i0, int i1, int i2, cudaStream_t st,
                                          int64_t *launches) {
    KifmmOps &ops = get(kernel, p, st, launches);
    const int K = ops.K, Kp = ops.Kp;
    const double *src = nullptr;
    std::vector<double> dense((size_t)Kp * Kp);
    double *tmp = nullptr;
    switch (which) {
    case 0:
    case 1: {
        tmp = ops.ws.get<double>("mat_tmp", (size_t)Kp * Kp);
        double *d_in = ops.ws.get<double>("surf_in", 3 * ops.n), *d_out = ops.ws.get<double>("surf_out", 3 * ops.n);
        PK_CUDA(cudaMemsetAsync(tmp, 0, (size_t)Kp * Kp * sizeof(double), st));
        kernel_block_device(kernel, which == 0 ? d_out : d_in, ops.n, which == 0 ? d_in : d_out, ops.n, tmp, Kp, st);
        src = tmp;
        break;
    }
    case 2: src = ops.m2m + (size_t)(i0 & 7) * Kp * Kp; break;
    case 3: src = ops.l2l + (size_t)(i0 & 7) * Kp * Kp; break;
    case 4: {
        if (std::max({std::abs(i0), std::abs(i1), std::abs(i2)}) < 2 || std::abs(i0) > 3 || std::abs(i1) > 3 ||
            std::abs(i2) > 3)
            throw InvalidArgument("apply_m2l: offset outside the well-separated range");
        src = ops.m2l + (size_t)ops.h_slot_of_code[offset_code(i0, i1, i2)] * Kp * Kp;
        break;
    }
    case 5: {
        const int axes[3] = {i0 & 1, (i0 >> 1) & 1, (i0 >> 2) & 1};
        src = image_operator(ops, axes, i1, st, launches);
        break;
    }
    default: throw InvalidArgument("kifmm_matrix: unknown matrix kind");
    }
    PK_CUDA(cudaMemcpyAsync(dense.data(), src, dense.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    std::vector<double> out((size_t)K * K);
    for (int i = 0; i < K; i++) std::memcpy(&out[(size_t)i * K], &dense[(size_t)i * Kp], K * sizeof(double));
    return out;
}

} // namespace pkgpu
