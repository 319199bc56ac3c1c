// FFT-accelerated M2L (see m2l_fft.h).
#include <algorithm>
#include <cmath>
#include <string>

#include <cub/cub.cuh>
#include <cufft.h>

#include "kernels.cuh"
#include "m2l_fft.h"
#include "operators.h"

namespace pkgpu {

#define PK_FFT(x)                                                                                                   \
    do {                                                                                                            \
        cufftResult r_ = (x);                                                                                       \
        if (r_ != CUFFT_SUCCESS)                                                                                    \
            throw ::pkgpu::CudaError(std::string("cuFFT error ") + std::to_string((int)r_) + " at " + __FILE__ + ":" + \
                                     std::to_string(__LINE__));                                                     \
    } while (0)

FftOps::~FftOps() {
    for (auto &kv : plans_r2c) cufftDestroy((cufftHandle)kv.second);
    for (auto &kv : plans_c2r) cufftDestroy((cufftHandle)kv.second);
}

namespace {

constexpr int kSlots = kNumM2L;
constexpr int FFT_THREADS = 128;
constexpr int FFT_TC = 8; // target columns per CTA: each K^ load feeds TC columns

// lattice kernel grids k_{d,ab}(dg) = K_ab(dg D - d) at the root scale, one N^3 grid per
// (slot, a, b); dg = i for i < p, i - N otherwise (N = 2p: every surface difference in [-(p-1), p-1])
__global__ void kgrid_kernel(int kernel, int N, int p, const int *__restrict__ code_of_slot, double *grid) {
    const int ks = kernel == 0 ? 1 : 3;
    const int sab = blockIdx.y;
    const int slot = sab / (ks * ks), a = (sab / ks) % ks, b = sab % ks;
    const int code = code_of_slot[slot];
    const double dx = code / 49 - 3, dy = (code / 7) % 7 - 3, dz = code % 7 - 3;
    const double D = 1.05 / (p - 1);
    const int64_t N3 = (int64_t)N * N * N;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < N3; idx += (int64_t)gridDim.x * blockDim.x) {
        const int ix = (int)(idx / (N * N)), iy = (int)((idx / N) % N), iz = (int)(idx % N);
        const int gx = ix < p ? ix : ix - N, gy = iy < p ? iy : iy - N, gz = iz < p ? iz : iz - N;
        const double r[3] = {gx * D - dx, gy * D - dy, gz * D - dz};
        const double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
        const double rinv = 1.0 / sqrt(r2);
        double v;
        if (kernel == 0)
            v = rinv;
        else
            v = kOneOver8Pi * ((a == b ? rinv : 0.0) + r[a] * r[b] * rinv * rinv * rinv);
        grid[(int64_t)sab * N3 + idx] = v;
    }
}

// scatter phi of the window's source boxes onto their grids (interior points stay zero)
__global__ void fft_scatter_kernel(const double *__restrict__ X, int64_t Kp, const int *__restrict__ srcs, int nsrc,
                                   int n, int ks, const int *__restrict__ gidx, int64_t N3, double *grid) {
    const int64_t total = (int64_t)nsrc * n * ks;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / (n * ks);
        const int r = (int)(t % (n * ks)), i = r / ks, c = r % ks;
        grid[(k * ks + c) * N3 + gidx[i]] = X[(int64_t)srcs[k] * Kp + ks * i + c];
    }
}

// check potentials at the surface points: Y[out(col)][kt i + a] += scale * grid[col][a][g_i]
__global__ void fft_gather_kernel(const double *__restrict__ grid, const int *__restrict__ out_box, int W, int n, int kt,
                                  const int *__restrict__ gidx, int64_t N3, double scale, int64_t Kp,
                                  double *__restrict__ Y) {
    const int64_t total = (int64_t)W * n * kt;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int col = (int)(t / (n * kt));
        const int r = (int)(t % (n * kt)), i = r / kt, a = r % kt;
        const int ob = out_box[col];
        if (ob < 0) continue;
        Y[(int64_t)ob * Kp + kt * i + a] += scale * grid[((int64_t)col * kt + a) * N3 + gidx[i]];
    }
}

// Q^[col][a][w] = sum_slots sum_b K^[slot][a][b][w] Phi^[map(src)][b][w]; a thread per
// frequency, FFT_TC columns per CTA (one K^ read serves them all)
template <int KS>
__global__ void __launch_bounds__(FFT_THREADS) fft_hadamard_kernel(const double2 *__restrict__ khat,
                                                                   const double2 *__restrict__ phat,
                                                                   const int *__restrict__ smap,
                                                                   const int *__restrict__ table, int64_t ld,
                                                                   int nw, double2 *__restrict__ qhat) {
    constexpr int KT = KS;
    const int w = blockIdx.x * FFT_THREADS + threadIdx.x;
    const int c0 = blockIdx.y * FFT_TC;
    double2 acc[FFT_TC][KT];
#pragma unroll
    for (int c = 0; c < FFT_TC; c++)
#pragma unroll
        for (int a = 0; a < KT; a++) acc[c][a] = make_double2(0.0, 0.0);
    const bool on = w < nw;
    for (int s = 0; s < kSlots; s++) {
        int src[FFT_TC];
        bool any = false;
#pragma unroll
        for (int c = 0; c < FFT_TC; c++) {
            const int b = table[(int64_t)s * ld + c0 + c];
            src[c] = b >= 0 ? smap[b] : -1;
            any |= b >= 0;
        }
        if (!any || !on) continue;
        double2 kh[KT][KS];
#pragma unroll
        for (int a = 0; a < KT; a++)
#pragma unroll
            for (int b = 0; b < KS; b++) kh[a][b] = khat[((int64_t)(s * KT + a) * KS + b) * nw + w];
#pragma unroll
        for (int c = 0; c < FFT_TC; c++) {
            if (src[c] < 0) continue;
            double2 ph[KS];
#pragma unroll
            for (int b = 0; b < KS; b++) ph[b] = phat[((int64_t)src[c] * KS + b) * nw + w];
#pragma unroll
            for (int a = 0; a < KT; a++)
#pragma unroll
                for (int b = 0; b < KS; b++) {
                    acc[c][a].x = fma(kh[a][b].x, ph[b].x, fma(-kh[a][b].y, ph[b].y, acc[c][a].x));
                    acc[c][a].y = fma(kh[a][b].x, ph[b].y, fma(kh[a][b].y, ph[b].x, acc[c][a].y));
                }
        }
    }
    if (!on) return;
#pragma unroll
    for (int c = 0; c < FFT_TC; c++)
#pragma unroll
        for (int a = 0; a < KT; a++) qhat[((int64_t)(c0 + c) * KT + a) * nw + w] = acc[c][a];
}

// unique source boxes of a window: flags over the level's boxes
__global__ void fft_mark_kernel(const int *__restrict__ table, int64_t ld, int ncols, int64_t box0, int *flags) {
    const int64_t total = (int64_t)kSlots * ncols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t / ncols), c = (int)(t % ncols);
        const int b = table[(int64_t)s * ld + c];
        if (b >= 0) flags[b - box0] = 1;
    }
}
__global__ void fft_map_kernel(const int *__restrict__ list, int n, int64_t box0, int *smap, int value_is_index) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) smap[list[k]] = value_is_index ? k : -1;
    (void)box0;
}
__global__ void offset_list_kernel(int *list, int n, int64_t box0) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) list[k] += (int)box0;
}

cufftHandle plan_for(std::map<int, long long> &cache, int N, int batch, bool r2c) {
    auto it = cache.find(batch);
    if (it != cache.end()) return (cufftHandle)it->second;
    cufftHandle h;
    int dims[3] = {N, N, N};
    PK_FFT(cufftPlanMany(&h, 3, dims, nullptr, 1, 0, nullptr, 1, 0, r2c ? CUFFT_D2Z : CUFFT_Z2D, batch));
    cache[batch] = (long long)h;
    return h;
}

// batched transforms in chunks of at most `chunk` grids (cached plans: chunk and the tail)
void exec_batched(FftOps &f, bool r2c, void *in, void *out, int64_t nbatch, cudaStream_t st) {
    const int64_t N3 = (int64_t)f.N * f.N * f.N, chunk = 1024;
    for (int64_t b0 = 0; b0 < nbatch; b0 += chunk) {
        const int nb = (int)std::min<int64_t>(chunk, nbatch - b0);
        cufftHandle h = plan_for(r2c ? f.plans_r2c : f.plans_c2r, f.N, nb, r2c);
        PK_FFT(cufftSetStream(h, st));
        if (r2c)
            PK_FFT(cufftExecD2Z(h, static_cast<double *>(in) + b0 * N3,
                                reinterpret_cast<cufftDoubleComplex *>(out) + b0 * f.nw));
        else
            PK_FFT(cufftExecZ2D(h, reinterpret_cast<cufftDoubleComplex *>(in) + b0 * f.nw,
                                static_cast<double *>(out) + b0 * N3));
    }
}

} // namespace

int m2l_fft_prepare(KifmmOps &ops, Workspace &ws, cudaStream_t st) {
    FftOps &f = ops.fft;
    if (f.ready) return 0;
    const int p = ops.p, ks = ops.ks, kt = ops.kt;
    f.N = 2 * p;
    f.nw = f.N * f.N * (f.N / 2 + 1);
    const int64_t N3 = (int64_t)f.N * f.N * f.N;
    // surface point -> grid index (the lattice of src/geometry.cpp:41-71)
    const std::vector<int> g = surface_grid(p);
    std::vector<int> gi(ops.n);
    for (int i = 0; i < ops.n; i++) gi[i] = (g[3 * i] * f.N + g[3 * i + 1]) * f.N + g[3 * i + 2];
    f.gidx = ops.ws.get<int>("fft_gidx", ops.n);
    PK_CUDA(cudaMemcpyAsync(f.gidx, gi.data(), gi.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    int *d_code = ops.ws.get<int>("fft_code", kSlots);
    PK_CUDA(cudaMemcpyAsync(d_code, ops.h_code_of_slot.data(), kSlots * sizeof(int), cudaMemcpyHostToDevice, st));
    const int64_t ngrids = (int64_t)kSlots * kt * ks;
    double *kg = ws.get<double>("fft_kgrid", ngrids * N3);
    kgrid_kernel<<<dim3(std::max<int64_t>(1, N3 / 256), (unsigned)ngrids), 256, 0, st>>>(ops.kernel, f.N, p, d_code, kg);
    PK_CUDA(cudaGetLastError());
    f.khat = ops.ws.get<double>("fft_khat", ngrids * f.nw * 2);
    exec_batched(f, true, kg, f.khat, ngrids, st);
    PK_CUDA(cudaStreamSynchronize(st)); // the host vectors above are read by async copies
    f.ready = true;
    return 2;
}

int m2l_fft_level(KifmmOps &ops, const FftLevelArgs &a, Workspace &ws, cudaStream_t st) {
    if (a.ncols == 0) return 0;
    if (a.ncols % FFT_TC != 0) throw RuntimeError("m2l_fft: columns must be a multiple of 8");
    FftOps &f = ops.fft;
    const int ks = ops.ks, kt = ops.kt, n = ops.n;
    const int64_t N3 = (int64_t)f.N * f.N * f.N, nlev = a.box1 - a.box0;
    int launches = 0;
    // columns per window: spectra of the window's targets and of their (unique) sources
    const int64_t per_col = (int64_t)(kt + 2 * ks) * (f.nw * 16 + N3 * 8);
    const int W = (int)std::max<int64_t>(FFT_TC, std::min<int64_t>(a.ncols, (int64_t)12e9 / per_col) / FFT_TC * FFT_TC);
    int *flags = ws.get<int>("fft_flags", nlev), *list = ws.get<int>("fft_list", nlev), *cnt = ws.get<int>("fft_cnt", 1);
    int *smap = ws.get<int>("fft_smap", nlev);
    PK_CUDA(cudaMemsetAsync(smap, 0xff, nlev * sizeof(int), st));
    for (int c0 = 0; c0 < a.ncols; c0 += W) {
        const int wc = std::min(W, a.ncols - c0);
        const int *tab = a.src + c0;
        // unique sources of the window (periodic wraps reach the far end of the level)
        PK_CUDA(cudaMemsetAsync(flags, 0, nlev * sizeof(int), st));
        fft_mark_kernel<<<(unsigned)std::min<int64_t>(((int64_t)kSlots * wc + 255) / 256, 148 * 16), 256, 0, st>>>(
            tab, a.ld, wc, a.box0, flags);
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, cub::CountingInputIterator<int>(0), flags, list, cnt, (int)nlev, st);
        void *tmp = ws.get<char>("fft_sel", tb);
        PK_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cub::CountingInputIterator<int>(0), flags, list, cnt, (int)nlev, st));
        int nsrc = 0;
        PK_CUDA(cudaMemcpyAsync(&nsrc, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        launches += 3;
        if (nsrc == 0) continue;
        // smap: level-relative source -> its row in the window's spectra (box ids offset by box0)
        offset_list_kernel<<<(nsrc + 255) / 256, 256, 0, st>>>(list, nsrc, a.box0);
        int *smap_abs = smap - a.box0; // indexed by absolute box id
        fft_map_kernel<<<(nsrc + 255) / 256, 256, 0, st>>>(list, nsrc, 0, smap_abs, 1);
        // forward: source grids (interior zero, kept zero across windows) -> spectra
        const int64_t ngs = (int64_t)nsrc * ks;
        const size_t gbytes = (size_t)ngs * N3 * sizeof(double);
        double *gin = ws.get<double>("fft_gin", ngs * N3);
        PK_CUDA(cudaMemsetAsync(gin, 0, gbytes, st));
        fft_scatter_kernel<<<(unsigned)std::min<int64_t>((ngs * n + 255) / 256, 148 * 32), 256, 0, st>>>(
            a.X, ops.Kp, list, nsrc, n, ks, f.gidx, N3, gin);
        double *phat = ws.get<double>("fft_phat", ngs * f.nw * 2);
        exec_batched(f, true, gin, phat, ngs, st);
        // frequency-domain accumulation over the V lists
        double *qhat = ws.get<double>("fft_qhat", (int64_t)wc * kt * f.nw * 2);
        const dim3 grid((f.nw + FFT_THREADS - 1) / FFT_THREADS, wc / FFT_TC);
        if (ks == 1)
            fft_hadamard_kernel<1><<<grid, FFT_THREADS, 0, st>>>(reinterpret_cast<const double2 *>(f.khat),
                                                                 reinterpret_cast<const double2 *>(phat), smap_abs, tab,
                                                                 a.ld, f.nw, reinterpret_cast<double2 *>(qhat));
        else
            fft_hadamard_kernel<3><<<grid, FFT_THREADS, 0, st>>>(reinterpret_cast<const double2 *>(f.khat),
                                                                 reinterpret_cast<const double2 *>(phat), smap_abs, tab,
                                                                 a.ld, f.nw, reinterpret_cast<double2 *>(qhat));
        // inverse, then the check potentials at the surface points (1 / N^3: cuFFT is unnormalised)
        double *gout = ws.get<double>("fft_gout", (int64_t)wc * kt * N3);
        exec_batched(f, false, qhat, gout, (int64_t)wc * kt, st);
        fft_gather_kernel<<<(unsigned)std::min<int64_t>(((int64_t)wc * n * kt + 255) / 256, 148 * 32), 256, 0, st>>>(
            gout, a.out_box + c0, wc, n, kt, f.gidx, N3, a.alpha / (double)N3, ops.Kp, a.Y);
        fft_map_kernel<<<(nsrc + 255) / 256, 256, 0, st>>>(list, nsrc, 0, smap_abs, 0); // reset the map
        PK_CUDA(cudaGetLastError());
        launches += 9;
    }
    return launches;
}

} // namespace pkgpu
