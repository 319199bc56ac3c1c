// FFT-accelerated M2L (see m2l_fft.h).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <string>
#include <type_traits>

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

// Edge of the cyclic surface grid. The surface differences g_i - g_j lie in [-(p-1), p-1]:
// 2p - 1 distinct values, so a cyclic convolution of that size is already the linear one at
// every surface point (round 2: N = 2p - 1 instead of 2p -- 22% fewer surface frequencies at
// p = 8; the pruned surface DFTs are direct sums and cuFFT takes any size for K^).
__host__ __device__ constexpr int fft_edge(int p) { return 2 * p - 1; }

// lattice kernel grids k_{d,ab}(dg) = K_ab(dg D - d) at the root scale, one N^3 grid per
// (slot, a, b); dg = i for i < p, i - N otherwise (N = fft_edge(p): every surface difference in [-(p-1), p-1])
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
// (only_tiles: the 64-column tiles with tile_nsrc < 0, whose sources overflowed the staging)
template <int KS>
__global__ void __launch_bounds__(FFT_THREADS) fft_hadamard_kernel(const double2 *__restrict__ khat,
                                                                   const double2 *__restrict__ phat,
                                                                   const int *__restrict__ smap,
                                                                   const int *__restrict__ table, int64_t ld,
                                                                   int nw, double2 *__restrict__ qhat,
                                                                   const int *__restrict__ only_tiles) {
    constexpr int KT = KS;
    const int w = blockIdx.x * FFT_THREADS + threadIdx.x;
    const int c0 = blockIdx.y * FFT_TC;
    if (only_tiles && only_tiles[c0 / 64] >= 0) return;
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

// ---------------------------------------------------------------------------
// Source-staged accumulation (the main kernel). A tile is 64 consecutive target columns
// (Morton order: a compact block of boxes whose V lists share most sources -- ~512 unique
// sources for the 64 x 189 entries of a uniform level). fft_tile_sources_kernel dedups a
// tile's sources (shared-memory hash) into tile_srcs and maps every (slot, target) entry to
// its position there (srcmap, int16). fft_stage_kernel then runs one CTA per (tile, block of
// 4 frequencies), two CTAs per SM: the tile's source spectra for those frequencies are
// staged in shared memory once (chunks of 448 sources), the kernel spectra 32 slots at a
// time, and every (target, slot) entry reads both from there -- the kernel spectrum of a
// slot is the same address across a warp (32 targets, one frequency): a broadcast.
constexpr int FT_TILE = 64;   // targets per tile
constexpr int FT_WB = 4;      // frequencies per CTA (a warp of 32 targets per frequency)
constexpr int FT_CH = 320;    // staged sources per chunk (Stokes: 320 x 13 x 16 B = 67 KB)
constexpr int FT_SCH = 32;    // slots whose kernel spectra are staged at a time (18 KB)
constexpr int FT_HS = 4096;   // dedup hash slots per tile
constexpr int FT_MAXU = 3072; // unique sources per tile handled by staging (more: the direct kernel)
constexpr int FT_THREADS = 256;

__device__ __forceinline__ int ft_hash(int k) { return (int)(((unsigned)k * 2654435761u) >> 20) & (FT_HS - 1); }

__global__ void __launch_bounds__(FT_THREADS) fft_tile_sources_kernel(const int *__restrict__ table, int64_t ld,
                                                                       const int *__restrict__ smap, int *tile_nsrc,
                                                                       int *tile_srcs, short *srcmap) {
    __shared__ int keys[FT_HS], vals[FT_HS];
    __shared__ int s_count, s_over;
    const int tile = blockIdx.x, tid = threadIdx.x;
    const int c0 = tile * FT_TILE;
    for (int h = tid; h < FT_HS; h += FT_THREADS) keys[h] = -1;
    if (tid == 0) s_count = 0, s_over = 0;
    __syncthreads();
    constexpr int NE = kSlots * FT_TILE;
    for (int e = tid; e < NE; e += FT_THREADS) {
        const int b = table[(int64_t)(e / FT_TILE) * ld + c0 + e % FT_TILE];
        if (b < 0) continue;
        const int key = smap[b];
        int h = ft_hash(key);
        for (int probe = 0; probe < FT_HS; probe++) {
            const int old = atomicCAS(&keys[h], -1, key);
            if (old == -1 || old == key) break;
            h = (h + 1) & (FT_HS - 1);
        }
    }
    __syncthreads();
    // positions in slot order of the hash table (deterministic for a given key set)
    for (int h = tid; h < FT_HS; h += FT_THREADS)
        if (keys[h] >= 0) {
            const int idx = atomicAdd(&s_count, 1);
            vals[h] = idx;
        }
    __syncthreads();
    const int u = s_count;
    if (u > FT_MAXU) {
        if (tid == 0) tile_nsrc[tile] = -1; // too many: this tile takes the direct kernel
        return;
    }
    for (int h = tid; h < FT_HS; h += FT_THREADS)
        if (keys[h] >= 0) tile_srcs[(int64_t)tile * FT_MAXU + vals[h]] = keys[h];
    for (int e = tid; e < NE; e += FT_THREADS) {
        const int b = table[(int64_t)(e / FT_TILE) * ld + c0 + e % FT_TILE];
        short v = -1;
        if (b >= 0) {
            const int key = smap[b];
            int h = ft_hash(key);
            while (keys[h] != key) h = (h + 1) & (FT_HS - 1);
            v = (short)vals[h];
        }
        srcmap[(int64_t)tile * NE + e] = v;
    }
    if (tid == 0) tile_nsrc[tile] = u;
}

__device__ __forceinline__ void ft_cp16(void *smem, const void *gmem, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void ft_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void ft_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int KS>
__global__ void __launch_bounds__(FT_THREADS, 2) fft_stage_kernel(const double2 *__restrict__ khat,
                                                                   const double2 *__restrict__ phat,
                                                                   const int *__restrict__ tile_nsrc,
                                                                   const int *__restrict__ tile_srcs,
                                                                   const short *__restrict__ srcmap, int nw,
                                                                   double2 *__restrict__ qhat) {
    constexpr int KT = KS;
    constexpr int SST = KS * FT_WB + 1;            // source stride (double2): odd, so 32 random sources
                                                   // spread over all eight 16-byte bank groups
    constexpr int KCH = FT_SCH * KT * KS * FT_WB;  // double2 per kernel-spectrum chunk
    constexpr int MCH = FT_SCH * FT_TILE / 8;      // srcmap chunk in 16-byte units (8 shorts)
    extern __shared__ __align__(16) double2 ft_smem[];
    double2 *stage = ft_smem;                      // [FT_CH][SST] source spectra
    double2 *kst = stage + FT_CH * SST;            // 2 x [FT_SCH][KT][KS][FT_WB] kernel spectra
    short *mst = reinterpret_cast<short *>(kst + 2 * KCH); // 2 x [FT_SCH][FT_TILE] source positions
    const int tile = blockIdx.y, tid = threadIdx.x;
    const int u = tile_nsrc[tile];
    if (u < 0) return; // overflow tile: the direct kernel covers it
    const int t = tid % FT_TILE, wl = tid / FT_TILE; // warp = 32 targets, one frequency
    const int w0 = blockIdx.x * FT_WB, w = w0 + wl;
    double2 acc[KT], acc2[KT];
#pragma unroll
    for (int a = 0; a < KT; a++) acc[a] = acc2[a] = make_double2(0.0, 0.0);
    const short *smg = srcmap + (int64_t)tile * kSlots * FT_TILE;
    constexpr int NSC = (kSlots + FT_SCH - 1) / FT_SCH;
    auto load_chunk = [&](int c, int buf) { // kernel spectra + source positions of slot chunk c
        const int s0 = c * FT_SCH, ns = min(FT_SCH, kSlots - s0);
        double2 *kd = kst + buf * KCH;
        for (int e = tid; e < ns * KT * KS * FT_WB; e += FT_THREADS) {
            const int sab = e / FT_WB, ww = e % FT_WB;
            const bool ok = w0 + ww < nw;
            ft_cp16(kd + e, khat + ((int64_t)s0 * KT * KS + sab) * nw + (ok ? w0 + ww : 0), ok);
        }
        short *md = mst + buf * FT_SCH * FT_TILE;
        for (int e = tid; e < ns * FT_TILE / 8; e += FT_THREADS) ft_cp16(md + 8 * e, smg + (int64_t)s0 * FT_TILE + 8 * e, true);
    };
    for (int k0 = 0; k0 < u; k0 += FT_CH) {
        const int nk = min(FT_CH, u - k0);
        __syncthreads(); // previous chunk's readers are done with the buffers
        for (int e = tid; e < nk * KS * FT_WB; e += FT_THREADS) {
            const int k = e / (KS * FT_WB), cw = e % (KS * FT_WB), c = cw / FT_WB, ww = cw % FT_WB;
            const int src = tile_srcs[(int64_t)tile * FT_MAXU + k0 + k];
            const bool ok = w0 + ww < nw;
            ft_cp16(stage + k * SST + cw, phat + ((int64_t)src * KS + c) * nw + (ok ? w0 + ww : 0), ok);
        }
        load_chunk(0, 0);
        ft_commit();
        for (int c = 0; c < NSC; c++) {
            if (c + 1 < NSC) load_chunk(c + 1, (c + 1) & 1);
            ft_commit();
            ft_wait<1>(); // chunk c (and the sources) landed
            __syncthreads();
            const int ns = min(FT_SCH, kSlots - c * FT_SCH);
            const double2 *kb = kst + (c & 1) * KCH + wl;
            const short *mb = mst + (c & 1) * FT_SCH * FT_TILE + t;
            // two slots per step into two accumulator sets: twice the independent DFMA chains
            // (the dependent chain per set is 2 KS DFMAs long; "wait" stalls dominated with one set)
            for (int s = 0; s < ns; s += 2) {
                const int li0 = (int)mb[s * FT_TILE] - k0;
                const int li1 = s + 1 < ns ? (int)mb[(s + 1) * FT_TILE] - k0 : -1;
                const bool on0 = li0 >= 0 && li0 < nk, on1 = li1 >= 0 && li1 < nk;
                if (on0) {
                    const double2 *st = stage + (int64_t)li0 * SST + wl;
                    const double2 *kk = kb + (int64_t)s * KT * KS * FT_WB;
#pragma unroll
                    for (int b = 0; b < KS; b++) {
                        const double2 p = st[b * FT_WB];
#pragma unroll
                        for (int a = 0; a < KT; a++) {
                            const double2 k = kk[(a * KS + b) * FT_WB]; // same address across the warp
                            acc[a].x = fma(k.x, p.x, fma(-k.y, p.y, acc[a].x));
                            acc[a].y = fma(k.x, p.y, fma(k.y, p.x, acc[a].y));
                        }
                    }
                }
                if (on1) {
                    const double2 *st = stage + (int64_t)li1 * SST + wl;
                    const double2 *kk = kb + (int64_t)(s + 1) * KT * KS * FT_WB;
#pragma unroll
                    for (int b = 0; b < KS; b++) {
                        const double2 p = st[b * FT_WB];
#pragma unroll
                        for (int a = 0; a < KT; a++) {
                            const double2 k = kk[(a * KS + b) * FT_WB];
                            acc2[a].x = fma(k.x, p.x, fma(-k.y, p.y, acc2[a].x));
                            acc2[a].y = fma(k.x, p.y, fma(k.y, p.x, acc2[a].y));
                        }
                    }
                }
            }
            __syncthreads(); // chunk c's buffers are refilled two chunks later
        }
    }
    if (w >= nw) return;
    const int col = tile * FT_TILE + t;
#pragma unroll
    for (int a = 0; a < KT; a++)
        qhat[((int64_t)col * KT + a) * nw + w] = make_double2(acc[a].x + acc2[a].x, acc[a].y + acc2[a].y);
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

template <class F> void set_smem_once(F *kernel, size_t bytes) {
    static std::mutex mtx;
    static std::map<std::pair<const void *, int>, size_t> done;
    int dev = 0;
    PK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mtx);
    size_t &d = done[{reinterpret_cast<const void *>(kernel), dev}];
    if (d >= bytes) return;
    PK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    d = bytes;
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


namespace {

constexpr int LAT_E = 14; // stored offset classes e = c - o with code (ex+1) 9 + (ey+1) 3 + (ez+1) >= 13

__host__ __device__ inline int sym_index(int a, int b, int ks) { // (a, b) -> packed upper triangle
    if (a > b) {
        const int t = a;
        a = b;
        b = t;
    }
    return ks == 1 ? 0 : (a == 0 ? b : (a == 1 ? 2 + b : 5));
}

// M[kappa][e'][comp][w] = sum_{D, |2D + e| >= 2} K^_{2D+e}[a][b][w] exp(+2 pi i kappa.D / m)
__global__ void lat_build_kernel(const double2 *__restrict__ khat, const int *__restrict__ slot_of_code, int ks,
                                 int nw, int mx, int my, int mz, double2 *__restrict__ M) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int nc = ks * (ks + 1) / 2;
    const int ec = blockIdx.y / nc, comp = blockIdx.y % nc;
    const int64_t kap = blockIdx.z;
    if (w >= nw) return;
    int a = 0, b = 0;
    if (ks == 3) {
        const int A[6] = {0, 0, 0, 1, 1, 2}, B[6] = {0, 1, 2, 1, 2, 2};
        a = A[comp];
        b = B[comp];
    }
    const int code = 13 + ec;
    const int ex = code / 9 - 1, ey = (code / 3) % 3 - 1, ez = code % 3 - 1;
    const int kx = (int)(kap / ((int64_t)my * mz)), ky = (int)((kap / mz) % my), kz = (int)(kap % mz);
    double re = 0.0, im = 0.0;
    for (int Dx = -1; Dx <= 1; Dx++)
        for (int Dy = -1; Dy <= 1; Dy++)
            for (int Dz = -1; Dz <= 1; Dz++) {
                const int dx = 2 * Dx + ex, dy = 2 * Dy + ey, dz = 2 * Dz + ez;
                if (max(abs(dx), max(abs(dy), abs(dz))) < 2) continue; // adjacent: U / W / X lists
                const int slot = slot_of_code[(dx + 3) * 49 + (dy + 3) * 7 + (dz + 3)];
                const double2 k = khat[((int64_t)(slot * ks + a) * ks + b) * nw + w];
                // exp(+2 pi i (kx Dx / mx + ky Dy / my + kz Dz / mz)), exact for the period
                const double ph = (double)kx * Dx / mx + (double)ky * Dy / my + (double)kz * Dz / mz;
                double s, c;
                sincospi(2.0 * ph, &s, &c);
                re += k.x * c - k.y * s;
                im += k.x * s + k.y * c;
            }
    M[((kap * LAT_E + ec) * nc + comp) * nw + w] = make_double2(re, im);
}

// box of each (parent-lattice point u, octant c); -1 for absent boxes and padding
__global__ void lat_boxmap_kernel(const int4 *__restrict__ cell, int64_t box0, int64_t nl, int my, int mz,
                                  int *__restrict__ box_of) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nl) return;
    const int4 c = cell[box0 + k];
    const int64_t u = ((int64_t)(c.x >> 1) * my + (c.y >> 1)) * mz + (c.z >> 1);
    box_of[u * 8 + ((c.x & 1) | (c.y & 1) << 1 | (c.z & 1) << 2)] = (int)(box0 + k);
}

// the dense layout's V-list entries against the lattice stencil: bad += mismatches, plus
// level boxes that are not output columns
__global__ void lat_check_kernel(const int *__restrict__ table, int64_t ld, const int *__restrict__ out_box, int ncols,
                                 const int *__restrict__ code_of_slot, const int4 *__restrict__ cell,
                                 const int *__restrict__ box_of, int n, int px, int py, int pz, int my, int mz,
                                 int64_t box0, int64_t nl, const int2 *__restrict__ srng,
                                 const int2 *__restrict__ trng, const int *__restrict__ mask,
                                 int *__restrict__ seen, int *bad, int *dbg) {
    const int64_t total = (int64_t)kNumM2L * ncols;
    int nbad = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(t / ncols), col = (int)(t % ncols);
        const int tb = out_box[col];
        const int got = table[(int64_t)s * ld + col];
        if (tb < 0) {
            nbad += got >= 0;
            continue;
        }
        if (tb < box0 || tb >= box0 + nl) { // not a box of this level
            nbad++;
            continue;
        }
        if (s == 0) seen[tb - box0] = 1;
        const int code = code_of_slot[s];
        const int4 c = cell[tb];
        const int dx = code / 49 - 3, dy = (code / 7) % 7 - 3, dz = code % 7 - 3;
        int x = c.x + dx, y = c.y + dy, z = c.z + dz;
        int want = -1;
        // the octant's stencil: the parents adjacent, d + o in [-2, 3] per axis
        bool in = dx + (c.x & 1) >= -2 && dx + (c.x & 1) <= 3 && dy + (c.y & 1) >= -2 && dy + (c.y & 1) <= 3 &&
                  dz + (c.z & 1) >= -2 && dz + (c.z & 1) <= 3;
        if (px) x = ((x % n) + n) % n; else in &= x >= 0 && x < n;
        if (py) y = ((y % n) + n) % n; else in &= y >= 0 && y < n;
        if (pz) z = ((z % n) + n) % n; else in &= z >= 0 && z < n;
        if (in) want = box_of[(((int64_t)(x >> 1) * my + (y >> 1)) * mz + (z >> 1)) * 8 + ((x & 1) | (y & 1) << 1 | (z & 1) << 2)];
        // the evaluate lists omit sources without source points (zero densities on the lattice)
        // and give boxes without target points no list at all (their results are never read)
        const bool omitted = got < 0 && ((want >= 0 && srng && srng[want].y <= srng[want].x) ||
                                         (trng && trng[tb].y <= trng[tb].x) || (mask && !mask[tb]));
        if (want != got && !omitted) {
            nbad++;
            if (dbg) {
                const int k = atomicAdd(dbg, 1);
                if (k < 8) {
                    dbg[1 + 4 * k] = s;
                    dbg[2 + 4 * k] = tb;
                    dbg[3 + 4 * k] = want;
                    dbg[4 + 4 * k] = got;
                }
            }
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}
__global__ void lat_seen_kernel(const int *__restrict__ seen, int64_t nl, int *bad) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < nl && !seen[k]) atomicAdd(bad, 1);
}

// Q~[kappa][o][a][w] = sum_c sum_b M_{c-o}[a][b](kappa, w) Psi~[kappa][c][b][w]; a thread per
// (kappa, w), the 8 octants' spectra in shared memory, the 8 outputs in registers; each
// offset class e is loaded once and applied to every (o, c) pair with c - o = e
template <int KS>
__global__ void __launch_bounds__(128) lat_mul_kernel(const double2 *__restrict__ M, const double2 *__restrict__ Psi,
                                                      double2 *__restrict__ Q, int nw, int64_t total) {
    constexpr int NC = KS * (KS + 1) / 2;
    __shared__ double2 ps[8 * KS][128];
    // flat (kappa, w) index: nw = N N (N / 2 + 1) is odd-sized, so a block may span two kappa
    const int64_t t = blockIdx.x * (int64_t)128 + threadIdx.x;
    const bool on = t < total;
    const int64_t kap = on ? t / nw : 0;
    const int w = on ? (int)(t % nw) : 0;
    const int64_t base = kap * 8 * KS * nw;
#pragma unroll
    for (int j = 0; j < 8 * KS; j++) ps[j][threadIdx.x] = on ? Psi[base + (int64_t)j * nw + w] : make_double2(0.0, 0.0);
    double2 acc[8][KS];
#pragma unroll
    for (int o = 0; o < 8; o++)
#pragma unroll
        for (int a = 0; a < KS; a++) acc[o][a] = make_double2(0.0, 0.0);
    // one offset class e (code) with its spectra m (conjugated for -e)
    auto apply = [&](int code, const double2 (&m)[NC], bool cj) {
        const int ex = code / 9 - 1, ey = (code / 3) % 3 - 1, ez = code % 3 - 1;
        const double sg = cj ? -1.0 : 1.0;
#pragma unroll
        for (int o = 0; o < 8; o++) {
            const int cx = (o & 1) + ex, cy = ((o >> 1) & 1) + ey, cz = ((o >> 2) & 1) + ez;
            if (cx < 0 || cx > 1 || cy < 0 || cy > 1 || cz < 0 || cz > 1) continue;
            const int c = cx | cy << 1 | cz << 2;
#pragma unroll
            for (int b = 0; b < KS; b++) {
                const double2 p = ps[c * KS + b][threadIdx.x];
#pragma unroll
                for (int a = 0; a < KS; a++) {
                    const double2 k = m[sym_index(a, b, KS)];
                    const double ky = sg * k.y;
                    acc[o][a].x = fma(k.x, p.x, fma(-ky, p.y, acc[o][a].x));
                    acc[o][a].y = fma(k.x, p.y, fma(ky, p.x, acc[o][a].y));
                }
            }
        }
    };
    if (on) {
        // each stored class serves e and -e (M_{-e} = conj(M_e)): one load per class
        // (fully unrolled: the octant pairs of each class resolve at compile time, and the
        // next class's spectra are in flight while this one is applied)
        double2 m[NC], mn[NC];
#pragma unroll
        for (int k = 0; k < NC; k++) m[k] = M[(kap * LAT_E * NC + k) * nw + w];
#pragma unroll
        for (int ec = 0; ec < LAT_E; ec++) {
            if (ec + 1 < LAT_E) {
#pragma unroll
                for (int k = 0; k < NC; k++) mn[k] = M[((kap * LAT_E + ec + 1) * NC + k) * nw + w];
            }
            apply(13 + ec, m, false);
            if (ec) apply(13 - ec, m, true);
#pragma unroll
            for (int k = 0; k < NC; k++) m[k] = mn[k];
        }
    }
    if (!on) return;
#pragma unroll
    for (int o = 0; o < 8; o++)
#pragma unroll
        for (int a = 0; a < KS; a++) Q[base + (int64_t)(o * KS + a) * nw + w] = acc[o][a];
}

// In-register radix-2 FFT of M points (M a power of two <= 32), sign -1 forward / +1 inverse
__host__ __device__ constexpr int bit_reverse(int i, int M) {
    int r = 0;
    for (int b = 1; b < M; b <<= 1) r = (r << 1) | ((i & b) ? 1 : 0);
    return r;
}
template <int M> __device__ __forceinline__ void reg_fft(double2 (&v)[M], double sign) {
#pragma unroll
    for (int i = 0; i < M; i++) { // bit reversal (compile-time indices)
        const int j = bit_reverse(i, M);
        if (i < j) {
            const double2 t = v[i];
            v[i] = v[j];
            v[j] = t;
        }
    }
#pragma unroll
    for (int len = 2; len <= M; len <<= 1) {
#pragma unroll
        for (int k = 0; k < len / 2; k++) {
            double s, c;
            sincospi(sign * 2.0 * k / len, &s, &c);
#pragma unroll
            for (int i = 0; i < M; i += len) {
                const double2 a = v[i + k], b = v[i + k + len / 2];
                const double2 t = make_double2(b.x * c - b.y * s, b.x * s + b.y * c);
                v[i + k] = make_double2(a.x + t.x, a.y + t.y);
                v[i + k + len / 2] = make_double2(a.x - t.x, a.y - t.y);
            }
        }
    }
}

// One axis of the 3D lattice transform, in place: X[u][j] (j fastest, S columns); a thread
// per (column j, line along the axis), M points per line at u stride `ustride`
template <int M>
__global__ void __launch_bounds__(128) lat_fft_axis_kernel(double2 *__restrict__ X, int64_t S, int64_t nlines,
                                                           int64_t ustride, int64_t inner, double sign) {
    const int64_t j = blockIdx.x * 128 + threadIdx.x;
    const int64_t line = blockIdx.y;
    if (j >= S) return;
    // line -> base u: lines enumerate (outer, inner) around the axis
    const int64_t u0 = (line / inner) * (inner * M) + (line % inner);
    double2 v[M];
#pragma unroll
    for (int i = 0; i < M; i++) v[i] = X[(u0 + i * ustride) * S + j];
    reg_fft<M>(v, sign);
#pragma unroll
    for (int i = 0; i < M; i++) X[(u0 + i * ustride) * S + j] = v[i];
    (void)nlines;
}

// the whole 3D transform of small lattices (M3 <= 512) in shared memory: a CTA per block of
// JB consecutive columns, one read and one write of the data
template <int MX, int MY, int MZ, int JB>
__global__ void __launch_bounds__(256) lat_fft_smem_kernel(double2 *__restrict__ X, int64_t S, double sign) {
    constexpr int M3 = MX * MY * MZ;
    extern __shared__ double2 lat_sm[]; // [M3][JB]
    const int64_t j0 = (int64_t)blockIdx.x * JB;
    const int tid = threadIdx.x;
    for (int e = tid; e < M3 * JB; e += 256) {
        const int u = e / JB, jj = e % JB;
        lat_sm[e] = j0 + jj < S ? X[(int64_t)u * S + j0 + jj] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    auto pass = [&](auto mc, int stride, int inner) {
        constexpr int M = decltype(mc)::value;
        constexpr int L = M3 / M; // lines per column
        for (int e = tid; e < L * JB; e += 256) {
            const int line = e / JB, jj = e % JB;
            const int u0 = (line / inner) * (inner * M) + (line % inner);
            double2 v[M];
#pragma unroll
            for (int i = 0; i < M; i++) v[i] = lat_sm[(u0 + i * stride) * JB + jj];
            reg_fft<M>(v, sign);
#pragma unroll
            for (int i = 0; i < M; i++) lat_sm[(u0 + i * stride) * JB + jj] = v[i];
        }
        __syncthreads();
    };
    if (MZ > 1) pass(std::integral_constant<int, MZ>{}, 1, 1);
    if (MY > 1) pass(std::integral_constant<int, MY>{}, MZ, MZ);
    if (MX > 1) pass(std::integral_constant<int, MX>{}, MY * MZ, MY * MZ);
    for (int e = tid; e < M3 * JB; e += 256) {
        const int u = e / JB, jj = e % JB;
        if (j0 + jj < S) X[(int64_t)u * S + j0 + jj] = lat_sm[e];
    }
}

template <int MX, int MY, int MZ> void lat_fft_smem(double2 *X, int64_t S, double sign, cudaStream_t st) {
    constexpr int JB = 16;
    constexpr size_t smem = (size_t)MX * MY * MZ * JB * sizeof(double2);
    auto k = lat_fft_smem_kernel<MX, MY, MZ, JB>;
    set_smem_once(k, smem);
    k<<<(unsigned)((S + JB - 1) / JB), 256, smem, st>>>(X, S, sign);
}

template <int M> void lat_fft_axis(double2 *X, int64_t S, int64_t M3, int64_t ustride, double sign, cudaStream_t st) {
    const int64_t nlines = M3 / M;
    lat_fft_axis_kernel<M><<<dim3((unsigned)((S + 127) / 128), (unsigned)nlines), 128, 0, st>>>(X, S, nlines, ustride,
                                                                                                  ustride, sign);
}

// 3D transform over the lattice (mx, my, mz) of every column: in place, unnormalised
int lat_fft(double2 *X, int64_t S, const int m[3], double sign, cudaStream_t st) {
    const int64_t M3 = (int64_t)m[0] * m[1] * m[2];
    if (M3 == 1) return 0;
#define LAT_SMEM(a, b, c)                                                                                              \
    if (m[0] == a && m[1] == b && m[2] == c) {                                                                         \
        lat_fft_smem<a, b, c>(X, S, sign, st);                                                                         \
        return 1;                                                                                                      \
    }
    LAT_SMEM(2, 2, 2) LAT_SMEM(4, 4, 4) LAT_SMEM(8, 8, 8)
    LAT_SMEM(2, 2, 1) LAT_SMEM(2, 1, 2) LAT_SMEM(1, 2, 2) LAT_SMEM(2, 1, 1) LAT_SMEM(1, 2, 1) LAT_SMEM(1, 1, 2)
    LAT_SMEM(4, 4, 8) LAT_SMEM(4, 8, 4) LAT_SMEM(8, 4, 4) LAT_SMEM(2, 2, 4) LAT_SMEM(2, 4, 2) LAT_SMEM(4, 2, 2)
#undef LAT_SMEM
    int launches = 0;
    const int64_t inner[3] = {(int64_t)m[1] * m[2], m[2], 1};
    for (int ax = 2; ax >= 0; ax--) {
        const int64_t stride = inner[ax];
        switch (m[ax]) {
        case 1: break;
        case 2: lat_fft_axis<2>(X, S, M3, stride, sign, st), launches++; break;
        case 4: lat_fft_axis<4>(X, S, M3, stride, sign, st), launches++; break;
        case 8: lat_fft_axis<8>(X, S, M3, stride, sign, st), launches++; break;
        case 16: lat_fft_axis<16>(X, S, M3, stride, sign, st), launches++; break;
        case 32: lat_fft_axis<32>(X, S, M3, stride, sign, st), launches++; break;
        default: throw RuntimeError("lattice M2L: lattice edge " + std::to_string(m[ax]) + " unsupported");
        }
    }
    return launches;
}

// ---- surface transforms of the lattice path -------------------------------------------
// The lattice and surface transforms commute, so the lattice FFT runs on the raw surface
// values (n per box and component, 8x less data than spectra) and the surface transforms
// run per lattice frequency kappa on complex data. A density lives on the p^3 corner of
// its N^3 grid (N = fft_edge(p)), only at the surface points, and the check potentials are needed
// only there: each surface transform is three direct DFT stages over the nonzero / needed
// index ranges (sums of p terms), one CTA per (kappa, octant, component), with cuFFT's D2Z
// half-spectrum layout and sign ([kx][ky][kz], kz <= N/2, exp(-2 pi i k.g / N)).
constexpr int LS_THREADS = 256;

// A[u][(c ks + b) n + i] = phi of box (u, c), component b, surface point i (0: absent box)
__global__ void lat_gather_surface_kernel(const double *__restrict__ X, int64_t Kp, const int *__restrict__ box_of,
                                          int64_t M3, int ks, int n, double2 *__restrict__ A) {
    const int64_t S = (int64_t)8 * ks * n, total = M3 * S;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = t / S;
        const int j = (int)(t % S), c = j / (ks * n), r = j % (ks * n), b = r / n, i = r % n;
        const int box = box_of[u * 8 + c];
        A[t] = make_double2(box >= 0 ? X[(int64_t)box * Kp + ks * i + b] : 0.0, 0.0);
    }
}

// Y[box (u, o)][kt i + a] += scale * Re A[u][(o kt + a) n + i]
__global__ void lat_scatter_surface_kernel(const double2 *__restrict__ A, const int *__restrict__ box_of, int64_t M3,
                                           int kt, int n, double scale, int64_t Kp, double *__restrict__ Y) {
    const int64_t S = (int64_t)8 * kt * n, total = M3 * S;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = t / S;
        const int j = (int)(t % S), o = j / (kt * n), r = j % (kt * n), a = r / n, i = r % n;
        const int box = box_of[u * 8 + o];
        if (box >= 0) Y[(int64_t)box * Kp + kt * i + a] += scale * A[t].x;
    }
}

// Psi[g][w] = surface DFT of the n complex values A[g][i], g = (kappa 8 + c) ks + b
__global__ void __launch_bounds__(LS_THREADS) lat_surface_fwd_kernel(const double2 *__restrict__ A, int p, int n,
                                                                     const int *__restrict__ gidx,
                                                                     double2 *__restrict__ Psi) {
    extern __shared__ double2 ls_sm[];
    const int N = fft_edge(p), NH = N / 2 + 1, nw = N * N * NH;
    double2 *tw = ls_sm;                 // [N] exp(-2 pi i k / N)
    double2 *cube = tw + N;              // [x][y][z] (p^3)
    double2 *f1 = cube + p * p * p;      // [x][y][kz]  (p p NH)
    double2 *f2 = f1 + p * p * NH;       // [x][ky][kz] (p N NH)
    const int64_t g = blockIdx.x;
    const double2 *in = A + g * n;
    double2 *out = Psi + g * nw;
    const int tid = threadIdx.x;
    for (int k = tid; k < N; k += LS_THREADS) {
        double s, c;
        sincospi(-2.0 * k / N, &s, &c);
        tw[k] = make_double2(c, s);
    }
    for (int e = tid; e < p * p * p; e += LS_THREADS) cube[e] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int i = tid; i < n; i += LS_THREADS) {
        const int gi = gidx[i], x = gi / (N * N), y = (gi / N) % N, z = gi % N;
        cube[(x * p + y) * p + z] = in[i];
    }
    __syncthreads();
    // z: p -> kz <= N/2 (the half spectrum; the rest is the conjugate at -kappa)
    for (int e = tid; e < p * p * NH; e += LS_THREADS) {
        const int xy = e / NH, kz = e % NH;
        const double2 *line = cube + xy * p;
        double re = 0.0, im = 0.0;
        for (int z = 0; z < p; z++) {
            const double2 a = line[z], t = tw[(kz * z) % N];
            re = fma(a.x, t.x, fma(-a.y, t.y, re));
            im = fma(a.x, t.y, fma(a.y, t.x, im));
        }
        f1[e] = make_double2(re, im);
    }
    __syncthreads();
    // y: p -> N
    for (int e = tid; e < p * N * NH; e += LS_THREADS) {
        const int x = e / (N * NH), ky = (e / NH) % N, kz = e % NH;
        double re = 0.0, im = 0.0;
        for (int y = 0; y < p; y++) {
            const double2 a = f1[(x * p + y) * NH + kz], t = tw[(ky * y) % N];
            re = fma(a.x, t.x, fma(-a.y, t.y, re));
            im = fma(a.x, t.y, fma(a.y, t.x, im));
        }
        f2[e] = make_double2(re, im);
    }
    __syncthreads();
    // x: p -> N, straight to the spectrum
    for (int w = tid; w < nw; w += LS_THREADS) {
        const int kx = w / (N * NH), r = w % (N * NH);
        double re = 0.0, im = 0.0;
        for (int x = 0; x < p; x++) {
            const double2 a = f2[x * N * NH + r], t = tw[(kx * x) % N];
            re = fma(a.x, t.x, fma(-a.y, t.y, re));
            im = fma(a.x, t.y, fma(a.y, t.x, im));
        }
        out[w] = make_double2(re, im);
    }
}

// A[g][i] = inverse surface DFT at the surface points of the full spectrum of lattice
// frequency kappa, g = (kappa 8 + o) kt + a. Only kz <= N/2 is stored: the other half is
// conj(Q(-kappa, -w)), so a CTA takes the pair (kappa, -kappa) and writes both.
__global__ void __launch_bounds__(LS_THREADS) lat_surface_inv_kernel(const double2 *__restrict__ Q,
                                                                     const int64_t *__restrict__ pairs, int kt, int p,
                                                                     int n, const int *__restrict__ gidx,
                                                                     double2 *__restrict__ A) {
    extern __shared__ double2 ls_sm[];
    const int N = fft_edge(p), NH = N / 2 + 1, nw = N * N * NH;
    double2 *tw = ls_sm;                 // [N] exp(+2 pi i k / N)
    double2 *b1 = tw + N;                // 2 x [x][ky][kz] (p N NH)
    double2 *b2 = b1 + 2 * p * N * NH;   // 2 x [x][y][kz]  (p p NH)
    const int64_t pr = pairs[blockIdx.x / (8 * kt)];
    const int oa = blockIdx.x % (8 * kt);
    const int64_t kap[2] = {pr & 0xffffffffLL, pr >> 32};
    const int tid = threadIdx.x;
    for (int k = tid; k < N; k += LS_THREADS) {
        double s, c;
        sincospi(2.0 * k / N, &s, &c);
        tw[k] = make_double2(c, s);
    }
    __syncthreads();
    const int nh = kap[0] == kap[1] ? 1 : 2;
    // x: N -> p, then y: N -> p, for kappa and -kappa
    for (int e = tid; e < nh * p * N * NH; e += LS_THREADS) {
        const int h = e / (p * N * NH), r0 = e % (p * N * NH), x = r0 / (N * NH), r = r0 % (N * NH);
        const double2 *in = Q + (kap[h] * 8 * kt + oa) * nw;
        double re = 0.0, im = 0.0;
        for (int kx = 0; kx < N; kx++) {
            const double2 q = in[kx * N * NH + r], t = tw[(kx * x) % N];
            re = fma(q.x, t.x, fma(-q.y, t.y, re));
            im = fma(q.x, t.y, fma(q.y, t.x, im));
        }
        b1[e] = make_double2(re, im);
    }
    __syncthreads();
    for (int e = tid; e < nh * p * p * NH; e += LS_THREADS) {
        const int h = e / (p * p * NH), r0 = e % (p * p * NH), x = r0 / (p * NH), y = (r0 / NH) % p, kz = r0 % NH;
        const double2 *src = b1 + h * p * N * NH;
        double re = 0.0, im = 0.0;
        for (int ky = 0; ky < N; ky++) {
            const double2 q = src[(x * N + ky) * NH + kz], t = tw[(ky * y) % N];
            re = fma(q.x, t.x, fma(-q.y, t.y, re));
            im = fma(q.x, t.y, fma(q.y, t.x, im));
        }
        b2[e] = make_double2(re, im);
    }
    __syncthreads();
    // z: the full line of kappa is B(kappa, kz) for kz <= N/2 and conj(B(-kappa, N - kz)) above
    for (int e = tid; e < nh * n; e += LS_THREADS) {
        const int h = e / n, i = e % n;
        const int gi = gidx[i], x = gi / (N * N), y = (gi / N) % N, z = gi % N;
        const double2 *own = b2 + h * p * p * NH + (x * p + y) * NH;
        const double2 *oth = b2 + (nh == 2 ? 1 - h : 0) * p * p * NH + (x * p + y) * NH;
        double re = 0.0, im = 0.0;
        for (int kz = 0; kz < NH; kz++) {
            const double2 q = own[kz], t = tw[(kz * z) % N];
            re = fma(q.x, t.x, fma(-q.y, t.y, re));
            im = fma(q.x, t.y, fma(q.y, t.x, im));
        }
        for (int kz = NH; kz < N; kz++) {
            const double2 q = oth[N - kz], t = tw[(kz * z) % N]; // conj(q) * t
            re = fma(q.x, t.x, fma(q.y, t.y, re));
            im = fma(q.x, t.y, fma(-q.y, t.x, im));
        }
        A[(kap[h] * 8 * kt + oa) * n + i] = make_double2(re, im);
    }
}

// The same two transforms with p a compile-time constant: every twiddle index is a
// constant, each thread keeps one input column in registers and produces all its outputs
// (no per-term index arithmetic, one shared-memory read per input).
// exp(-2 pi i k / N), N = fft_edge(P), per compile-time P: with constant indices the twiddles
// are constant-bank operands of the DFMAs themselves (no shared-memory load per term)
constexpr int kLatTwMaxP = 10, kLatTwMaxN = 32;
__constant__ double2 c_lat_tw[kLatTwMaxP + 1][kLatTwMaxN];
template <int P, int SIGN> __device__ __forceinline__ double2 ctw(int k) {
    const double2 t = c_lat_tw[P][k];
    return SIGN < 0 ? t : make_double2(t.x, -t.y);
}
__device__ __forceinline__ void cmac(double2 &acc, double2 a, double2 t) {
    acc.x = fma(a.x, t.x, fma(-a.y, t.y, acc.x));
    acc.y = fma(a.x, t.y, fma(a.y, t.x, acc.y));
}

// Two groups g (lattice frequency, octant, component) per CTA, side by side: stages 1 and 2
// have P^2 and P NH columns per group -- 64 each at p = 8, half of a 128-thread CTA, always
// the same two warps (the same two of the SM's four schedulers) -- so the second group takes
// the other half; stage 3 runs both groups' columns over all threads.
template <int P>
__global__ void __launch_bounds__(256) lat_surface_fwd_t(const double2 *__restrict__ A, int n,
                                                         const int *__restrict__ gidx, double2 *__restrict__ Psi,
                                                         int64_t ngroups) {
    constexpr int N = fft_edge(P), NH = N / 2 + 1, NW = N * N * NH;
    constexpr int NS = P * P * P - (P - 2) * (P - 2) * (P - 2); // surface points (= n: constant divisors)
    // rows of 8 complex values are 128 bytes: threads that walk one row each would all start in
    // the same bank (8-way conflicts on every access), so those rows get one element of padding
    constexpr int PZ = P + 1, NHP = NH + 1;
    constexpr int CUBE = P * P * PZ, F1 = P * P * NHP, F2 = P * N * NH;
    constexpr int RA = CUBE > F2 ? CUBE : F2; // the cube is dead when stage 2 writes f2: one region for both
    extern __shared__ double2 lt_sm[];
    double2 *cube = lt_sm;           // 2 x [x][y][z (padded)], stride RA
    double2 *f2 = lt_sm;             // 2 x [x][ky][kz], stride RA (over the cube)
    double2 *f1 = lt_sm + 2 * RA;    // 2 x [x][y][kz (padded)]
    const int64_t g0 = 2 * (int64_t)blockIdx.x;
    const int ng = g0 + 1 < ngroups ? 2 : 1;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < 2 * RA; e += nt) cube[e] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int e = tid; e < ng * NS; e += nt) {
        const int h = e / NS, i = e % NS;
        const int gi = gidx[i], x = gi / (N * N), y = (gi / N) % N, z = gi % N;
        cube[h * RA + (x * P + y) * PZ + z] = A[(g0 + h) * NS + i];
    }
    __syncthreads();
    const int half = nt / 2; // threads per group in stages 1 and 2
    {
        const int h = tid / half, t = tid % half;
        if (h < ng) {
            const double2 *cb = cube + h * RA;
            double2 *o1 = f1 + h * F1;
            for (int xy = t; xy < P * P; xy += half) { // z: P -> NH
                double2 v[P];
#pragma unroll
                for (int z = 0; z < P; z++) v[z] = cb[xy * PZ + z];
#pragma unroll
                for (int kz = 0; kz < NH; kz++) {
                    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int z = 0; z < P; z++) cmac(acc, v[z], ctw<P, -1>((kz * z) % N));
                    o1[xy * NHP + kz] = acc;
                }
            }
        }
    }
    __syncthreads();
    {
        const int h = tid / half, t = tid % half;
        if (h < ng) {
            const double2 *i1 = f1 + h * F1;
            double2 *o2 = f2 + h * RA;
            for (int col = t; col < P * NH; col += half) { // y: P -> N, column (x, kz)
                const int x = col / NH, kz = col % NH;
                double2 v[P];
#pragma unroll
                for (int y = 0; y < P; y++) v[y] = i1[(x * P + y) * NHP + kz];
#pragma unroll
                for (int ky = 0; ky < N; ky++) {
                    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int y = 0; y < P; y++) cmac(acc, v[y], ctw<P, -1>((ky * y) % N));
                    o2[(x * N + ky) * NH + kz] = acc;
                }
            }
        }
    }
    __syncthreads();
    for (int e = tid; e < ng * N * NH; e += nt) { // x: P -> N, column (h, ky, kz), straight out
        const int h = e / (N * NH), r = e % (N * NH);
        const double2 *i2 = f2 + h * RA;
        double2 *out = Psi + (g0 + h) * NW;
        double2 v[P];
#pragma unroll
        for (int x = 0; x < P; x++) v[x] = i2[x * N * NH + r];
#pragma unroll
        for (int kx = 0; kx < N; kx++) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int x = 0; x < P; x++) cmac(acc, v[x], ctw<P, -1>((kx * x) % N));
            out[kx * N * NH + r] = acc;
        }
    }
}

template <int P>
__global__ void __launch_bounds__(256) lat_surface_inv_t(const double2 *__restrict__ Q, const int64_t *__restrict__ pairs,
                                                         int kt, int n, const int *__restrict__ gidx,
                                                         double2 *__restrict__ A) {
    constexpr int N = fft_edge(P), NH = N / 2 + 1, NW = N * N * NH;
    extern __shared__ double2 lt_sm[];
    double2 *tw = lt_sm;                             // [N]
    constexpr int NHP = NH + 1;                  // padded row of b2 (see lat_surface_fwd_t)
    double2 *const b1 = tw + N;                  // 2 x [x][ky][kz] (per half)
    double2 *const b2 = b1 + 2 * P * N * NH;     // 2 x [x][y][kz (padded)]
    const int64_t pr = pairs[blockIdx.x / (8 * kt)];
    const int oa = blockIdx.x % (8 * kt);
    const int64_t kap[2] = {pr & 0xffffffffLL, pr >> 32};
    const int nh = kap[0] == kap[1] ? 1 : 2;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int k = tid; k < N; k += nt) {
        double s, c;
        sincospi(2.0 * k / N, &s, &c);
        tw[k] = make_double2(c, s);
    }
    __syncthreads();
    for (int e = tid; e < nh * N * NH; e += nt) { // x: N -> P, column (h, ky, kz)
        const int h = e / (N * NH), r = e % (N * NH);
        const double2 *in = Q + (kap[h] * 8 * kt + oa) * NW + r;
        double2 v[N];
#pragma unroll
        for (int kx = 0; kx < N; kx++) v[kx] = in[kx * N * NH];
#pragma unroll
        for (int x = 0; x < P; x++) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int kx = 0; kx < N; kx++) cmac(acc, v[kx], ctw<P, 1>((kx * x) % N));
            b1[h * P * N * NH + x * N * NH + r] = acc;
        }
    }
    __syncthreads();
    for (int e = tid; e < nh * P * NH; e += nt) { // y: N -> P, column (h, x, kz)
        const int h = e / (P * NH), x = (e / NH) % P, kz = e % NH;
        double2 v[N];
#pragma unroll
        for (int ky = 0; ky < N; ky++) v[ky] = b1[h * P * N * NH + (x * N + ky) * NH + kz];
#pragma unroll
        for (int y = 0; y < P; y++) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int ky = 0; ky < N; ky++) cmac(acc, v[ky], ctw<P, 1>((ky * y) % N));
            b2[h * P * P * NHP + (x * P + y) * NHP + kz] = acc;
        }
    }
    __syncthreads();
    constexpr int NS = P * P * P - (P - 2) * (P - 2) * (P - 2); // surface points (= n: constant divisors)
    for (int e = tid; e < nh * NS; e += nt) { // z at the surface points
        const int h = e / NS, i = e % NS;
        const int gi = gidx[i], x = gi / (N * N), y = (gi / N) % N, z = gi % N;
        const double2 *own = b2 + h * P * P * NHP + (x * P + y) * NHP;
        const double2 *oth = b2 + (nh == 2 ? 1 - h : 0) * P * P * NHP + (x * P + y) * NHP;
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int kz = 0; kz < NH; kz++) cmac(acc, own[kz], tw[(kz * z) % N]);
#pragma unroll
        for (int kz = NH; kz < N; kz++) {
            const double2 q = oth[N - kz];
            cmac(acc, make_double2(q.x, -q.y), tw[(kz * z) % N]);
        }
        A[(kap[h] * 8 * kt + oa) * NS + i] = acc;
    }
}

// the lattice frequencies as (kappa, -kappa) pairs, each pair once (self-conjugate: kappa twice)
std::vector<int64_t> conjugate_pairs(const int m[3]) {
    std::vector<int64_t> out;
    const int64_t M3 = (int64_t)m[0] * m[1] * m[2];
    for (int64_t k = 0; k < M3; k++) {
        const int kx = (int)(k / ((int64_t)m[1] * m[2])), ky = (int)((k / m[2]) % m[1]), kz = (int)(k % m[2]);
        const int64_t c = ((int64_t)((m[0] - kx) % m[0]) * m[1] + (m[1] - ky) % m[1]) * m[2] + (m[2] - kz) % m[2];
        if (c < k) continue;
        out.push_back(k | (c << 32));
    }
    return out;
}

std::array<int, 3> lattice_dims(int level, const int periodic[3]) {
    const int m = 1 << (level - 1);
    return {periodic[0] ? m : 2 * m, periodic[1] ? m : 2 * m, periodic[2] ? m : 2 * m};
}

LatticeShape &lattice_shape(KifmmOps &ops, const std::array<int, 3> &m, cudaStream_t st, int *launches) {
    FftOps &f = ops.fft;
    LatticeShape &S = f.lattice[m];
    if (S.M) return S;
    S.m[0] = m[0], S.m[1] = m[1], S.m[2] = m[2];
    S.M3 = (int64_t)m[0] * m[1] * m[2];
    const int nc = ops.ks * (ops.ks + 1) / 2;
    S.M = ops.ws.get<double>("lat_M_" + std::to_string(m[0]) + "_" + std::to_string(m[1]) + "_" + std::to_string(m[2]),
                             (size_t)S.M3 * LAT_E * nc * f.nw * 2);
    const dim3 grid((f.nw + 127) / 128, LAT_E * nc, (unsigned)S.M3);
    lat_build_kernel<<<grid, 128, 0, st>>>(reinterpret_cast<const double2 *>(f.khat), ops.slot_of_code, ops.ks, f.nw,
                                           m[0], m[1], m[2], reinterpret_cast<double2 *>(S.M));
    PK_CUDA(cudaGetLastError());
    *launches += 1;
    const std::vector<int64_t> pr = conjugate_pairs(S.m);
    S.npairs = (int64_t)pr.size();
    S.pairs = ops.ws.get<int64_t>("lat_pairs_" + std::to_string(m[0]) + "_" + std::to_string(m[1]) + "_" +
                                      std::to_string(m[2]),
                                  pr.size());
    PK_CUDA(cudaMemcpyAsync(S.pairs, pr.data(), pr.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaStreamSynchronize(st)); // pr is a host temporary
    return S;
}

} // namespace

int64_t m2l_lattice_bytes(const KifmmOps &ops, int level, const int periodic[3]) {
    const int p = ops.p, N = fft_edge(p), nw = N * N * (N / 2 + 1);
    const auto m = lattice_dims(level, periodic);
    const int64_t M3 = (int64_t)m[0] * m[1] * m[2];
    const int nc = ops.ks * (ops.ks + 1) / 2;
    const int64_t spectra = M3 * LAT_E * nc * nw * 16;            // M
    const int64_t lat = 2 * M3 * 8 * ops.ks * (int64_t)nw * 16;   // Psi~, Q~
    return spectra + lat;
}

int m2l_lattice_check(KifmmOps &ops, const LatticeLevelArgs &a, const int *table, int64_t ld, const int *out_box,
                      int ncols, int *bad, Workspace &ws, cudaStream_t st) {
    const auto m = lattice_dims(a.level, a.periodic);
    const int64_t M3 = (int64_t)m[0] * m[1] * m[2], nl = a.box1 - a.box0;
    const int n = 1 << a.level;
    int *box_of = ws.get<int>("lat_boxof_chk", M3 * 8);
    int *seen = ws.get<int>("lat_seen", std::max<int64_t>(nl, 1));
    int *d_code = ops.ws.get<int>("fft_code", kNumM2L); // uploaded by m2l_fft_prepare
    static const bool debug = std::getenv("PKGPU_LATTICE_DEBUG") != nullptr;
    int *dbg = nullptr;
    if (debug) {
        dbg = ws.get<int>("lat_dbg", 33);
        PK_CUDA(cudaMemsetAsync(dbg, 0, 33 * sizeof(int), st));
    }
    PK_CUDA(cudaMemsetAsync(box_of, 0xff, M3 * 8 * sizeof(int), st));
    PK_CUDA(cudaMemsetAsync(seen, 0, nl * sizeof(int), st));
    lat_boxmap_kernel<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(a.cell, a.box0, nl, m[1], m[2], box_of);
    const int64_t total = (int64_t)kNumM2L * ncols;
    lat_check_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
        table, ld, out_box, ncols, d_code, a.cell, box_of, n, a.periodic[0], a.periodic[1], a.periodic[2], m[1], m[2],
        a.box0, nl, a.srng, a.trng, a.mask, seen, bad, dbg);
    if (!a.mask) lat_seen_kernel<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(seen, nl, bad);
    PK_CUDA(cudaGetLastError());
    if (debug) {
        int h[33];
        PK_CUDA(cudaMemcpyAsync(h, dbg, sizeof h, cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        std::vector<int> cells(4 * 8 * 2);
        for (int k = 0; k < std::min(h[0], 8); k++) {
            int4 ct{}, cw{}, cg{};
            PK_CUDA(cudaMemcpy(&ct, a.cell + h[2 + 4 * k], sizeof ct, cudaMemcpyDeviceToHost));
            if (h[3 + 4 * k] >= 0) PK_CUDA(cudaMemcpy(&cw, a.cell + h[3 + 4 * k], sizeof cw, cudaMemcpyDeviceToHost));
            if (h[4 + 4 * k] >= 0) PK_CUDA(cudaMemcpy(&cg, a.cell + h[4 + 4 * k], sizeof cg, cudaMemcpyDeviceToHost));
            const int code = ops.h_code_of_slot[h[1 + 4 * k]];
            std::fprintf(stderr, "  level %d slot %d d=(%d,%d,%d) target %d (%d,%d,%d) want %d (%d,%d,%d) got %d (%d,%d,%d)\n",
                         a.level, h[1 + 4 * k], code / 49 - 3, (code / 7) % 7 - 3, code % 7 - 3, h[2 + 4 * k], ct.x, ct.y,
                         ct.z, h[3 + 4 * k], cw.x, cw.y, cw.z, h[4 + 4 * k], cg.x, cg.y, cg.z);
        }
    }
    return 3;
}

int m2l_lattice_level(KifmmOps &ops, const LatticeLevelArgs &a, Workspace &ws, cudaStream_t st) {
    FftOps &f = ops.fft;
    int launches = 0;
    const auto m = lattice_dims(a.level, a.periodic);
    LatticeShape &S = lattice_shape(ops, m, st, &launches);
    const int ks = ops.ks, kt = ops.kt, n = ops.n;
    if (n != ops.p * ops.p * ops.p - (ops.p - 2) * (ops.p - 2) * (ops.p - 2))
        throw RuntimeError("lattice M2L: surface point count does not match p"); // the kernels' constant
    const int64_t M3 = S.M3, N3 = (int64_t)f.N * f.N * f.N, nl = a.box1 - a.box0;
    int *box_of = ws.get<int>("lat_boxof", M3 * 8);
    auto mark = [&](const char *stage, int begin) {
        if (a.mark) a.mark(a.user, stage, begin);
    };
    mark("lat_fwd", 1);
    PK_CUDA(cudaMemsetAsync(box_of, 0xff, M3 * 8 * sizeof(int), st));
    lat_boxmap_kernel<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(a.cell, a.box0, nl, m[1], m[2], box_of);
    // surface values -> lattice spectra (in place) -> surface spectra Psi~[kappa][c][b][w]
    const int p = ops.p, NH = f.N / 2 + 1;
    const int64_t Ss = (int64_t)8 * ks * n, St = (int64_t)8 * kt * n;
    double2 *A = reinterpret_cast<double2 *>(ws.get<double>("lat_surf", (size_t)M3 * std::max(Ss, St) * 2));
    lat_gather_surface_kernel<<<(unsigned)std::min<int64_t>((M3 * Ss + 255) / 256, 148 * 32), 256, 0, st>>>(
        a.X, ops.Kp, box_of, M3, ks, n, A);
    launches += lat_fft(A, Ss, S.m, -1.0, st);
    const int64_t ng = M3 * 8 * ks;
    double *psi = ws.get<double>("lat_psi", (size_t)ng * f.nw * 2);
    const int tpb = std::min(256, (f.N * NH + 31) / 32 * 32);
    switch (p) {
#define LAT_FWD(PP)                                                                                                    \
    case PP: {                                                                                                         \
        constexpr int NN = fft_edge(PP), HH = NN / 2 + 1;                                                              \
        const size_t sm = (size_t)(2 * (std::max(PP * PP * (PP + 1), PP * NN * HH) + PP * PP * (HH + 1))) * 16;        \
        set_smem_once(lat_surface_fwd_t<PP>, sm);                                                                      \
        lat_surface_fwd_t<PP><<<(unsigned)((ng + 1) / 2), tpb, sm, st>>>(A, n, f.gidx,                                 \
                                                                         reinterpret_cast<double2 *>(psi), ng);        \
        break;                                                                                                         \
    }
        LAT_FWD(4) LAT_FWD(5) LAT_FWD(6) LAT_FWD(7) LAT_FWD(8) LAT_FWD(9) LAT_FWD(10)
#undef LAT_FWD
    default: {
        const size_t fsm = (size_t)(f.N + p * p * p + p * p * NH + p * f.N * NH) * 16;
        set_smem_once(lat_surface_fwd_kernel, fsm);
        lat_surface_fwd_kernel<<<(unsigned)ng, LS_THREADS, fsm, st>>>(A, p, n, f.gidx, reinterpret_cast<double2 *>(psi));
    }
    }
    mark("lat_fwd", 0);
    // pointwise products over (kappa, w): one pass over the stencil spectra, Psi~ and Q~
    double *q = ws.get<double>("lat_q", (size_t)M3 * 8 * kt * f.nw * 2);
    mark("lat_mul", 1);
    const int64_t total = M3 * f.nw;
    const unsigned grid = (unsigned)((total + 127) / 128);
    if (ks == 1)
        lat_mul_kernel<1><<<grid, 128, 0, st>>>(reinterpret_cast<const double2 *>(S.M),
                                                reinterpret_cast<const double2 *>(psi), reinterpret_cast<double2 *>(q),
                                                f.nw, total);
    else
        lat_mul_kernel<3><<<grid, 128, 0, st>>>(reinterpret_cast<const double2 *>(S.M),
                                                reinterpret_cast<const double2 *>(psi), reinterpret_cast<double2 *>(q),
                                                f.nw, total);
    mark("lat_mul", 0);
    if (a.work) // algorithmic bytes: M (14 classes x symmetric components) + Psi~ in, Q~ out, 16 B each
        a.work(a.user, "lat_mul", (double)M3 * f.nw, 16.0 * (LAT_E * (ks * (ks + 1) / 2) + 8 * ks + 8 * kt));
    mark("lat_inv", 1);
    // (a CTA takes a conjugate pair of lattice frequencies: 2 N NH first-stage columns, one round
    // of global loads with twice the threads)
    const int tpb_inv = std::min(256, (2 * f.N * NH + 31) / 32 * 32);
    // surface values per lattice frequency -> inverse lattice transform -> check potentials
    // (unnormalised transforms: 1 / (N^3 M3))
    switch (p) {
#define LAT_INV(PP)                                                                                                    \
    case PP: {                                                                                                         \
        constexpr int NN = fft_edge(PP), HH = NN / 2 + 1;                                                              \
        const size_t sm = (size_t)(NN + 2 * PP * NN * HH + 2 * PP * PP * (HH + 1)) * 16;                               \
        set_smem_once(lat_surface_inv_t<PP>, sm);                                                                      \
        lat_surface_inv_t<PP><<<(unsigned)(S.npairs * 8 * kt), tpb_inv, sm, st>>>(reinterpret_cast<const double2 *>(q),\
                                                                               S.pairs, kt, n, f.gidx, A);             \
        break;                                                                                                         \
    }
        LAT_INV(4) LAT_INV(5) LAT_INV(6) LAT_INV(7) LAT_INV(8) LAT_INV(9) LAT_INV(10)
#undef LAT_INV
    default: {
        const size_t ism = (size_t)(f.N + 2 * p * f.N * NH + 2 * p * p * NH) * 16;
        set_smem_once(lat_surface_inv_kernel, ism);
        lat_surface_inv_kernel<<<(unsigned)(S.npairs * 8 * kt), LS_THREADS, ism, st>>>(
            reinterpret_cast<const double2 *>(q), S.pairs, kt, p, n, f.gidx, A);
    }
    }
    launches += lat_fft(A, St, S.m, 1.0, st);
    if (!a.defer_scatter) {
        lat_scatter_surface_kernel<<<(unsigned)std::min<int64_t>((M3 * St + 255) / 256, 148 * 32), 256, 0, st>>>(
            A, box_of, M3, kt, n, a.alpha / ((double)N3 * (double)M3), ops.Kp, a.Y);
        launches += 1;
    }
    PK_CUDA(cudaGetLastError());
    mark("lat_inv", 0);
    return launches + 5;
}

int m2l_lattice_scatter(KifmmOps &ops, const LatticeLevelArgs &a, Workspace &ws, cudaStream_t st) {
    FftOps &f = ops.fft;
    int launches = 0;
    const auto m = lattice_dims(a.level, a.periodic);
    LatticeShape &S = lattice_shape(ops, m, st, &launches);
    const int ks = ops.ks, kt = ops.kt, n = ops.n;
    const int64_t M3 = S.M3, N3 = (int64_t)f.N * f.N * f.N;
    const int64_t Ss = (int64_t)8 * ks * n, St = (int64_t)8 * kt * n;
    // the buffers m2l_lattice_level left (same names and sizes: no reallocation)
    int *box_of = ws.get<int>("lat_boxof", M3 * 8);
    double2 *A = reinterpret_cast<double2 *>(ws.get<double>("lat_surf", (size_t)M3 * std::max(Ss, St) * 2));
    lat_scatter_surface_kernel<<<(unsigned)std::min<int64_t>((M3 * St + 255) / 256, 148 * 32), 256, 0, st>>>(
        A, box_of, M3, kt, n, a.alpha / ((double)N3 * (double)M3), ops.Kp, a.Y);
    PK_CUDA(cudaGetLastError());
    return launches + 1;
}

// the constant twiddle tables of the templated surface transforms, once per device
void upload_lattice_twiddles() {
    static std::mutex mtx;
    static bool done[64] = {false};
    int dev = 0;
    PK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mtx);
    if (dev < 64 && done[dev]) return;
    static double2 h[kLatTwMaxP + 1][kLatTwMaxN];
    const double pi = 3.14159265358979323846;
    for (int p = 2; p <= kLatTwMaxP; p++) {
        const int N = fft_edge(p);
        for (int k = 0; k < N && k < kLatTwMaxN; k++)
            h[p][k] = make_double2(std::cos(-2.0 * pi * k / N), std::sin(-2.0 * pi * k / N));
    }
    PK_CUDA(cudaMemcpyToSymbol(c_lat_tw, h, sizeof h));
    if (dev < 64) done[dev] = true;
}

int m2l_fft_prepare(KifmmOps &ops, Workspace &ws, cudaStream_t st) {
    FftOps &f = ops.fft;
    if (f.ready) return 0;
    upload_lattice_twiddles();
    const int p = ops.p, ks = ops.ks, kt = ops.kt;
    f.N = fft_edge(p);
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
    if (a.ncols % FT_TILE != 0) throw RuntimeError("m2l_fft: columns must be a multiple of 64");
    FftOps &f = ops.fft;
    const int ks = ops.ks, kt = ops.kt, n = ops.n;
    const int64_t N3 = (int64_t)f.N * f.N * f.N, nlev = a.box1 - a.box0;
    int launches = 0;
    // columns per window: spectra of the window's targets and of their (unique) sources
    const int64_t per_col = (int64_t)(kt + 2 * ks) * (f.nw * 16 + N3 * 8);
    const int W = (int)std::max<int64_t>(FT_TILE, std::min<int64_t>(a.ncols, (int64_t)12e9 / per_col) / FT_TILE * FT_TILE);
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
        // frequency-domain accumulation over the V lists: source-staged tiles of 64 targets,
        // the direct kernel for tiles whose sources overflow the staging
        double *qhat = ws.get<double>("fft_qhat", (int64_t)wc * kt * f.nw * 2);
        const int ntiles = wc / FT_TILE;
        int *tile_nsrc = ws.get<int>("fft_tile_nsrc", ntiles);
        int *tile_srcs = ws.get<int>("fft_tile_srcs", (int64_t)ntiles * FT_MAXU);
        short *srcmap = ws.get<short>("fft_srcmap", (int64_t)ntiles * kSlots * FT_TILE);
        fft_tile_sources_kernel<<<ntiles, FT_THREADS, 0, st>>>(tab, a.ld, smap_abs, tile_nsrc, tile_srcs, srcmap);
        const dim3 sgrid((f.nw + FT_WB - 1) / FT_WB, ntiles);
        const size_t ssm = ((size_t)FT_CH * (ks * FT_WB + 1) + 2 * FT_SCH * kt * ks * FT_WB) * sizeof(double2) +
                           2 * FT_SCH * FT_TILE * sizeof(short);
        const dim3 grid((f.nw + FFT_THREADS - 1) / FFT_THREADS, wc / FFT_TC);
        if (ks == 1) {
            set_smem_once(fft_stage_kernel<1>, ssm);
            fft_stage_kernel<1><<<sgrid, FT_THREADS, ssm, st>>>(reinterpret_cast<const double2 *>(f.khat),
                                                                reinterpret_cast<const double2 *>(phat), tile_nsrc,
                                                                tile_srcs, srcmap, f.nw, reinterpret_cast<double2 *>(qhat));
            fft_hadamard_kernel<1><<<grid, FFT_THREADS, 0, st>>>(reinterpret_cast<const double2 *>(f.khat),
                                                                 reinterpret_cast<const double2 *>(phat), smap_abs, tab,
                                                                 a.ld, f.nw, reinterpret_cast<double2 *>(qhat), tile_nsrc);
        } else {
            set_smem_once(fft_stage_kernel<3>, ssm);
            fft_stage_kernel<3><<<sgrid, FT_THREADS, ssm, st>>>(reinterpret_cast<const double2 *>(f.khat),
                                                                reinterpret_cast<const double2 *>(phat), tile_nsrc,
                                                                tile_srcs, srcmap, f.nw, reinterpret_cast<double2 *>(qhat));
            fft_hadamard_kernel<3><<<grid, FFT_THREADS, 0, st>>>(reinterpret_cast<const double2 *>(f.khat),
                                                                 reinterpret_cast<const double2 *>(phat), smap_abs, tab,
                                                                 a.ld, f.nw, reinterpret_cast<double2 *>(qhat), tile_nsrc);
        }
        launches += 3;
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
