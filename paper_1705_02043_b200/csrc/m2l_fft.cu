// FFT-accelerated M2L (see m2l_fft.h).
#include <algorithm>
#include <cmath>
#include <mutex>
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
