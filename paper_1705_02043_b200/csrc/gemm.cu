// Gather-GEMM on DMMA (mma.sync.aligned.m8n8k4.row.col.f64 -> SASS DMMA.8x8x4).
//
// CTA tile BM x 64 (rows x box columns), BK = 16 deep k-chunks, cp.async multistage
// pipeline. The reduction runs over (active slot, k-chunk); a slot is active for a
// tile when any of its 64 columns has a source box, so octant-homogeneous M2L tiles
// only stream the ~189 offsets that occur. Operand rows are padded to BK+4 doubles,
// which makes the 8-row x 4-double fragment reads hit distinct bank groups.
// Load balance: the slot range is split across CTAs when the tile grid is small
// (split partials reduced in a fixed order -> deterministic results).
#include <algorithm>

#include "gemm.h"

namespace pkgpu {

namespace {

constexpr int BN = kGemmBN;
constexpr int BK = 16;
constexpr int PAD = BK + 4;
constexpr int STAGES = 3;
constexpr int MAX_SLOTS = 320;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

struct KParams {
    GemmArgs a;
    int nsplit;
    double *part; // [nsplit][ncols][Kp] when nsplit > 1
};

__device__ __forceinline__ int col_out(const GemmArgs &a, int c) {
    if (a.out_box) return a.out_box[c];
    return c < a.nvalid ? a.box0 + c : -1;
}
__device__ __forceinline__ int col_src(const GemmArgs &a, int slot, int c) {
    if (a.src) return a.src[(int64_t)slot * a.ld_src + c];
    return col_out(a, c);
}

// BM rows per CTA; warps arranged (BM/32) x 2, warp tile 32 x 32.
template <int BM>
__global__ void __launch_bounds__(BM / 32 * 2 * 32) gather_gemm_kernel(KParams kp) {
    constexpr int WARPS_M = BM / 32;
    constexpr int NT = WARPS_M * 2 * 32;
    const GemmArgs &a = kp.a;
    extern __shared__ __align__(16) double smem[];
    double *As = smem;                          // [STAGES][BM][PAD]
    double *Bs = smem + STAGES * BM * PAD;      // [STAGES][BN][PAD]
    __shared__ int s_slots[MAX_SLOTS];
    __shared__ int s_flag[MAX_SLOTS];
    __shared__ int s_nact;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row0 = blockIdx.x * BM;
    const int col0 = blockIdx.y * BN;
    const int split = blockIdx.z;
    const int s_begin = (int)((int64_t)a.nslots * split / kp.nsplit);
    const int s_end = (int)((int64_t)a.nslots * (split + 1) / kp.nsplit);
    const int ns = s_end - s_begin;

    // active slots for this tile (deterministic order)
    for (int s = warp; s < ns; s += NT / 32) {
        const int slot = s_begin + s;
        bool any = false;
        for (int j = lane; j < BN; j += 32) any |= col_src(a, slot, col0 + j) >= 0;
        any = __any_sync(0xffffffffu, any);
        if (lane == 0) s_flag[s] = any ? 1 : 0;
    }
    __syncthreads();
    if (tid == 0) {
        int n = 0;
        for (int s = 0; s < ns; s++)
            if (s_flag[s]) s_slots[n++] = s_begin + s;
        s_nact = n;
    }
    __syncthreads();
    const int nact = s_nact;
    const int nk = a.Kp / BK;
    const int niter = nact * nk;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto load_stage = [&](int it, int stage) {
        const int slot = s_slots[it / nk];
        const int k0 = (it % nk) * BK;
        const int mat = a.tile_mat ? a.tile_mat[blockIdx.y] : (a.slot_mat ? a.slot_mat[slot] : slot);
        const double *Am = a.A + (int64_t)mat * a.Kp * a.Kp;
        double *as = As + stage * BM * PAD;
        double *bs = Bs + stage * BN * PAD;
        // A: BM rows x 16 doubles = BM*8 chunks of 16 B
        for (int ch = tid; ch < BM * (BK / 2); ch += NT) {
            const int r = ch / (BK / 2), cc = ch % (BK / 2);
            cp_async16(as + r * PAD + cc * 2, Am + (int64_t)(row0 + r) * a.Kp + k0 + cc * 2, 16);
        }
        // B: 64 gathered box vectors x 16 doubles
        for (int ch = tid; ch < BN * (BK / 2); ch += NT) {
            const int j = ch / (BK / 2), cc = ch % (BK / 2);
            const int sb = col_src(a, slot, col0 + j);
            const double *g = sb >= 0 ? a.X + (int64_t)sb * a.Kp + k0 + cc * 2 : a.X;
            cp_async16(bs + j * PAD + cc * 2, g, sb >= 0 ? 16 : 0);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
        if (s < niter) load_stage(s, s);
        cp_async_commit();
    }
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    for (int it = 0; it < niter; it++) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = it + STAGES - 1;
        if (nxt < niter) load_stage(nxt, nxt % STAGES);
        cp_async_commit();
        const double *as = As + (it % STAGES) * BM * PAD + (wm * 32 + (lane >> 2)) * PAD + (lane & 3);
        const double *bs = Bs + (it % STAGES) * BN * PAD + (wn * 32 + (lane >> 2)) * PAD + (lane & 3);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; i++) af[i] = as[i * 8 * PAD + kk];
#pragma unroll
            for (int j = 0; j < 4; j++) bf[j] = bs[j * 8 * PAD + kk];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) dmma(acc[i][j], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // epilogue: C fragment (row = lane/4, cols = 2*(lane%4) + {0,1})
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int r = row0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < 4; j++) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int c = col0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
                const double v = acc[i][j][h];
                if (kp.nsplit > 1) {
                    kp.part[((int64_t)split * a.ncols + c) * a.Kp + r] = v;
                    continue;
                }
                const int ob = col_out(a, c);
                if (ob < 0) continue;
                double *y = a.Y + (int64_t)ob * a.Kp + r;
                if (a.rdiv) {
                    const double d = a.rdiv[r];
                    *y = d > a.rdiv_eps ? v / d : 0.0;
                } else {
                    *y = (a.beta != 0.0 ? a.beta * *y : 0.0) + a.alpha * v;
                }
            }
        }
    }
}

__global__ void split_reduce_kernel(KParams kp) {
    const GemmArgs &a = kp.a;
    const int64_t total = (int64_t)a.ncols * a.Kp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / a.Kp), r = (int)(i % a.Kp);
        const int ob = col_out(a, c);
        if (ob < 0) continue;
        double v = 0.0;
        for (int s = 0; s < kp.nsplit; s++) v += kp.part[((int64_t)s * a.ncols + c) * a.Kp + r];
        double *y = a.Y + (int64_t)ob * a.Kp + r;
        if (a.rdiv) {
            const double d = a.rdiv[r];
            *y = d > a.rdiv_eps ? v / d : 0.0;
        } else {
            *y = (a.beta != 0.0 ? a.beta * *y : 0.0) + a.alpha * v;
        }
    }
}

// one warp per row
__global__ void gemv_kernel(const double *__restrict__ A, int rows, int cols, int lda, const double *__restrict__ x,
                            double *__restrict__ y, double alpha, double beta, const double *rdiv, double eps) {
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    double s = 0.0;
    for (int j = lane; j < cols; j += 32) s = fma(A[(int64_t)row * lda + j], x[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        if (rdiv)
            y[row] = rdiv[row] > eps ? s / rdiv[row] : 0.0;
        else
            y[row] = (beta != 0.0 ? beta * y[row] : 0.0) + alpha * s;
    }
}

template <int BM> size_t smem_bytes() { return (size_t)STAGES * (BM + BN) * PAD * sizeof(double); }

template <int BM> void configure() {
    static bool done = false;
    if (!done) {
        PK_CUDA(cudaFuncSetAttribute(gather_gemm_kernel<BM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_bytes<BM>()));
        done = true;
    }
}

} // namespace

int gather_gemm(const GemmArgs &a, Workspace &ws, cudaStream_t st, int num_sms) {
    if (a.ncols == 0 || a.nslots == 0) return 0;
    if (a.Kp % 64 != 0 || a.ncols % BN != 0 || a.nslots > MAX_SLOTS)
        throw RuntimeError("gather_gemm: bad shape");
    const int BMsel = (a.Kp % 128 == 0) ? 128 : 64;
    const int rowtiles = a.Kp / BMsel, coltiles = a.ncols / BN;
    const int64_t base = (int64_t)rowtiles * coltiles;
    const int64_t target = (int64_t)num_sms * 2 * 4;
    int nsplit = 1;
    if (base < target && a.nslots >= 8) nsplit = (int)std::min<int64_t>((target + base - 1) / base, a.nslots / 4);
    nsplit = std::max(nsplit, 1);
    KParams kp{a, nsplit, nullptr};
    if (nsplit > 1) kp.part = ws.get<double>("gemm_part", (size_t)nsplit * a.ncols * a.Kp);
    dim3 grid(rowtiles, coltiles, nsplit);
    if (BMsel == 128) {
        configure<128>();
        gather_gemm_kernel<128><<<grid, 256, smem_bytes<128>(), st>>>(kp);
    } else {
        configure<64>();
        gather_gemm_kernel<64><<<grid, 128, smem_bytes<64>(), st>>>(kp);
    }
    PK_CUDA(cudaGetLastError());
    if (nsplit > 1) {
        const int64_t total = (int64_t)a.ncols * a.Kp;
        split_reduce_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, num_sms * 16), 256, 0, st>>>(kp);
        PK_CUDA(cudaGetLastError());
        return 2;
    }
    return 1;
}

void gemv(const double *A, int rows, int cols, int lda, const double *x, double *y, double alpha, double beta,
          const double *rdiv, double rdiv_eps, cudaStream_t st) {
    gemv_kernel<<<(rows + 7) / 8, 256, 0, st>>>(A, rows, cols, lda, x, y, alpha, beta, rdiv, rdiv_eps);
    PK_CUDA(cudaGetLastError());
}

} // namespace pkgpu
