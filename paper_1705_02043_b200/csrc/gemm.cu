// Gather-GEMM on DMMA (mma.sync.aligned.m8n8k4.row.col.f64 -> SASS DMMA.8x8x4).
//
// Work unit: a BM x 64 output tile (rows x box columns) over one contiguous chunk of
// its reduction space (active slot, 16-deep k-chunk). A slot is active for a column
// tile when any of its 64 columns has a source box (a prepass writes the per-tile
// active-slot lists), so octant-homogeneous M2L tiles stream only their ~189 offsets.
//
// Default mainloop ("tma"): persistent CTAs (2 per SM) pull units from an atomic
// counter. One producer warp streams each stage:
//   A  BM x 16 operator tile   -> cp.async.bulk.tensor.2d (TMA), 128B swizzle
//   B  64 x 16 gathered box rows -> cp.async 16 B (zero-fill for absent sources),
//                                   tracked by cp.async.mbarrier.arrive.noinc
// onto a "full" mbarrier; eight consumer warps run DMMA on 32x32 warp tiles and hand
// the stage back through an "empty" mbarrier (4-stage ring). Units that split a tile's
// reduction write partials reduced in a fixed order -> bitwise deterministic results.
// Fallback mainloop ("cpasync", PKGPU_GEMM=cpasync): all threads stage with cp.async,
// __syncthreads pipeline, one CTA per unit.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <tuple>

#include <cudaTypedefs.h>

#include "gemm.h"
#include "gemm_tma.cuh"
#include "tuning.h"

namespace pkgpu {

namespace {

constexpr int BN = kGemmBN;
constexpr int BK = 16;
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
    double *part;           // [nsplit][ncols][Kp] when nsplit > 1
    const int *tile_slots;  // [coltiles][MAX_SLOTS] active slots per column tile (null: slot si = si)
    const int *tile_nact;   // [coltiles] (null: every tile has the one slot of an identity gather)
    int rowtiles, coltiles; // unit = row + rowtiles * (col + coltiles * split)
    int total_units;
    int *counter;           // persistent scheduler (self-resetting: the CTA taking the last fetch zeroes it)
    // hybrid schedule (plan_hybrid below): whole tiles for the full waves, then the rest of the
    // iteration space cut into one equal chunk per resident CTA; a chunk is 1-3 pieces, each
    // inside one tile. Null: the uniform split above.
    const int4 *pieces;     // (tile = row + rowtiles * col, it0, it1 of nit_nom, partial index or -1: whole tile)
    const int2 *chunks;     // [total_units] piece range [x, y)
    const int *tile_parts;  // [rowtiles * coltiles] partials per tile (0: written directly)
    int nit_nom;            // nominal iterations per tile the plan was cut in (nslots * Kp / 16)
    int reduce_col0;        // first column holding a split tile
};

struct TmaParams {
    CUtensorMap tmA; // 2D view of the stacked operators: (Kp cols) x (nmat*Kp rows), 128B swizzle
    KParams kp;
};

__device__ __forceinline__ int col_out(const GemmArgs &a, int c) {
    if (a.out_box) return a.out_box[c];
    return c < a.nvalid ? a.box0 + c : -1;
}
__device__ __forceinline__ int col_src(const GemmArgs &a, int slot, int c) {
    if (a.src) return a.src[(int64_t)slot * a.ld_src + c];
    return col_out(a, c);
}
__device__ __forceinline__ int slot_matrix(const GemmArgs &a, int slot, int coltile) {
    return a.tile_mat ? a.tile_mat[coltile] : (a.slot_mat ? a.slot_mat[slot] : slot);
}

// prepass: active slots per column tile, in slot order (one block per column tile)
__global__ void slot_scan_kernel(GemmArgs a, int bn, int *tile_slots, int *tile_nact) {
    __shared__ int flag[MAX_SLOTS];
    const int ct = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < a.nslots; s += blockDim.x / 32) {
        bool any = false;
        for (int j = lane; j < bn; j += 32) any |= col_src(a, s, ct * bn + j) >= 0;
        any = __any_sync(0xffffffffu, any);
        if (lane == 0) flag[s] = any ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int n = 0;
        for (int s = 0; s < a.nslots; s++)
            if (flag[s]) tile_slots[ct * MAX_SLOTS + n++] = s;
        tile_nact[ct] = n;
    }
}

// epilogue of one output element (row r, column c) from its full sum
__device__ __forceinline__ void store_final(const GemmArgs &a, int r, int c, double v) {
    if (r >= a.Kp) return; // zero-filled operator rows of the last row tile
    const int ob = col_out(a, c);
    if (ob < 0) return;
    double *y = a.Y + (int64_t)ob * a.Kp + r;
    if (a.rdiv) {
        const double d = a.rdiv[r];
        *y = d > a.rdiv_eps ? v / d : 0.0;
    } else {
        *y = (a.beta != 0.0 ? a.beta * *y : 0.0) + a.alpha * v;
    }
}

// epilogue of one accumulator element: a split unit's partial, or the final value
__device__ __forceinline__ void store_out(const KParams &kp, int split, int r, int c, double v) {
    if (split >= 0) {
        if (r < kp.a.Kp) kp.part[((int64_t)split * kp.a.ncols + c) * kp.a.Kp + r] = v;
        return;
    }
    store_final(kp.a, r, c, v);
}

__device__ __forceinline__ void unit_range(const KParams &kp, int nact, int split, int &it0, int &it1) {
    const int64_t niter = (int64_t)nact * (kp.a.Kp / BK);
    it0 = (int)(niter * split / kp.nsplit);
    it1 = (int)(niter * (split + 1) / kp.nsplit);
}

// ---------------------------------------------------------------------------
// persistent TMA / mbarrier warp-specialised mainloop: NCW consumer warps + 1 producer.
//   BNT =  64, NCW =  8: two CTAs per SM (4-stage ring each)
//   BNT = 128, NCW = 16: one CTA per SM (6-stage ring), each operator tile feeds 128
//                        columns -> half the operator traffic per FLOP (big M2L levels)
constexpr int TMA_BROW = 160; // bytes per gathered B row in shared memory (128 B data + pad)

template <int BM, int BNT> constexpr int tma_stage_bytes() { return BM * BK * 8 + BNT * TMA_BROW; }

// register cap so the intended residency fits the 64K-register file; measured with
// cudaOccupancyMaxActiveBlocksPerMultiprocessor (PKGPU_GEMM_VERBOSE): 96 keeps 2 x 9-warp
// CTAs (104 drops to 1) and is the most a 17-warp CTA can launch with
template <int BM, int NSTAGE, int BNT, int NCW>
__global__ void __maxnreg__(96)
    gather_gemm_tma_kernel(const __grid_constant__ TmaParams tp) {
    constexpr int WARPS_M = BM / 32;       // 4 (BM = 128)
    constexpr int WARPS_N = NCW / WARPS_M; // 2 or 4
    constexpr int WTN = BNT / WARPS_N;     // 32
    constexpr int NTL = WTN / 8;           // 4
    constexpr int A_BYTES = BM * BK * 8;
    constexpr int STAGE = tma_stage_bytes<BM, BNT>();
    constexpr int RPL = BNT / 4; // B rows per producer lane
    static_assert(STAGE % 1024 == 0, "stage must keep 1024-byte alignment for the 128B swizzle");
    const KParams &kp = tp.kp;
    const GemmArgs &a = kp.a;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];
    __shared__ int s_unit;
    __shared__ int s_rowsrc[BNT]; // producer: source box of each B row for the current slot

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; s++) {
            tma::mbar_init(&full[s], 33); // producer lane 0 expect_tx + 32 cp.async arrivals
            tma::mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    const int nk = a.Kp / BK;
    // consumer fragment addressing. A (128B-swizzled): element (r, k) at
    // r*128 + (((k>>1) ^ (r&7)) << 4) + ((k&1) << 3); fragment rows have r&7 == lane>>2.
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    const int swz = lane >> 2;
    int aoff[4];
#pragma unroll
    for (int kk = 0; kk < 4; kk++) aoff[kk] = (((2 * kk) + ((lane & 3) >> 1)) ^ swz) * 16 + (lane & 1) * 8;
    const int arow = (wm * 32 + (lane >> 2)) * 128;
    const int brow = (wn * WTN + (lane >> 2)) * TMA_BROW + (lane & 3) * 8;

    int g = 0; // pipeline iterations issued/consumed so far by this CTA (stage ring position)
    for (;;) {
        if (tid == 0) {
            const int u = atomicAdd(kp.counter, 1);
            // every CTA ends on one failed fetch: total_units + gridDim.x fetches in all, so the
            // last one leaves the counter at zero for the next launch on the stream
            if (u == kp.total_units + (int)gridDim.x - 1) *kp.counter = 0;
            s_unit = u;
        }
        __syncthreads();
        const int unit = s_unit;
        __syncthreads();
        if (unit >= kp.total_units) break;
        int pc0 = unit, pc1 = unit + 1;
        if (kp.chunks) {
            const int2 ch = kp.chunks[unit];
            pc0 = ch.x, pc1 = ch.y;
        }
      for (int pc = pc0; pc < pc1; pc++) {
        int rt, ct, split, it0, it1;
        if (kp.pieces) {
            const int4 pd = kp.pieces[pc];
            rt = pd.x % kp.rowtiles, ct = pd.x / kp.rowtiles;
            const int64_t niter = (int64_t)(kp.tile_nact ? kp.tile_nact[ct] : 1) * (a.Kp / BK);
            it0 = (int)(niter * pd.y / kp.nit_nom);
            it1 = (int)(niter * pd.z / kp.nit_nom);
            split = pd.w;
        } else {
            rt = unit % kp.rowtiles;
            const int rest = unit / kp.rowtiles;
            ct = rest % kp.coltiles;
            split = rest / kp.coltiles;
            unit_range(kp, kp.tile_nact ? kp.tile_nact[ct] : 1, split, it0, it1);
            if (kp.nsplit <= 1) split = -1; // the whole tile: final values
        }
        const int row0 = rt * BM, col0 = ct * BNT;
        const int *slots = kp.tile_slots ? kp.tile_slots + ct * MAX_SLOTS : nullptr;
        const int n = it1 - it0;
        if (warp == NCW) {
            // ---------------- producer ----------------
            // this lane's B rows for the current slot, cached in registers (reloaded on
            // slot change, every Kp/16 iterations): no dependent loads in the issue loop
            int cur = -1, mat = 0;
            for (int i = 0; i < n; i++) {
                const int gi = g + i, st = gi % NSTAGE;
                const int it = it0 + i;
                const int si = it / nk, k0 = (it % nk) * BK;
                if (si != cur) {
                    cur = si;
                    const int slot = slots ? slots[si] : si;
                    mat = slot_matrix(a, slot, ct);
                    __syncwarp();
                    for (int j = lane; j < BNT; j += 32) s_rowsrc[j] = col_src(a, slot, col0 + j);
                    __syncwarp();
                }
                tma::mbar_wait(&empty[st], ((gi / NSTAGE) & 1) ^ 1);
                unsigned char *as = smem + st * STAGE;
                unsigned char *bs = as + A_BYTES;
                if (lane == 0) {
                    tma::mbar_expect_tx(&full[st], A_BYTES);
                    tma::tma_load_3d(as, &tp.tmA, k0, row0, mat, &full[st]);
                }
#pragma unroll
                for (int m = 0; m < RPL; m++) {
                    const int j = (lane >> 3) + 4 * m;
                    const int rb = s_rowsrc[j];
                    const double *src = rb >= 0 ? a.X + (int64_t)rb * a.Kp + k0 + 2 * (lane & 7) : a.X;
                    tma::cp_async16(bs + j * TMA_BROW + 16 * (lane & 7), src, rb >= 0 ? 16 : 0);
                }
                tma::cp_async_mbar_arrive(&full[st]);
            }
        } else {
            // ---------------- consumers ----------------
            double acc[4][NTL][2];
#pragma unroll
            for (int m = 0; m < 4; m++)
#pragma unroll
                for (int q = 0; q < NTL; q++) acc[m][q][0] = acc[m][q][1] = 0.0;
            for (int i = 0; i < n; i++) {
                const int gi = g + i, st = gi % NSTAGE;
                tma::mbar_wait(&full[st], (gi / NSTAGE) & 1);
                const unsigned char *as = smem + st * STAGE + arow;
                const unsigned char *bs = smem + st * STAGE + A_BYTES + brow;
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    double af[4], bf[NTL];
#pragma unroll
                    for (int m = 0; m < 4; m++) af[m] = *reinterpret_cast<const double *>(as + m * 8 * 128 + aoff[kk]);
#pragma unroll
                    for (int q = 0; q < NTL; q++)
                        bf[q] = *reinterpret_cast<const double *>(bs + q * 8 * TMA_BROW + kk * 32);
#pragma unroll
                    for (int m = 0; m < 4; m++)
#pragma unroll
                        for (int q = 0; q < NTL; q++) dmma(acc[m][q], af[m], bf[q]);
                }
                __syncwarp();
                if (lane == 0) tma::mbar_arrive(&empty[st]);
            }
#pragma unroll
            for (int m = 0; m < 4; m++) {
                const int r = row0 + wm * 32 + m * 8 + (lane >> 2);
#pragma unroll
                for (int q = 0; q < NTL; q++)
#pragma unroll
                    for (int h = 0; h < 2; h++)
                        store_out(kp, split, r, col0 + wn * WTN + q * 8 + 2 * (lane & 3) + h, acc[m][q][h]);
            }
        }
        g += n;
      }
    }
}

__global__ void split_reduce_kernel(KParams kp, int bm, int bnt) {
    const GemmArgs &a = kp.a;
    const int64_t total = (int64_t)(a.ncols - kp.reduce_col0) * a.Kp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = kp.reduce_col0 + (int)(i / a.Kp), r = (int)(i % a.Kp);
        const int ob = col_out(a, c);
        if (ob < 0) continue;
        int np = kp.nsplit;
        if (kp.tile_parts) {
            np = kp.tile_parts[r / bm + kp.rowtiles * (c / bnt)];
            if (np == 0) continue; // a whole tile, written by the GEMM
        }
        double v = 0.0;
        for (int s = 0; s < np; s++) v += kp.part[((int64_t)s * a.ncols + c) * a.Kp + r];
        double *y = a.Y + (int64_t)ob * a.Kp + r;
        if (a.rdiv) {
            const double d = a.rdiv[r];
            *y = d > a.rdiv_eps ? v / d : 0.0;
        } else {
            *y = (a.beta != 0.0 ? a.beta * *y : 0.0) + a.alpha * v;
        }
    }
}

// ---------------------------------------------------------------------------
// Skinny launches (the top levels of the tree: at most SK_MAXAPP (column, slot) pairs, e.g.
// the 8 + 64 M2M translations into levels 0 and 1 or the pseudo-inverse of 1-64 boxes) are
// bound by streaming the operator matrices once, not by the FLOPs: on the tile kernel they
// cost 40-75 us each at cfg2 (a 128 x 64 tile per unit whatever the column count, split-K
// partials, three launches). Here a warp owns one output row for every column: it streams
// that row of each matrix the pairs use (all rows prefetched into L2 up front, then held in
// registers), takes the dot product with each pair's source vector (L1 / L2 hits) and sums a
// column's slots in slot order -- one launch, no partials, bitwise deterministic.
constexpr int SK_MAXAPP = 64;  // (column, slot) pairs
constexpr int SK_MAXC = 1024;  // columns of the (padded) layout
constexpr int SK_MAXJ = 24;    // Kp / 64
constexpr int SK_WARPS = 4;

__global__ void __launch_bounds__(SK_WARPS * 32) skinny_gemm_kernel(GemmArgs a) {
    __shared__ int s_ci[SK_MAXAPP], s_src[SK_MAXAPP], s_mat[SK_MAXAPP]; // pair: column index, source box, matrix
    __shared__ int s_col[SK_MAXAPP];                                    // valid columns
    __shared__ short s_cmap[SK_MAXC];                                   // column -> index in s_col
    __shared__ int s_wcnt[SK_WARPS], s_napp, s_ncol;
    __shared__ double s_acc[SK_WARPS][SK_MAXAPP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NT = SK_WARPS * 32;
    if (tid == 0) s_napp = s_ncol = 0;
    for (int i = tid; i < SK_WARPS * SK_MAXAPP; i += NT) (&s_acc[0][0])[i] = 0.0;
    __syncthreads();
    // ordered compaction of the valid columns, then of the pairs (slot-major, column order)
    for (int c0 = 0; c0 < a.ncols; c0 += NT) {
        const int c = c0 + tid;
        const bool v = c < a.ncols && col_out(a, c) >= 0;
        const unsigned b = __ballot_sync(0xffffffffu, v);
        if (lane == 0) s_wcnt[warp] = __popc(b);
        __syncthreads();
        int base = s_ncol;
        for (int w = 0; w < warp; w++) base += s_wcnt[w];
        const int pos = base + __popc(b & ((1u << lane) - 1));
        if (c < a.ncols) s_cmap[c] = v ? (short)min(pos, SK_MAXAPP - 1) : (short)-1;
        if (v && pos < SK_MAXAPP) s_col[pos] = c;
        __syncthreads();
        if (tid == 0) {
            int n = s_ncol;
            for (int w = 0; w < SK_WARPS; w++) n += s_wcnt[w];
            s_ncol = min(n, SK_MAXAPP);
        }
        __syncthreads();
    }
    const int total = a.nslots * a.ncols;
    for (int e0 = 0; e0 < total; e0 += NT) {
        const int e = e0 + tid;
        int slot = 0, c = 0, sb = -1;
        if (e < total) {
            slot = e / a.ncols, c = e % a.ncols;
            if (col_out(a, c) >= 0) sb = col_src(a, slot, c);
        }
        const bool v = sb >= 0;
        const unsigned b = __ballot_sync(0xffffffffu, v);
        if (lane == 0) s_wcnt[warp] = __popc(b);
        __syncthreads();
        int base = s_napp;
        for (int w = 0; w < warp; w++) base += s_wcnt[w];
        const int pos = base + __popc(b & ((1u << lane) - 1));
        if (v && pos < SK_MAXAPP) {
            s_ci[pos] = s_cmap[c];
            s_src[pos] = sb;
            s_mat[pos] = slot_matrix(a, slot, c / BN);
        }
        __syncthreads();
        if (tid == 0) {
            int n = s_napp;
            for (int w = 0; w < SK_WARPS; w++) n += s_wcnt[w];
            s_napp = min(n, SK_MAXAPP);
        }
        __syncthreads();
    }
    const int napp = s_napp, ncolv = s_ncol;
    const int r = blockIdx.x * SK_WARPS + warp;
    if (r >= a.Kp) return;
    const int nj = a.Kp / 64;
    // every matrix row this warp will read, requested from DRAM at once
    for (int p = 0, prev = -1; p < napp; p++) {
        const int m = s_mat[p];
        if (m == prev) continue;
        prev = m;
        const char *row = reinterpret_cast<const char *>(a.A + ((int64_t)m * a.Kp + r) * a.Kp);
        for (int off = lane * 128; off < a.Kp * 8; off += 32 * 128)
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(row + off));
    }
    double2 ar[SK_MAXJ];
    int cur = -1;
    for (int p = 0; p < napp; p++) {
        const int m = s_mat[p];
        if (m != cur) {
            cur = m;
            const double2 *row = reinterpret_cast<const double2 *>(a.A + ((int64_t)m * a.Kp + r) * a.Kp) + lane;
#pragma unroll
            for (int j = 0; j < SK_MAXJ; j++)
                if (j < nj) ar[j] = __ldg(row + 32 * j);
        }
        const double2 *x = reinterpret_cast<const double2 *>(a.X + (int64_t)s_src[p] * a.Kp) + lane;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int j = 0; j < SK_MAXJ; j++)
            if (j < nj) {
                const double2 xv = __ldg(x + 32 * j);
                d0 = fma(ar[j].x, xv.x, d0);
                d1 = fma(ar[j].y, xv.y, d1);
            }
        double d = d0 + d1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0) s_acc[warp][s_ci[p]] += d; // a column's slots in slot order
    }
    __syncwarp();
    for (int ci = lane; ci < ncolv; ci += 32) store_final(a, r, s_col[ci], s_acc[warp][ci]);
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

// (BNT, stages): 64 -> 4 x 26 KB, two CTAs per SM; 128 -> 6 x 36 KB, one CTA per SM
template <int BNT> constexpr int tma_stages() { return BNT == 64 ? 4 : 6; }
template <int BNT> size_t tma_smem_bytes() { return (size_t)tma_stages<BNT>() * tma_stage_bytes<128, BNT>() + 1024; }

// dynamic shared memory opt-in, once per (kernel, device): the attribute is per device
template <class K> void set_smem(K kernel, size_t bytes) {
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        PK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// tensor map over the stacked operator array, cached per (pointer, nmat, Kp, BM)
CUtensorMap operator_map(const double *A, int nmat, int Kp, int BM) {
    static std::map<std::tuple<const double *, int, int, int>, CUtensorMap> cache;
    static std::mutex mtx; // contexts may run on several host threads
    std::lock_guard<std::mutex> lock(mtx);
    const auto key = std::make_tuple(A, nmat, Kp, BM);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    CUtensorMap m;
    const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)Kp, (cuuint64_t)nmat};
    const cuuint64_t strides[2] = {(cuuint64_t)Kp * sizeof(double), (cuuint64_t)Kp * Kp * sizeof(double)};
    const cuuint32_t box[3] = {BK, (cuuint32_t)BM, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(A), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return cache.emplace(key, m).first->second;
}

// int counters that every launch leaves at zero: zeroed here only when (re)allocated
int *zeroed_counters(Workspace &ws, const char *name, size_t n, cudaStream_t st) {
    auto &b = ws.bufs[name];
    if (!b) b = std::make_unique<DevBuf>();
    const size_t before = b->bytes;
    int *p = b->as<int>(n);
    if (b->bytes != before) PK_CUDA(cudaMemsetAsync(p, 0, b->bytes, st)); // new allocation
    return p;
}

// Hybrid schedule for launches of one to a few waves of tiles (cfg2's level-4 pseudo-inverse:
// 448 tiles on 296 resident CTAs). A uniform split-K (three units per tile there) pays
// partials for every tile and still ends on a ragged wave. Here the full waves run whole
// tiles, written directly, and the remaining tiles' iteration space is cut into one equal
// chunk per resident CTA (a chunk crosses at most two tile boundaries; each piece writes a
// partial, summed per tile in piece order by split_reduce_kernel: deterministic).
struct HybridPlan {
    const int4 *pieces = nullptr;
    const int2 *chunks = nullptr;
    const int *tile_parts = nullptr;
    int nchunks = 0, maxparts = 0, reduce_col0 = 0;
};

HybridPlan plan_hybrid(Workspace &ws, int rowtiles, int coltiles, int bnt, int resident, int nit, cudaStream_t st) {
    const std::string key = "gemm_plan_" + std::to_string(rowtiles) + "_" + std::to_string(coltiles) + "_" +
                            std::to_string(resident) + "_" + std::to_string(nit);
    const int base = rowtiles * coltiles;
    const int full = base / resident * resident, rest = base - full;
    std::vector<int4> pieces;
    std::vector<int2> chunks;
    std::vector<int> parts(base, 0);
    for (int t = 0; t < full; t++) {
        chunks.push_back(make_int2((int)pieces.size(), (int)pieces.size() + 1));
        pieces.push_back(make_int4(t, 0, nit, -1));
    }
    const int64_t total = (int64_t)rest * nit;
    for (int k = 0; k < resident; k++) {
        int64_t pos = total * k / resident;
        const int64_t hi = total * (k + 1) / resident;
        if (hi <= pos) continue;
        const int first = (int)pieces.size();
        while (pos < hi) {
            const int tl = (int)(pos / nit);
            const int64_t tend = std::min<int64_t>(hi, (int64_t)(tl + 1) * nit);
            const int a0 = (int)(pos - (int64_t)tl * nit), a1 = (int)(tend - (int64_t)tl * nit);
            const bool whole = a0 == 0 && a1 == nit;
            pieces.push_back(make_int4(full + tl, a0, a1, whole ? -1 : parts[full + tl]++));
            pos = tend;
        }
        chunks.push_back(make_int2(first, (int)pieces.size()));
    }
    HybridPlan P;
    P.nchunks = (int)chunks.size();
    for (int v : parts) P.maxparts = std::max(P.maxparts, v);
    P.reduce_col0 = full / rowtiles * bnt; // tiles are numbered row-fastest: the first column with a split tile
    const bool fresh = ws.bufs.find(key + "_p") == ws.bufs.end();
    int4 *dp = ws.get<int4>(key + "_p", pieces.size());
    int2 *dc = ws.get<int2>(key + "_c", chunks.size());
    int *dt = ws.get<int>(key + "_t", parts.size());
    if (fresh) {
        PK_CUDA(cudaMemcpyAsync(dp, pieces.data(), pieces.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
        PK_CUDA(cudaMemcpyAsync(dc, chunks.data(), chunks.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
        PK_CUDA(cudaMemcpyAsync(dt, parts.data(), parts.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        PK_CUDA(cudaStreamSynchronize(st)); // host temporaries
    }
    P.pieces = dp, P.chunks = dc, P.tile_parts = dt;
    return P;
}

} // namespace

int gather_gemm(const GemmArgs &a, Workspace &ws, cudaStream_t st, int num_sms) {
    if (a.ncols == 0 || a.nslots == 0) return 0;
    if (a.Kp % 64 != 0 || a.ncols % BN != 0 || a.nslots > MAX_SLOTS)
        throw RuntimeError("gather_gemm: bad shape");
    if (a.napps > 0 && a.napps <= std::min<int64_t>(tuning().gemm_skinny_apps, SK_MAXAPP) && a.ncols <= SK_MAXC &&
        a.Kp / 64 <= SK_MAXJ) {
        skinny_gemm_kernel<<<(a.Kp + SK_WARPS - 1) / SK_WARPS, SK_WARPS * 32, 0, st>>>(a);
        PK_CUDA(cudaGetLastError());
        return 1;
    }
    // 128-row tiles for every K: the TMA zero-fills operator rows past Kp (3D tensor map,
    // out-of-bounds) and the epilogue drops them
    constexpr int BMsel = 128;
    // 128-column tiles when the caller's column layout allows (big octant-grouped levels)
    const int bnt = (a.bn == 128 && a.ncols % 128 == 0) ? 128 : BN;
    const int rowtiles = (a.Kp + BMsel - 1) / BMsel, coltiles = a.ncols / bnt;
    const int64_t base = (int64_t)rowtiles * coltiles;
    const int resident = num_sms * (bnt == 128 ? 1 : 2);
    // enough units for ~32 per resident CTA (dynamic scheduling evens them out), each
    // still at least gemm_min_iters (default 16) iterations long (shorter units measured
    // slower at cfg2: more partials to reduce, no gain on the small levels)
    const int64_t iters = (int64_t)a.nslots * (a.Kp / BK);
    const Tuning &tu = tuning();
    const int64_t want = tu.gemm_units_per_cta * resident;
    int nsplit = 1;
    // pseudo-inverse factors (one slot) on grids smaller than the resident CTAs (the top
    // levels: 1-512 columns) are latency-bound -- shorter units spread them over the machine
    // (measured at cfg2: pinv 1.06 -> 0.91 ms per direction with 4; the 8-slot M2M / L2L
    // lose with shorter units: more partials to reduce)
    const int64_t mi = (base < resident && a.nslots == 1) ? tu.gemm_min_iters_small : tu.gemm_min_iters;
    if (base < want)
        nsplit = (int)std::min<int64_t>({(want + base - 1) / base, std::max<int64_t>(1, iters / mi), 64});
    nsplit = std::max(nsplit, 1);
    KParams kp{};
    kp.a = a;
    kp.nsplit = nsplit;
    kp.rowtiles = rowtiles;
    kp.coltiles = coltiles;
    kp.total_units = (int)(base * nsplit);
    // one to a few waves of tiles that the uniform split would cut: the hybrid schedule, when
    // its tail chunks are still at least gemm_min_iters long
    bool hybrid = false;
    const bool sub_wave = base < resident && a.nslots == 1 && base * iters / resident >= 2 * tu.gemm_min_iters_small;
    if (tu.gemm_hybrid && nsplit > 1 && (base >= resident || sub_wave) && base < 8 * (int64_t)resident &&
        base % resident != 0 && (sub_wave || (base % resident) * iters / resident >= tu.gemm_min_iters)) {
        const HybridPlan P = plan_hybrid(ws, rowtiles, coltiles, bnt, resident, (int)iters, st);
        kp.pieces = P.pieces, kp.chunks = P.chunks, kp.tile_parts = P.tile_parts;
        kp.nit_nom = (int)iters;
        kp.reduce_col0 = P.reduce_col0;
        kp.total_units = P.nchunks;
        kp.nsplit = nsplit = std::max(P.maxparts, 1);
        hybrid = P.maxparts > 0;
    }
    if (nsplit > 1 || hybrid) kp.part = ws.get<double>("gemm_part", (size_t)nsplit * a.ncols * a.Kp);
    int launches = 0;
    if (a.src || a.nslots != 1) { // an identity gather's one slot is active in every tile
        int *tslots = ws.get<int>("gemm_tile_slots", (size_t)coltiles * MAX_SLOTS);
        int *tnact = ws.get<int>("gemm_tile_nact", coltiles);
        slot_scan_kernel<<<coltiles, 256, 0, st>>>(a, bnt, tslots, tnact);
        kp.tile_slots = tslots;
        kp.tile_nact = tnact;
        launches = 1;
    }
    kp.counter = zeroed_counters(ws, "gemm_counter", 1, st);
    TmaParams tp;
    std::memset(&tp, 0, sizeof tp);
    tp.kp = kp;
    tp.tmA = operator_map(a.A, a.nmat > 0 ? a.nmat : 1, a.Kp, BMsel);
    const unsigned grid = (unsigned)std::min<int64_t>(kp.total_units, resident);
    if (bnt == 128) {
        constexpr auto k = gather_gemm_tma_kernel<128, tma_stages<128>(), 128, 16>;
        set_smem(k, tma_smem_bytes<128>());
        k<<<grid, 17 * 32, tma_smem_bytes<128>(), st>>>(tp);
    } else {
        constexpr auto k = gather_gemm_tma_kernel<128, tma_stages<64>(), 64, 8>;
        set_smem(k, tma_smem_bytes<64>());
        k<<<grid, 9 * 32, tma_smem_bytes<64>(), st>>>(tp);
    }
    PK_CUDA(cudaGetLastError());
    launches++;
    if (nsplit > 1 || hybrid) {
        const int64_t total = (int64_t)(a.ncols - kp.reduce_col0) * a.Kp;
        split_reduce_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, num_sms * 16), 256, 0, st>>>(kp, BMsel,
                                                                                                            bnt);
        PK_CUDA(cudaGetLastError());
        launches++;
    }
    return launches;
}

void gemv(const double *A, int rows, int cols, int lda, const double *x, double *y, double alpha, double beta,
          const double *rdiv, double rdiv_eps, cudaStream_t st) {
    gemv_kernel<<<(rows + 7) / 8, 256, 0, st>>>(A, rows, cols, lda, x, y, alpha, beta, rdiv, rdiv_eps);
    PK_CUDA(cudaGetLastError());
}

} // namespace pkgpu
