// M2L on the int8 tensor pipe (see m2l_i8.h for the arithmetic).
//
// Kernel m2l_i8_kernel: persistent, one CTA per SM, 7 warps.
//   Tile: 128 gathered boxes (MMA M) x Nt operator rows (MMA N, Nt <= 256, Ki / Nt tiles)
//   per modulus, reduced over the tile's active V-list slots x 128-byte k-chunks.
//   warps 0-1  producers: per stage, 16 cp.async of 16 B per thread gather the 128 box
//              residue rows (128 B each, 128B swizzle applied by hand: chunk c of row j
//              lands at j*128 + ((c ^ (j & 7)) << 4)); thread 0 also issues the TMA 3D
//              load of the Nt x 128 operator residue tile (hardware 128B swizzle).
//              Completion: cp.async.mbarrier.arrive.noinc x 64 + expect_tx on "full".
//   warp 2     MMA issuer: allocates 512 TMEM columns (two 128 x 256 int32 accumulators);
//              one thread waits "full", fences the cp.async (generic proxy) writes into
//              the async proxy, issues 4 x tcgen05.mma.cta_group::1.kind::i8 (K = 32 B
//              each) and tcgen05.commit's the stage back to "empty".
//   warps 3-6  epilogue: tcgen05.ld (lane quarter = warp % 4: 32 boxes) 32 columns at a
//              time, reduce mod m_t, transpose through shared memory and red.add into
//              R[t][col][row] with 128-byte coalesced atomics; the second accumulator
//              lets the next unit's MMAs run meanwhile.
// Work unit = (modulus, operator row tile, 128-column tile, chunk of the tile's active
// slots); chunks keep |int32 accumulator| <= slots * Ki * 128^2 < 2^31.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include <cudaTypedefs.h>

#include "gemm_tma.cuh"
#include "m2l_i8.h"
#include "tuning.h"

namespace pkgpu {

namespace {

constexpr int BKI = 128;            // k-chunk (bytes = int8 elements) per stage
constexpr int TBM = 128;            // gathered boxes per tile (MMA M)
constexpr int A_BYTES = TBM * BKI;  // gathered tile
constexpr int B_BYTES = 256 * BKI;  // operator tile, Nt <= 256 rows
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NST = 4;
constexpr int NST_MAX = 8;
constexpr int NPROD = 2; // producer warps
constexpr int MMA_WARP = NPROD;
constexpr int NTHREADS = (NPROD + 1 + 4) * 32;
constexpr int MAX_SLOTS = 320;
constexpr int EPI_PITCH = 33; // transpose tile row pitch (ints), conflict-free

const int kModuli[kI8MaxModuli] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227,
                                   223, 217, 211, 199, 197, 193, 191, 181, 179, 173};

__constant__ int c_mod[kI8MaxModuli];
__constant__ int c_pm[kI8MaxModuli][kI8MaxModuli]; // (prod_{s' < s} m_s') mod m_t, s < t
__constant__ int c_pinv[kI8MaxModuli];              // (prod_{s < t} m_s)^-1 mod m_t
__constant__ int c_c21[kI8MaxModuli], c_c42[kI8MaxModuli]; // 2^21 mod m_t, 2^42 mod m_t
__constant__ float c_finv[kI8MaxModuli];            // 1 / m_t

struct Params {
    CUtensorMap tmB; // operators: (Ki, Ki, nmod * nmat) int8, box (128, Nt, 1), 128B swizzle
    const int8_t *X; // box residues [nmod][rows_per_mod][Ki]
    const int *src;
    int64_t ld_src, box0;
    int zero_row, rows_per_mod;
    const int *tile_slots, *tile_nact;
    const int *tile_below; // [tile][MAX_SLOTS + 1]: active slots of the tile with index < s
    int nslots, by_index;
    int direct; // single-kernel epilogue stores the partial residues (one unit per output tile)
    const uint8_t *half_mask; // dual kernel: [pair tile][slot] bit h = half h has a source
    const int *tile_partial;  // dual kernel: [pair tile] 1 if some active slot misses a half
    int nmat, nmod, KC, Nt, rowtiles, coltiles, nchunk, total_units, ncols, Ki;
    uint32_t idesc;
    int nst, stage_bytes; // single-CTA kernel: stage ring depth and stride
    int tile_fast;        // unit order: column tile fastest (decode_unit)
    int *sched;           // dynamic schedule: global unit counter (zeroed per launch), or null
    int t_base;           // first modulus of this launch (the small-level run split by modulus across ranks)
    int epi_transpose;    // epilogue atomics through a shared-memory transpose (coalesced)
    int *R; // [nmod][ncols][Ki]
};

// ---- tcgen05 helpers ----
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    // K-major, 128B swizzle: start >> 4, LBO 16 B (unused), SBO 1024 B (8-row groups),
    // descriptor version 1 (bit 46), layout SWIZZLE_128B = 2 (bits 61-63)
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     tma::smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                 "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                   "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                   "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                   "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// warp index the compiler can prove warp-uniform (a shuffle from lane 0): branches on it
// keep the MMA warp's loop on the uniform datapath, so descriptors live in uniform
// registers and tcgen05.mma issues without per-instruction R2UR / waterfall loops
__device__ __forceinline__ int warp_uniform() { return __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0); }
// whole-warp MMA / commit, one elected lane issues (the warp must be converged)
__device__ __forceinline__ void mma_i8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t *bar) {
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                     tma::smem_u32(bar))
                 : "memory");
}

// Chunk c of a column tile = its active slots with slot index in [nslots c / nchunk,
// nslots (c + 1) / nchunk): every tile walks the SAME slot-index window at the same time,
// so the concurrently running units of one (modulus, chunk) share each operator tile
// through L2 instead of streaming it from DRAM once per tile.
// Otherwise (by_index = 0) chunk c = the c-th equal share of the tile's active list: equal
// unit sizes, which the static round-robin schedule of the big levels needs.
__device__ __forceinline__ void chunk_range(const Params &p, int tile, int chunk, int &s0, int &s1) {
    if (p.by_index) {
        const int *below = p.tile_below + tile * (MAX_SLOTS + 1);
        s0 = below[p.nslots * chunk / p.nchunk];
        s1 = below[p.nslots * (chunk + 1) / p.nchunk];
    } else {
        const int nact = p.tile_nact[tile];
        s0 = nact * chunk / p.nchunk;
        s1 = nact * (chunk + 1) / p.nchunk;
    }
}

// unit index -> (modulus t, operator row tile rt, column tile ct, chunk). Default order:
// row tile fastest (concurrent units share their gathered rows); tile_fast: column tile
// fastest (the concurrent units of one (t, rt, chunk) walk the same operator tiles --
// with slot-index chunks, one DRAM read of each tile serves them all through L2)
__device__ __forceinline__ void decode_unit(const Params &p, int u, int ntiles, int &t, int &rt, int &ct, int &chunk) {
    if (p.tile_fast) {
        ct = u % ntiles;
        u /= ntiles;
        rt = u % p.rowtiles;
        u /= p.rowtiles;
    } else {
        rt = u % p.rowtiles;
        u /= p.rowtiles;
        ct = u % ntiles;
        u /= ntiles;
    }
    chunk = u % p.nchunk;
    t = p.t_base + u / p.nchunk;
}

struct Unit {
    int t, rt, ct, s0, s1;
};
__device__ __forceinline__ Unit decode(const Params &p, int u) {
    // row tile fastest: consecutive units (running concurrently) share their gathered rows
    Unit x;
    int chunk;
    decode_unit(p, u, p.coltiles, x.t, x.rt, x.ct, chunk);
    chunk_range(p, x.ct, chunk, x.s0, x.s1);
    return x;
}

__global__ void __launch_bounds__(NTHREADS, 1) m2l_i8_kernel(const __grid_constant__ Params p) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    // stage ring: p.nst stages of p.stage_bytes (16 KB gathered rows + the operator tile)
    const int NS = p.nst, SB = p.stage_bytes;
    int *s_epi = reinterpret_cast<int *>(smem + NS * SB); // [4 warps][32][33] when transposing
    __shared__ __align__(8) uint64_t full[NST_MAX], empty[NST_MAX], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    constexpr int NPT = NPROD * 32;
    if (tid == 0) {
        for (int s = 0; s < NS; s++) {
            tma::mbar_init(&full[s], NPT + 1); // cp.async arrivals + the TMA expect_tx arrival
            tma::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            tma::mbar_init(&tfull[b], 1);
            tma::mbar_init(&tempty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         tma::smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    int g = 0;  // pipeline stages so far
    int jb = 0; // non-empty units so far (accumulator ring position)
    for (int u = blockIdx.x; u < p.total_units; u += gridDim.x) {
        const Unit x = decode(p, u);
        const int n = (x.s1 - x.s0) * p.KC;
        if (n == 0) continue;
        const int *slots = p.tile_slots + x.ct * MAX_SLOTS;
        if (warp < NPROD) {
            // ---------------- producers ----------------
            // thread -> 16-byte chunk c = lane & 7 of rows j = (tid >> 3) + 8 i, i < 16
            const int c = lane & 7, j0 = tid >> 3;
            const int8_t *Xt = p.X + (int64_t)x.t * p.rows_per_mod * p.Ki + c * 16;
            for (int si = x.s0; si < x.s1; si++) {
                const int slot = slots[si];
                const int *srow = p.src + (int64_t)slot * p.ld_src + x.ct * TBM;
                int64_t off[16];
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const int b = srow[j0 + 8 * i];
                    off[i] = (int64_t)(b >= 0 ? (int)(b - p.box0) : p.zero_row) * p.Ki;
                }
                for (int kc = 0; kc < p.KC; kc++) {
                    const int gi = g + (si - x.s0) * p.KC + kc, st = gi % NS;
                    tma::mbar_wait(&empty[st], ((gi / NS) & 1) ^ 1);
                    unsigned char *as = smem + st * SB;
                    if (tid == 0) {
                        tma::mbar_expect_tx(&full[st], p.Nt * BKI);
                        tma::tma_load_4d(as + A_BYTES, &p.tmB, 0, 0, kc, (x.t * p.nmat + slot) * p.rowtiles + x.rt,
                                         &full[st]);
                    }
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int j = j0 + 8 * i;
                        tma::cp_async16(as + j * BKI + ((c ^ (j & 7)) << 4), Xt + off[i] + kc * BKI, 16);
                    }
                    tma::cp_async_mbar_arrive(&full[st]);
                }
            }
        } else if (warp == MMA_WARP) {
            // ---------------- MMA issuer: the whole warp runs the loop (warp-uniform), one
            // elected lane issues each tcgen05.mma / commit ----------------
            const int buf = jb & 1;
            tma::mbar_wait(&tempty[buf], ((jb >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t dt = tmem + buf * 256;
            int st = g % NS;
            uint32_t ph = (g / NS) & 1;
            const uint32_t sbase = tma::smem_u32(smem);
            for (int i = 0; i < n; i++) {
                tma::mbar_wait(&full[st], ph);
                // the gathered rows were written by cp.async through the generic proxy
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                tc_fence_after();
                const uint32_t a0 = sbase + st * SB;
                const uint64_t ad = sw128_desc(a0), bd = sw128_desc(a0 + A_BYTES);
#pragma unroll
                for (int kk = 0; kk < BKI / 32; kk++) // K = 32 bytes per MMA: +2 in the 16-byte start field
                    mma_i8_elect(dt, ad + 2 * kk, bd + 2 * kk, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
                commit_elect(&empty[st]);
                if (++st == NS) st = 0, ph ^= 1;
            }
            commit_elect(&tfull[buf]);
            __syncwarp();
        } else {
            // ---------------- epilogue: TMEM lane = box, column = operator row ----------------
            const int buf = jb & 1, q = warp & 3;
            int *tile = s_epi + (warp - MMA_WARP - 1) * 32 * EPI_PITCH;
            tma::mbar_wait(&tfull[buf], (jb >> 1) & 1);
            tc_fence_after();
            const int m = c_mod[x.t];
            const float inv = 1.0f / (float)m;
            const int col0 = x.ct * TBM + q * 32;
            const int r0 = x.rt * p.Nt;
            const int nr = min(p.Nt, p.Ki - r0);
            int *Rt = p.R + ((int64_t)x.t * p.ncols + col0) * p.Ki + r0;
            for (int j0 = 0; j0 < p.Nt; j0 += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * 256 + j0, v);
                if (!p.epi_transpose) {
                    // direct: thread = box, 32 consecutive rows (one 128-byte line per thread)
                    int *Rb = Rt + (int64_t)lane * p.Ki + j0;
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        const int a = (int)v[j];
                        const int r = a - __float2int_rn((float)a * inv) * m;
                        if (r && j0 + j < nr) atomicAdd(Rb + j, r);
                    }
                    continue;
                }
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    // |a| < 2^31: float quotient is off by at most one; r in (-3m/2, 3m/2)
                    const int a = (int)v[j];
                    tile[lane * EPI_PITCH + j] = a - __float2int_rn((float)a * inv) * m;
                }
                __syncwarp();
                const bool ok = j0 + lane < nr;
#pragma unroll 8
                for (int b = 0; b < 32; b++) {
                    const int r = tile[b * EPI_PITCH + lane]; // box col0 + b, row r0 + j0 + lane
                    if (ok) {
                        if (p.direct)
                            Rt[(int64_t)b * p.Ki + j0 + lane] = r;
                        else if (r)
                            atomicAdd(Rt + (int64_t)b * p.Ki + j0 + lane, r);
                    }
                }
                __syncwarp();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&tempty[buf]);
        }
        g += n;
        jb++;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
    }
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(tma::smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void remote_arrive(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// CTA-scope release (the PTX default): what a stage relay needs -- the relaying thread has
// observed the stage's cp.async completion on its own barrier
__device__ __forceinline__ void remote_arrive_cta(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

// ---------------------------------------------------------------------------
// Dynamic unit schedule (p.sched != null): one scheduler warp per CTA / CTA pair hands out
// unit indices from a global counter in increasing order, so the concurrently running units
// always form one contiguous window of the unit order -- with the column-tile-fastest order
// and slot-index chunks, the operator tiles of that window are read from DRAM once and
// served from L2 to every tile (the static round robin lets CTAs drift apart on adaptive
// levels, whose tiles have very different slot counts). Every role warp of both CTAs pops
// the same sequence from a small queue in its own shared memory; slots are released on the
// leader's "empty" barrier (remote arrivals from the peer).
constexpr int UQ = 4;
struct UnitQueue {
    int u[UQ];
    uint64_t full[UQ], empty[UQ];
};
__device__ __forceinline__ void uq_init(UnitQueue &q, unsigned consumers) {
    for (int s = 0; s < UQ; s++) {
        tma::mbar_init(&q.full[s], 1);
        tma::mbar_init(&q.empty[s], consumers);
    }
}
// k-th unit of the sequence (whole warp); `remote`: this CTA is the pair's peer
__device__ __forceinline__ int uq_pop(UnitQueue &q, int k, bool remote) {
    const int s = k % UQ;
    tma::mbar_wait(&q.full[s], (k / UQ) & 1);
    const int u = *reinterpret_cast<volatile int *>(&q.u[s]);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        if (remote)
            remote_arrive(map_to_rank(&q.empty[s], 0));
        else
            tma::mbar_arrive(&q.empty[s]);
    }
    return u;
}
// the scheduler warp (leader CTA): pushes units until it has pushed one >= total
__device__ __forceinline__ void uq_schedule(UnitQueue &q, int *counter, int total, bool pair) {
    for (int k = 0;; k++) {
        const int s = k % UQ;
        tma::mbar_wait(&q.empty[s], ((k / UQ) & 1) ^ 1);
        int u = 0;
        if ((threadIdx.x & 31) == 0) {
            u = min(atomicAdd(counter, 1), total);
            q.u[s] = u;
            tma::mbar_arrive(&q.full[s]);
            if (pair) {
                asm volatile("st.shared::cluster.b32 [%0], %1;\n" ::"r"(map_to_rank(&q.u[s], 1)), "r"(u) : "memory");
                remote_arrive(map_to_rank(&q.full[s], 1));
            }
        }
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= total) break;
    }
}
// ---------------------------------------------------------------------------
// Dual-tile variant (one CTA per SM): a unit covers TWO 128-box column tiles (a 256-column
// pair tile with one slot list) and one operator row tile. Per stage: 2 x 16 KB gathered
// rows (four producer warps) + one Nt x 128 B operator tile, consumed by two M128 x Nt MMAs
// (one per column tile, two TMEM accumulators at columns 0 and 256). Bytes per MAC drop
// from (128 + Nt) / (128 Nt) to (256 + Nt) / (256 Nt): 60 KB per 2 x 3.7 M MACs at Nt =
// 224, which the per-SM L2 ingest (~69 B/clk measured) sustains at the MMA rate. The
// accumulators fill TMEM, so the epilogue of a unit is not overlapped with the next.
constexpr int DUAL_NPROD = 4;
constexpr int DUAL_MMA_WARP = DUAL_NPROD;
constexpr int DUAL_THREADS = (DUAL_NPROD + 1 + 4) * 32;
constexpr int DUAL_SCHED_WARP = DUAL_THREADS / 32;    // warp 9: unit scheduler (dynamic schedule)
constexpr int DUAL_THREADS_DYN = DUAL_THREADS + 32;
constexpr int DUAL_A_BYTES = 2 * A_BYTES;
constexpr int DUAL_STAGE = DUAL_A_BYTES + B_BYTES;
constexpr int DUAL_NST = 3;

__global__ void __launch_bounds__(DUAL_THREADS_DYN, 1) m2l_i8_dual_kernel(const __grid_constant__ Params p) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    int *s_epi = reinterpret_cast<int *>(smem + DUAL_NST * DUAL_STAGE); // [4 warps][32][33]
    __shared__ __align__(8) uint64_t full[DUAL_NST], empty[DUAL_NST], tfull, tempty;
    __shared__ UnitQueue uq;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    constexpr int NPT = DUAL_NPROD * 32;
    const bool dyn = p.sched != nullptr;
    if (tid == 0) {
        for (int s = 0; s < DUAL_NST; s++) {
            tma::mbar_init(&full[s], NPT + 1);
            tma::mbar_init(&empty[s], 1);
        }
        tma::mbar_init(&tfull, 1);
        tma::mbar_init(&tempty, 4);
        uq_init(uq, DUAL_THREADS / 32);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == DUAL_MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         tma::smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    int g = 0, jb = 0;
    const int npairs = p.coltiles / 2;
    if (warp == DUAL_SCHED_WARP) {
        if (dyn) uq_schedule(uq, p.sched, p.total_units, false);
    } else
    for (int k = 0, us = blockIdx.x;; k++, us += gridDim.x) {
        const int u = dyn ? uq_pop(uq, k, false) : us;
        if (u >= p.total_units) break;
        int t, rt, pr, chunk;
        decode_unit(p, u, npairs, t, rt, pr, chunk);
        int s0, s1;
        chunk_range(p, pr, chunk, s0, s1);
        const int n = (s1 - s0) * p.KC;
        if (n == 0) continue;
        const int *slots = p.tile_slots + pr * MAX_SLOTS;
        const int colp = pr * 2 * TBM; // first of the 256 columns
        if (warp < DUAL_NPROD) {
            // ---------------- producers: 256 rows, 16 cp.async of 16 B per thread ----------------
            const int c = lane & 7, j0 = tid >> 3; // rows j0 + 16 i, i < 16
            const int8_t *Xt = p.X + (int64_t)t * p.rows_per_mod * p.Ki + c * 16;
            for (int si = s0; si < s1; si++) {
                const int slot = slots[si];
                const int *srow = p.src + (int64_t)slot * p.ld_src + colp;
                // halves without a source for this slot are neither gathered nor multiplied
                const int hm = p.half_mask[pr * MAX_SLOTS + slot]; // loaded alongside the rows (no extra latency)
                int bx[16];
#pragma unroll
                for (int i = 0; i < 16; i++) bx[i] = srow[j0 + 16 * i];
                int64_t off[16];
#pragma unroll
                for (int i = 0; i < 16; i++)
                    off[i] = (int64_t)(bx[i] >= 0 ? (int)(bx[i] - p.box0) : p.zero_row) * p.Ki;
                for (int kc = 0; kc < p.KC; kc++) {
                    const int gi = g + (si - s0) * p.KC + kc, st = gi % DUAL_NST;
                    tma::mbar_wait(&empty[st], ((gi / DUAL_NST) & 1) ^ 1);
                    unsigned char *as = smem + st * DUAL_STAGE;
                    if (tid == 0) {
                        tma::mbar_expect_tx(&full[st], p.Nt * BKI);
                        tma::tma_load_4d(as + DUAL_A_BYTES, &p.tmB, 0, 0, kc, (t * p.nmat + slot) * p.rowtiles + rt,
                                         &full[st]);
                    }
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int j = j0 + 16 * i; // rows 0..127: tile 0, 128..255: tile 1 (contiguous)
                        if ((hm >> (i >> 3)) & 1)
                            tma::cp_async16(as + j * BKI + ((c ^ (j & 7)) << 4), Xt + off[i] + kc * BKI, 16);
                    }
                    tma::cp_async_mbar_arrive(&full[st]);
                }
            }
        } else if (warp == DUAL_MMA_WARP) {
            // ---------------- MMA issuer: two M128 x Nt MMAs per k-step (whole warp,
            // elected lane issues) ----------------
            tma::mbar_wait(&tempty, (jb & 1) ^ 1);
            tc_fence_after();
            int st = g % DUAL_NST;
            uint32_t ph = (g / DUAL_NST) & 1;
            const uint32_t sbase = tma::smem_u32(smem);
            bool started0 = false, started1 = false; // first MMA of a half overwrites its accumulator
            const uint8_t *hmt = p.half_mask + pr * MAX_SLOTS;
            // tiles whose every active slot feeds both halves (uniform levels) take the
            // unconditional loop; the masked one costs a few percent per stage
            if (__reduce_or_sync(0xffffffffu, (unsigned)p.tile_partial[pr]) == 0u) {
                for (int i = 0; i < n; i++) {
                    tma::mbar_wait(&full[st], ph);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    tc_fence_after();
                    const uint32_t a0 = sbase + st * DUAL_STAGE;
                    const uint64_t ad0 = sw128_desc(a0), ad1 = sw128_desc(a0 + A_BYTES),
                                   bd = sw128_desc(a0 + DUAL_A_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BKI / 32; kk++) {
                        const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                        mma_i8_elect(tmem, ad0 + 2 * kk, bd + 2 * kk, p.idesc, acc);
                        mma_i8_elect(tmem + 256, ad1 + 2 * kk, bd + 2 * kk, p.idesc, acc);
                    }
                    commit_elect(&empty[st]);
                    if (++st == DUAL_NST) st = 0, ph ^= 1;
                }
                commit_elect(&tfull);
                __syncwarp();
                g += n;
                jb++;
                continue;
            }
            int hm = hmt[slots[s0]];
            int hm_next = s0 + 1 < s1 ? hmt[slots[s0 + 1]] : 0;
            for (int i = 0, kc = 0, si = s0; i < n; i++) {
                tma::mbar_wait(&full[st], ph);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                tc_fence_after();
                const uint32_t a0 = sbase + st * DUAL_STAGE;
                const uint64_t ad0 = sw128_desc(a0), ad1 = sw128_desc(a0 + A_BYTES), bd = sw128_desc(a0 + DUAL_A_BYTES);
                // REDUX writes a uniform register: the conditional MMAs stay on the uniform datapath
                // (a branch on a loaded value would bring back the per-MMA R2UR waterfall)
                const unsigned hu = __reduce_or_sync(0xffffffffu, (unsigned)hm);
                const bool on0 = (hu & 1u) != 0, on1 = (hu & 2u) != 0;
#pragma unroll
                for (int kk = 0; kk < BKI / 32; kk++) {
                    if (on0) mma_i8_elect(tmem, ad0 + 2 * kk, bd + 2 * kk, p.idesc, (started0 || kk > 0) ? 1u : 0u);
                    if (on1) mma_i8_elect(tmem + 256, ad1 + 2 * kk, bd + 2 * kk, p.idesc, (started1 || kk > 0) ? 1u : 0u);
                }
                started0 |= on0;
                started1 |= on1;
                commit_elect(&empty[st]);
                if (++st == DUAL_NST) st = 0, ph ^= 1;
                if (++kc == p.KC) { // next slot: its mask was loaded a slot ahead
                    kc = 0;
                    si++;
                    hm = hm_next;
                    hm_next = si + 1 < s1 ? hmt[slots[si + 1]] : 0;
                }
            }
            commit_elect(&tfull);
            __syncwarp();
        } else {
            // ---------------- epilogue: both accumulators ----------------
            const int q = warp & 3;
            int *tile = s_epi + (warp - DUAL_MMA_WARP - 1) * 32 * EPI_PITCH;
            tma::mbar_wait(&tfull, jb & 1);
            tc_fence_after();
            const int m = c_mod[t];
            const float inv = 1.0f / (float)m;
            const int r0 = rt * p.Nt;
            const int nr = min(p.Nt, p.Ki - r0);
            int used = 0; // halves that received an MMA in this unit (others hold stale TMEM)
            for (int si = s0 + lane; si < s1; si += 32) used |= p.half_mask[pr * MAX_SLOTS + slots[si]];
            for (int o = 16; o; o >>= 1) used |= __shfl_xor_sync(0xffffffffu, used, o);
            for (int h = 0; h < 2; h++) {
                if (!((used >> h) & 1)) continue;
                int *Rt = p.R + ((int64_t)t * p.ncols + colp + h * TBM + q * 32) * p.Ki + r0;
                for (int j0 = 0; j0 < p.Nt; j0 += 32) {
                    uint32_t vv[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + h * 256 + j0, vv);
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        const int a = (int)vv[j];
                        tile[lane * EPI_PITCH + j] = a - __float2int_rn((float)a * inv) * m;
                    }
                    __syncwarp();
                    const bool ok = j0 + lane < nr;
#pragma unroll 8
                    for (int b = 0; b < 32; b++) {
                        const int r = tile[b * EPI_PITCH + lane];
                        if (ok && r) atomicAdd(Rt + (int64_t)b * p.Ki + j0 + lane, r);
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&tempty);
        }
        g += n;
        jb++;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == DUAL_MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
    }
}

// ---------------------------------------------------------------------------
// Pair-dual (cluster of 2, cta_group::2): a 512-column quad per unit, two M256 x Nt MMAs per
// k-step issued by the leader. MMA h covers quad columns 256 h .. 256 h + 255: its rows
// 0-127 come from CTA 0's shared memory, 128-255 from CTA 1's, and each CTA holds half of
// the operator tile (Nt / 2 rows). Per SM and stage: 256 gathered rows + Nt / 2 operator
// rows (46 KB at Nt = 224) for the same MACs as the dual kernel's 256 + Nt rows (60 KB) --
// the dual kernel is bound by the per-SM L2 ingest, so the MMA rate rises with it.
// Both CTAs gather with cp.async onto their own "full" barrier; the peer's MMA-warp lane
// relays its completed stages to the leader ("pfull"), which issues once both are in and
// commits "empty" / "tfull" to both CTAs (multicast). Quarter masks (bit b = quad columns
// 128 b .. 128 b + 127 have a source) pick which MMAs run: MMA h if bit 2h or 2h+1.
__device__ __forceinline__ void mma_i8_pair_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// commit to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void commit_pair_elect(uint64_t *bar) {
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
                     tma::smem_u32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}
constexpr int PD_B_BYTES = 128 * BKI; // half operator tile, Nt / 2 <= 128 rows
constexpr int PD_NA = 4;               // gathered-row ring (32 KB stages)
constexpr int PD_NB = 5;               // operator ring (16 KB stages): runs further ahead
constexpr int PD_OPER_WARP = DUAL_THREADS / 32; // warp 9: operator TMA producer
constexpr int PD_SCHED_WARP = PD_OPER_WARP + 1;         // warp 10: unit scheduler (leader, dynamic schedule)
constexpr int PD_THREADS = DUAL_THREADS + 64;
constexpr size_t PD_RING_BYTES = (size_t)PD_NA * DUAL_A_BYTES + (size_t)PD_NB * PD_B_BYTES;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PD_THREADS, 1)
    m2l_i8_pairdual_kernel(const __grid_constant__ Params p) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    unsigned char *ringB = smem + PD_NA * DUAL_A_BYTES;
    int *s_epi = reinterpret_cast<int *>(smem + PD_RING_BYTES); // [4 warps][32][33]
    __shared__ __align__(8) uint64_t fullA[PD_NA], pfullA[PD_NA], emptyA[PD_NA], fullB[PD_NB], emptyB[PD_NB], tfull,
        tempty;
    __shared__ UnitQueue uq;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    constexpr int NPT = DUAL_NPROD * 32;
    const int half = p.Nt / 2;
    if (tid == 0) {
        for (int s = 0; s < PD_NA; s++) {
            tma::mbar_init(&fullA[s], NPT);  // local cp.async arrivals
            tma::mbar_init(&pfullA[s], 1);   // leader: the peer's relayed "rows landed"
            tma::mbar_init(&emptyA[s], 1);   // the leader's multicast MMA commit
        }
        for (int s = 0; s < PD_NB; s++) {
            tma::mbar_init(&fullB[s], 1);    // leader: its expect_tx (both halves' bytes land on it)
            tma::mbar_init(&emptyB[s], 1);   // the leader's multicast MMA commit
        }
        tma::mbar_init(&tfull, 1);
        tma::mbar_init(&tempty, 8); // leader: 4 local + 4 remote epilogue warps
        uq_init(uq, 2 * (PD_OPER_WARP + 1)); // leader: the role warps of both CTAs
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == DUAL_MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         tma::smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    int g = 0, jb = 0;
    const int nquads = p.coltiles / 4;
    const bool dyn = p.sched != nullptr;
    if (warp == PD_SCHED_WARP) {
        if (dyn && leader) uq_schedule(uq, p.sched, p.total_units, true);
    } else
    for (int k = 0, us = blockIdx.x / 2;; k++, us += gridDim.x / 2) {
        const int u = dyn ? uq_pop(uq, k, !leader) : us;
        if (u >= p.total_units) break;
        int t, rt, qd, chunk;
        decode_unit(p, u, nquads, t, rt, qd, chunk);
        int s0, s1;
        chunk_range(p, qd, chunk, s0, s1);
        const int n = (s1 - s0) * p.KC;
        if (n == 0) continue;
        const int *slots = p.tile_slots + qd * MAX_SLOTS;
        const int colq = qd * 4 * TBM;
        const uint8_t *hmt = p.half_mask + qd * MAX_SLOTS;
        if (warp < DUAL_NPROD) {
            // ---------------- gather producers (both CTAs): this CTA's 128 rows of each MMA ----------------
            const int c = lane & 7, j0 = tid >> 3; // stage rows j0 + 16 i, i < 16 (row j: MMA j / 128)
            const int8_t *Xt = p.X + (int64_t)t * p.rows_per_mod * p.Ki + c * 16;
            const int cbase = colq + (int)rank * TBM;
            for (int si = s0; si < s1; si++) {
                const int slot = slots[si];
                const int *srow = p.src + (int64_t)slot * p.ld_src + cbase;
                const int hm = hmt[slot];
                const int on = ((hm & 3) ? 1 : 0) | ((hm & 12) ? 2 : 0);
                int bx[16];
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const int j = j0 + 16 * i;
                    bx[i] = srow[(j & (TBM - 1)) + (j / TBM) * 2 * TBM];
                }
                int64_t off[16];
#pragma unroll
                for (int i = 0; i < 16; i++)
                    off[i] = (int64_t)(bx[i] >= 0 ? (int)(bx[i] - p.box0) : p.zero_row) * p.Ki;
                for (int kc = 0; kc < p.KC; kc++) {
                    const int gi = g + (si - s0) * p.KC + kc, st = gi % PD_NA;
                    tma::mbar_wait(&emptyA[st], ((gi / PD_NA) & 1) ^ 1);
                    unsigned char *as = smem + st * DUAL_A_BYTES;
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int j = j0 + 16 * i;
                        if ((on >> (i >> 3)) & 1)
                            tma::cp_async16(as + j * BKI + ((c ^ (j & 7)) << 4), Xt + off[i] + kc * BKI, 16);
                    }
                    tma::cp_async_mbar_arrive(&fullA[st]);
                }
            }
        } else if (warp == PD_OPER_WARP) {
            // ---------------- operator producer (both CTAs): own half tile, onto the leader's barrier ----------------
            for (int i = 0; i < n; i++) {
                const int gi = g + i, st = gi % PD_NB;
                const int slot = slots[s0 + i / p.KC], kc = i % p.KC;
                tma::mbar_wait(&emptyB[st], ((gi / PD_NB) & 1) ^ 1);
                if (lane == 0) {
                    const uint32_t bar = map_to_rank(&fullB[st], 0);
                    if (leader)
                        asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;\n" ::"r"(bar),
                                     "r"(2 * half * BKI)
                                     : "memory");
                    asm volatile("cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
                                 "bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(tma::smem_u32(ringB + st * PD_B_BYTES)),
                                 "l"(reinterpret_cast<uint64_t>(&p.tmB)), "r"(0), "r"((int)rank * half), "r"(kc),
                                 "r"((t * p.nmat + slot) * p.rowtiles + rt), "r"(bar)
                                 : "memory");
                }
                __syncwarp();
            }
        } else if (warp == DUAL_MMA_WARP) {
            if (!leader) {
                // ---------------- relay (peer): own rows landed -> leader's pfullA ----------------
                for (int i = 0; i < n; i++) {
                    const int gi = g + i, st = gi % PD_NA;
                    tma::mbar_wait(&fullA[st], (gi / PD_NA) & 1);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    if (lane == 0) remote_arrive_cta(map_to_rank(&pfullA[st], 0));
                    __syncwarp();
                }
            } else {
                // ---------------- MMA issuer (leader; whole warp, elected lane) ----------------
                tma::mbar_wait(&tempty, (jb & 1) ^ 1);
                tc_fence_after();
                const uint32_t abase = tma::smem_u32(smem), bbase = tma::smem_u32(ringB);
                // tiles whose every active slot feeds all four quarters issue unconditionally
                const bool all = __reduce_or_sync(0xffffffffu, (unsigned)p.tile_partial[qd]) == 0u;
                bool started0 = false, started1 = false;
                int hm = hmt[slots[s0]];
                int hm_next = s0 + 1 < s1 ? hmt[slots[s0 + 1]] : 0;
                for (int i = 0, kc = 0, si = s0; i < n; i++) {
                    const int gi = g + i, sa = gi % PD_NA, sb = gi % PD_NB;
                    tma::mbar_wait(&fullA[sa], (gi / PD_NA) & 1);
                    tma::mbar_wait(&pfullA[sa], (gi / PD_NA) & 1);
                    tma::mbar_wait(&fullB[sb], (gi / PD_NB) & 1);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    tc_fence_after();
                    const uint32_t a0 = abase + sa * DUAL_A_BYTES;
                    const uint64_t ad0 = sw128_desc(a0), ad1 = sw128_desc(a0 + A_BYTES),
                                   bd = sw128_desc(bbase + sb * PD_B_BYTES);
                    if (all) {
#pragma unroll
                        for (int kk = 0; kk < BKI / 32; kk++) {
                            const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                            mma_i8_pair_elect(tmem, ad0 + 2 * kk, bd + 2 * kk, p.idesc, acc);
                            mma_i8_pair_elect(tmem + 256, ad1 + 2 * kk, bd + 2 * kk, p.idesc, acc);
                        }
                    } else {
                        const unsigned hu = __reduce_or_sync(0xffffffffu, (unsigned)hm);
                        const bool on0 = (hu & 3u) != 0, on1 = (hu & 12u) != 0;
#pragma unroll
                        for (int kk = 0; kk < BKI / 32; kk++) {
                            if (on0)
                                mma_i8_pair_elect(tmem, ad0 + 2 * kk, bd + 2 * kk, p.idesc,
                                                  (started0 || kk > 0) ? 1u : 0u);
                            if (on1)
                                mma_i8_pair_elect(tmem + 256, ad1 + 2 * kk, bd + 2 * kk, p.idesc,
                                                  (started1 || kk > 0) ? 1u : 0u);
                        }
                        started0 |= on0;
                        started1 |= on1;
                        if (++kc == p.KC) {
                            kc = 0;
                            si++;
                            hm = hm_next;
                            hm_next = si + 1 < s1 ? hmt[slots[si + 1]] : 0;
                        }
                    }
                    commit_pair_elect(&emptyA[sa]);
                    commit_pair_elect(&emptyB[sb]);
                }
                commit_pair_elect(&tfull);
            }
            __syncwarp();
        } else {
            // ---------------- epilogue (both CTAs: own 128 lanes of each accumulator) ----------------
            const int q = warp & 3;
            int *tile = s_epi + (warp - DUAL_MMA_WARP - 1) * 32 * EPI_PITCH;
            tma::mbar_wait(&tfull, jb & 1);
            tc_fence_after();
            const int m = c_mod[t];
            const float inv = 1.0f / (float)m;
            const int r0 = rt * p.Nt;
            const int nr = min(p.Nt, p.Ki - r0);
            int used = 0; // MMAs issued in this unit (the others' TMEM is stale)
            for (int si = s0 + lane; si < s1; si += 32) used |= hmt[slots[si]];
            for (int o = 16; o; o >>= 1) used |= __shfl_xor_sync(0xffffffffu, used, o);
            for (int h = 0; h < 2; h++) {
                if (!((used >> (2 * h)) & 3)) continue;
                int *Rt = p.R + ((int64_t)t * p.ncols + colq + h * 2 * TBM + (int)rank * TBM + q * 32) * p.Ki + r0;
                for (int j0 = 0; j0 < p.Nt; j0 += 32) {
                    uint32_t vv[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + h * 256 + j0, vv);
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        const int a = (int)vv[j];
                        tile[lane * EPI_PITCH + j] = a - __float2int_rn((float)a * inv) * m;
                    }
                    __syncwarp();
                    const bool ok = j0 + lane < nr;
#pragma unroll 8
                    for (int b = 0; b < 32; b++) {
                        const int r = tile[b * EPI_PITCH + lane];
                        if (ok && r) atomicAdd(Rt + (int64_t)b * p.Ki + j0 + lane, r);
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) remote_arrive(map_to_rank(&tempty, 0));
        }
        g += n;
        jb++;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == DUAL_MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
    }
}


// active slots per column tile of `bn` columns, in slot order
// half_mask (bn = 256 / 512): bit q set when the 128-column quarter q has a source
__global__ void slot_scan_kernel(const int *__restrict__ src, int64_t ld_src, int nslots, int bn, int *tile_slots,
                                 int *tile_nact, int *tile_below, uint8_t *half_mask, int *tile_partial) {
    __shared__ unsigned qm[MAX_SLOTS];
    const int ct = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < nslots; s += blockDim.x / 32) {
        unsigned m = 0; // bit q: the 128-column quarter q of the tile has a source
#pragma unroll 4
        for (int j = lane; j < bn; j += 32)
            if (src[(int64_t)s * ld_src + (int64_t)ct * bn + j] >= 0) m |= 1u << (j / TBM);
        m = __reduce_or_sync(0xffffffffu, m);
        if (lane == 0) {
            qm[s] = m;
            if (half_mask) half_mask[ct * MAX_SLOTS + s] = (uint8_t)m;
        }
    }
    __syncthreads();
    if (warp == 0) { // active-slot list, "below" prefix counts and the partial flag, 32 slots per step
        int n = 0;
        unsigned partial = 0;
        int *below = tile_below + ct * (MAX_SLOTS + 1);
        const unsigned fullm = (1u << (bn / TBM)) - 1;
        for (int s0 = 0; s0 < nslots; s0 += 32) {
            const int s = s0 + lane;
            const unsigned m = s < nslots ? qm[s] : 0u;
            const unsigned bal = __ballot_sync(0xffffffffu, m != 0);
            const int pre = n + __popc(bal & ((1u << lane) - 1));
            if (s < nslots) {
                below[s] = pre;
                if (m) tile_slots[ct * MAX_SLOTS + pre] = s;
            }
            partial |= (m && m != fullm) ? 1u : 0u;
            n += __popc(bal);
        }
        partial = __reduce_or_sync(0xffffffffu, partial);
        if (lane == 0) {
            below[nslots] = n;
            tile_nact[ct] = n;
            if (tile_partial) tile_partial[ct] = (int)partial;
        }
    }
}

// ---- residues ----
__device__ __forceinline__ int mod_pos(long long a, int m, double inv) {
    // a in (-2^50, 2^50): floor division in double, one correction step
    long long q = (long long)floor((double)a * inv);
    long long r = a - q * m;
    if (r < 0) r += m;
    if (r >= m) r -= m;
    return (int)r;
}
__device__ __forceinline__ int mod_small(int a, int m, float inv) {
    // |a| < 2^22: float quotient off by at most one
    int r = a - __float2int_rd((float)a * inv) * m;
    if (r < 0) r += m;
    if (r >= m) r -= m;
    return r;
}
__device__ __forceinline__ int balanced(int r, int m) { return r >= (m + 1) / 2 ? r - m : r; }

// residues of v (|v| <= 2^62) for all moduli, via v = a2 2^42 + a1 2^21 + a0: the folded
// value a2 (2^42 mod m) + a1 (2^21 mod m) + a0 has |.| < 2^30, reduced with a float quotient
// (off by at most one or two) and corrections -- 32-bit integer work only
__device__ __forceinline__ void residues(long long v, int nmod, int8_t *out, int64_t stride) {
    const int a0 = (int)(v & ((1ll << 21) - 1)), a1 = (int)((v >> 21) & ((1ll << 21) - 1)), a2 = (int)(v >> 42);
    for (int t = 0; t < nmod; t++) {
        const int m = c_mod[t];
        const int f = a2 * c_c42[t] + a1 * c_c21[t] + a0;
        int r = f - __float2int_rd(__int2float_rn(f) * c_finv[t]) * m;
        if (r < 0) r += m;
        if (r < 0) r += m;
        if (r >= m) r -= m;
        if (r >= m) r -= m;
        out[t * stride] = (int8_t)balanced(r, m);
    }
}

__global__ void rowmax_kernel(const double *__restrict__ A, int nmat, int K, int Kp, unsigned long long *mx) {
    const int r = blockIdx.x, o = blockIdx.y;
    double m = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(A[((size_t)o * Kp + r) * Kp + k]));
    for (int s = 16; s; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) atomicMax(&mx[r], (unsigned long long)__double_as_longlong(m));
}

__global__ void rowexp_kernel(const unsigned long long *__restrict__ mx, int K, int Ki, int *rowexp) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= Ki) return;
    const double m = r < K ? __longlong_as_double((long long)mx[r]) : 0.0;
    rowexp[r] = m > 0 ? ilogb(m) + 1 : 0;
}

// operator residues, tile-contiguous: [t][mat][row tile][k chunk][Nt rows][128 B], so every
// TMA box (an Nt x 128 B operator tile, or half of it) is one contiguous range
__global__ void op_residue_kernel(const double *__restrict__ A, int nmat, int K, int Kp, int Ki, int nmod, int beta,
                                  const int *__restrict__ rowexp, int Nt, int rowtiles, int8_t *__restrict__ res) {
    const int r = blockIdx.x, o = blockIdx.y; // r < rowtiles * Nt
    const int KC = Ki / 128;
    const int64_t stride = (int64_t)nmat * rowtiles * KC * Nt * 128;
    const int rt = r / Nt, rr = r % Nt;
    int8_t *out = res + (((int64_t)o * rowtiles + rt) * KC * Nt + rr) * 128;
    for (int k = threadIdx.x; k < Ki; k += blockDim.x) {
        const double a = (r < K && k < K) ? A[((size_t)o * Kp + r) * Kp + k] : 0.0;
        residues(llrint(ldexp(a, beta - (r < K ? rowexp[r] : 0))), nmod, out + (int64_t)(k / 128) * Nt * 128 + (k % 128),
                 stride);
    }
}

// plain [t][mat][Ki][Ki] int8 -> the tile-contiguous layout (the i8_gather_gemm test entry)
__global__ void op_tile_kernel(const int8_t *__restrict__ A, int nmm, int Ki, int Nt, int rowtiles,
                               int8_t *__restrict__ out) {
    const int r = blockIdx.x, o = blockIdx.y; // o < nmod * nmat
    const int KC = Ki / 128, rt = r / Nt, rr = r % Nt;
    (void)nmm;
    for (int k = threadIdx.x; k < Ki; k += blockDim.x)
        out[(((int64_t)o * rowtiles + rt) * KC + k / 128) * Nt * 128 + (int64_t)rr * 128 + k % 128] =
            r < Ki ? A[((int64_t)o * Ki + r) * Ki + k] : 0;
}

__global__ void level_absmax_kernel(const double *__restrict__ X, int64_t nbox, int K, int Kp,
                                    unsigned long long *mx) {
    double m = 0;
    const int64_t n = nbox * Kp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (i % Kp < K) m = fmax(m, fabs(X[i]));
    for (int s = 16; s; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) atomicMax(mx, (unsigned long long)__double_as_longlong(m));
}

__device__ __forceinline__ int level_exp(const unsigned long long *mx) {
    const double m = __longlong_as_double((long long)*mx);
    return m > 0 ? ilogb(m) + 1 : 0;
}

// level of an index in a run of ranges start[0] <= ... < start[n]
__device__ __forceinline__ int level_of(const int64_t *start, int n, int64_t i) {
    int l = 0;
    while (l + 1 < n && i >= start[l + 1]) l++;
    return l;
}

// Xres[t][i][k] for boxes i < nbox of the run (row nbox: zeros), scaled by the box's level
__global__ void x_residue_kernel(const double *__restrict__ X, int64_t nbox, int K, int Kp, int Ki, int nmod,
                                 int beta, const unsigned long long *__restrict__ mx, I8Levels lv,
                                 int8_t *__restrict__ res) {
    const int64_t rows = nbox + 1, n = rows * Ki, stride = rows * Ki;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / Ki;
        const int k = (int)(i % Ki);
        double x = 0.0;
        int e = 0;
        if (b < nbox && k < K) {
            x = X[b * Kp + k];
            e = level_exp(mx + level_of(lv.box0, lv.n, lv.box0[0] + b));
        }
        residues(llrint(ldexp(x, beta - e)), nmod, res + i, stride);
    }
}

// Garner (balanced mixed-radix digits) + Horner in FP64:
//   Y[out(c)][r] += alpha 2^(e_r + E - beta_a - beta_b) S,  R = [t][c][r]
template <int NM>
__global__ void reconstruct_kernel(const int *__restrict__ R, int ncols, int Ki, int K, int Kp,
                                   const int *__restrict__ out_box, int64_t col_off, const int *__restrict__ rowexp,
                                   const unsigned long long *__restrict__ mx, int beta_sum, I8Levels lv,
                                   double *__restrict__ Y) {
    const int64_t n = (int64_t)ncols * Ki;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / Ki), r = (int)(i % Ki);
        if (r >= K) continue;
        const int ob = out_box[c];
        if (ob < 0) continue;
        const int l = level_of(lv.col0, lv.n, c + col_off);
        const int E = level_exp(mx + l);
        const double alpha = lv.alpha[l];
        int x[NM], acc[NM], v[NM];
#pragma unroll
        for (int t = 0; t < NM; t++) {
            x[t] = R[(int64_t)t * n + i];
            acc[t] = 0;
        }
#pragma unroll
        for (int t = 0; t < NM; t++) {
            const int m = c_mod[t];
            const float inv = c_finv[t];
            const int d = mod_small(x[t] - acc[t], m, inv);
            v[t] = balanced(mod_small(d * c_pinv[t], m, inv), m);
#pragma unroll
            for (int s = t + 1; s < NM; s++) acc[s] += v[t] * c_pm[t][s];
        }
        double h = v[NM - 1];
#pragma unroll
        for (int t = NM - 2; t >= 0; t--) h = fma(h, (double)c_mod[t], (double)v[t]);
        Y[(int64_t)ob * Kp + r] += alpha * ldexp(h, rowexp[r] + E - beta_sum);
    }
}

// ---- i8_translate: per-column fixed-point scale ----
// Block per column c: E_c from max |X| over the column's sources, then the residues of those
// source rows at scale 2^(beta - E_c) (a source shared by several columns is written with
// the same E by each of them), and R[.][c][.] = 0. Block 0 also zeroes the zero row.
__global__ void tr_prepare_kernel(const int *__restrict__ src, int64_t ld_src, int nslots, int64_t src_lo,
                                  int64_t nsrc, const double *__restrict__ X, int K, int Kp, int Ki, int nmod, int beta,
                                  int ncols, int8_t *__restrict__ xres, int *__restrict__ ecol, int *__restrict__ R,
                                  int zero_r) {
    __shared__ double red[32];
    __shared__ int sb[8];
    const int c = blockIdx.x, tid = threadIdx.x;
    const int64_t stride = (nsrc + 1) * Ki;
    if (tid < nslots) sb[tid] = src[(int64_t)tid * ld_src + c];
    __syncthreads();
    double m = 0.0;
    for (int s = 0; s < nslots; s++) {
        const int b = sb[s];
        if (b < 0) continue;
        for (int k = tid; k < K; k += blockDim.x) m = fmax(m, fabs(X[(int64_t)b * Kp + k]));
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    if (tid < 32) {
        m = tid < (int)(blockDim.x >> 5) ? red[tid] : 0.0;
        for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (tid == 0) red[0] = m;
    }
    __syncthreads();
    m = red[0];
    const int E = m > 0 ? ilogb(m) + 1 : 0;
    if (tid == 0) ecol[c] = E;
    for (int s = 0; s < nslots; s++) {
        const int b = sb[s];
        if (b < 0) continue;
        int8_t *row = xres + (int64_t)(b - src_lo) * Ki;
        for (int k = tid; k < Ki; k += blockDim.x) {
            const double x = k < K ? X[(int64_t)b * Kp + k] : 0.0;
            residues(llrint(ldexp(x, beta - E)), nmod, row + k, stride);
        }
    }
    if (zero_r)
        for (int t = 0; t < nmod; t++)
            for (int k = tid; k < Ki; k += blockDim.x) R[((int64_t)t * ncols + c) * Ki + k] = 0;
    if (c == 0)
        for (int i = tid; i < nmod * Ki; i += blockDim.x) xres[(int64_t)(i / Ki) * stride + nsrc * Ki + i % Ki] = 0;
}

// CRT rebuild of one residue vector (Garner balanced mixed radix, Horner in FP64)
template <int NM> __device__ __forceinline__ double crt_value(const int *__restrict__ R, int64_t i, int64_t n) {
    int x[NM], acc[NM], v[NM];
#pragma unroll
    for (int t = 0; t < NM; t++) {
        x[t] = R[(int64_t)t * n + i];
        acc[t] = 0;
    }
#pragma unroll
    for (int t = 0; t < NM; t++) {
        const int m = c_mod[t];
        const float inv = c_finv[t];
        const int d = mod_small(x[t] - acc[t], m, inv);
        v[t] = balanced(mod_small(d * c_pinv[t], m, inv), m);
#pragma unroll
        for (int s = t + 1; s < NM; s++) acc[s] += v[t] * c_pm[t][s];
    }
    double h = v[NM - 1];
#pragma unroll
    for (int t = NM - 2; t >= 0; t--) h = fma(h, (double)c_mod[t], (double)v[t]);
    return h;
}

template <int NM>
__global__ void tr_finish_kernel(const int *__restrict__ R, int ncols, int Ki, int K, int Kp,
                                 const int *__restrict__ out_box, const int *__restrict__ rowexp,
                                 const int *__restrict__ ecol, int beta_sum, double alpha, double beta,
                                 const double *__restrict__ rdiv, double rdiv_eps, double *__restrict__ Y) {
    const int64_t n = (int64_t)ncols * Ki;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / Ki), r = (int)(i % Ki);
        if (r >= K) continue;
        const int ob = out_box[c];
        if (ob < 0) continue;
        const double v = ldexp(crt_value<NM>(R, i, n), rowexp[r] + ecol[c] - beta_sum);
        double *y = Y + (int64_t)ob * Kp + r;
        if (rdiv) {
            const double d = rdiv[r];
            *y = d > rdiv_eps ? v / d : 0.0;
        } else {
            *y = (beta != 0.0 ? beta * *y : 0.0) + alpha * v;
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        PK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
        if (!ptr || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// CRT tables: pm[s][t] = prod_{s' < s} m_s' mod m_t ; pinv[t] = (prod_{s < t} m_s)^-1 mod m_t
void upload_tables() {
    static int dev_done[64] = {0};
    int dev = 0;
    PK_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && dev_done[dev]) return;
    int pm[kI8MaxModuli][kI8MaxModuli] = {}, pinv[kI8MaxModuli] = {};
    for (int t = 0; t < kI8MaxModuli; t++) {
        const int m = kModuli[t];
        long long P = 1 % m;
        for (int s = 0; s < t; s++) {
            pm[s][t] = (int)P;
            P = P * (kModuli[s] % m) % m;
        }
        int inv = 0;
        for (int c = 1; c < m; c++)
            if ((P * c) % m == 1) inv = c;
        if (t > 0 && inv == 0) throw RuntimeError("m2l_i8: moduli not coprime");
        pinv[t] = t == 0 ? 1 : inv;
    }
    PK_CUDA(cudaMemcpyToSymbol(c_mod, kModuli, sizeof kModuli));
    PK_CUDA(cudaMemcpyToSymbol(c_pm, pm, sizeof pm));
    PK_CUDA(cudaMemcpyToSymbol(c_pinv, pinv, sizeof pinv));
    int c21[kI8MaxModuli], c42[kI8MaxModuli];
    float finv[kI8MaxModuli];
    for (int t = 0; t < kI8MaxModuli; t++) {
        const int m = kModuli[t];
        c21[t] = (int)((1ll << 21) % m);
        c42[t] = (int)((long long)c21[t] * c21[t] % m);
        finv[t] = 1.0f / (float)m;
    }
    PK_CUDA(cudaMemcpyToSymbol(c_c21, c21, sizeof c21));
    PK_CUDA(cudaMemcpyToSymbol(c_c42, c42, sizeof c42));
    PK_CUDA(cudaMemcpyToSymbol(c_finv, finv, sizeof finv));
    if (dev < 64) dev_done[dev] = 1;
}

int sm_count() {
    int dev = 0, n = 0;
    PK_CUDA(cudaGetDevice(&dev));
    PK_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

} // namespace

const int *i8_moduli() { return kModuli; }

int64_t i8_window(int nmod, int Ki) {
    (void)nmod;
    // default: 65,536 columns; 8,192 at p >= 10 (Ki >= 1536), where a smaller window keeps
    // the gathered source rows of a window L2-resident (cfg3 513 -> 506 ms, cfg5 19.7 -> 18.6 s)
    const int64_t w = tuning().i8_window > 0 ? tuning().i8_window : (Ki >= 1536 ? 8192 : kI8Window);
    return std::max<int64_t>(kI8Tile, w / kI8Tile * kI8Tile);
}

const I8Settings &i8_settings() {
    static const I8Settings s = [] {
        const Tuning &t = tuning();
        I8Settings r;
        r.enabled = t.m2l_int8;
        // measured at cfg2: the int8 translations lose to the DMMA gather-GEMM (the per-column
        // residue / CRT traffic outweighs the GEMM for 1-8 slots), so they are opt-in
        r.trans = r.enabled && t.trans_int8;
        r.nmod = std::max(14, std::min(t.nmod, kI8MaxModuli));
        r.beta_a = t.beta_a;
        r.beta_b = t.beta_b;
        r.min_boxes = t.i8_min_boxes;
        r.lattice = t.m2l_int8 && t.m2l_lattice;
        return r;
    }();
    return s;
}

I8Settings i8_settings_for(const I8Settings &s, int64_t nslots, int K) {
    I8Settings r = s;
    if (!r.enabled) return r;
    const double need = r.beta_a + r.beta_b + std::log2((double)nslots * K) + 1.0;
    auto bits = [](int nmod) {
        double b = 0;
        for (int t = 0; t < nmod; t++) b += std::log2((double)kModuli[t]);
        return b;
    };
    while (bits(r.nmod) <= need && r.nmod < kI8MaxModuli) r.nmod++;
    if (bits(r.nmod) <= need) r.enabled = r.trans = false;
    return r;
}

void i8_build_operators(I8Operators &o, Workspace &ws, const double *A, int nmat, int K, int Kp, int nmod,
                        int beta_a, cudaStream_t st, const char *tag) {
    const std::string pre = std::string("i8_") + tag + "_";
    upload_tables();
    o.nmod = nmod;
    o.beta_a = beta_a;
    o.K = K;
    o.Ki = (K + BKI - 1) / BKI * BKI;
    o.nmat = nmat;
    unsigned long long *mx = ws.get<unsigned long long>(pre + "rowmax", o.Ki);
    PK_CUDA(cudaMemsetAsync(mx, 0, o.Ki * sizeof(unsigned long long), st));
    rowmax_kernel<<<dim3(K, nmat), 32, 0, st>>>(A, nmat, K, Kp, mx);
    o.rowexp = ws.get<int>(pre + "rowexp", o.Ki);
    rowexp_kernel<<<(o.Ki + 127) / 128, 128, 0, st>>>(mx, K, o.Ki, o.rowexp);
    const int nt = nt_of(K), rtl = rowtiles_of(K);
    o.res = ws.get<int8_t>(pre + "res", (size_t)nmod * nmat * rtl * nt * o.Ki);
    op_residue_kernel<<<dim3(rtl * nt, nmat), 128, 0, st>>>(A, nmat, K, Kp, o.Ki, nmod, beta_a, o.rowexp, nt, rtl,
                                                             o.res);
    PK_CUDA(cudaGetLastError());
}

namespace {

// Kernel variant per launch (I8Kernel): pair-dual (cta_group::2, 512-column quads) for big
// levels (cfg2 level 4: 6.86 -> 6.63 ms against the dual kernel, cfg3 608 -> 518 ms per
// evaluate); dual for the packed small-level runs (the pair-dual kernel's 1024-column run
// streams the operators as often and balances worse: 2.6 -> 3.9 ms at cfg2). A tile's
// quarters / halves with no source for a slot skip their gather and MMA. i8_gather_gemm
// (tests) keeps the single-CTA kernel below 2048 columns so all three stay covered.
// PKGPU_I8_KERNEL forces one variant everywhere. See DESIGN.md §4.
I8Kernel select_kernel(bool big) {
    const I8Kernel forced = tuning().i8_kernel;
    if (forced != I8Kernel::automatic) return forced;
    return big ? I8Kernel::pairdual : I8Kernel::dual;
}
// the pair-dual kernel needs whole 512-column quads and Nt / 2 a multiple of 16
I8Kernel window_kernel(I8Kernel k, int ncols, int K) {
    if (k == I8Kernel::pairdual && (ncols % (4 * TBM) != 0 || nt_of(K) % 32 != 0)) return I8Kernel::dual;
    return k;
}
int column_tile(I8Kernel k) { return k == I8Kernel::pairdual ? 4 * TBM : k == I8Kernel::dual ? 2 * TBM : TBM; }
bool masked(I8Kernel k) { return k != I8Kernel::single; }

inline size_t partial_offset(int tiles) { return ((size_t)tiles * MAX_SLOTS + 15) / 16 * 16; }

// active-slot lists per column tile (ncols / column_tile(k) tiles)
void scan_tiles(const int *src, int64_t ld_src, int nslots, int ncols, I8Kernel k, Workspace &ws, cudaStream_t st,
                int **tslots, int **tnact, int **tbelow, uint8_t **thmask = nullptr) {
    const int bn = column_tile(k), tiles = ncols / bn;
    *tslots = ws.get<int>("i8_tile_slots", (size_t)tiles * MAX_SLOTS);
    *tnact = ws.get<int>("i8_tile_nact", tiles);
    *tbelow = ws.get<int>("i8_tile_below", (size_t)tiles * (MAX_SLOTS + 1));
    // per-tile masks [tiles][MAX_SLOTS] followed by the per-tile partial flags (int)
    uint8_t *hmask = masked(k) ? ws.get<uint8_t>("i8_tile_hmask", partial_offset(tiles) + (size_t)tiles * 4) : nullptr;
    int *partial = masked(k) ? reinterpret_cast<int *>(hmask + partial_offset(tiles)) : nullptr;
    slot_scan_kernel<<<tiles, 1024, 0, st>>>(src, ld_src, nslots, bn, *tslots, *tnact, *tbelow, hmask, partial);
    if (thmask) *thmask = hmask;
    PK_CUDA(cudaGetLastError());
}

// dynamic shared memory opt-in, per device (the attribute is per device; one process may
// drive several GPUs)
template <class F> void ensure_smem(F *kernel, size_t bytes) {
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

void launch_gemm(const int8_t *A, int nmat, const int8_t *B, int rows_per_mod, int zero_row, int Ki, int nmod,
                 const int *src, int64_t ld_src, int64_t box0, int nslots, int ncols, int *R, const int *tslots,
                 const int *tnact, const int *tbelow, I8Kernel kind, cudaStream_t st, bool direct = false,
                 const uint8_t *thmask = nullptr, int K = 0, int *sched = nullptr, int t0 = 0, int t1 = -1) {
    if (masked(kind) && !thmask) throw RuntimeError("i8 gemm: the dual-tile kernels need the half masks");
    const int num_sms = sm_count();
    Params p;
    std::memset(&p, 0, sizeof p);
    p.X = B;
    p.src = src;
    p.ld_src = ld_src;
    p.box0 = box0;
    p.zero_row = zero_row;
    p.rows_per_mod = rows_per_mod;
    p.nmat = nmat;
    p.nmod = nmod;
    p.KC = Ki / BKI;
    if (K <= 0) K = Ki;
    p.rowtiles = rowtiles_of(K);
    p.Nt = nt_of(K);
    p.coltiles = ncols / TBM;
    p.ncols = ncols;
    p.Ki = Ki;
    p.R = R;
    // instruction descriptor: D s32 (bits 4-5 = 2), A / B signed int8 (bits 7-9 / 10-12 = 1),
    // both K-major, N >> 3 at bit 17, M >> 4 at bit 24 (M = 256 for the CTA pair)
    const int M = kind == I8Kernel::pairdual ? 2 * TBM : TBM;
    p.idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.Nt >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    // chunks keep |int32 accumulator| <= slots * Ki * 128^2 < 2^31
    const int64_t cmax = std::max<int64_t>(1, 2147483647LL / ((int64_t)Ki * 16384));
    int nchunk = (int)((nslots + cmax - 1) / cmax);
    if (t1 < 0) t1 = nmod;
    p.t_base = t0;
    const int64_t base = (int64_t)(t1 - t0) * p.rowtiles * (ncols / column_tile(kind));
    const int64_t resident = kind == I8Kernel::pairdual ? num_sms / 2 : num_sms;
    // enough units for ~4 per resident CTA (cfg2's small-level run: 3 -> 4 chunks, 2.57 -> 2.43 ms)
    while (base * nchunk < 4 * resident && nchunk * 16 < nslots) nchunk++;
    p.nchunk = nchunk;
    p.total_units = (int)(base * nchunk);
    if (direct && (nchunk != 1 || kind != I8Kernel::single))
        throw RuntimeError("i8 gemm: direct stores need one unit per tile");
    p.direct = direct ? 1 : 0;
    p.epi_transpose = 1;
    p.tile_slots = tslots;
    p.tile_nact = tnact;
    p.tile_below = tbelow;
    p.nslots = nslots;
    p.half_mask = thmask;
    p.tile_partial = thmask ? reinterpret_cast<const int *>(thmask + partial_offset(ncols / column_tile(kind))) : nullptr;
    // slot-index windows for the single-CTA kernel (operator reuse through L2 across its
    // tiles); equal list shares for the dual-tile kernels (balanced static schedule)
    const Tuning &tu = tuning();
    p.by_index = tu.i8_by_index >= 0 ? tu.i8_by_index : (masked(kind) ? 0 : 1);
    p.tile_fast = tu.i8_tile_fast >= 0 ? tu.i8_tile_fast : 0;
    // dynamic unit schedule (dual-tile kernels): the caller's zeroed counter
    if (sched && kind != I8Kernel::single) {
        PK_CUDA(cudaMemsetAsync(sched, 0, sizeof(int), st));
        p.sched = sched;
    }
    if (tu.i8_min_chunks > nchunk) {
        p.nchunk = nchunk = tu.i8_min_chunks;
        p.total_units = (int)(base * nchunk);
    }
    // operator residues, tile-contiguous [t][mat][row tile][k chunk][Nt][128 B] (op_residue_kernel)
    const cuuint64_t dims[4] = {(cuuint64_t)BKI, (cuuint64_t)p.Nt, (cuuint64_t)p.KC,
                                (cuuint64_t)nmod * nmat * p.rowtiles};
    const cuuint64_t strides[3] = {(cuuint64_t)BKI, (cuuint64_t)BKI * p.Nt, (cuuint64_t)BKI * p.Nt * p.KC};
    // the CTA-pair kernel stages half of the operator tile per CTA
    const cuuint32_t box[4] = {BKI, (cuuint32_t)(kind == I8Kernel::pairdual ? p.Nt / 2 : p.Nt), 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&p.tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t *>(A), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (int8) failed (" + std::to_string((int)r) + ")");
    const size_t epi = 4 * 32 * EPI_PITCH * sizeof(int) + 1024;
    if (kind == I8Kernel::pairdual) {
        if (ncols % (4 * TBM) != 0) throw RuntimeError("i8 gemm: the pair-dual kernel needs 512-column multiples");
        if (p.Nt % 32 != 0 || p.Nt / 2 > 128) throw RuntimeError("i8 pair-dual kernel: Nt / 2 must be a multiple of 16");
        const size_t smem = PD_RING_BYTES + epi;
        ensure_smem(m2l_i8_pairdual_kernel, smem);
        const unsigned grid = 2 * (unsigned)std::min<int64_t>(p.total_units, num_sms / 2);
        m2l_i8_pairdual_kernel<<<grid, PD_THREADS, smem, st>>>(p);
    } else if (kind == I8Kernel::dual) {
        const size_t smem = (size_t)DUAL_NST * DUAL_STAGE + epi;
        ensure_smem(m2l_i8_dual_kernel, smem);
        const unsigned grid = (unsigned)std::min<int64_t>(p.total_units, num_sms);
        m2l_i8_dual_kernel<<<grid, DUAL_THREADS_DYN, smem, st>>>(p);
    } else {
        // stage = 16 KB gathered rows + the operator tile rounded to 1 KB; as many stages as
        // the 227 KB of shared memory allow (the transposing epilogue costs 16.5 KB)
        p.stage_bytes = A_BYTES + (p.Nt * BKI + 1023) / 1024 * 1024;
        const size_t epi_bytes = 4 * 32 * EPI_PITCH * sizeof(int);
        const size_t avail = 227 * 1024 - 1024 - 512 - epi_bytes;
        p.nst = (int)std::min<size_t>(NST_MAX, avail / p.stage_bytes);
        const size_t smem = (size_t)p.nst * p.stage_bytes + epi_bytes + 1024;
        ensure_smem(m2l_i8_kernel, smem);
        const unsigned grid = (unsigned)std::min<int64_t>(p.total_units, num_sms);
        m2l_i8_kernel<<<grid, NTHREADS, smem, st>>>(p);
    }
    PK_CUDA(cudaGetLastError());
}

} // namespace

int i8_gather_gemm(const int8_t *A, int nmat, const int8_t *B, int rows_per_mod, int zero_row, int Ki, int nmod,
                   const int *src, int64_t ld_src, int64_t box0, int nslots, int ncols, int *R, Workspace &ws,
                   cudaStream_t st) {
    if (ncols == 0 || nslots == 0) return 0;
    if (ncols % kI8Tile != 0 || Ki % BKI != 0 || nslots > MAX_SLOTS || nmod < 1 || nmod > kI8MaxModuli)
        throw RuntimeError("i8_gather_gemm: bad shape");
    upload_tables();
    int *tslots = nullptr, *tnact = nullptr, *tbelow = nullptr;
    const I8Kernel kind = window_kernel(ncols >= 2048 ? select_kernel(true) : I8Kernel::single, ncols, Ki);
    // the kernels read operator residues tile-contiguous; the test input is [t][slot][Ki][Ki]
    const int nt = nt_of(Ki), rtl = rowtiles_of(Ki);
    int8_t *At = ws.get<int8_t>("i8_gg_tiled", (size_t)nmod * nmat * rtl * nt * Ki);
    op_tile_kernel<<<dim3(rtl * nt, nmod * nmat), 128, 0, st>>>(A, nmod * nmat, Ki, nt, rtl, At);
    PK_CUDA(cudaGetLastError());
    A = At;
    uint8_t *thmask = nullptr;
    scan_tiles(src, ld_src, nslots, ncols, kind, ws, st, &tslots, &tnact, &tbelow, &thmask);
    launch_gemm(A, nmat, B, rows_per_mod, zero_row, Ki, nmod, src, ld_src, box0, nslots, ncols, R, tslots, tnact,
                tbelow, kind, st, false, thmask, 0, tuning().i8_dynamic > 0 ? ws.get<int>("i8_sched", 1) : nullptr);
    return 2;
}

I8LevelWork m2l_i8_prepare(const I8Operators &o, const I8LevelArgs &a, int beta_b, Workspace &ws, cudaStream_t st,
                           int64_t *launches) {
    I8LevelWork w;
    if (a.ncols == 0) return w;
    if (a.lv.n < 1 || a.lv.n > kI8MaxLevels) throw RuntimeError("m2l_i8: bad level run");
    const int nmod = o.nmod, Ki = o.Ki;
    const int64_t box0 = a.lv.box0[0], nbox = a.lv.box0[a.lv.n] - box0;
    w.rows = nbox + 1;
    w.mx = ws.get<unsigned long long>("i8_level_max", kI8MaxLevels);
    PK_CUDA(cudaMemsetAsync(w.mx, 0, kI8MaxLevels * sizeof(unsigned long long), st));
    for (int l = 0; l < a.lv.n; l++) {
        const int64_t nb = a.lv.box0[l + 1] - a.lv.box0[l];
        if (nb > 0)
            level_absmax_kernel<<<(unsigned)std::min<int64_t>((nb * a.Kp + 255) / 256, 296), 256, 0, st>>>(
                a.X + a.lv.box0[l] * a.Kp, nb, a.K, a.Kp, w.mx + l);
    }
    int8_t *xres = ws.get<int8_t>("i8_xres", (size_t)nmod * w.rows * Ki);
    x_residue_kernel<<<(unsigned)std::min<int64_t>((w.rows * Ki + 255) / 256, 148 * 16), 256, 0, st>>>(
        a.X + box0 * a.Kp, nbox, a.K, a.Kp, Ki, nmod, beta_b, w.mx, a.lv, xres);
    w.xres = xres;
    upload_tables();
    w.kind = select_kernel(a.big);
    PK_CUDA(cudaGetLastError());
    if (launches) *launches += 1 + a.lv.n;
    return w;
}

// profiling: MMA rows issued (128 per active half per slot) -- padding and union waste show
// against the V-list applications
__global__ void mma_rows_kernel(const uint8_t *__restrict__ hmask, int nslots, unsigned long long *rows) {
    int c = 0;
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) c += __popc(hmask[blockIdx.x * MAX_SLOTS + s]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(rows, 128ull * c);
}

int m2l_i8_window(const I8Operators &o, const I8LevelArgs &a, I8LevelWork &w, int64_t c0, int64_t c1, Workspace &ws,
                  cudaStream_t st) {
    const int ncols = (int)(c1 - c0);
    if (ncols <= 0) return 0;
    if (c0 % kI8Tile != 0 || ncols % kI8Tile != 0) throw RuntimeError("m2l_i8: column window not tile aligned");
    // residue sums of this column window only (the window bounds R: 4 nmod Ki bytes per column);
    // a modulus-split run (partitioned) sums into the caller's collective-visible buffer
    w.R = w.R_ext ? w.R_ext : ws.get<int>("i8_R", (size_t)o.nmod * ncols * o.Ki);
    PK_CUDA(cudaMemsetAsync(w.R, 0, (size_t)o.nmod * ncols * o.Ki * sizeof(int), st));
    // the multicast variant needs whole 512-column quads; other windows use the dual kernel
    w.win_kind = window_kernel(w.kind, ncols, o.K);
    scan_tiles(a.src + c0, a.ld_src, a.nslots, ncols, w.win_kind, ws, st, &w.tile_slots, &w.tile_nact,
               &w.tile_below, &w.tile_hmask);
    if (a.mma_rows && w.tile_hmask) {
        mma_rows_kernel<<<ncols / (2 * TBM), 32, 0, st>>>(w.tile_hmask, a.nslots, a.mma_rows);
        PK_CUDA(cudaGetLastError());
        return 2;
    }
    return 1;
}

int m2l_i8_gemm(const I8Operators &o, const I8LevelArgs &a, I8LevelWork &w, int64_t c0, int64_t c1, Workspace &ws,
                cudaStream_t st) {
    const int ncols = (int)(c1 - c0);
    if (ncols <= 0) return 0;
    const int dyn = tuning().i8_dynamic;
    launch_gemm(o.res, o.nmat, w.xres, (int)w.rows, (int)(w.rows - 1), o.Ki, o.nmod, a.src + c0, a.ld_src,
                a.lv.box0[0], a.nslots, ncols, w.R, w.tile_slots, w.tile_nact, w.tile_below, w.win_kind, st, false,
                w.tile_hmask, o.K, dyn > 0 ? ws.get<int>("i8_sched", 1) : nullptr, w.t0, w.t1 < 0 ? o.nmod : w.t1);
    return 1;
}

int m2l_i8_finish(const I8Operators &o, const I8LevelArgs &a, const I8LevelWork &w, int64_t c0, int64_t c1,
                  int beta_b, cudaStream_t st) {
    const int ncols = (int)(c1 - c0);
    if (ncols <= 0) return 0;
    const int64_t n = (int64_t)ncols * o.Ki;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    const int bs = o.beta_a + beta_b;
    switch (o.nmod) {
#define PK_RC(NM)                                                                                                      \
    case NM:                                                                                                           \
        reconstruct_kernel<NM><<<grid, 256, 0, st>>>(w.R, ncols, o.Ki, a.K, a.Kp, a.out_box + c0, c0, o.rowexp, w.mx, \
                                                     bs, a.lv, a.Y);                                                   \
        break;
        PK_RC(14) PK_RC(15) PK_RC(16) PK_RC(17) PK_RC(18) PK_RC(19) PK_RC(20)
#undef PK_RC
    default:
        throw RuntimeError("m2l_i8: unsupported modulus count " + std::to_string(o.nmod));
    }
    PK_CUDA(cudaGetLastError());
    return 1;
}

int i8_translate(const I8Operators &o, const I8TransArgs &a, int beta_b, Workspace &ws, cudaStream_t st) {
    if (a.ncols == 0) return 0;
    if (a.ncols % kI8Tile != 0 || a.nslots < 1 || a.nslots > 8 || a.nslots > o.nmat || a.src_hi < a.src_lo)
        throw RuntimeError("i8_translate: bad shape");
    upload_tables();
    const int nmod = o.nmod, Ki = o.Ki;
    const int64_t nsrc = a.src_hi - a.src_lo;
    int8_t *xres = ws.get<int8_t>("tr_xres", (size_t)nmod * (nsrc + 1) * Ki);
    int *ecol = ws.get<int>("tr_ecol", a.ncols);
    int *R = ws.get<int>("tr_R", (size_t)nmod * a.ncols * Ki);
    // <= 16 slots: one work unit per output tile (launch_gemm), whose epilogue stores the
    // partial residues directly -- no R zeroing, no atomics
    const bool direct = a.nslots <= 16;
    tr_prepare_kernel<<<a.ncols, 256, 0, st>>>(a.src, a.ld_src, a.nslots, a.src_lo, nsrc, a.X, a.K, a.Kp, Ki, nmod,
                                                beta_b, a.ncols, xres, ecol, R, direct ? 0 : 1);
    PK_CUDA(cudaGetLastError());
    int *tslots = nullptr, *tnact = nullptr, *tbelow = nullptr;
    scan_tiles(a.src, a.ld_src, a.nslots, a.ncols, I8Kernel::single, ws, st, &tslots, &tnact, &tbelow);
    launch_gemm(o.res, o.nmat, xres, (int)(nsrc + 1), (int)nsrc, Ki, nmod, a.src, a.ld_src, a.src_lo, a.nslots,
                a.ncols, R, tslots, tnact, tbelow, I8Kernel::single, st, direct, nullptr, o.K);
    const int64_t n = (int64_t)a.ncols * Ki;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    const int bs = o.beta_a + beta_b;
    switch (nmod) {
#define PK_TF(NM)                                                                                                      \
    case NM:                                                                                                           \
        tr_finish_kernel<NM><<<grid, 256, 0, st>>>(R, a.ncols, Ki, a.K, a.Kp, a.out_box, o.rowexp, ecol, bs, a.alpha,  \
                                                   a.beta, a.rdiv, a.rdiv_eps, a.Y);                                   \
        break;
        PK_TF(14) PK_TF(15) PK_TF(16) PK_TF(17) PK_TF(18) PK_TF(19) PK_TF(20)
#undef PK_TF
    default:
        throw RuntimeError("i8_translate: unsupported modulus count " + std::to_string(nmod));
    }
    PK_CUDA(cudaGetLastError());
    return 4;
}

int m2l_i8_level(const I8Operators &o, const I8LevelArgs &a, int beta_b, Workspace &ws, cudaStream_t st) {
    int64_t l = 0;
    I8LevelWork w = m2l_i8_prepare(o, a, beta_b, ws, st, &l);
    const int64_t win = i8_window(o.nmod, o.Ki);
    for (int64_t c0 = 0; c0 < a.ncols; c0 += win) {
        const int64_t c1 = std::min<int64_t>(a.ncols, c0 + win);
        l += m2l_i8_window(o, a, w, c0, c1, ws, st);
        l += m2l_i8_gemm(o, a, w, c0, c1, ws, st);
        l += m2l_i8_finish(o, a, w, c0, c1, beta_b, st);
    }
    return (int)l;
}

} // namespace pkgpu
