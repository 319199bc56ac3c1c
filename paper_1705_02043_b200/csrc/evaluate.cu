// The evaluate pipeline (pkifmm::evaluate, src/fmm.cpp:690-742) on one B200.
//
//   validate + compatibility gate (src/fmm.cpp:693-706, src/refsum.cpp:733-756)
//   tree (Morton keys, radix sort, level-synchronous split)           -> timings.tree
//   column layout + lists (U/W/X CSR, V straight into the M2L table)
//   upward:   S2M (pairs) ; per level M2M (gather-GEMM) + pinv (2 GEMMs)
//   downward: X (pairs) ; per level M2L + L2L (gather-GEMMs) + pinv
//   periodizing step: phi_far = T_M2L phi_up[0] (+ pinv(a_dn, M_img phi_up[0]))  -> m2l_apply
//   leaf pass: L2T + W + U + far field, fused, one write per target
// All device work is on the context stream; timings are CUDA events.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>

#include "context.h"
#include "tuning.h"
#include "gemm.h"
#include "pairs.h"

namespace pkgpu {

namespace {

constexpr int BN = kGemmBN;

__global__ void compat_partial_kernel(const double *__restrict__ s, int64_t n, int ks, double *__restrict__ part) {
    // part[block][0] = sum |s|, part[block][1+a] = sum s_a ; fixed partition -> deterministic
    __shared__ double red[4][256];
    double a[4] = {0, 0, 0, 0};
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b = per * blockIdx.x, e = min(n, b + per);
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x)
        for (int c = 0; c < ks; c++) {
            const double v = s[i * ks + c];
            a[0] += fabs(v);
            a[1 + c] += v;
        }
    for (int c = 0; c < 4; c++) red[c][threadIdx.x] = a[c];
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o)
            for (int c = 0; c < 4; c++) red[c][threadIdx.x] += red[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 4; c++) part[4 * blockIdx.x + c] = red[c][0];
}

__global__ void layout_keys_kernel(TreeView T, int *keys, int *vals) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < T.nboxes) {
        const int4 c = T.cell[b];
        keys[b] = c.w * 8 + ((c.x & 1) | ((c.y & 1) << 1) | ((c.z & 1) << 2));
        vals[b] = b;
    }
}

// Two column layouts per level (see build_layout):
//   oct  : boxes grouped by octant, each group padded to 64 -> octant-homogeneous tiles (L2L)
//   m2l  : the oct layout on big levels, plain Morton order (= BFS order) on small ones
__global__ void layout_fill_kernel(TreeView T, const int *__restrict__ skeys, const int *__restrict__ sboxes,
                                   const int *__restrict__ group_start, const int *__restrict__ oct_gcol,
                                   const int *__restrict__ m2l_gcol, const int *__restrict__ m2l_base,
                                   const int *__restrict__ grouped, int *col_of_box, int *out_box, int *out_oct,
                                   int *l2l_src, int *tile_oct) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T.nboxes) return;
    const int key = skeys[i], b = sboxes[i];
    const int lvl = key / 8;
    const int rank = i - group_start[key];
    const int ocol = oct_gcol[key] + rank;
    out_oct[ocol] = b;
    l2l_src[ocol] = T.parent[b];
    tile_oct[ocol / BN] = key & 7;
    const int col = grouped[lvl] ? m2l_gcol[key] + rank : m2l_base[lvl] + (int)(b - T.level_off[lvl]);
    col_of_box[b] = col;
    out_box[col] = b;
}

// M2M columns: internal boxes with sources only (src/fmm.cpp:536, 546), BFS order,
// per level padded to 64 (restricted to `mask` boxes in partitioned runs)
__global__ void m2m_flags_kernel(TreeView T, const int *__restrict__ mask, int *flags, int *level_count) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const bool f = !T.isleaf[b] && T.srng[b].y > T.srng[b].x && (!mask || mask[b]);
    flags[b] = f ? 1 : 0;
    if (f) atomicAdd(&level_count[T.cell[b].w], 1);
}

// ---- Morton-range partition (pkgpu_evaluate_partitioned) ----
// leaves -> full 36-bit Morton start key (DFS order once sorted)
__global__ void leaf_key_kernel(TreeView T, const int *__restrict__ leaves, int nleaves, unsigned long long *keys,
                                int *vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nleaves) return;
    const int b = leaves[i];
    keys[i] = T.prefix[b] << (3 * (kMaxDepth - T.cell[b].w));
    vals[i] = b;
}

// box -> does its DFS leaf interval meet [lo, hi)?  own[b]: leaf owned by this rank
__global__ void part_mask_kernel(TreeView T, const unsigned long long *__restrict__ lkeys, int nleaves, int lo, int hi,
                                 int nranks, int *in, int *own, int *rlo, int *rhi) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const int sh = 3 * (kMaxDepth - T.cell[b].w);
    const unsigned long long k0 = T.prefix[b] << sh, k1 = (T.prefix[b] + 1ull) << sh;
    int a = 0, e = nleaves;
    while (a < e) { // first leaf key >= k0
        const int m = (a + e) >> 1;
        if (lkeys[m] < k0)
            a = m + 1;
        else
            e = m;
    }
    int c = a, f = nleaves;
    while (c < f) { // first leaf key >= k1
        const int m = (c + f) >> 1;
        if (lkeys[m] < k1)
            c = m + 1;
        else
            f = m;
    }
    in[b] = (a < hi && c > lo) ? 1 : 0;
    own[b] = (T.isleaf[b] && a >= lo && a < hi) ? 1 : 0;
    // ranks of the box's first and last leaf: rank(i) = ceil((i + 1) R / L) - 1 for the
    // equal split lo_r = floor(L r / R)
    auto rank_of = [&](int i) { return (int)((((int64_t)i + 1) * nranks + nleaves - 1) / nleaves) - 1; };
    rlo[b] = rank_of(min(a, nleaves - 1));
    rhi[b] = rank_of(max(a, c - 1));
}

// boxes of the small levels (the packed int8 run) join every rank's mask when that run is
// split by modulus: all ranks then lay out and compute the same columns
__global__ void small_or_kernel(TreeView T, const int *__restrict__ in, int64_t small_max, int *out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const int l = T.cell[b].w;
    out[b] = in[b] || (l >= 1 && T.level_off[l + 1] - T.level_off[l] <= small_max);
}
__global__ void need_small_kernel(TreeView T, int64_t small_max, unsigned long long all, unsigned long long *need) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const int l = T.cell[b].w;
    if (l >= 1 && T.level_off[l + 1] - T.level_off[l] <= small_max) need[b] |= all;
}

// ---- equivalent-density exchange of the partitioned run ----
__global__ void strad_flags_kernel(const int *__restrict__ rlo, const int *__restrict__ rhi, int n, int *flags) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < n) flags[b] = rlo[b] != rhi[b];
}
// send (dir 0): boxes this rank owns that rank q needs; recv (dir 1): boxes rank q owns that this rank needs
__global__ void halo_flags_kernel(const int *__restrict__ rlo, const int *__restrict__ rhi,
                                  const unsigned long long *__restrict__ need, int n, int me, int q, int dir,
                                  int *flags) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int o = rlo[b];
    const bool single = o == rhi[b];
    flags[b] = dir == 0 ? (single && o == me && ((need[b] >> q) & 1ull)) : (single && o == q && ((need[b] >> me) & 1ull));
}
__global__ void rows_pack_kernel(const double *__restrict__ X, const int *__restrict__ list, int n, int Kp,
                                 double *__restrict__ buf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * Kp) return;
    buf[i] = X[(int64_t)list[i / Kp] * Kp + i % Kp];
}
__global__ void rows_unpack_kernel(const double *__restrict__ buf, const int *__restrict__ list, int n, int Kp,
                                   double *__restrict__ X) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * Kp) return;
    X[(int64_t)list[i / Kp] * Kp + i % Kp] = buf[i];
}

__global__ void flags_by_level_kernel(TreeView T, const int *__restrict__ mask, int *level_count) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    if (mask[b]) atomicAdd(&level_count[T.cell[b].w], 1);
}

__global__ void level_list_fill_kernel(TreeView T, const int *__restrict__ list, int n, const int *__restrict__ start,
                                       const int *__restrict__ base, int *out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int b = list[p];
    const int l = T.cell[b].w;
    out[base[l] + (p - start[l])] = b;
}

__global__ void mask_oct_kernel(const int *__restrict__ mask, int64_t n, int *out_oct, int *l2l_src) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    const int b = out_oct[c];
    if (b >= 0 && !mask[b]) out_oct[c] = -1, l2l_src[c] = -1;
}

__global__ void m2m_fill_kernel(TreeView T, const int *__restrict__ list, int n, const int *__restrict__ list_start,
                                const int *__restrict__ col_base, int64_t ncols, int *out, int *src) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int b = list[p];
    const int l = T.cell[b].w;
    const int col = col_base[l] + (p - list_start[l]);
    out[col] = b;
    for (int o = 0; o < 8; o++) {
        const int c = T.child[8 * b + o];
        src[(int64_t)o * ncols + col] = (c >= 0 && T.srng[c].y > T.srng[c].x) ? c : -1;
    }
}

// buf[(b - lo) Kp + k] = phi_up[b][k] on the rank of the box's first leaf, 0 elsewhere
__global__ void level_contrib_kernel(const double *__restrict__ X, const int *__restrict__ rlo, int me, int64_t lo,
                                     int64_t hi, int Kp, double *__restrict__ buf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (hi - lo) * Kp) return;
    const int64_t b = lo + i / Kp;
    buf[i] = rlo[b] == me ? X[b * Kp + i % Kp] : 0.0;
}

__global__ void add_kernel(double *y, const double *x, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += x[i];
}

// stage profiler: CUDA events on the work stream around each stage (profiling on)
struct Prof {
    pkgpu_context &ctx;
    cudaStream_t st;
    struct Mark {
        std::string stage;
        cudaEvent_t a, b;
        int64_t l0, l1;
    };
    std::vector<Mark> marks;
    size_t next = 0;
    Prof(pkgpu_context &c, cudaStream_t s) : ctx(c), st(s) {}
    cudaEvent_t ev() {
        if (next == ctx.evpool.size()) {
            cudaEvent_t e;
            PK_CUDA(cudaEventCreate(&e));
            ctx.evpool.push_back(e);
        }
        return ctx.evpool[next++];
    }
    int begin(const char *stage) {
        if (!ctx.profiling) return -1;
        Mark m{stage, ev(), ev(), ctx.launches, 0};
        PK_CUDA(cudaEventRecord(m.a, st));
        marks.push_back(m);
        return (int)marks.size() - 1;
    }
    void end(int i) {
        if (i < 0) return;
        PK_CUDA(cudaEventRecord(marks[i].b, st));
        marks[i].l1 = ctx.launches;
    }
    void finish() {
        if (marks.empty()) return;
        PK_CUDA(cudaStreamSynchronize(st));
        for (auto &m : marks) {
            float ms = 0;
            PK_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
            auto &s = ctx.stats[m.stage];
            s.seconds += ms * 1e-3;
            s.launches += m.l1 - m.l0;
        }
    }
    void work(const char *stage, double units, double flops_per_unit) {
        if (!ctx.profiling) return;
        auto &s = ctx.stats[stage];
        s.units += units;
        s.flops += units * flops_per_unit;
    }
};

// algorithmic work of one evaluate (pairs / applications), reference conventions
__global__ void work_count_kernel(TreeView T, int n, const int64_t *__restrict__ u_off, const int2 *__restrict__ u_ent,
                                  const int64_t *__restrict__ w_off, const int64_t *__restrict__ x_off,
                                  const int2 *__restrict__ x_ent, unsigned long long *cnt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const int2 sr = T.srng[b], tr = T.trng[b];
    const long long ns = sr.y - sr.x, nt = tr.y - tr.x;
    unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (T.isleaf[b]) {
        if (nt > 0) {
            long long su = 0;
            for (int64_t e = u_off[b]; e < u_off[b + 1]; e++) {
                const int2 r = T.srng[u_ent[e].x];
                su += r.y - r.x;
            }
            c[0] = nt * su;                              // U pairs
            c[1] = nt * (w_off[b + 1] - w_off[b]) * n;   // W pairs
            c[2] = nt * n;                               // L2T pairs
        }
        if (ns > 0) c[3] = ns * n;                       // S2M pairs
    } else if (ns > 0) {
        for (int o = 0; o < 8; o++) {
            const int ch = T.child[8 * b + o];
            if (ch >= 0 && T.srng[ch].y > T.srng[ch].x) c[5]++; // M2M applications
        }
    }
    if (nt > 0) {
        long long sx = 0;
        for (int64_t e = x_off[b]; e < x_off[b + 1]; e++) {
            const int2 r = T.srng[x_ent[e].x];
            sx += r.y - r.x;
        }
        c[4] = sx * n;                                   // X pairs
        if (T.parent[b] >= 0) c[6] = 1;                  // pinv_dn / L2L boxes
    }
    if (ns > 0) c[7] = 1;                                // pinv_up boxes
    for (int k = 0; k < 8; k++)
        if (c[k]) atomicAdd(cnt + k, c[k]);
}

struct Layout {
    std::vector<int64_t> colbase, octbase, m2mbase; // per level (size depth + 2): m2l, oct, m2m layouts
    int wide[kMaxLevels + 1] = {0};                // m2l layout padded to 128-column tiles
    int i8[kMaxLevels + 1] = {0};                  // M2L on the int8 tensor pipe (256-column tiles)
    int i8_last[kMaxLevels + 1] = {0};             // int8 run starting at this level ends at i8_last
    int i8_big[kMaxLevels + 1] = {0};              // ... and is one big level (dual-tile kernel)
    int lat[kMaxLevels + 1] = {0};                 // M2L by the lattice FFT (m2l_lattice_level)
    int64_t ncols = 0, noct = 0, nm2m = 0;
    int *col_of_box = nullptr, *out_box = nullptr, *out_m2m = nullptr, *m2m_src = nullptr, *m2l_table = nullptr;
    int *out_oct = nullptr, *l2l_src = nullptr, *tile_oct = nullptr;
    int *l2l_src8 = nullptr;          // [8][noct]: parent per (octant slot, column) for i8_translate
    std::vector<int64_t> lvbase;      // per-level columns of lvcol (levels padded to kI8Tile)
    int *lvcol = nullptr;             // box per column, -1 padding (pseudo-inverse columns)
};

__global__ void lvcol_fill_kernel(TreeView T, const int *__restrict__ lvbase, int *lvcol) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const int l = T.cell[b].w;
    lvcol[lvbase[l] + (b - T.level_off[l])] = b;
}
__global__ void l2l_src8_kernel(const int *__restrict__ l2l_src, const int *__restrict__ tile_oct, int64_t noct,
                                int *src8) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= noct) return;
    const int b = l2l_src[c];
    if (b >= 0) src8[(int64_t)tile_oct[c / BN] * noct + c] = b;
}

// Columns of the gather-GEMMs. Octant grouping makes every 64-column M2L tile share
// one offset set (~189 of 316 slots active, no zero columns) at the price of padding
// each octant group to 64; a level uses it when that streams fewer (column x slot)
// pairs than Morton order with (nearly) all 316 offsets active. L2L always uses the
// octant layout so each tile has a single L2L matrix. M2M gets its own compact layout
// of internal boxes with sources.
Layout build_layout(pkgpu_context &ctx, const DeviceTree &T, const int *mask, const int *lat, cudaStream_t st) {
    Workspace &ws = ctx.ws;
    const int nb = (int)T.nboxes;
    const TreeView tv = T.view();
    int *keys = ws.get<int>("lay_keys", nb), *vals = ws.get<int>("lay_vals", nb);
    int *skeys = ws.get<int>("lay_skeys", nb), *svals = ws.get<int>("lay_svals", nb);
    constexpr int NK = kMaxLevels * 8;
    layout_keys_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(tv, keys, vals);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, skeys, vals, svals, nb, 0, 7, st);
    void *tmp = ws.get<char>("lay_temp", tb);
    PK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, skeys, vals, svals, nb, 0, 7, st));
    ctx.launches += 4;
    // boxes per (level, octant): counted by the tree build and read back with its header (no
    // round trip here); the small tables below go up from pinned staging (no wait either)
    std::vector<int> count(T.oct_hist), start(NK, 0), ogcol(NK, 0), mgcol(NK, 0), mbase(kMaxLevels + 1, 0),
        grouped(kMaxLevels + 1, 0);
    count.resize(NK, 0);
    constexpr int kStage = 4 * NK + 4 * (kMaxLevels + 1) + kMaxLevels + 2;
    if (!ctx.h_layout) PK_CUDA(cudaMallocHost(&ctx.h_layout, kStage * sizeof(int)));
    int *h_stage = ctx.h_layout;
    Layout L;
    L.colbase.assign(T.depth + 2, 0);
    L.octbase.assign(T.depth + 2, 0);
    int s = 0;
    int64_t co = 0, cm = 0;
    // int8 runs: consecutive small levels (<= PKGPU_I8_SMALL boxes, default 1024: nearly all
    // 316 offsets active, few columns, bound by streaming the operator residues) share one
    // launch and are packed into as few 128-column tiles as possible; a big level runs alone
    const int64_t small_max = tuning().i8_small_boxes;
    const I8Settings &is = ctx.i8;
    auto i8_level = [&](int lv) {
        return is.enabled && lv >= 1 && lv <= T.depth && !lat[lv] &&
               T.level_off[lv + 1] - T.level_off[lv] >= is.min_boxes;
    };
    for (int l = 0; l <= T.depth; l++) L.lat[l] = lat[l];
    auto small_level = [&](int lv) { return T.level_off[lv + 1] - T.level_off[lv] <= small_max; };
    int run_first = -1; // first level of the int8 run being laid out
    for (int l = 0; l <= T.depth; l++) {
        const int64_t nl = T.level_off[l + 1] - T.level_off[l];
        // octant grouping streams ~189 offsets over padded groups; Morton order streams
        // (nearly) all 316 over the level's boxes: pick the cheaper column count x slots
        int64_t padded = 0, padded128 = 0;
        for (int o = 0; o < 8; o++) {
            padded += (count[l * 8 + o] + BN - 1) / BN * BN;
            padded128 += (count[l * 8 + o] + 127) / 128 * 128;
        }
        // (the FFT M2L wants Morton order: 64-box tiles of compact blocks share their sources)
        grouped[l] = !is.fft && padded * 189 <= (nl + BN - 1) / BN * BN * 316 ? 1 : 0;
        // 128-column DMMA M2L tiles (one 17-warp CTA per SM) measured slower than two
        // 64-column CTAs per SM on cfg2/3/4 (49.3 vs 46.3 ms M2L at cfg2): not used
        (void)padded128;
        L.wide[l] = 0;
        const int padm = L.wide[l] ? 128 : BN;
        L.i8[l] = i8_level(l) ? 1 : 0;
        const bool in_run = L.i8[l] && run_first >= 0; // continues the current int8 run
        if (L.i8[l] && !in_run) run_first = l;
        // inside an int8 run an ungrouped level is packed (8-column granularity) after the
        // previous one; grouped levels keep 64-aligned octant groups
        if (grouped[l] || !L.i8[l]) cm = (cm + BN - 1) / BN * BN;
        co = (co + kI8Tile - 1) / kI8Tile * kI8Tile; // levels in whole int8 tiles (i8_translate L2L)
        L.octbase[l] = co;
        L.colbase[l] = cm;
        mbase[l] = (int)cm;
        for (int o = 0; o < 8; o++) {
            const int k = l * 8 + o;
            start[k] = s;
            ogcol[k] = (int)co;
            mgcol[k] = (int)cm;
            s += count[k];
            co += (count[k] + BN - 1) / BN * BN;
            if (grouped[l]) cm += (count[k] + padm - 1) / padm * padm;
        }
        if (!grouped[l]) cm += L.i8[l] ? (nl + 7) / 8 * 8 : (nl + BN - 1) / BN * BN;
        if (L.i8[l]) {
            // close the run unless the next level is small too. Runs are whole 256-column pair
            // tiles (the dual kernel's); a big level is whole 512-column quads (the pair-dual
            // kernel's tile; quarters without sources are skipped by the masks)
            const bool cont = small_level(l) && i8_level(l + 1) && small_level(l + 1) && l + 1 - run_first < kI8MaxLevels;
            if (!cont) {
                L.i8_last[run_first] = l;
                L.i8_big[run_first] = run_first == l && !small_level(l) ? 1 : 0;
                const int64_t q = L.i8_big[run_first] ? 2 * kI8Tile : kI8Tile;
                cm = L.colbase[run_first] + (cm - L.colbase[run_first] + q - 1) / q * q;
                run_first = -1;
            }
        }
    }
    co = (co + kI8Tile - 1) / kI8Tile * kI8Tile;
    L.octbase[T.depth + 1] = co;
    L.colbase[T.depth + 1] = cm;
    L.noct = co;
    L.ncols = cm;
    int *d_small = ws.get<int>("lay_small", 4 * NK + 2 * (kMaxLevels + 1));
    {
        int *h = h_stage;
        h = std::copy(start.begin(), start.end(), h);
        h = std::copy(ogcol.begin(), ogcol.end(), h);
        h = std::copy(mgcol.begin(), mgcol.end(), h);
        h = std::copy(mbase.begin(), mbase.end(), h);
        h = std::copy(grouped.begin(), grouped.end(), h);
        PK_CUDA(cudaMemcpyAsync(d_small, h_stage, (h - h_stage) * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    int *h_stage2 = h_stage + 4 * NK + 2 * (kMaxLevels + 1); // the M2M tables and lvbase below
    const int64_t C = std::max<int64_t>(cm, 1), CO = std::max<int64_t>(co, 1);
    L.col_of_box = ws.get<int>("col_of_box", nb);
    // the -1-initialised tables share one buffer (one memset instead of four; C, CO are
    // multiples of 64, so every table stays 256-byte aligned)
    int *ff = ws.get<int>("lay_ff", (size_t)C + 2 * (size_t)CO + (size_t)kNumM2L * C);
    L.out_box = ff;
    L.out_oct = ff + C;
    L.l2l_src = L.out_oct + CO;
    L.m2l_table = L.l2l_src + CO;
    L.tile_oct = ws.get<int>("tile_oct", CO / BN + 1);
    PK_CUDA(cudaMemsetAsync(L.tile_oct, 0, (CO / BN + 1) * sizeof(int), st));
    PK_CUDA(cudaMemsetAsync(ff, 0xff, ((size_t)C + 2 * (size_t)CO + (size_t)kNumM2L * C) * sizeof(int), st));
    layout_fill_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(
        tv, skeys, svals, d_small, d_small + NK, d_small + 2 * NK, d_small + 3 * NK, d_small + 3 * NK + kMaxLevels + 1,
        L.col_of_box, L.out_box, L.out_oct, L.l2l_src, L.tile_oct);
    PK_CUDA(cudaGetLastError());
    if (ctx.i8.trans) {
        if (mask) {
            mask_oct_kernel<<<blocks_for(CO, 256), 256, 0, st>>>(mask, CO, L.out_oct, L.l2l_src);
            ctx.launches += 1;
        }
        L.l2l_src8 = ws.get<int>("l2l_src8", (size_t)8 * CO);
        PK_CUDA(cudaMemsetAsync(L.l2l_src8, 0xff, (size_t)8 * CO * sizeof(int), st));
        l2l_src8_kernel<<<blocks_for(CO, 256), 256, 0, st>>>(L.l2l_src, L.tile_oct, CO, L.l2l_src8);
        // pseudo-inverse columns: each level's boxes, padded to whole int8 tiles
        L.lvbase.assign(T.depth + 2, 0);
        for (int l = 0; l <= T.depth; l++)
            L.lvbase[l + 1] = L.lvbase[l] + (T.level_off[l + 1] - T.level_off[l] + kI8Tile - 1) / kI8Tile * kI8Tile;
        int *hb = h_stage2 + 2 * (kMaxLevels + 1);
        std::copy(L.lvbase.begin(), L.lvbase.end(), hb);
        int *d_lvbase = ws.get<int>("lvbase", L.lvbase.size());
        PK_CUDA(cudaMemcpyAsync(d_lvbase, hb, L.lvbase.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        L.lvcol = ws.get<int>("lvcol", std::max<int64_t>(L.lvbase[T.depth + 1], 1));
        PK_CUDA(cudaMemsetAsync(L.lvcol, 0xff, std::max<int64_t>(L.lvbase[T.depth + 1], 1) * sizeof(int), st));
        lvcol_fill_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(tv, d_lvbase, L.lvcol);
        PK_CUDA(cudaGetLastError());
        ctx.launches += 2;
    }
    // ---- M2M layout: internal boxes with sources, compacted in BFS order ----
    // (unmasked: the tree build has listed and counted them; a partition's mask selects here)
    const int *list = T.m2m_list;
    std::vector<int> lc(T.m2m_count);
    lc.resize(kMaxLevels + 1, 0);
    if (mask) {
        int *flags = ws.get<int>("m2m_flags", nb), *sel = ws.get<int>("m2m_list", nb);
        int *lcount = ws.get<int>("m2m_lcount", kMaxLevels + 1), *nsel = ws.get<int>("m2m_nsel", 1);
        PK_CUDA(cudaMemsetAsync(lcount, 0, (kMaxLevels + 1) * sizeof(int), st));
        if (!ctx.i8.trans) {
            mask_oct_kernel<<<blocks_for(CO, 256), 256, 0, st>>>(mask, CO, L.out_oct, L.l2l_src);
            ctx.launches += 1;
        }
        m2m_flags_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(tv, mask, flags, lcount);
        size_t fb = 0;
        cub::DeviceSelect::Flagged(nullptr, fb, cub::CountingInputIterator<int>(0), flags, sel, nsel, nb, st);
        void *ftmp = ws.get<char>("m2m_sel_temp", fb);
        PK_CUDA(cub::DeviceSelect::Flagged(ftmp, fb, cub::CountingInputIterator<int>(0), flags, sel, nsel, nb, st));
        PK_CUDA(cudaMemcpyAsync(lc.data(), lcount, lc.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        list = sel;
        ctx.launches += 4;
    }
    std::vector<int> lstart(kMaxLevels + 1, 0), cbase(kMaxLevels + 1, 0);
    L.m2mbase.assign(T.depth + 2, 0);
    int64_t cmm = 0;
    int nint = 0;
    for (int l = 0; l <= T.depth; l++) {
        lstart[l] = nint;
        cbase[l] = (int)cmm;
        L.m2mbase[l] = cmm;
        nint += lc[l];
        cmm += (lc[l] + kI8Tile - 1) / kI8Tile * kI8Tile; // whole int8 tiles (i8_translate)
    }
    L.m2mbase[T.depth + 1] = cmm;
    L.nm2m = cmm;
    const int64_t CM = std::max<int64_t>(cmm, 1);
    L.out_m2m = ws.get<int>("m2m_ff", 9 * CM); // out_m2m [CM] and m2m_src [8][CM]: one -1 fill
    L.m2m_src = L.out_m2m + CM;
    int *d_m2m_small = ws.get<int>("m2m_small", 2 * (kMaxLevels + 1));
    std::copy(cbase.begin(), cbase.end(), std::copy(lstart.begin(), lstart.end(), h_stage2));
    PK_CUDA(cudaMemcpyAsync(d_m2m_small, h_stage2, 2 * (kMaxLevels + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemsetAsync(L.out_m2m, 0xff, 9 * CM * sizeof(int), st));
    if (nint > 0)
        m2m_fill_kernel<<<blocks_for(nint, 256), 256, 0, st>>>(tv, list, nint, d_m2m_small, d_m2m_small + kMaxLevels + 1,
                                                               CM, L.out_m2m, L.m2m_src);
    PK_CUDA(cudaGetLastError());
    ctx.launches += 6;
    return L;
}

// Morton-range partition of the leaves for rank r of R (pkgpu_evaluate_partitioned):
// `in` marks boxes whose subtree meets the rank's leaves, `own` its leaves; `act`
// lists the `in` boxes per level (padded to 64 with -1) for the pseudo-inverses, and
// `leaves` the owned leaves for the leaf pass.
struct Partition {
    bool on = false;
    int *in = nullptr, *own = nullptr;
    int *rlo = nullptr, *rhi = nullptr; // ranks of each box's first and last leaf
    int *act = nullptr;
    std::vector<int64_t> actbase; // per level column base into act
    int *leaves = nullptr;
    int nleaves = 0;
};

void compact(pkgpu_context &ctx, const int *flags, int n, int *list, int *count_dev, const char *tag, cudaStream_t st) {
    size_t fb = 0;
    cub::DeviceSelect::Flagged(nullptr, fb, cub::CountingInputIterator<int>(0), flags, list, count_dev, n, st);
    void *tmp = ctx.ws.get<char>(std::string("cmp_") + tag, fb);
    PK_CUDA(cub::DeviceSelect::Flagged(tmp, fb, cub::CountingInputIterator<int>(0), flags, list, count_dev, n, st));
    ctx.launches += 2;
}

Partition build_partition(pkgpu_context &ctx, const DeviceTree &T, int rank, int nranks, cudaStream_t st) {
    Workspace &ws = ctx.ws;
    Partition P;
    P.on = true;
    const int nb = (int)T.nboxes, nl = (int)T.nleaves;
    const TreeView tv = T.view();
    // leaves in DFS (Morton) order; equal leaf counts per rank
    unsigned long long *k_in = ws.get<unsigned long long>("pt_kin", nl), *k_out = ws.get<unsigned long long>("pt_kout", nl);
    int *v_in = ws.get<int>("pt_vin", nl), *v_out = ws.get<int>("pt_vout", nl);
    leaf_key_kernel<<<blocks_for(nl, 256), 256, 0, st>>>(tv, T.leaves, nl, k_in, v_in);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, v_out, nl, 0, 36, st);
    void *tmp = ws.get<char>("pt_sort", tb);
    PK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, v_out, nl, 0, 36, st));
    const int lo = (int)((int64_t)nl * rank / nranks), hi = (int)((int64_t)nl * (rank + 1) / nranks);
    P.in = ws.get<int>("pt_in", nb);
    P.own = ws.get<int>("pt_own", nb);
    P.rlo = ws.get<int>("pt_rlo", nb);
    P.rhi = ws.get<int>("pt_rhi", nb);
    part_mask_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(tv, k_out, nl, lo, hi, nranks, P.in, P.own, P.rlo, P.rhi);
    // owned leaves
    P.leaves = ws.get<int>("pt_leaves", std::max(nl, 1));
    int *cnt = ws.get<int>("pt_cnt", 2);
    compact(ctx, P.own, nb, P.leaves, cnt, "own", st);
    // per-level lists of boxes meeting the range
    int *lcount = ws.get<int>("pt_lcount", kMaxLevels + 1), *list = ws.get<int>("pt_list", nb);
    PK_CUDA(cudaMemsetAsync(lcount, 0, (kMaxLevels + 1) * sizeof(int), st));
    flags_by_level_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(tv, P.in, lcount);
    compact(ctx, P.in, nb, list, cnt + 1, "in", st);
    int h[2];
    std::vector<int> lc(kMaxLevels + 1);
    PK_CUDA(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaMemcpyAsync(lc.data(), lcount, lc.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    P.nleaves = h[0];
    std::vector<int> start(kMaxLevels + 1, 0), base(kMaxLevels + 1, 0);
    P.actbase.assign(T.depth + 2, 0);
    int s = 0;
    int64_t c = 0;
    for (int l = 0; l <= T.depth; l++) {
        start[l] = s, base[l] = (int)c, P.actbase[l] = c;
        s += lc[l];
        c += (lc[l] + kI8Tile - 1) / kI8Tile * kI8Tile;
    }
    P.actbase[T.depth + 1] = c;
    P.act = ws.get<int>("pt_act", std::max<int64_t>(c, 1));
    PK_CUDA(cudaMemsetAsync(P.act, 0xff, std::max<int64_t>(c, 1) * sizeof(int), st));
    int *d_sb = ws.get<int>("pt_sb", 2 * (kMaxLevels + 1));
    std::vector<int> sb(start);
    sb.insert(sb.end(), base.begin(), base.end());
    PK_CUDA(cudaMemcpyAsync(d_sb, sb.data(), sb.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    if (h[1] > 0)
        level_list_fill_kernel<<<blocks_for(h[1], 256), 256, 0, st>>>(tv, list, h[1], d_sb, d_sb + kMaxLevels + 1,
                                                                      P.act);
    ctx.launches += 6;
    PK_CUDA(cudaStreamSynchronize(st));
    return P;
}

// Equivalent-density exchange after the upward pass (pkgpu_partition, include/pkgpu.h):
// straddling boxes summed by one allreduce, then the halo -- each rank receives from their
// owners the densities of the V / W sources of its own target boxes (alltoallv). Returns
// the doubles this rank received (the bytes-moved statistic of the stage profiler).
int64_t exchange_up(pkgpu_context &ctx, const DeviceTree &T, const Partition &P, const ListSetup &ls, double *Pup,
                    int Kp, const pkgpu_partition *part, int64_t small_all, cudaStream_t st, unsigned lat_levels = 0) {
    Workspace &ws = ctx.ws;
    const int nb = (int)T.nboxes, R = part->nranks, me = part->rank;
    if (R > 64) throw InvalidArgument("evaluate_partitioned: at most 64 ranks");
    int *flags = ws.get<int>("ex_flags", nb), *cnt = ws.get<int>("ex_cnt", 2 * R + 1);
    int64_t moved = 0;
    // 1. straddlers (identical list on every rank)
    int *slist = ws.get<int>("ex_slist", nb);
    strad_flags_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(P.rlo, P.rhi, nb, flags);
    compact(ctx, flags, nb, slist, cnt + 2 * R, "exs", st);
    // 2. who needs what, from the replicated tree
    unsigned long long *need = ws.get<unsigned long long>("ex_need", nb);
    need_masks(T, ls, P.rlo, P.rhi, need, st, lat_levels); // lattice levels' V sources come with the level gather
    if (small_all > 0) // modulus-split small-level run: every rank computes every small-level column
        need_small_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(T.view(), small_all,
                                                                R == 64 ? ~0ull : (1ull << R) - 1ull, need);
    std::vector<int *> lists(2 * R, nullptr);
    for (int q = 0; q < R; q++)
        for (int dir = 0; dir < 2; dir++) {
            int *l = lists[2 * q + dir] = ws.get<int>("ex_l" + std::to_string(2 * q + dir), nb);
            if (q == me) {
                PK_CUDA(cudaMemsetAsync(cnt + 2 * q + dir, 0, sizeof(int), st));
                continue;
            }
            halo_flags_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(P.rlo, P.rhi, need, nb, me, q, dir, flags);
            compact(ctx, flags, nb, l, cnt + 2 * q + dir, ("exh" + std::to_string(2 * q + dir)).c_str(), st);
        }
    ctx.launches += 2 + 2 * (R - 1);
    std::vector<int> h(2 * R + 1);
    PK_CUDA(cudaMemcpyAsync(h.data(), cnt, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    const int ns = h[2 * R];
    if (ns > 0) {
        double *buf = static_cast<double *>(part->alloc(part->user, (size_t)ns * Kp * sizeof(double)));
        if (!buf) throw RuntimeError("evaluate_partitioned: allocation callback failed");
        const int64_t n = (int64_t)ns * Kp;
        rows_pack_kernel<<<blocks_for(n, 256), 256, 0, st>>>(Pup, slist, ns, Kp, buf);
        PK_CUDA(cudaStreamSynchronize(st));
        if (part->allreduce(part->user, buf, n, st) != 0)
            throw RuntimeError("evaluate_partitioned: allreduce of straddling equivalent densities failed");
        rows_unpack_kernel<<<blocks_for(n, 256), 256, 0, st>>>(buf, slist, ns, Kp, Pup);
        ctx.launches += 2;
        moved += n;
    }
    std::vector<int64_t> sc(R), rc(R);
    int64_t st_tot = 0, rt_tot = 0;
    for (int q = 0; q < R; q++) {
        sc[q] = (int64_t)h[2 * q] * Kp, rc[q] = (int64_t)h[2 * q + 1] * Kp;
        st_tot += sc[q], rt_tot += rc[q];
    }
    double *sbuf = static_cast<double *>(part->alloc(part->user, (size_t)std::max<int64_t>(st_tot, 1) * sizeof(double)));
    double *rbuf = static_cast<double *>(part->alloc(part->user, (size_t)std::max<int64_t>(rt_tot, 1) * sizeof(double)));
    if (!sbuf || !rbuf) throw RuntimeError("evaluate_partitioned: allocation callback failed");
    for (int q = 0, o = 0; q < R; q++) {
        if (h[2 * q]) {
            rows_pack_kernel<<<blocks_for(sc[q], 256), 256, 0, st>>>(Pup, lists[2 * q], h[2 * q], Kp, sbuf + o);
            ctx.launches++;
        }
        o += (int)sc[q];
    }
    PK_CUDA(cudaStreamSynchronize(st));
    if (part->alltoallv(part->user, sbuf, sc.data(), rbuf, rc.data(), st) != 0)
        throw RuntimeError("evaluate_partitioned: halo exchange of equivalent densities failed");
    for (int q = 0; q < R; q++) {
        int64_t o = 0;
        for (int k = 0; k < q; k++) o += rc[k];
        if (h[2 * q + 1]) {
            rows_unpack_kernel<<<blocks_for(rc[q], 256), 256, 0, st>>>(rbuf + o, lists[2 * q + 1], h[2 * q + 1], Kp,
                                                                       Pup);
            ctx.launches++;
        }
    }
    return moved + rt_tot;
}

// int8 operator sets for i8_translate, built on first use
I8Operators &i8_ops(pkgpu_context &ctx, KifmmOps &ops, I8Operators &o, const double *A, int nmat, const char *tag,
                    cudaStream_t st) {
    const I8Settings &is = ctx.i8;
    if (!o.res || o.nmod != is.nmod || o.beta_a != is.beta_a) {
        i8_build_operators(o, ops.ws, A, nmat, ops.K, ops.Kp, is.nmod, is.beta_a, st, tag);
        ctx.launches += 3;
    }
    return o;
}

void pinv_level(pkgpu_context &ctx, KifmmOps &ops, bool up, int64_t lo, int64_t hi, int level, double *Q, double *Tmp,
                double *Phi, cudaStream_t st, const Partition *P, const Layout &Lay) {
    if (ctx.i8.trans) {
        // x = V (S+ (U^T b)) as two int8-pipe translations (nested order kept)
        I8TransArgs a;
        a.K = ops.K;
        a.Kp = ops.Kp;
        if (P && P->on) {
            a.out_box = P->act + P->actbase[level];
            a.ncols = (int)(P->actbase[level + 1] - P->actbase[level]);
        } else {
            a.out_box = Lay.lvcol + Lay.lvbase[level];
            a.ncols = (int)(Lay.lvbase[level + 1] - Lay.lvbase[level]);
        }
        if (a.ncols <= 0) return;
        a.nslots = 1;
        a.src = a.out_box;
        a.ld_src = a.ncols;
        a.src_lo = lo;
        a.src_hi = hi;
        a.X = Q;
        a.Y = Tmp;
        a.rdiv = up ? ops.s_up : ops.s_dn;
        a.rdiv_eps = up ? ops.up.eps : ops.dn.eps;
        I8Operators &u = up ? i8_ops(ctx, ops, ops.i8_ut_up, ops.Ut_up, 1, "ut_up", st)
                            : i8_ops(ctx, ops, ops.i8_ut_dn, ops.Ut_dn, 1, "ut_dn", st);
        ctx.launches += i8_translate(u, a, ctx.i8.beta_b, ctx.ws, st);
        a.X = Tmp;
        a.Y = Phi;
        a.rdiv = nullptr;
        a.alpha = std::ldexp(1.0, -level); // phi /= 2^l (src/fmm.cpp:550-551, 595-596)
        a.beta = 0.0;
        I8Operators &v = up ? i8_ops(ctx, ops, ops.i8_v_up, ops.V_up, 1, "v_up", st)
                            : i8_ops(ctx, ops, ops.i8_v_dn, ops.V_dn, 1, "v_dn", st);
        ctx.launches += i8_translate(v, a, ctx.i8.beta_b, ctx.ws, st);
        return;
    }
    GemmArgs a;
    a.Kp = ops.Kp;
    if (P && P->on) { // only the boxes meeting this rank's leaves
        a.out_box = P->act + P->actbase[level];
        a.ncols = (int)(P->actbase[level + 1] - P->actbase[level]);
    } else {
        a.nvalid = (int)(hi - lo);
        a.box0 = (int)lo;
        a.ncols = round_up(a.nvalid, BN);
        a.napps = a.nvalid;
    }
    if (a.ncols <= 0) return;
    a.A = up ? ops.Ut_up : ops.Ut_dn;
    a.X = Q;
    a.Y = Tmp;
    a.rdiv = up ? ops.s_up : ops.s_dn;
    a.rdiv_eps = up ? ops.up.eps : ops.dn.eps;
    ctx.launches += gather_gemm(a, ctx.ws, st, ctx.num_sms);
    if (ctx.profiling) ctx.stats["dmma_gemm"].units += 1; // gather_gemm_tma_kernel launches
    GemmArgs b = a;
    b.A = up ? ops.V_up : ops.V_dn;
    b.X = Tmp;
    b.Y = Phi;
    b.rdiv = nullptr;
    b.alpha = std::ldexp(1.0, -level); // phi /= 2^l (src/fmm.cpp:550-551, 595-596)
    b.beta = 0.0;
    ctx.launches += gather_gemm(b, ctx.ws, st, ctx.num_sms);
    if (ctx.profiling) ctx.stats["dmma_gemm"].units += 1; // gather_gemm_tma_kernel launches
}

// single-vector pinv: x = V (S+ (U^T b)) (src/linalg.cpp:78-87)
void pinv_vec(pkgpu_context &ctx, KifmmOps &ops, bool up, const double *b, double *tmp, double *x, cudaStream_t st) {
    gemv(up ? ops.Ut_up : ops.Ut_dn, ops.K, ops.K, ops.Kp, b, tmp, 1.0, 0.0, up ? ops.s_up : ops.s_dn,
         up ? ops.up.eps : ops.dn.eps, st);
    gemv(up ? ops.V_up : ops.V_dn, ops.K, ops.K, ops.Kp, tmp, x, 1.0, 0.0, nullptr, 0.0, st);
    ctx.launches += 2;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    PK_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3f;
}

bool same_setup(const pkgpu_setup &a, const pkgpu_setup &b) {
    return a.periodicity == b.periodicity && (a.axes[0] != 0) == (b.axes[0] != 0) &&
           (a.axes[1] != 0) == (b.axes[1] != 0) && (a.axes[2] != 0) == (b.axes[2] != 0) &&
           a.box_length == b.box_length && a.ell == b.ell;
}

} // namespace

void evaluate(pkgpu_context &ctx, const pkgpu_request &req, double *out, pkgpu_timings *timings,
              pkgpu_compat *compat, const pkgpu_partition *part) {
    cudaStream_t st = ctx.stream;
    const bool partitioned = part && part->nranks > 1;
    // A caller's stream (pkgpu_context_set_stream) keeps its ordering but not the work: the
    // evaluate runs on the context's own high-priority stream between two events on the
    // caller's stream, so that the overlapped low-priority lattice M2L yields to the
    // latency-bound chain (a caller's stream usually has the lowest priority itself).
    // Partitioned evaluates hand `st` to the caller's collectives and stay on it.
    struct HandBack {
        pkgpu_context &c;
        cudaStream_t user, work;
        ~HandBack() {
            if (user == work) return;
            if (cudaEventRecord(c.ev_user, work) == cudaSuccess) cudaStreamWaitEvent(user, c.ev_user, 0);
        }
    } hand_back{ctx, st, st};
    if (!partitioned && st != ctx.own_stream && ctx.own_stream && ctx.ev_user && tuning().overlap_m2l) {
        PK_CUDA(cudaEventRecord(ctx.ev_user, st));
        PK_CUDA(cudaStreamWaitEvent(ctx.own_stream, ctx.ev_user, 0));
        st = hand_back.work = ctx.own_stream;
    }
    if (partitioned) {
        if (part->rank < 0 || part->rank >= part->nranks || !part->alloc || !part->allreduce)
            throw InvalidArgument("evaluate_partitioned: bad partition descriptor");
        if (req.mode == PKGPU_MODE_DIRECT)
            throw InvalidArgument("evaluate_partitioned: direct mode is not partitioned");
    }
    const int kernel = req.kernel;
    if (kernel != PKGPU_LAPLACE && kernel != PKGPU_STOKESLET) throw InvalidArgument("unknown kernel");
    const int ks = kernel == PKGPU_LAPLACE ? 1 : 3, kt = ks;
    // src/fmm.cpp:693-701
    if (req.n_strengths != req.n_sources * ks)
        throw InvalidArgument("evaluate: strengths length does not match sources");
    const bool periodic = req.setup.periodicity != PKGPU_NONE;
    if (periodic) {
        if (!req.op) throw ConfigError("evaluate: a periodizing operator is required for periodic runs");
        const pkgpu_operator &op = *req.op;
        if (op.kernel != kernel || op.p != req.p || !same_setup(op.setup, req.setup))
            throw ConfigError("evaluate: operator provenance (kernel/p/ell/periodicity) does not match the request");
    }
    if (req.p < 2) throw InvalidArgument("surface grid requires p >= 2");
    const int64_t ns = req.n_sources, nt = req.n_targets;
    Workspace &ws = ctx.ws;
    // inputs on the device
    const double *d_src = req.sources, *d_str = req.strengths, *d_trg = req.targets;
    double *d_out = out;
    bool str_pending = false; // strengths still in flight on the auxiliary stream
    auto need_strengths = [&]() {
        if (str_pending) PK_CUDA(cudaStreamWaitEvent(st, ctx.ev_join, 0));
        str_pending = false;
    };
    if (!req.device_pointers) {
        // targets passed as the sources' own buffer (the usual self-evaluation) go over once
        const bool same = req.targets == req.sources && nt == ns;
        double *s = ws.get<double>("in_src", 3 * ns + 1), *q = ws.get<double>("in_str", ks * ns + 1),
               *t = same ? s : ws.get<double>("in_trg", 3 * nt + 1);
        if (ns) PK_CUDA(cudaMemcpyAsync(s, req.sources, 3 * ns * sizeof(double), cudaMemcpyHostToDevice, st));
        // the tree needs only the positions: the strengths go over on the auxiliary stream, beside
        // the tree build (awaited before their first use)
        if (ns && ctx.aux_stream && !partitioned) {
            PK_CUDA(cudaEventRecord(ctx.ev_fork, st)); // the staging buffer's previous readers are done
            PK_CUDA(cudaStreamWaitEvent(ctx.aux_stream, ctx.ev_fork, 0));
            PK_CUDA(cudaMemcpyAsync(q, req.strengths, ks * ns * sizeof(double), cudaMemcpyHostToDevice, ctx.aux_stream));
            PK_CUDA(cudaEventRecord(ctx.ev_join, ctx.aux_stream));
            str_pending = true;
        } else if (ns) {
            PK_CUDA(cudaMemcpyAsync(q, req.strengths, ks * ns * sizeof(double), cudaMemcpyHostToDevice, st));
        }
        if (nt && !same) PK_CUDA(cudaMemcpyAsync(t, req.targets, 3 * nt * sizeof(double), cudaMemcpyHostToDevice, st));
        d_src = s, d_str = q, d_trg = t;
        d_out = ws.get<double>("out", kt * nt + 1);
    }
    // compatibility gate (src/refsum.cpp:733-756)
    pkgpu_compat rep{1, 0.0, {0}};
    if (periodic && !(kernel == PKGPU_STOKESLET && req.setup.periodicity == PKGPU_TP) && ns > 0) {
        const int nblk = 256;
        double *part = ws.get<double>("compat_part", 4 * nblk);
        need_strengths();
        compat_partial_kernel<<<nblk, 256, 0, st>>>(d_str, ns, ks, part);
        std::vector<double> h(4 * nblk);
        PK_CUDA(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        ctx.launches += 1;
        double abs_total = 0, sums[3] = {0, 0, 0};
        for (int b = 0; b < nblk; b++) {
            abs_total += h[4 * b];
            for (int c = 0; c < ks; c++) sums[c] += h[4 * b + 1 + c];
        }
        double worst = 0;
        for (int c = 0; c < ks; c++) worst = std::max(worst, std::fabs(sums[c]));
        if (worst > 1e-12 * abs_total) {
            rep.ok = 0;
            rep.residual = worst;
            std::snprintf(rep.violated, sizeof rep.violated, "%s",
                          kernel == PKGPU_LAPLACE ? "neutrality: net charge must vanish"
                                                  : "neutrality: net force must vanish");
        }
    }
    if (compat) *compat = rep;
    if (!rep.ok && !req.force)
        throw ConfigError(std::string("evaluate: compatibility violation (") + rep.violated + ")");
    pkgpu_timings tm{0, 0, 0, 0};
    const int axes[3] = {req.setup.axes[0] != 0, req.setup.axes[1] != 0, req.setup.axes[2] != 0};
    const int ell = req.setup.ell;

    if (req.mode == PKGPU_MODE_DIRECT) {
        // src/fmm.cpp:711-721: all image offsets with max-norm <= ell, skip coincident at 0
        need_strengths();
        PK_CUDA(cudaEventRecord(ctx.ev[0], st));
        std::vector<std::array<int, 3>> offs =
            periodic ? image_offsets(axes, 0, ell) : std::vector<std::array<int, 3>>{{0, 0, 0}};
        std::vector<double> hoffs;
        for (auto &d : offs) hoffs.insert(hoffs.end(), {(double)d[0], (double)d[1], (double)d[2]});
        double *d_offs = ws.get<double>("direct_offs", hoffs.size());
        int *d_coin = ws.get<int>("direct_coin", offs.size());
        PK_CUDA(cudaMemcpyAsync(d_offs, hoffs.data(), hoffs.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        PK_CUDA(cudaMemsetAsync(d_coin, 0, offs.size() * sizeof(int), st));
        KifmmOps &ops = ctx.ops.get(kernel, req.p, st, &ctx.launches);
        PairGeom g{kernel, req.p, ops.n, ops.Kp, ops.d_tmpl};
        // one launch per offset keeps per-offset coincidence counts (error text)
        for (size_t o = 0; o < offs.size(); o++) {
            direct_pairs(kernel, d_trg, nt, d_src, d_str, ns, d_offs + 3 * o, 1, 1, nullptr, nullptr, d_out,
                         o > 0 ? 1 : 0, d_coin + o, ws, st);
            ctx.launches += 1;
        }
        std::vector<int> coin(offs.size());
        PK_CUDA(cudaMemcpyAsync(coin.data(), d_coin, coin.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
        // direct_root_upward_density (src/fmm.cpp:676-686)
        double *q = ws.get<double>("root_q", ops.Kp), *tmp = ws.get<double>("root_t", ops.Kp),
               *up = ws.get<double>("root_up", ops.Kp);
        PK_CUDA(cudaMemsetAsync(q, 0, ops.Kp * sizeof(double), st));
        if (ns) root_check_potential(g, d_src, d_str, ns, q, ws, st);
        pinv_vec(ctx, ops, true, q, tmp, up, st);
        PK_CUDA(cudaEventRecord(ctx.ev[1], st));
        PK_CUDA(cudaStreamSynchronize(st));
        for (size_t o = 0; o < offs.size(); o++)
            if (coin[o] > 0)
                throw InvalidArgument("kernel_block_apply: " + std::to_string(coin[o]) +
                                      " coincident target/source pairs");
        tm.near = elapsed(ctx.ev[0], ctx.ev[1]);
        if (periodic) {
            double *far = ws.get<double>("far_dn", ops.Kp);
            PK_CUDA(cudaEventRecord(ctx.ev[2], st));
            gemv(req.op->device_matrix(ctx.device, st), ops.K, ops.K, ops.K, up, far, 1.0, 0.0, nullptr, 0.0, st);
            PK_CUDA(cudaEventRecord(ctx.ev[3], st));
            direct_pairs(kernel, d_trg, nt, d_src, d_str, 0, nullptr, 0, 1, &g, far, d_out, 1, d_coin, ws, st);
            PK_CUDA(cudaEventRecord(ctx.ev[4], st));
            ctx.launches += 2;
            PK_CUDA(cudaStreamSynchronize(st));
            tm.m2l_apply = elapsed(ctx.ev[2], ctx.ev[3]);
            tm.far = elapsed(ctx.ev[3], ctx.ev[4]);
        }
    } else {
        // ---------------- FMM mode ----------------
        Prof prof(ctx, st);
        PK_CUDA(cudaEventRecord(ctx.ev[0], st));
        int pm = prof.begin("tree");
        DeviceTree &T = ctx.tree;
        build_tree(T, d_src, ns, d_trg, nt, req.leaf_capacity, st, &ctx.launches);
        need_strengths();
        gather_strengths(T, d_str, ks, st, &ctx.launches);
        prof.end(pm);
        PK_CUDA(cudaEventRecord(ctx.ev[1], st));
        KifmmOps &ops = ctx.ops.get(kernel, req.p, st, &ctx.launches);
        // residue range of the int8 M2L for this K (m2l_i8.h): more moduli, or DMMA, when
        // |S| <= 316 K 2^(beta_a + beta_b) could reach M / 2; restored when the call ends
        struct I8Restore {
            pkgpu_context &c;
            I8Settings saved;
            ~I8Restore() { c.i8 = saved; }
        } i8_restore{ctx, ctx.i8};
        ctx.i8 = i8_settings_for(ctx.i8, kNumM2L, ops.K);
        const int Kp = ops.Kp;
        const int64_t nb = T.nboxes;
        PairGeom g{kernel, req.p, ops.n, Kp, ops.d_tmpl};
        pm = prof.begin("lists");
        Partition Part;
        if (partitioned) Part = build_partition(ctx, T, part->rank, part->nranks, st);
        const Partition *PP = partitioned ? &Part : nullptr;
        // the small-level int8 run split by modulus across ranks (allgather given): every
        // rank lays out all of that run's columns
        const bool msplit = partitioned && part->allgather && ctx.i8.enabled;
        const int64_t small_max = tuning().i8_small_boxes;
        int *lmask = partitioned ? Part.in : nullptr;
        if (msplit) {
            lmask = ws.get<int>("pt_in_small", nb);
            small_or_kernel<<<blocks_for(nb, 256), 256, 0, st>>>(T.view(), Part.in, small_max, lmask);
            ctx.launches++;
        }
        ListSetup ls{};
        if (periodic && ell >= 1)
            for (int a = 0; a < 3; a++) ls.periodic[a] = axes[a];
        // levels whose M2L runs as a lattice convolution (m2l_fft.h): filled lattices within
        // the device budget. A partitioned evaluate runs them too, replicated on every rank
        // (a level is one convolution): the level's equivalent densities are gathered after
        // the upward exchange (below)
        // -- up to lattice_max_ranks ranks: beyond, a rank's share of the dense products costs
        // less than the whole level's convolution plus the gather
        int lat[kMaxLevels + 1] = {0};
        if (ctx.i8.lattice && (!partitioned || part->nranks <= tuning().lattice_max_ranks)) {
            const Tuning &tu = tuning();
            int64_t used = 0;
            for (int l = 1; l <= T.depth; l++) {
                const double cells = std::ldexp(1.0, 3 * l);
                const int64_t nl = T.level_off[l + 1] - T.level_off[l];
                const int64_t bytes = m2l_lattice_bytes(ops, l, ls.periodic);
                if (nl >= tu.lattice_fill * cells && used + bytes <= tu.lattice_budget) {
                    lat[l] = 1;
                    used += bytes;
                }
            }
        }
        Layout Lay = build_layout(ctx, T, lmask, lat, st);
        // U / W / X lists, the M2L gather table and the lattice check feed the downward pass only:
        // on a single rank they run on the context's auxiliary stream while the upward pass
        // (S2M, M2M, pinv: layout only) runs on the work stream -- forked here, joined before
        // the X pass. Profiling keeps everything on the work stream (stage times add up).
        const bool overlap_lists = !partitioned && !ctx.profiling && tuning().overlap_lists && ctx.aux_stream;
        auto lists_stage = [&](cudaStream_t ls_st) {
            build_lists_eval(T, ls, ctx.lists, Lay.m2l_table, Lay.ncols, Lay.col_of_box, ops.slot_of_code, ls_st,
                             &ctx.launches, lmask);
            // the lattice levels' V lists must be exactly the stencil (they are for filled levels;
            // a level that is not falls back to the dense product)
            if (std::any_of(Lay.lat, Lay.lat + T.depth + 1, [](int v) { return v != 0; })) {
                ctx.launches += m2l_fft_prepare(ops, ws, ls_st);
                int *bad = ws.get<int>("lat_bad", kMaxLevels + 1);
                PK_CUDA(cudaMemsetAsync(bad, 0, (kMaxLevels + 1) * sizeof(int), ls_st));
                for (int l = 1; l <= T.depth; l++) {
                    if (!Lay.lat[l]) continue;
                    LatticeLevelArgs la;
                    la.level = l;
                    for (int a = 0; a < 3; a++) la.periodic[a] = ls.periodic[a];
                    la.box0 = T.level_off[l];
                    la.box1 = T.level_off[l + 1];
                    la.cell = T.cell;
                    la.srng = T.srng;
                    la.trng = T.trng;
                    la.mask = lmask;
                    ctx.launches += m2l_lattice_check(ops, la, Lay.m2l_table + Lay.colbase[l], Lay.ncols,
                                                      Lay.out_box + Lay.colbase[l],
                                                      (int)(Lay.colbase[l + 1] - Lay.colbase[l]), bad + l, ws, ls_st);
                }
                int hb[kMaxLevels + 1];
                PK_CUDA(cudaMemcpyAsync(hb, bad, sizeof hb, cudaMemcpyDeviceToHost, ls_st));
                PK_CUDA(cudaStreamSynchronize(ls_st));
                static const bool dbg = std::getenv("PKGPU_LATTICE_DEBUG") != nullptr;
                for (int l = 1; l <= T.depth; l++) {
                    if (dbg && Lay.lat[l])
                        std::fprintf(stderr, "lattice level %d: %lld boxes, %d V-list mismatches\n", l,
                                     (long long)(T.level_off[l + 1] - T.level_off[l]), hb[l]);
                    if (Lay.lat[l] && hb[l]) Lay.lat[l] = 0; // dense fallback (DMMA)
                }
            }
        };
        if (overlap_lists)
            PK_CUDA(cudaEventRecord(ctx.ev_fork, st)); // tree + layout complete
        else
            lists_stage(st);
        prof.end(pm);
        // pseudo-inverse scratch: one level at a time (indexed by box id through a level offset)
        int64_t maxlev = 1;
        for (int l = 0; l <= T.depth; l++) maxlev = std::max<int64_t>(maxlev, T.level_off[l + 1] - T.level_off[l]);
        double *Q = ws.get<double>("Q", nb * Kp), *Tm = ws.get<double>("Tmp", maxlev * Kp),
               *Pdn = ws.get<double>("phi_dn", nb * Kp);
        // phi_up lives in collective-visible memory when partitioned without a halo exchange
        // (then summed over ranks in one allreduce)
        const bool halo = partitioned && part->alltoallv;
        double *Pup = partitioned && !halo ? static_cast<double *>(part->alloc(part->user, nb * Kp * sizeof(double)))
                                           : ws.get<double>("phi_up", nb * Kp);
        if (!Pup) throw RuntimeError("evaluate_partitioned: allocation callback failed");
        if (partitioned) PK_CUDA(cudaMemsetAsync(Pup, 0, nb * Kp * sizeof(double), st));
        // The deepest lattice level's M2L (the bulk of the M2L) depends only on that level's
        // phi_up: it runs on a second auxiliary stream (own workspace) from the moment its
        // pinv_up is queued, beside the M2M / pinv chain of the coarser levels, the lists and the
        // coarse levels' downward chain, whose small launches leave most of the GPU idle. The
        // result stays in the workspace; the scatter into q runs on the work stream where the
        // downward pass reaches the level (after the X pass: q has one writer at a time). The
        // lattice check of the lists stage still decides: a level it rejects drops the result.
        auto lat_args = [&](int l, bool defer) {
            LatticeLevelArgs la;
            la.level = l;
            for (int a = 0; a < 3; a++) la.periodic[a] = ls.periodic[a];
            la.box0 = T.level_off[l];
            la.box1 = T.level_off[l + 1];
            la.cell = T.cell;
            la.X = Pup;
            la.Y = Q;
            la.alpha = std::ldexp(1.0, l); // q += 2^l M_d phi_src (src/fmm.cpp:573)
            la.defer_scatter = defer;
            return la;
        };
        // (the coarser lattice levels likewise, on a third stream of middle priority: small, but
        // they sat on the chain, which ends the overlapped region once the deepest level's M2L
        // has become cheaper than it)
        int lat_async = -1;
        bool lat_early[kMaxLevels + 1] = {false};
        if (overlap_lists && tuning().overlap_m2l && ctx.aux2_stream && ctx.aux3_stream) {
            for (int l = 2; l <= T.depth; l++)
                if (Lay.lat[l]) lat_async = l, lat_early[l] = true;
            if (lat_async >= 2) ctx.launches += m2l_fft_prepare(ops, ws, st); // kernel spectra (first use)
        }
        // ---- upward pass (src/fmm.cpp:532-553) ----
        PK_CUDA(cudaMemsetAsync(Q, 0, nb * Kp * sizeof(double), st));
        pm = prof.begin("s2m");
        s2m_pass(g, T, Q, st, partitioned ? Part.leaves : nullptr, partitioned ? Part.nleaves : 0);
        ctx.launches += 1;
        prof.end(pm);
        for (int l = T.depth; l >= 0; l--) {
            const int64_t lo = T.level_off[l], hi = T.level_off[l + 1];
            const int64_t c0 = Lay.m2mbase[l], c1 = Lay.m2mbase[l + 1];
            if (c1 > c0 && ctx.i8.trans) {
                I8TransArgs a;
                a.K = ops.K;
                a.Kp = Kp;
                a.ncols = (int)(c1 - c0);
                a.out_box = Lay.out_m2m + c0;
                a.nslots = 8;
                a.src = Lay.m2m_src + c0;
                a.ld_src = Lay.nm2m;
                a.src_lo = T.level_off[l + 1]; // children
                a.src_hi = T.level_off[l + 2];
                a.X = Pup;
                a.Y = Q;
                a.alpha = std::ldexp(1.0, l); // q += 2^l M2M_o phi_child (src/fmm.cpp:547)
                a.beta = 0.0;
                pm = prof.begin("m2m");
                ctx.launches += i8_translate(i8_ops(ctx, ops, ops.i8_m2m, ops.m2m, 8, "m2m", st), a, ctx.i8.beta_b, ws, st);
                prof.end(pm);
            } else if (c1 > c0) {
                GemmArgs a;
                a.Kp = Kp;
                a.ncols = (int)(c1 - c0);
                a.out_box = Lay.out_m2m + c0;
                a.nslots = 8;
                a.src = Lay.m2m_src + c0;
                a.ld_src = Lay.nm2m;
                a.A = ops.m2m;
                a.nmat = 8;
                a.X = Pup;
                a.Y = Q;
                a.alpha = std::ldexp(1.0, l); // q += 2^l M2M_o phi_child (src/fmm.cpp:547)
                a.beta = 0.0;
                a.napps = (int)std::min<int64_t>(8 * (hi - lo), 1 << 30); // the level's parents x 8 children
                pm = prof.begin("m2m");
                ctx.launches += gather_gemm(a, ws, st, ctx.num_sms);
                if (ctx.profiling) ctx.stats["dmma_gemm"].units += 1; // gather_gemm_tma_kernel launches
                prof.end(pm);
            }
            pm = prof.begin("pinv_up");
            pinv_level(ctx, ops, true, lo, hi, l, Q, Tm - lo * Kp, Pup, st, PP, Lay);
            prof.end(pm);
            if (lat_early[l]) {
                // phi_up of this lattice level is final: its M2L starts here, beside the rest of
                // the upward pass, the lists and the coarse levels' downward chain
                cudaStream_t ls = l == lat_async ? ctx.aux2_stream : ctx.aux3_stream;
                PK_CUDA(cudaEventRecord(ctx.ev_lat_fork[l], st));
                PK_CUDA(cudaStreamWaitEvent(ls, ctx.ev_lat_fork[l], 0));
                ctx.launches += m2l_lattice_level(ops, lat_args(l, true), ctx.ws_lat[l], ls);
                PK_CUDA(cudaEventRecord(ctx.ev_lat_join[l], ls));
            }
        }
        if (overlap_lists) {
            // the upward pass is queued; build the lists beside it and join
            PK_CUDA(cudaStreamWaitEvent(ctx.aux_stream, ctx.ev_fork, 0));
            lists_stage(ctx.aux_stream);
            PK_CUDA(cudaEventRecord(ctx.ev_join, ctx.aux_stream));
            PK_CUDA(cudaStreamWaitEvent(st, ctx.ev_join, 0));
        }
        if (halo) {
            // straddlers summed, then the halo of V / W sources from their owners
            pm = prof.begin("comm");
            unsigned lat_levels = 0;
            for (int l = 1; l <= T.depth; l++)
                if (Lay.lat[l]) lat_levels |= 1u << l;
            const int64_t moved = exchange_up(ctx, T, Part, ls, Pup, Kp, part, msplit ? small_max : 0, st, lat_levels);
            prof.end(pm);
            prof.work("comm", 8.0 * moved, 0.0);
        } else if (partitioned) {
            // the upward chain is linear in the sources: the complete equivalent densities
            // (root included, feeding the periodizing step) are the sum over ranks
            pm = prof.begin("comm");
            PK_CUDA(cudaStreamSynchronize(st));
            if (part->allreduce(part->user, Pup, nb * Kp, st) != 0)
                throw RuntimeError("evaluate_partitioned: allreduce of equivalent densities failed");
            prof.end(pm);
            prof.work("comm", 8.0 * nb * Kp, 0.0);
        }
        if (halo) {
            // lattice levels need every box's density on every rank: each row is contributed by
            // the rank of its first leaf (complete there: an owner's box, or a straddler after
            // the straddler allreduce) and summed -- an allgather through the allreduce callback
            for (int l = 1; l <= T.depth; l++) {
                if (!Lay.lat[l]) continue;
                const int64_t lo = T.level_off[l], hi = T.level_off[l + 1], cnt = (hi - lo) * Kp;
                pm = prof.begin("comm");
                double *buf = static_cast<double *>(part->alloc(part->user, cnt * sizeof(double)));
                if (!buf) throw RuntimeError("evaluate_partitioned: allocation callback failed");
                level_contrib_kernel<<<blocks_for(cnt, 256), 256, 0, st>>>(Pup, Part.rlo, part->rank, lo, hi, Kp, buf);
                PK_CUDA(cudaStreamSynchronize(st));
                if (part->allreduce(part->user, buf, cnt, st) != 0)
                    throw RuntimeError("evaluate_partitioned: allreduce of a lattice level's densities failed");
                PK_CUDA(cudaMemcpyAsync(Pup + lo * Kp, buf, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
                ctx.launches += 1;
                prof.end(pm);
                prof.work("comm", 8.0 * cnt, 0.0);
            }
        }
        PK_CUDA(cudaEventRecord(ctx.ev[2], st));
        // ---- periodizing step: far density on the root outer surface. It needs only the root's
        // phi_up: queued here, ahead of the downward pass, its five small launches run while the
        // overlapped lattice M2L keeps the GPU busy instead of between the downward pass and
        // the leaf pass (cfg2: 0.05 ms off the critical path) ----
        double *far = nullptr;
        pm = prof.begin("periodic");
        if (periodic) {
            far = ws.get<double>("far_dn", Kp);
            gemv(req.op->device_matrix(ctx.device, st), ops.K, ops.K, ops.K, Pup, far, 1.0, 0.0, nullptr, 0.0, st);
            ctx.launches += 1;
            if (ell >= 2 && ns > 0) {
                // image layers 2..ell (src/fmm.cpp:635-645): pinv(a_dn, M_img phi_up[0])
                const double *mimg = ctx.ops.image_operator(ops, axes, ell, st, &ctx.launches);
                double *qi = ws.get<double>("img_q", Kp), *ti = ws.get<double>("img_t", Kp),
                       *pi = ws.get<double>("img_phi", Kp);
                gemv(mimg, ops.K, ops.K, Kp, Pup, qi, 1.0, 0.0, nullptr, 0.0, st);
                pinv_vec(ctx, ops, false, qi, ti, pi, st);
                add_kernel<<<(ops.K + 255) / 256, 256, 0, st>>>(far, pi, ops.K);
                ctx.launches += 2;
            }
        }
        prof.end(pm);
        PK_CUDA(cudaEventRecord(ctx.ev[3], st));
        // ---- downward pass (src/fmm.cpp:557-601) ----
        PK_CUDA(cudaMemsetAsync(Q, 0, nb * Kp * sizeof(double), st));
        pm = prof.begin("x");
        x_pass(g, T, ctx.lists, Q, st);
        ctx.launches += ctx.lists.x.count ? 1 : 0;
        prof.end(pm);
        int i8_apps[kMaxLevels + 1] = {0}; // levels whose M2L ran on the int8 pipe
        int lat_apps[kMaxLevels + 1] = {0}; // levels whose M2L ran as a lattice convolution
        bool mma_rows_zeroed = false;
        // ---- M2L on the int8 pipe: every int8 level in ONE launch (M2L reads only phi_up,
        // so it can precede the L2L chain; one pass streams each operator tile once for all
        // levels), in runs of consecutive int8 levels ----
        for (int l = 1; l <= T.depth;) {
            if (!Lay.i8[l]) {
                l++;
                continue;
            }
            // one launch per int8 run (build_layout): the small levels together, each big
            // level alone (measured: one launch for every level is slower at cfg2)
            const int l1 = Lay.i8_last[l];
            const I8Settings &is = ctx.i8;
            if (!ops.i8.res || ops.i8.nmod != is.nmod || ops.i8.beta_a != is.beta_a) {
                i8_build_operators(ops.i8, ops.ws, ops.m2l, kNumM2L, ops.K, Kp, is.nmod, is.beta_a, st);
                ctx.launches += 3;
            }
            I8LevelArgs a;
            a.K = ops.K;
            a.Kp = Kp;
            const int64_t c0 = Lay.colbase[l];
            a.ncols = (int)(Lay.colbase[l1 + 1] - c0);
            a.out_box = Lay.out_box + c0;
            a.nslots = kNumM2L;
            a.src = Lay.m2l_table + c0;
            a.ld_src = Lay.ncols;
            a.lv.n = l1 - l + 1;
            for (int j = 0; j <= a.lv.n; j++) {
                a.lv.box0[j] = T.level_off[l + j];
                a.lv.col0[j] = Lay.colbase[l + j] - c0;
                if (j < a.lv.n) a.lv.alpha[j] = std::ldexp(1.0, l + j); // q += 2^l M_d phi_src (src/fmm.cpp:573)
            }
            a.X = Pup;
            a.Y = Q;
            a.big = Lay.i8_big[l] != 0;
            if (ctx.profiling) {
                a.mma_rows = ws.get<unsigned long long>("i8_mma_rows", 1);
                if (!mma_rows_zeroed) PK_CUDA(cudaMemsetAsync(a.mma_rows, 0, sizeof(unsigned long long), st));
                mma_rows_zeroed = true;
            }
            pm = prof.begin("m2l");
            int ps = prof.begin("m2l_prep");
            I8LevelWork w = m2l_i8_prepare(ops.i8, a, is.beta_b, ws, st, &ctx.launches);
            prof.end(ps);
            const int64_t win = i8_window(ops.i8.nmod, ops.i8.Ki);
            // split by modulus across ranks: ceil(nmod / R) moduli here, the residue sums of
            // all columns gathered before the CRT (the run streams 1 / R of the operators)
            const bool split_run = msplit && !a.big && a.ncols <= win;
            int64_t split_block = 0;
            if (split_run) {
                const int R = part->nranks, B = (ops.i8.nmod + R - 1) / R;
                split_block = (int64_t)B * a.ncols * ops.i8.Ki * (int64_t)sizeof(int);
                w.R_ext = static_cast<int *>(part->alloc(part->user, (size_t)split_block * R));
                if (!w.R_ext) throw RuntimeError("evaluate_partitioned: allocation callback failed");
                w.t0 = std::min(ops.i8.nmod, part->rank * B);
                w.t1 = std::min(ops.i8.nmod, (part->rank + 1) * B);
            }
            for (int64_t w0 = 0; w0 < a.ncols; w0 += win) { // column windows bound the residue sums
                const int64_t w1 = std::min<int64_t>(a.ncols, w0 + win);
                ps = prof.begin("m2l_prep");
                ctx.launches += m2l_i8_window(ops.i8, a, w, w0, w1, ws, st);
                prof.end(ps);
                ps = prof.begin("m2l_i8");
                if (!split_run || w.t1 > w.t0) ctx.launches += m2l_i8_gemm(ops.i8, a, w, w0, w1, ws, st);
                prof.end(ps);
                if (split_run) {
                    ps = prof.begin("comm");
                    PK_CUDA(cudaStreamSynchronize(st));
                    if (part->allgather(part->user, w.R_ext, split_block, st) != 0)
                        throw RuntimeError("evaluate_partitioned: allgather of residue sums failed");
                    prof.end(ps);
                    prof.work("comm", (double)split_block * (part->nranks - 1), 0.0);
                }
                ps = prof.begin("m2l_crt");
                ctx.launches += m2l_i8_finish(ops.i8, a, w, w0, w1, is.beta_b, st);
                prof.end(ps);
            }
            prof.end(pm);
            for (int j = l; j <= l1; j++) i8_apps[j] = 1;
            l = l1 + 1;
        }
        for (int l = 0; l <= T.depth; l++) {
            const int64_t lo = T.level_off[l], hi = T.level_off[l + 1];
            const int64_t c0 = Lay.colbase[l], c1 = Lay.colbase[l + 1];
            if (lat_early[l]) PK_CUDA(cudaStreamWaitEvent(st, ctx.ev_lat_join[l], 0)); // also when dropped
            if (lat_early[l] && Lay.lat[l]) {
                // computed on an auxiliary stream: add it into q
                pm = prof.begin("m2l");
                ctx.launches += m2l_lattice_scatter(ops, lat_args(l, true), ctx.ws_lat[l], st);
                prof.end(pm);
                lat_apps[l] = 1;
            } else if (l >= 1 && Lay.lat[l]) {
                // M2L as a convolution on the level's lattice (m2l_fft.h)
                pm = prof.begin("m2l");
                LatticeLevelArgs la;
                la.level = l;
                for (int a = 0; a < 3; a++) la.periodic[a] = ls.periodic[a];
                la.box0 = lo;
                la.box1 = hi;
                la.cell = T.cell;
                la.X = Pup;
                la.Y = Q;
                la.alpha = std::ldexp(1.0, l); // q += 2^l M_d phi_src (src/fmm.cpp:573)
                struct Hook {
                    Prof *prof;
                    int open;
                } hook{&prof, -1};
                la.user = &hook;
                la.mark = [](void *u, const char *stage, int begin) {
                    Hook *h = static_cast<Hook *>(u);
                    if (begin) {
                        h->open = h->prof->begin(stage);
                    } else {
                        h->prof->end(h->open);
                        // lat_mul is one kernel launch (the level's launches are added afterwards)
                        if (h->open >= 0 && !std::strcmp(stage, "lat_mul")) h->prof->ctx.stats[stage].launches += 1;
                    }
                };
                la.work = [](void *u, const char *stage, double units, double per_unit) {
                    static_cast<Hook *>(u)->prof->work(stage, units, per_unit);
                };
                ctx.launches += m2l_lattice_level(ops, la, ws, st);
                prof.end(pm);
                lat_apps[l] = 1;
            } else if (l >= 1 && Lay.i8[l]) {
                // M2L done above
            } else if (l >= 1 && ctx.i8.fft) {
                // M2L by FFT on the surface lattice (m2l_fft.h)
                pm = prof.begin("m2l");
                ctx.launches += m2l_fft_prepare(ops, ws, st);
                FftLevelArgs fa;
                fa.ncols = (int)(c1 - c0);
                fa.out_box = Lay.out_box + c0;
                fa.src = Lay.m2l_table + c0;
                fa.ld = Lay.ncols;
                fa.box0 = T.level_off[l];
                fa.box1 = T.level_off[l + 1];
                fa.X = Pup;
                fa.Y = Q;
                fa.alpha = std::ldexp(1.0, l); // q += 2^l M_d phi_src (src/fmm.cpp:573)
                ctx.launches += m2l_fft_level(ops, fa, ws, st);
                prof.end(pm);
            } else if (l >= 1) {
                GemmArgs a;
                a.Kp = Kp;
                a.ncols = (int)(c1 - c0);
                a.out_box = Lay.out_box + c0;
                a.nslots = kNumM2L;
                a.src = Lay.m2l_table + c0;
                a.ld_src = Lay.ncols;
                a.A = ops.m2l;
                a.nmat = kNumM2L;
                a.bn = Lay.wide[l] ? 128 : 64;
                a.X = Pup;
                a.Y = Q;
                a.alpha = std::ldexp(1.0, l); // q += 2^l M_d phi_src (src/fmm.cpp:573, 168-171)
                a.beta = 1.0;
                pm = prof.begin("m2l");
                ctx.launches += gather_gemm(a, ws, st, ctx.num_sms);
                if (ctx.profiling) ctx.stats["dmma_gemm"].units += 1; // gather_gemm_tma_kernel launches
                prof.end(pm);
            }
            if (l >= 1 && ctx.i8.trans) {
                const int64_t o0 = Lay.octbase[l], o1 = Lay.octbase[l + 1];
                I8TransArgs b;
                b.K = ops.K;
                b.Kp = Kp;
                b.ncols = (int)(o1 - o0);
                b.out_box = Lay.out_oct + o0;
                b.nslots = 8;
                b.src = Lay.l2l_src8 + o0;
                b.ld_src = Lay.noct;
                b.src_lo = T.level_off[l - 1]; // parents
                b.src_hi = T.level_off[l];
                b.X = Pdn;
                b.Y = Q;
                b.alpha = std::ldexp(1.0, l) * 0.5; // q += (2^l / 2) L2L_o phi_parent (src/fmm.cpp:590-591)
                b.beta = 1.0;
                pm = prof.begin("l2l");
                ctx.launches += i8_translate(i8_ops(ctx, ops, ops.i8_l2l, ops.l2l, 8, "l2l", st), b, ctx.i8.beta_b, ws, st);
                prof.end(pm);
            } else if (l >= 1) {
                const int64_t o0 = Lay.octbase[l], o1 = Lay.octbase[l + 1];
                GemmArgs b;
                b.Kp = Kp;
                b.ncols = (int)(o1 - o0);
                b.out_box = Lay.out_oct + o0;
                b.nslots = 1;
                b.src = Lay.l2l_src + o0;
                b.ld_src = Lay.noct;
                b.tile_mat = Lay.tile_oct + o0 / BN;
                b.A = ops.l2l;
                b.nmat = 8;
                b.X = Pdn;
                b.Y = Q;
                b.alpha = std::ldexp(1.0, l) * 0.5; // q += (2^l / 2) L2L_o phi_parent (src/fmm.cpp:590-591)
                b.beta = 1.0;
                b.napps = (int)std::min<int64_t>(hi - lo, 1 << 30); // one parent per box of the level
                pm = prof.begin("l2l");
                ctx.launches += gather_gemm(b, ws, st, ctx.num_sms);
                if (ctx.profiling) ctx.stats["dmma_gemm"].units += 1; // gather_gemm_tma_kernel launches
                prof.end(pm);
            }
            pm = prof.begin("pinv_dn");
            pinv_level(ctx, ops, false, lo, hi, l, Q, Tm - lo * Kp, Pdn, st, PP, Lay);
            prof.end(pm);
        }
        // ---- leaf pass: L2T + W + U + far ----
        pm = prof.begin("leaf");
        if (partitioned) {
            // each target is written by exactly one rank; the sum over ranks is the result
            double *pout = static_cast<double *>(part->alloc(part->user, std::max<int64_t>(kt * nt, 1) * sizeof(double)));
            if (!pout) throw RuntimeError("evaluate_partitioned: allocation callback failed");
            PK_CUDA(cudaMemsetAsync(pout, 0, kt * nt * sizeof(double), st));
            leaf_pass(g, T, ctx.lists, Pdn, Pup, far, pout, st, Part.leaves, Part.nleaves);
            prof.end(pm);
            pm = prof.begin("comm");
            PK_CUDA(cudaStreamSynchronize(st));
            if (part->allreduce(part->user, pout, kt * nt, st) != 0)
                throw RuntimeError("evaluate_partitioned: allreduce of potentials failed");
            if (nt) PK_CUDA(cudaMemcpyAsync(d_out, pout, kt * nt * sizeof(double), cudaMemcpyDeviceToDevice, st));
        } else {
            leaf_pass(g, T, ctx.lists, Pdn, Pup, far, d_out, st);
        }
        ctx.launches += 1;
        prof.end(pm);
        PK_CUDA(cudaEventRecord(ctx.ev[4], st));
        PK_CUDA(cudaStreamSynchronize(st));
        prof.finish();
        if (ctx.profiling) {
            unsigned long long *cnt = ws.get<unsigned long long>("work_cnt", 8);
            PK_CUDA(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), st));
            work_count_kernel<<<blocks_for(nb, 128), 128, 0, st>>>(T.view(), ops.n, ctx.lists.u.off,
                                                                   ctx.lists.u.ent, ctx.lists.w.off,
                                                                   ctx.lists.x.off, ctx.lists.x.ent, cnt);
            unsigned long long h[8];
            PK_CUDA(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
            PK_CUDA(cudaStreamSynchronize(st));
            const double pf = kernel == PKGPU_LAPLACE ? 11.0 : 28.0;
            const double K = ops.K, dense = 2.0 * K * K, pinv = 4.0 * K * K + K;
            const double far_pairs = periodic ? (double)nt * ops.n : 0.0;
            prof.work("leaf", (double)(h[0] + h[1] + h[2]) + far_pairs, pf);
            prof.work("s2m", (double)h[3], pf);
            prof.work("x", (double)h[4], pf);
            prof.work("m2m", (double)h[5], dense);
            prof.work("m2l", (double)ctx.lists.v_total, dense);
            // int8 levels: V applications there (CSR offsets at the level bounds); the
            // algorithmic int8 work is nmod K^2 MACs per application (2 ops per MAC)
            double v_i8 = 0, v_lat = 0;
            for (int l = 1; l <= T.depth; l++) {
                if (lat_apps[l]) {
                    int64_t o2[2];
                    PK_CUDA(cudaMemcpy(&o2[0], ctx.lists.v.off + T.level_off[l], sizeof(int64_t), cudaMemcpyDeviceToHost));
                    PK_CUDA(cudaMemcpy(&o2[1], ctx.lists.v.off + T.level_off[l + 1], sizeof(int64_t),
                                       cudaMemcpyDeviceToHost));
                    v_lat += (double)(o2[1] - o2[0]);
                }
                if (!i8_apps[l]) continue;
                int64_t o2[2];
                PK_CUDA(cudaMemcpy(&o2[0], ctx.lists.v.off + T.level_off[l], sizeof(int64_t), cudaMemcpyDeviceToHost));
                PK_CUDA(cudaMemcpy(&o2[1], ctx.lists.v.off + T.level_off[l + 1], sizeof(int64_t),
                                   cudaMemcpyDeviceToHost));
                v_i8 += (double)(o2[1] - o2[0]);
            }
            // lattice levels: V applications served by the convolution (dense-equivalent FLOP)
            if (v_lat > 0) prof.work("m2l_lattice", v_lat, dense);
            if (v_i8 > 0) {
                prof.work("m2l_i8", v_i8, 2.0 * ctx.i8.nmod * K * K);
                if (mma_rows_zeroed) { // MMA rows issued vs V applications (tile padding / union waste)
                    unsigned long long rows = 0;
                    PK_CUDA(cudaMemcpyAsync(&rows, ws.get<unsigned long long>("i8_mma_rows", 1), sizeof rows,
                                            cudaMemcpyDeviceToHost, st));
                    PK_CUDA(cudaStreamSynchronize(st));
                    prof.work("m2l_mma_rows", (double)rows, 0.0);
                }
                prof.work("m2l_prep", v_i8, 0.0);
                prof.work("m2l_crt", v_i8, 0.0);
            }
            prof.work("l2l", (double)h[6], dense);
            prof.work("pinv_dn", (double)h[6], pinv);
            prof.work("pinv_up", (double)h[7], pinv);
            prof.work("periodic", periodic ? 1.0 : 0.0, dense + (ell >= 2 ? dense + pinv : 0.0));
            auto &u = ctx.stats["u_pairs"];
            u.units += (double)h[0];
            u.flops += (double)h[0] * pf;
        }
        tm.tree = elapsed(ctx.ev[0], ctx.ev[1]);
        tm.near = elapsed(ctx.ev[1], ctx.ev[2]) + elapsed(ctx.ev[3], ctx.ev[4]);
        tm.m2l_apply = elapsed(ctx.ev[2], ctx.ev[3]);
        tm.far = 0.0; // fused into the leaf pass
    }
    if (!req.device_pointers && nt) {
        PK_CUDA(cudaMemcpyAsync(out, d_out, kt * nt * sizeof(double), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
    }
    if (timings) *timings = tm;
}

void kernel_block_apply_device(pkgpu_context &ctx, int kernel, const double *targets, int64_t nt,
                               const double *sources, int64_t ns, const double *shift, const double *density,
                               double *out, int skip) {
    cudaStream_t st = ctx.stream;
    Workspace &ws = ctx.ws;
    const int ks = kernel == 0 ? 1 : 3;
    double *t = ws.get<double>("kba_t", 3 * nt + 1), *s = ws.get<double>("kba_s", 3 * ns + 1),
           *d = ws.get<double>("kba_d", ks * ns + 1), *o = ws.get<double>("kba_o", ks * nt + 1),
           *sh = ws.get<double>("kba_sh", 3);
    int *coin = ws.get<int>("kba_coin", 1);
    if (nt) PK_CUDA(cudaMemcpyAsync(t, targets, 3 * nt * sizeof(double), cudaMemcpyHostToDevice, st));
    if (ns) PK_CUDA(cudaMemcpyAsync(s, sources, 3 * ns * sizeof(double), cudaMemcpyHostToDevice, st));
    if (ns) PK_CUDA(cudaMemcpyAsync(d, density, ks * ns * sizeof(double), cudaMemcpyHostToDevice, st));
    if (nt) PK_CUDA(cudaMemcpyAsync(o, out, ks * nt * sizeof(double), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemcpyAsync(sh, shift, 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaMemsetAsync(coin, 0, sizeof(int), st));
    // shift == 0 with skip -> coincident pairs contribute 0; anything else is counted
    direct_pairs(kernel, t, nt, s, d, ns, sh, 1, skip, nullptr, nullptr, o, 1, coin, ws, st);
    ctx.launches += 1;
    int hcoin = 0;
    PK_CUDA(cudaMemcpyAsync(&hcoin, coin, sizeof(int), cudaMemcpyDeviceToHost, st));
    std::vector<double> res(ks * nt);
    if (nt) PK_CUDA(cudaMemcpyAsync(res.data(), o, ks * nt * sizeof(double), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    // src/kernel.cpp:125-127: coincident pairs are an error unless skip was requested
    // (the sum itself is still computed with their contribution set to zero)
    if (hcoin > 0 && !skip)
        throw InvalidArgument("kernel_block_apply: " + std::to_string(hcoin) + " coincident target/source pairs");
    std::memcpy(out, res.data(), res.size() * sizeof(double));
}

} // namespace pkgpu
