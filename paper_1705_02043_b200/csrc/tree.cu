// Device octree build: FmmTree::FmmTree (src/fmm.cpp:301-389) restated as
//   36-bit Morton keys (x = least significant bit of each triple) from floor(x*4096)
//   -> stable radix sort of (key, index) for sources and targets (the key bits of the first
//      8 levels; all 36 once a tree has needed more)
//   -> level-synchronous splitting: a box splits iff |src| > s or |trg| > s; its
//      children are the non-empty next-octant-digit sub-ranges, emitted in octant
//      order, so boxes come out level-major and Morton-ordered within a level —
//      exactly the reference's BFS numbering. All levels run in ONE cooperative kernel
//      (tree_loop_kernel: grid barriers between levels, one header read back at the end).
// x >= box_center  <=>  the (l+1)-th most significant bit of floor(x*4096) is set,
// because box centers (c+1/2)2^-l are exact dyadics (SURVEY.md §8a "Tree semantics").
#include <algorithm>
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <sstream>

#include "tree.h"
#include "tuning.h"

namespace pkgpu {

namespace cg = cooperative_groups;

namespace {

__device__ __forceinline__ unsigned long long spread3(unsigned v) {
    unsigned long long x = v & 0xfffu;
    unsigned long long r = 0;
#pragma unroll
    for (int b = 0; b < 12; b++) r |= ((x >> b) & 1ull) << (3 * b);
    return r;
}

__global__ void keys_kernel(const double *__restrict__ pts, int64_t n, unsigned long long *__restrict__ keys,
                            int *__restrict__ idx, int *__restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    // same predicate as src/fmm.cpp:310 (NaN passes it there, and lands in octant 0
    // at every split since NaN >= c is false — floor(NaN) converts to 0 here)
    const bool outside = x < 0 || x >= 1 || y < 0 || y >= 1 || z < 0 || z >= 1;
    if (outside) {
        atomicAdd(bad, 1);
        keys[i] = 0;
    } else {
        const unsigned qx = (unsigned)floor(x * 4096.0), qy = (unsigned)floor(y * 4096.0),
                       qz = (unsigned)floor(z * 4096.0);
        keys[i] = spread3(qx) | (spread3(qy) << 1) | (spread3(qz) << 2);
    }
    idx[i] = (int)i;
}

// first position in [lo, hi) whose octant digit (at `shift`) is >= o
__device__ __forceinline__ int lower_digit(const unsigned long long *__restrict__ keys, int lo, int hi, int shift,
                                           unsigned o) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (((keys[mid] >> shift) & 7u) < o)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void gather_pos_kernel(const double *__restrict__ pts, const int *__restrict__ perm, int64_t n,
                                  double4 *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t j = perm[i];
    out[i] = make_double4(pts[3 * j], pts[3 * j + 1], pts[3 * j + 2], 0.0);
}

__global__ void gather_str_kernel(const double *__restrict__ str, const int *__restrict__ perm, int64_t n, int ks,
                                  double4 *__restrict__ pos, double4 *__restrict__ f) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t j = perm[i];
    if (ks == 1)
        pos[i].w = str[j];
    else
        f[i] = make_double4(str[3 * j], str[3 * j + 1], str[3 * j + 2], 0.0);
}

// ---------------------------------------------------------------------------
// The level loop as ONE cooperative kernel (grid-wide barriers instead of a host round trip
// per level: the level's box count decides the next level's launch, and at cfg2 those seven
// round trips were 0.25 ms of a 3.9 ms evaluate). CTA c owns a contiguous chunk of the
// level's boxes, so child offsets are the CTA totals' prefix plus a block scan inside the
// chunk -- the same order as the exclusive sum over the whole level. The arrays have a
// capacity fixed at launch; a level that would not fit sets hdr->need and every CTA stops
// (the host grows the arrays and runs the kernel again). After the last level the same
// scheme compacts the leaves (BFS order).
struct TreeHeader {
    int depth, nboxes, nleaves, err_deep;
    long long need; // boxes needed when the capacity was exceeded (0: fits)
    int need_bits;  // a box had to split on key bits below the sorted ones (sort all 36 and rebuild)
    int pad_;
    int level_off[kMaxLevels + 2];
    int oct_hist[kMaxLevels * 8];    // boxes per (level, octant of the cell in its parent)
    int m2m_count[kMaxLevels + 1];   // internal boxes with sources per level
};

struct TreeLoopArgs {
    int cap, leaf_cap;
    int min_bit; // the keys are sorted on bits [min_bit, 36) only
    int ns, nt;  // the root's ranges
    const unsigned long long *skeys, *tkeys;
    unsigned long long *prefix;
    int4 *cell;
    int *parent, *child, *isleaf;
    int2 *srng, *trng;
    int *childcnt; // [cap]
    int4 *crange;  // [8 cap]
    int *ctatotal; // [2 gridDim.x]
    int *leaves;   // [cap]
    int *m2m_list; // [cap]: internal boxes with sources, BFS order (the evaluate's M2M columns)
    TreeHeader *hdr;
};

constexpr int TL_THREADS = 256;

// exclusive prefix of ctatotal at this CTA and the grid total (every thread gets both)
__device__ __forceinline__ void cta_offsets(const int *ctatotal, int &before, int &total, int *s_red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int b = 0, t = 0;
    for (int c = tid; c < (int)gridDim.x; c += TL_THREADS) {
        const int v = __ldcg(ctatotal + c);
        t += v;
        if (c < (int)blockIdx.x) b += v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        b += __shfl_xor_sync(0xffffffffu, b, o);
        t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    if (lane == 0) s_red[warp] = b, s_red[8 + warp] = t;
    __syncthreads();
    before = total = 0;
#pragma unroll
    for (int w = 0; w < TL_THREADS / 32; w++) before += s_red[w], total += s_red[8 + w];
}

// block-wide exclusive scan of one value per thread; returns the exclusive prefix, sum in `total`
__device__ __forceinline__ int block_excl_scan(int v, int &total, int *s_red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
    }
    __syncthreads();
    if (lane == 31) s_red[warp] = inc;
    __syncthreads();
    int wbase = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < TL_THREADS / 32; w++) {
        if (w < warp) wbase += s_red[w];
        total += s_red[w];
    }
    return wbase + inc - v;
}

__global__ void __launch_bounds__(TL_THREADS) tree_loop_kernel(TreeLoopArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int s_red[16];
    __shared__ int s_total;
    const int tid = threadIdx.x, G = gridDim.x, c = blockIdx.x;
    int base = 0, nl = 1, level = 0;
    bool overflow = false;
    // the root box (level 0: every point, no parent, no children yet); its ranges come from
    // the arguments at level 0, so no barrier is needed before the first split
    if (c == 0 && tid < 8) a.child[tid] = -1;
    if (c == 0 && tid == 0) {
        a.prefix[0] = 0ull;
        a.cell[0] = make_int4(0, 0, 0, 0);
        a.parent[0] = -1;
        a.isleaf[0] = 1;
        a.srng[0] = make_int2(0, a.ns);
        a.trng[0] = make_int2(0, a.nt);
    }
    for (;; level++) {
        if (c == 0 && tid == 0) a.hdr->level_off[level + 1] = base + nl;
        const int chunk = (nl + G - 1) / G;
        const int i0 = min(nl, c * chunk), i1 = min(nl, i0 + chunk);
        // ---- split: 16 lanes per box. Lane g searches one child boundary (g < 8: sources,
        // digit g; g >= 8: targets, digit g - 8) over the whole box range, so the boundaries
        // come from independent binary searches (one dependent chain of ~log2(n) loads)
        // instead of 14 chained ones: the top levels, one box spanning all points, are
        // latency-bound ----
        if (tid == 0) s_total = 0;
        __syncthreads();
        int mine = 0;
        const bool deep = level >= kMaxDepth;
        const int shift = deep ? 0 : 3 * (kMaxDepth - 1 - level);
        for (int ib = i0; ib < i1; ib += TL_THREADS / 16) {
            const int i = ib + (tid >> 4), g = tid & 15;
            const bool live = i < i1;
            const int2 s = !live ? make_int2(0, 0) : level == 0 ? make_int2(0, a.ns) : __ldcg(a.srng + base + i);
            const int2 t = !live ? make_int2(0, 0) : level == 0 ? make_int2(0, a.nt) : __ldcg(a.trng + base + i);
            const bool split = live && ((s.y - s.x) > a.leaf_cap || (t.y - t.x) > a.leaf_cap);
            int b = 0;
            if (split && !deep && shift < a.min_bit) {
                if (g == 0) atomicExch(&a.hdr->need_bits, 1);
            } else if (split && !deep) {
                const unsigned o = g & 7;
                b = g < 8 ? (o == 0 ? s.x : lower_digit(a.skeys, s.x, s.y, shift, o))
                          : (o == 0 ? t.x : lower_digit(a.tkeys, t.x, t.y, shift, o));
            }
            int sb[9], tb[9];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                sb[k] = __shfl_sync(0xffffffffu, b, (tid & 16) + k);
                tb[k] = __shfl_sync(0xffffffffu, b, (tid & 16) + 8 + k);
            }
            if (!live || g != 0) continue;
            int cnt = 0;
            if (split && deep) {
                atomicExch(&a.hdr->err_deep, 1);
            } else if (split) {
                sb[8] = s.y, tb[8] = t.y;
                for (int o = 0; o < 8; o++) {
                    a.crange[8 * (int64_t)i + o] = make_int4(sb[o], sb[o + 1], tb[o], tb[o + 1]);
                    cnt += (sb[o + 1] > sb[o] || tb[o + 1] > tb[o]) ? 1 : 0;
                }
            }
            a.childcnt[i] = cnt;
            mine += cnt;
        }
        if (mine) atomicAdd(&s_total, mine);
        __syncthreads();
        if (tid == 0) a.ctatotal[c] = s_total;
        grid.sync();
        // ---- emit: children in box order, octant order within a box ----
        int before, nnext;
        cta_offsets(a.ctatotal, before, nnext, s_red);
        if (a.min_bit > 0 && __ldcg(&a.hdr->need_bits)) {
            overflow = true;
            break; // uniform over the grid (written before the barrier)
        }
        if ((long long)base + nl + nnext > a.cap) {
            if (c == 0 && tid == 0) a.hdr->need = (long long)base + nl + nnext;
            overflow = true;
            break; // uniform over the grid
        }
        int run = before;
        for (int ib = i0; ib < i1; ib += TL_THREADS) {
            const int i = ib + tid;
            const bool live = i < i1;
            const int cnt = live ? a.childcnt[i] : 0;
            int tot;
            int j = run + block_excl_scan(cnt, tot, s_red);
            run += tot;
            if (!live) continue;
            const int gi = base + i;
            a.isleaf[gi] = cnt == 0 ? 1 : 0;
            if (cnt == 0) continue;
            const unsigned long long pf = __ldcg(a.prefix + gi);
            const int4 cc = __ldcg(a.cell + gi);
            for (int o = 0; o < 8; o++) {
                const int4 r = a.crange[8 * (int64_t)i + o];
                if (r.y == r.x && r.w == r.z) continue;
                const int gc = base + nl + j;
                a.prefix[gc] = (pf << 3) | (unsigned long long)o;
                a.cell[gc] = make_int4(2 * cc.x + (o & 1), 2 * cc.y + ((o >> 1) & 1), 2 * cc.z + ((o >> 2) & 1), cc.w + 1);
                a.parent[gc] = gi;
                a.srng[gc] = make_int2(r.x, r.y);
                a.trng[gc] = make_int2(r.z, r.w);
                int4 *ch = reinterpret_cast<int4 *>(a.child + 8 * (int64_t)gc);
                ch[0] = ch[1] = make_int4(-1, -1, -1, -1);
                a.child[8 * (int64_t)gi + o] = gc;
                j++;
            }
        }
        base += nl;
        nl = nnext;
        if (nnext == 0) break; // uniform
        grid.sync(); // the new level's ranges are read by every CTA
    }
    if (overflow) return;
    grid.sync(); // isleaf of the last level
    // ---- leaves, BFS order ----
    const int nb = base;
    const int chunk = (nb + G - 1) / G;
    const int i0 = min(nb, c * chunk), i1 = min(nb, i0 + chunk);
    // (the same pass counts what the column layouts of the evaluate need: boxes per level and
    // octant, internal boxes with sources per level)
    __shared__ int s_hist[kMaxLevels * 8 + kMaxLevels + 1];
    for (int k = tid; k < kMaxLevels * 8 + kMaxLevels + 1; k += TL_THREADS) s_hist[k] = 0;
    if (tid == 0) s_total = 0;
    __syncthreads();
    int mine = 0;
    for (int i = i0 + tid; i < i1; i += TL_THREADS) {
        const int leaf = __ldcg(a.isleaf + i);
        mine += leaf ? 1 : 0;
        const int4 cc = __ldcg(a.cell + i);
        atomicAdd(&s_hist[cc.w * 8 + ((cc.x & 1) | ((cc.y & 1) << 1) | ((cc.z & 1) << 2))], 1);
        const int2 sr = __ldcg(a.srng + i);
        if (!leaf && sr.y > sr.x) atomicAdd(&s_hist[kMaxLevels * 8 + cc.w], 1);
    }
    if (mine) atomicAdd(&s_total, mine);
    __syncthreads();
    for (int k = tid; k < kMaxLevels * 8 + kMaxLevels + 1; k += TL_THREADS)
        if (s_hist[k]) atomicAdd(k < kMaxLevels * 8 ? &a.hdr->oct_hist[k] : &a.hdr->m2m_count[k - kMaxLevels * 8], s_hist[k]);
    if (tid == 0) {
        a.ctatotal[c] = s_total;
        int m2m = 0; // this CTA's boxes are a BFS range: its per-level counts add up to its share
        for (int l = 0; l <= kMaxLevels; l++) m2m += s_hist[kMaxLevels * 8 + l];
        a.ctatotal[G + c] = m2m;
    }
    grid.sync();
    int before, nleaves, before2, nm2m;
    cta_offsets(a.ctatotal, before, nleaves, s_red);
    cta_offsets(a.ctatotal + G, before2, nm2m, s_red);
    int run = before, run2 = before2;
    for (int ib = i0; ib < i1; ib += TL_THREADS) {
        const int i = ib + tid;
        const int leaf = i < i1 && __ldcg(a.isleaf + i) ? 1 : 0;
        int f2 = 0;
        if (i < i1 && !leaf) {
            const int2 sr = __ldcg(a.srng + i);
            f2 = sr.y > sr.x ? 1 : 0;
        }
        int tot;
        const int j = run + block_excl_scan(leaf, tot, s_red);
        run += tot;
        if (leaf) a.leaves[j] = i;
        const int j2 = run2 + block_excl_scan(f2, tot, s_red);
        run2 += tot;
        if (f2) a.m2m_list[j2] = i;
    }
    if (c == 0 && tid == 0) {
        a.hdr->depth = level;
        a.hdr->nboxes = nb;
        a.hdr->nleaves = nleaves;
    }
}

std::string fmt_g(double v) {
    std::ostringstream os;
    os << v;
    return os.str();
}

void outside_message(const double *d_src, int64_t ns, const double *d_trg, int64_t nt, int bad_total) {
    // src/fmm.cpp:305-323: first 8 offenders, sources before targets
    std::string offenders;
    int bad = 0;
    auto scan = [&](const double *d, int64_t n, const char *what) {
        std::vector<double> h(3 * n);
        if (n) PK_CUDA(cudaMemcpy(h.data(), d, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n && bad < 8; i++) {
            const double x = h[3 * i], y = h[3 * i + 1], z = h[3 * i + 2];
            if (x < 0 || x >= 1 || y < 0 || y >= 1 || z < 0 || z >= 1) {
                offenders += " " + std::string(what) + "[" + std::to_string(i) + "]=(" + fmt_g(x) + "," + fmt_g(y) +
                             "," + fmt_g(z) + ")";
                bad++;
            }
        }
    };
    scan(d_src, ns, "source");
    scan(d_trg, nt, "target");
    throw InvalidArgument("FmmTree: " + std::to_string(bad_total) + " points outside [0,1)^3:" + offenders);
}

} // namespace

TreeView DeviceTree::view() const {
    TreeView v{};
    for (int l = 0; l <= kMaxLevels; l++)
        v.level_off[l] = l < (int)level_off.size() ? level_off[l] : (level_off.empty() ? 0 : level_off.back());
    v.depth = depth;
    v.nboxes = (int)nboxes;
    v.prefix = prefix;
    v.cell = cell;
    v.parent = parent;
    v.child = child;
    v.isleaf = isleaf;
    v.srng = srng;
    v.trng = trng;
    return v;
}

void build_tree(DeviceTree &T, const double *d_src, int64_t ns, const double *d_trg, int64_t nt, int leaf_capacity,
                cudaStream_t st, int64_t *launches) {
    if (leaf_capacity < 1) throw InvalidArgument("FmmTree: leaf capacity must be positive");
    if (ns >= (int64_t(1) << 31) - 1 || nt >= (int64_t(1) << 31) - 1)
        throw InvalidArgument("FmmTree: point count exceeds 2^31-1");
    T.ns = ns;
    T.nt = nt;
    T.leaf_capacity = leaf_capacity;
    Workspace &ws = T.ws;
    const int64_t nmax = std::max<int64_t>(std::max(ns, nt), 1);
    unsigned long long *k_in = ws.get<unsigned long long>("k_in", nmax);
    int *i_in = ws.get<int>("i_in", nmax);
    unsigned long long *skeys = ws.get<unsigned long long>("skeys", std::max<int64_t>(ns, 1));
    unsigned long long *tkeys = ws.get<unsigned long long>("tkeys", std::max<int64_t>(nt, 1));
    T.src_perm = ws.get<int>("src_perm", std::max<int64_t>(ns, 1));
    T.trg_perm = ws.get<int>("trg_perm", std::max<int64_t>(nt, 1));
    // the level loop's header and the outside-domain counter share one buffer (one memset)
    static_assert(sizeof(TreeHeader) % sizeof(int) == 0, "flags follow the header");
    TreeHeader *d_hdr = reinterpret_cast<TreeHeader *>(ws.get<char>("tree_header", sizeof(TreeHeader) + 4 * sizeof(int)));
    int *flags = reinterpret_cast<int *>(d_hdr + 1);
    if (!T.h_flags) PK_CUDA(cudaMallocHost(&T.h_flags, 4 * sizeof(int)));
    int *h_flags = T.h_flags;

    // keys + sort, sources then targets (the "bad" counter accumulates both). The sort covers
    // the key bits of the first 8 levels only (three 8-bit passes instead of five) unless a
    // tree of this context has needed more: a box that must split at level >= 8 makes the
    // level loop ask for the full sort (need_bits), once, and the context remembers.
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, k_in, skeys, i_in, T.src_perm, (int)nmax, 0, 36, st);
    void *temp = ws.get<char>("sort_temp", temp_bytes);
    // targets that are the sources (same buffer) sort once; the keys and order are copied
    const bool same = d_trg == d_src && nt == ns;
    T.src_pos = ws.get<double4>("src_pos", std::max<int64_t>(ns, 1));
    T.src_f = ws.get<double4>("src_f", std::max<int64_t>(ns, 1));
    // (readers of trg_pos use x, y, z only: the sources' w, the Laplace charge, does not matter)
    T.trg_pos = same ? T.src_pos : ws.get<double4>("trg_pos", std::max<int64_t>(nt, 1));
    if (same) {
        tkeys = skeys;
        T.trg_perm = T.src_perm;
    }
    auto sort_points = [&](int min_bit) {
        PK_CUDA(cudaMemsetAsync(d_hdr, 0, sizeof(TreeHeader) + 4 * sizeof(int), st));
        for (int pass = 0; pass < 2; pass++) {
            const int64_t n = pass == 0 ? ns : nt;
            if (n == 0) continue;
            if (pass == 1 && same) continue; // the targets alias the sources' keys, order and positions
            keys_kernel<<<blocks_for(n, 256), 256, 0, st>>>(pass == 0 ? d_src : d_trg, n, k_in, i_in, flags);
            size_t tb = temp_bytes;
            PK_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, k_in, pass == 0 ? skeys : tkeys, i_in,
                                                    pass == 0 ? T.src_perm : T.trg_perm, (int)n, min_bit, 36, st));
            *launches += 1 + 4;
        }
        // sorted point coordinates (need only the sort: queued before the level loop's read-back)
        if (ns) gather_pos_kernel<<<blocks_for(ns, 256), 256, 0, st>>>(d_src, T.src_perm, ns, T.src_pos);
        if (nt && !same) gather_pos_kernel<<<blocks_for(nt, 256), 256, 0, st>>>(d_trg, T.trg_perm, nt, T.trg_pos);
        *launches += same ? 1 : 2;
    };
    constexpr int kPartialSortBit = 3 * (kMaxDepth - 8); // levels 0..7 split on bits >= this
    int min_bit = T.full_sort ? 0 : kPartialSortBit;
    sort_points(min_bit);

    // level loop and leaf compaction: one cooperative kernel, one host round trip (the header,
    // with the outside-domain count). The box arrays keep their capacity between calls; the
    // first guess is four boxes per full leaf, and a tree that does not fit is rebuilt after
    // growing to what the overflowing level asked for.
    static_assert(sizeof(TreeHeader) % sizeof(int) == 0, "header is copied as ints");
    if (!T.h_header) PK_CUDA(cudaMallocHost(&T.h_header, sizeof(TreeHeader) + 4 * sizeof(int)));
    TreeHeader *hh = static_cast<TreeHeader *>(T.h_header);
    int dev = 0, nsm = 0, per_sm = 0;
    PK_CUDA(cudaGetDevice(&dev));
    PK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    PK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tree_loop_kernel, TL_THREADS, 0));
    if (per_sm < 1) throw RuntimeError("FmmTree: the level-loop kernel does not fit an SM");
    // CTAs per SM: the barriers cost more with more CTAs and a small tree is bound by them; a
    // large one by the latency of its boundary searches, which more resident warps hide
    const int64_t npts = ns + nt;
    const int grid = nsm * std::min(per_sm, npts > 4000000 ? 4 : npts > 400000 ? 2 : 1);
    size_t cap = std::max<size_t>(T.box_capacity,
                                  std::max<size_t>(1024, 4 * (size_t)((ns + nt) / leaf_capacity) + 64));
    if (tuning().tree_cap > 0) cap = std::max<size_t>(T.box_capacity, (size_t)tuning().tree_cap);
    for (bool first = true;; first = false) {
        T.prefix = ws.get<unsigned long long>("prefix", cap);
        T.cell = ws.get<int4>("cell", cap);
        T.parent = ws.get<int>("parent", cap);
        T.child = ws.get<int>("child", 8 * cap);
        T.isleaf = ws.get<int>("isleaf", cap);
        T.srng = ws.get<int2>("srng", cap);
        T.trng = ws.get<int2>("trng", cap);
        T.leaves = ws.get<int>("leaves", cap);
        T.m2m_list = ws.get<int>("m2m_list", cap);
        T.box_capacity = cap;
        TreeLoopArgs a;
        a.cap = (int)std::min<size_t>(cap, (size_t)INT32_MAX);
        a.leaf_cap = leaf_capacity;
        a.min_bit = min_bit;
        a.skeys = skeys;
        a.tkeys = tkeys;
        a.prefix = T.prefix;
        a.cell = T.cell;
        a.parent = T.parent;
        a.child = T.child;
        a.isleaf = T.isleaf;
        a.srng = T.srng;
        a.trng = T.trng;
        a.childcnt = ws.get<int>("childcnt", cap);
        a.crange = ws.get<int4>("crange", 8 * cap);
        a.ctatotal = ws.get<int>("ctatotal", 2 * grid);
        a.leaves = T.leaves;
        a.m2m_list = T.m2m_list;
        a.hdr = d_hdr;
        a.ns = (int)ns;
        a.nt = (int)nt;
        if (!first) PK_CUDA(cudaMemsetAsync(d_hdr, 0, sizeof(TreeHeader), st)); // (first: zeroed with the sort)
        void *kargs[] = {&a};
        PK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(tree_loop_kernel), dim3(grid), dim3(TL_THREADS), kargs,
                                            0, st));
        *launches += 1;
        PK_CUDA(cudaMemcpyAsync(hh, d_hdr, sizeof(TreeHeader) + 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        if (first) {
            h_flags[0] = reinterpret_cast<const int *>(hh + 1)[0]; // points outside the domain
            if (same) h_flags[0] *= 2; // the reference counts the targets' offenders as well
            if (h_flags[0] > 0) outside_message(d_src, ns, d_trg, nt, h_flags[0]);
        }
        if (hh->need_bits) {
            T.full_sort = true;
            min_bit = 0;
            sort_points(0);
            continue;
        }
        if (hh->need == 0) break;
        if (hh->need > (long long)INT32_MAX) throw RuntimeError("FmmTree: more than 2^31-1 boxes");
        cap = std::max<size_t>((size_t)hh->need + (size_t)hh->need / 2, 2 * cap);
        cap = std::min<size_t>(cap, (size_t)INT32_MAX);
    }
    if (hh->err_deep)
        throw RuntimeError("FmmTree: leaf over capacity at maximum depth " + std::to_string(kMaxDepth) +
                           " (duplicate point pathology)");
    T.depth = hh->depth;
    T.nboxes = hh->nboxes;
    T.nleaves = hh->nleaves;
    T.level_off.assign(hh->level_off, hh->level_off + T.depth + 2);
    T.oct_hist.assign(hh->oct_hist, hh->oct_hist + kMaxLevels * 8);
    T.m2m_count.assign(hh->m2m_count, hh->m2m_count + kMaxLevels + 1);
}

void gather_strengths(DeviceTree &T, const double *d_str, int ks, cudaStream_t st, int64_t *launches) {
    if (T.ns == 0) return;
    gather_str_kernel<<<blocks_for(T.ns, 256), 256, 0, st>>>(d_str, T.src_perm, T.ns, ks, T.src_pos, T.src_f);
    *launches += 1;
}

void export_tree(const DeviceTree &T, std::vector<int32_t> &table, std::vector<int32_t> &srcidx,
                 std::vector<int32_t> &trgidx, uint64_t &hash) {
    const int64_t nb = T.nboxes;
    std::vector<int4> cell(nb);
    std::vector<int> parent(nb), child(8 * nb), isleaf(nb);
    std::vector<int2> srng(nb), trng(nb);
    std::vector<int> sp(T.ns), tp(T.nt);
    PK_CUDA(cudaMemcpy(cell.data(), T.cell, nb * sizeof(int4), cudaMemcpyDeviceToHost));
    PK_CUDA(cudaMemcpy(parent.data(), T.parent, nb * sizeof(int), cudaMemcpyDeviceToHost));
    PK_CUDA(cudaMemcpy(child.data(), T.child, 8 * nb * sizeof(int), cudaMemcpyDeviceToHost));
    PK_CUDA(cudaMemcpy(isleaf.data(), T.isleaf, nb * sizeof(int), cudaMemcpyDeviceToHost));
    PK_CUDA(cudaMemcpy(srng.data(), T.srng, nb * sizeof(int2), cudaMemcpyDeviceToHost));
    PK_CUDA(cudaMemcpy(trng.data(), T.trng, nb * sizeof(int2), cudaMemcpyDeviceToHost));
    if (T.ns) PK_CUDA(cudaMemcpy(sp.data(), T.src_perm, T.ns * sizeof(int), cudaMemcpyDeviceToHost));
    if (T.nt) PK_CUDA(cudaMemcpy(tp.data(), T.trg_perm, T.nt * sizeof(int), cudaMemcpyDeviceToHost));
    table.assign(18 * nb, 0);
    srcidx.clear();
    trgidx.clear();
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t v) {
        h ^= v;
        h *= 1099511628211ull;
    };
    std::vector<int> seg;
    for (int64_t b = 0; b < nb; b++) {
        const bool leaf = isleaf[b] != 0;
        int32_t *t = &table[18 * b];
        t[0] = cell[b].w;
        t[1] = cell[b].x;
        t[2] = cell[b].y;
        t[3] = cell[b].z;
        t[4] = parent[b];
        t[5] = leaf ? 1 : 0;
        t[6] = leaf ? srng[b].y - srng[b].x : 0;
        t[7] = leaf ? trng[b].y - trng[b].x : 0;
        t[8] = srng[b].y - srng[b].x;
        t[9] = trng[b].y - trng[b].x;
        for (int o = 0; o < 8; o++) t[10 + o] = child[8 * b + o];
        mix((uint64_t)(int64_t)t[0]);
        mix((uint64_t)(int64_t)t[1]);
        mix((uint64_t)(int64_t)t[2]);
        mix((uint64_t)(int64_t)t[3]);
        mix(leaf ? 1 : 0);
        if (!leaf) continue;
        // leaf lists hold increasing original indices (stable partition in split())
        seg.assign(sp.begin() + srng[b].x, sp.begin() + srng[b].y);
        std::sort(seg.begin(), seg.end());
        for (int i : seg) mix(static_cast<uint64_t>(i) + 0x9e3779b97f4a7c15ull);
        srcidx.insert(srcidx.end(), seg.begin(), seg.end());
        seg.assign(tp.begin() + trng[b].x, tp.begin() + trng[b].y);
        std::sort(seg.begin(), seg.end());
        for (int i : seg) mix(static_cast<uint64_t>(i) + 0x517cc1b727220a95ull);
        trgidx.insert(trgidx.end(), seg.begin(), seg.end());
    }
    hash = h;
}

} // namespace pkgpu
