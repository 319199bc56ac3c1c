// Device octree build: FmmTree::FmmTree (src/fmm.cpp:301-389) restated as
//   36-bit Morton keys (x = least significant bit of each triple) from floor(x*4096)
//   -> stable radix sort of (key, index) for sources and targets
//   -> level-synchronous splitting: a box splits iff |src| > s or |trg| > s; its
//      children are the non-empty next-octant-digit sub-ranges, emitted in octant
//      order, so boxes come out level-major and Morton-ordered within a level —
//      exactly the reference's BFS numbering.
// x >= box_center  <=>  the (l+1)-th most significant bit of floor(x*4096) is set,
// because box centers (c+1/2)2^-l are exact dyadics (SURVEY.md §8a "Tree semantics").
#include <algorithm>
#include <cub/cub.cuh>
#include <sstream>

#include "tree.h"

namespace pkgpu {

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

// per box of level l: split decision and child ranges. 16 lanes per box: lane g searches
// one child boundary (g < 8: sources, digit g; g >= 8: targets, digit g - 8) over the whole
// box range, so the boundaries come from independent binary searches (one dependent chain
// of ~log2(n) loads) instead of 14 chained ones -- the top levels, where one box spans all
// points, were latency-bound
__global__ void split_kernel(int n, int level, int cap, const int2 *__restrict__ srng, const int2 *__restrict__ trng,
                             const unsigned long long *__restrict__ skeys, const unsigned long long *__restrict__ tkeys,
                             int *__restrict__ childcnt, int4 *__restrict__ crange, int *__restrict__ err) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = gt >> 4, g = gt & 15;
    const bool live = i < n;
    const int2 s = live ? srng[i] : make_int2(0, 0), t = live ? trng[i] : make_int2(0, 0);
    const bool split = live && ((s.y - s.x) > cap || (t.y - t.x) > cap);
    const bool deep = level >= kMaxDepth;
    int b = 0;
    if (split && !deep) {
        const int shift = 3 * (kMaxDepth - 1 - level);
        const unsigned o = g & 7;
        b = g < 8 ? (o == 0 ? s.x : lower_digit(skeys, s.x, s.y, shift, o))
                  : (o == 0 ? t.x : lower_digit(tkeys, t.x, t.y, shift, o));
    }
    // gather the 16 boundaries of the box into its first lane
    int sb[9], tb[9];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        sb[k] = __shfl_sync(0xffffffffu, b, (threadIdx.x & 16) + k);
        tb[k] = __shfl_sync(0xffffffffu, b, (threadIdx.x & 16) + 8 + k);
    }
    if (!live || g != 0) return;
    if (!split) {
        childcnt[i] = 0;
        return;
    }
    if (deep) {
        atomicExch(err, 1);
        childcnt[i] = 0;
        return;
    }
    sb[8] = s.y, tb[8] = t.y;
    int cnt = 0;
    for (int o = 0; o < 8; o++) {
        crange[8 * (int64_t)i + o] = make_int4(sb[o], sb[o + 1], tb[o], tb[o + 1]);
        cnt += (sb[o + 1] > sb[o] || tb[o + 1] > tb[o]) ? 1 : 0;
    }
    childcnt[i] = cnt;
}

__global__ void emit_kernel(int n, int64_t base_l, int64_t base_next, const int *__restrict__ childcnt,
                            const int *__restrict__ childoff, const int4 *__restrict__ crange,
                            unsigned long long *__restrict__ prefix, int4 *__restrict__ cell, int *__restrict__ parent,
                            int *__restrict__ child, int *__restrict__ isleaf, int2 *__restrict__ srng,
                            int2 *__restrict__ trng) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t gi = base_l + i;
    const int cnt = childcnt[i];
    isleaf[gi] = cnt == 0 ? 1 : 0;
    if (cnt == 0) return;
    int j = childoff[i];
    const unsigned long long pf = prefix[gi];
    const int4 c = cell[gi];
    for (int o = 0; o < 8; o++) {
        const int4 r = crange[8 * (int64_t)i + o];
        if (r.y == r.x && r.w == r.z) continue;
        const int64_t gc = base_next + j;
        prefix[gc] = (pf << 3) | (unsigned long long)o;
        cell[gc] = make_int4(2 * c.x + (o & 1), 2 * c.y + ((o >> 1) & 1), 2 * c.z + ((o >> 2) & 1), c.w + 1);
        parent[gc] = (int)gi;
        srng[gc] = make_int2(r.x, r.y);
        trng[gc] = make_int2(r.z, r.w);
        child[8 * gi + o] = (int)gc;
        j++;
    }
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

__global__ void leaf_flags_kernel(int n, const int *__restrict__ isleaf, int *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = isleaf[i];
}

// growable device array inside a Workspace (contents preserved on growth)
template <class T> T *grow(Workspace &ws, const std::string &name, size_t need, size_t used, cudaStream_t st) {
    auto &b = ws.bufs[name];
    if (!b) b = std::make_unique<DevBuf>();
    if (need * sizeof(T) <= b->bytes) return static_cast<T *>(b->ptr);
    const size_t nb = std::max(need * sizeof(T), b->bytes * 2);
    void *p = nullptr;
    PK_CUDA(cudaMalloc(&p, nb));
    if (used && b->ptr) PK_CUDA(cudaMemcpyAsync(p, b->ptr, used * sizeof(T), cudaMemcpyDeviceToDevice, st));
    PK_CUDA(cudaStreamSynchronize(st));
    if (b->ptr) PK_CUDA(cudaFree(b->ptr));
    b->ptr = p;
    b->bytes = nb;
    return static_cast<T *>(p);
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

// the root box (level 0: every point, no parent, no children yet)
__global__ void root_init_kernel(unsigned long long *prefix, int4 *cell, int *parent, int *child, int *isleaf,
                                 int2 *srng, int2 *trng, int ns, int nt) {
    const int t = threadIdx.x;
    if (t < 8) child[t] = -1;
    if (t == 0) {
        prefix[0] = 0ull;
        cell[0] = make_int4(0, 0, 0, 0);
        parent[0] = -1;
        isleaf[0] = 1;
        srng[0] = make_int2(0, ns);
        trng[0] = make_int2(0, nt);
    }
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
    int *flags = ws.get<int>("flags", 4);
    if (!T.h_flags) PK_CUDA(cudaMallocHost(&T.h_flags, 4 * sizeof(int)));
    int *h_flags = T.h_flags;

    PK_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(int), st));
    // keys + sort, sources then targets (the "bad" counter accumulates both)
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, k_in, skeys, i_in, T.src_perm, (int)nmax, 0, 36, st);
    void *temp = ws.get<char>("sort_temp", temp_bytes);
    // targets that are the sources (same buffer) sort once; the keys and order are copied
    const bool same = d_trg == d_src && nt == ns;
    for (int pass = 0; pass < 2; pass++) {
        const int64_t n = pass == 0 ? ns : nt;
        if (n == 0) continue;
        if (pass == 1 && same) {
            PK_CUDA(cudaMemcpyAsync(tkeys, skeys, n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
            PK_CUDA(cudaMemcpyAsync(T.trg_perm, T.src_perm, n * sizeof(int), cudaMemcpyDeviceToDevice, st));
            continue;
        }
        keys_kernel<<<blocks_for(n, 256), 256, 0, st>>>(pass == 0 ? d_src : d_trg, n, k_in, i_in, flags);
        size_t tb = temp_bytes;
        PK_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, k_in, pass == 0 ? skeys : tkeys, i_in,
                                                pass == 0 ? T.src_perm : T.trg_perm, (int)n, 0, 36, st));
        *launches += 1 + 4;
    }
    // (the outside-domain count is read back with the root level's counts below: one host
    // round trip fewer; nothing is allocated from the keys before that)

    // level-synchronous construction
    size_t cap = 1024, used = 0;
    auto arrays = [&](size_t need) {
        T.prefix = grow<unsigned long long>(ws, "prefix", need, used, st);
        T.cell = grow<int4>(ws, "cell", need, used, st);
        T.parent = grow<int>(ws, "parent", need, used, st);
        T.child = grow<int>(ws, "child", 8 * need, 8 * used, st);
        T.isleaf = grow<int>(ws, "isleaf", need, used, st);
        T.srng = grow<int2>(ws, "srng", need, used, st);
        T.trng = grow<int2>(ws, "trng", need, used, st);
    };
    arrays(cap);
    root_init_kernel<<<1, 32, 0, st>>>(T.prefix, T.cell, T.parent, T.child, T.isleaf, T.srng, T.trng, (int)ns, (int)nt);
    *launches += 1;
    T.level_off.assign(1, 0);
    int64_t nl = 1, base = 0;
    used = 1;
    int level = 0;
    for (;; level++) {
        T.level_off.push_back(base + nl);
        int *childcnt = ws.get<int>("childcnt", nl + 1);
        int *childoff = ws.get<int>("childoff", nl + 1);
        int4 *crange = ws.get<int4>("crange", 8 * nl);
        split_kernel<<<blocks_for(16 * nl, 128), 128, 0, st>>>((int)nl, level, leaf_capacity, T.srng + base,
                                                          T.trng + base, skeys, tkeys, childcnt, crange, flags + 1);
        size_t sb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, sb, childcnt, childoff, (int)nl + 1, st);
        void *stemp = ws.get<char>("scan_temp", sb);
        PK_CUDA(cudaMemsetAsync(childcnt + nl, 0, sizeof(int), st));
        PK_CUDA(cub::DeviceScan::ExclusiveSum(stemp, sb, childcnt, childoff, (int)nl + 1, st));
        PK_CUDA(cudaMemcpyAsync(h_flags, childoff + nl, sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaMemcpyAsync(h_flags + 1, flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        if (level == 0) PK_CUDA(cudaMemcpyAsync(h_flags + 2, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CUDA(cudaStreamSynchronize(st));
        *launches += 2;
        if (level == 0) {
            if (same) h_flags[2] *= 2; // the reference counts the targets' offenders as well
            if (h_flags[2] > 0) outside_message(d_src, ns, d_trg, nt, h_flags[2]);
        }
        if (h_flags[1])
            throw RuntimeError("FmmTree: leaf over capacity at maximum depth " + std::to_string(kMaxDepth) +
                               " (duplicate point pathology)");
        const int64_t nnext = h_flags[0];
        if (nnext > 0) {
            arrays(base + nl + nnext);
            PK_CUDA(cudaMemsetAsync(T.child + 8 * (base + nl), 0xff, 8 * nnext * sizeof(int), st));
        }
        emit_kernel<<<blocks_for(nl, 128), 128, 0, st>>>((int)nl, base, base + nl, childcnt, childoff, crange,
                                                         T.prefix, T.cell, T.parent, T.child, T.isleaf, T.srng,
                                                         T.trng);
        *launches += 1;
        used = base + nl + nnext;
        base += nl;
        nl = nnext;
        if (nnext == 0) break;
    }
    T.depth = level;
    T.nboxes = base;
    // leaves (BFS order)
    int *lflags = ws.get<int>("lflags", T.nboxes);
    T.leaves = ws.get<int>("leaves", T.nboxes);
    int *nsel = ws.get<int>("nsel", 1);
    leaf_flags_kernel<<<blocks_for(T.nboxes, 256), 256, 0, st>>>((int)T.nboxes, T.isleaf, lflags);
    size_t fb = 0;
    cub::DeviceSelect::Flagged(nullptr, fb, cub::CountingInputIterator<int>(0), lflags, T.leaves, nsel,
                               (int)T.nboxes, st);
    void *ftemp = ws.get<char>("flag_temp", fb);
    PK_CUDA(cub::DeviceSelect::Flagged(ftemp, fb, cub::CountingInputIterator<int>(0), lflags, T.leaves, nsel,
                                       (int)T.nboxes, st));
    PK_CUDA(cudaMemcpyAsync(h_flags, nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
    // sorted point coordinates
    T.src_pos = ws.get<double4>("src_pos", std::max<int64_t>(ns, 1));
    T.src_f = ws.get<double4>("src_f", std::max<int64_t>(ns, 1));
    T.trg_pos = ws.get<double4>("trg_pos", std::max<int64_t>(nt, 1));
    if (ns) gather_pos_kernel<<<blocks_for(ns, 256), 256, 0, st>>>(d_src, T.src_perm, ns, T.src_pos);
    if (nt) gather_pos_kernel<<<blocks_for(nt, 256), 256, 0, st>>>(d_trg, T.trg_perm, nt, T.trg_pos);
    *launches += 4;
    PK_CUDA(cudaStreamSynchronize(st));
    T.nleaves = h_flags[0];
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
