// Interaction lists with periodic image shifts (FmmTree::build_lists / traverse,
// src/fmm.cpp:422-503), built per box in parallel from the closed forms of the dual
// traversal (SURVEY.md §8a "List semantics"), for the shift set {0} ∪ image_offsets(1,1):
//   U(b) leaf b : leaves c adjacent to b (any level, incl. b itself at shift 0)
//   V(b)        : same-level c, parent(c) adjacent to parent(b), c not adjacent to b
//   W(b) leaf b : c finer than b, parent(c) adjacent to b, c not adjacent to b
//   X(b)        : leaves c coarser than b, adjacent to parent(b), not adjacent to b
// Every adjacent box at a coarser-or-equal level is found through the 27 neighbour
// cells (with periodic wrap -> shift), finer ones by descending adjacent internal
// same-level neighbours. Lookups are binary searches in the per-level Morton-sorted
// prefix arrays.
#include <cub/cub.cuh>

#include "tree.h"
#include "tuning.h"

namespace pkgpu {

namespace {

__device__ __forceinline__ unsigned long long morton_cell(int cx, int cy, int cz, int level) {
    unsigned long long r = 0;
    for (int b = 0; b < level; b++)
        r |= ((unsigned long long)((cx >> b) & 1) << (3 * b)) | ((unsigned long long)((cy >> b) & 1) << (3 * b + 1)) |
             ((unsigned long long)((cz >> b) & 1) << (3 * b + 2));
    return r;
}

__device__ int find_box(const TreeView &T, int l, int cx, int cy, int cz) {
    if (l > T.depth) return -1;
    int64_t lo = T.level_off[l], hi = T.level_off[l + 1];
    const unsigned long long key = morton_cell(cx, cy, cz, l);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const unsigned long long v = T.prefix[mid];
        if (v < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < T.level_off[l + 1] && T.prefix[lo] == key) ? (int)lo : -1;
}

// deepest existing box at level <= l containing cell (cx,cy,cz) of level l
__device__ int deepest_box(const TreeView &T, int l, int cx, int cy, int cz) {
    for (int k = min(l, T.depth); k >= 0; k--) {
        const int sh = l - k;
        const int b = find_box(T, k, cx >> sh, cy >> sh, cz >> sh);
        if (b >= 0) return b;
    }
    return 0;
}

// boxes_adjacent (src/fmm.cpp:422-433): closed boxes touch or overlap under the shift
__device__ __forceinline__ bool adjacent(int4 b, int4 c, int sx, int sy, int sz) {
    const int lf = max(b.w, c.w);
    const int bc[3] = {b.x, b.y, b.z}, cc[3] = {c.x, c.y, c.z}, s[3] = {sx, sy, sz};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const long long lob = (long long)bc[a] << (lf - b.w);
        const long long hib = (((long long)bc[a] + 1) << (lf - b.w)) - 1;
        const long long sc = (long long)cc[a] + ((long long)s[a] << c.w);
        const long long loc = sc << (lf - c.w);
        const long long hic = ((sc + 1) << (lf - c.w)) - 1;
        if (loc > hib + 1 || lob > hic + 1) return false;
    }
    return true;
}

__device__ __forceinline__ bool wrap1(int n, int size, int per, int &w, int &s) {
    if (n < 0) {
        if (!per) return false;
        w = n + size;
        s = -1;
    } else if (n >= size) {
        if (!per) return false;
        w = n - size;
        s = 1;
    } else {
        w = n;
        s = 0;
    }
    return true;
}

struct Params {
    int per[3];
    int eval_mode; // 1: skip boxes without targets and sources without sources (src/fmm.cpp:565-625)
    const int *mask; // optional: boxes with mask[b] == 0 get empty lists
};

__device__ __forceinline__ bool has_src(const TreeView &T, int c) { return T.srng[c].y > T.srng[c].x; }

// Enumerates all four lists of box b into the sink.
template <class Sink> __device__ void enumerate_box(const TreeView &T, const Params &P, int b, Sink &sink) {
    const int4 bc = T.cell[b];
    const int l = bc.w;
    const bool eval = P.eval_mode != 0;
    if (eval && T.trng[b].y == T.trng[b].x) return; // trg_subtree == 0
    if (P.mask && !P.mask[b]) return;
    const bool leaf = T.isleaf[b] != 0;
    // ---------------- U and W (leaf targets) ----------------
    if (leaf) {
        int seen_box[27], seen_code[27], nseen = 0;
        const int size = 1 << l;
        for (int dz = -1; dz <= 1; dz++)
            for (int dy = -1; dy <= 1; dy++)
                for (int dx = -1; dx <= 1; dx++) {
                    int wx, wy, wz, sx, sy, sz;
                    if (!wrap1(bc.x + dx, size, P.per[0], wx, sx) || !wrap1(bc.y + dy, size, P.per[1], wy, sy) ||
                        !wrap1(bc.z + dz, size, P.per[2], wz, sz))
                        continue;
                    const int scode = shift_code(sx, sy, sz);
                    const int k = deepest_box(T, l, wx, wy, wz);
                    const int4 kc = T.cell[k];
                    if (kc.w < l) { // coarser: a leaf there is adjacent; deduplicate over delta
                        if (!T.isleaf[k]) continue;
                        bool dup = false;
                        for (int q = 0; q < nseen; q++) dup |= (seen_box[q] == k && seen_code[q] == scode);
                        if (dup) continue;
                        seen_box[nseen] = k;
                        seen_code[nseen] = scode;
                        nseen++;
                        if (!eval || has_src(T, k)) sink.u(k, scode);
                        continue;
                    }
                    if (T.isleaf[k]) {
                        if (!eval || has_src(T, k)) sink.u(k, scode);
                        continue;
                    }
                    // same-level internal neighbour: descend the source side
                    int stack[12 * 8 + 8];
                    int top = 0;
                    stack[top++] = k;
                    while (top > 0) {
                        const int x = stack[--top];
                        for (int o = 0; o < 8; o++) {
                            const int cc = T.child[8 * x + o];
                            if (cc < 0) continue;
                            const int4 ccell = T.cell[cc];
                            if (adjacent(bc, ccell, sx, sy, sz)) {
                                if (T.isleaf[cc]) {
                                    if (!eval || has_src(T, cc)) sink.u(cc, scode);
                                } else {
                                    stack[top++] = cc;
                                }
                            } else {
                                if (!eval || has_src(T, cc)) sink.w(cc, scode);
                            }
                        }
                    }
                }
    }
    if (l == 0) return;
    // ---------------- V and X (through the parent's neighbourhood) ----------------
    const int pb = T.parent[b];
    const int4 pc = T.cell[pb];
    const int psize = 1 << (l - 1);
    int seen_box[27], seen_code[27], nseen = 0;
    for (int dz = -1; dz <= 1; dz++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
                int wx, wy, wz, sx, sy, sz;
                if (!wrap1(pc.x + dx, psize, P.per[0], wx, sx) || !wrap1(pc.y + dy, psize, P.per[1], wy, sy) ||
                    !wrap1(pc.z + dz, psize, P.per[2], wz, sz))
                    continue;
                const int scode = shift_code(sx, sy, sz);
                const int k = deepest_box(T, l - 1, wx, wy, wz);
                const int4 kc = T.cell[k];
                if (!T.isleaf[k]) {
                    if (kc.w != l - 1) continue; // region holds no points
                    // V: children of an adjacent same-level internal box, not adjacent to b
                    for (int o = 0; o < 8; o++) {
                        const int cc = T.child[8 * k + o];
                        if (cc < 0) continue;
                        const int4 ccell = T.cell[cc];
                        if (adjacent(bc, ccell, sx, sy, sz)) continue;
                        if (eval && !has_src(T, cc)) continue;
                        const int ddx = ccell.x + (sx << l) - bc.x, ddy = ccell.y + (sy << l) - bc.y,
                                  ddz = ccell.z + (sz << l) - bc.z;
                        sink.v(cc, offset_code(ddx, ddy, ddz));
                    }
                } else {
                    // X: coarser-or-equal leaf adjacent to the parent, not adjacent to b
                    bool dup = false;
                    for (int q = 0; q < nseen; q++) dup |= (seen_box[q] == k && seen_code[q] == scode);
                    if (dup) continue;
                    seen_box[nseen] = k;
                    seen_code[nseen] = scode;
                    nseen++;
                    if (adjacent(bc, kc, sx, sy, sz)) continue;
                    if (eval && !has_src(T, k)) continue;
                    sink.x(k, scode);
                }
            }
}

// ---------------------------------------------------------------------------
// Warp-per-box enumeration (evaluate path): lane d < 27 handles neighbour direction d of the
// serial enumerate_box, so the ~27 dependent deepest_box searches run concurrently instead
// of one after another. Entries keep the serial order (direction-major, the descent order
// within a direction): each lane counts its entries, an exclusive warp scan gives its
// offset, and the lane emits again at that offset. Coarse-leaf deduplication compares
// against the lower directions through shuffles.
struct LaneCount {
    int nu = 0, nv = 0, nw = 0, nx = 0;
    __device__ void u(int, int) { nu++; }
    __device__ void v(int, int) { nv++; }
    __device__ void w(int, int) { nw++; }
    __device__ void x(int, int) { nx++; }
};

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x - v;
}
__device__ __forceinline__ int warp_sum(int v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// direction d's U/W entries of leaf b (lanes >= 27 or invalid directions emit nothing)
template <class Sink>
__device__ void lane_uw(const TreeView &T, const Params &P, int b, int4 bc, int d, bool dup, int k, int scode,
                        bool valid, Sink &sink) {
    if (!valid) return;
    const bool eval = P.eval_mode != 0;
    const int l = bc.w;
    const int4 kc = T.cell[k];
    if (kc.w < l) {
        if (!T.isleaf[k] || dup) return;
        if (!eval || has_src(T, k)) sink.u(k, scode);
        return;
    }
    if (T.isleaf[k]) {
        if (!eval || has_src(T, k)) sink.u(k, scode);
        return;
    }
    int sx, sy, sz;
    shift_decode(scode, sx, sy, sz);
    int stack[12 * 8 + 8];
    int top = 0;
    stack[top++] = k;
    while (top > 0) {
        const int x = stack[--top];
        for (int o = 0; o < 8; o++) {
            const int cc = T.child[8 * x + o];
            if (cc < 0) continue;
            const int4 ccell = T.cell[cc];
            if (adjacent(bc, ccell, sx, sy, sz)) {
                if (T.isleaf[cc]) {
                    if (!eval || has_src(T, cc)) sink.u(cc, scode);
                } else {
                    stack[top++] = cc;
                }
            } else {
                if (!eval || has_src(T, cc)) sink.w(cc, scode);
            }
        }
    }
    (void)b;
    (void)d;
}

// direction d's V/X entries of box b
template <class Sink>
__device__ void lane_vx(const TreeView &T, const Params &P, int4 bc, bool dup, int k, int scode, bool valid,
                        Sink &sink) {
    if (!valid) return;
    const bool eval = P.eval_mode != 0;
    const int l = bc.w;
    const int4 kc = T.cell[k];
    int sx, sy, sz;
    shift_decode(scode, sx, sy, sz);
    if (!T.isleaf[k]) {
        if (kc.w != l - 1) return;
        for (int o = 0; o < 8; o++) {
            const int cc = T.child[8 * k + o];
            if (cc < 0) continue;
            const int4 ccell = T.cell[cc];
            if (adjacent(bc, ccell, sx, sy, sz)) continue;
            if (eval && !has_src(T, cc)) continue;
            sink.v(cc, offset_code(ccell.x + (sx << l) - bc.x, ccell.y + (sy << l) - bc.y, ccell.z + (sz << l) - bc.z));
        }
    } else {
        if (dup || adjacent(bc, kc, sx, sy, sz)) return;
        if (eval && !has_src(T, k)) return;
        sink.x(k, scode);
    }
}

// neighbour cell of direction d (27 directions, dz-major as the serial loop) around cell c
// of level lev: wrapped cell, its shift code and the deepest box holding it
__device__ __forceinline__ bool lane_neighbour(const TreeView &T, const Params &P, int4 c, int lev, int d, int &k,
                                               int &scode) {
    if (d >= 27) return false;
    const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
    const int size = 1 << lev;
    int wx, wy, wz, sx, sy, sz;
    if (!wrap1(c.x + dx, size, P.per[0], wx, sx) || !wrap1(c.y + dy, size, P.per[1], wy, sy) ||
        !wrap1(c.z + dz, size, P.per[2], wz, sz))
        return false;
    scode = shift_code(sx, sy, sz);
    k = deepest_box(T, lev, wx, wy, wz);
    return true;
}

// duplicate coarse candidate: a lower direction already produced the same (box, shift)
__device__ __forceinline__ bool lane_dup(bool coarse, int k, int scode, int lane) {
    bool dup = false;
    for (int q = 0; q < 27; q++) {
        const int qk = __shfl_sync(0xffffffffu, k, q), qs = __shfl_sync(0xffffffffu, scode, q);
        const int qc = __shfl_sync(0xffffffffu, coarse ? 1 : 0, q);
        dup |= q < lane && qc && qk == k && qs == scode;
    }
    return coarse && dup;
}

struct LaneFill {
    int2 *eu, *ew, *ex;
    int *table;
    int64_t ld;
    int col;
    const int *slot_of_code;
    __device__ void u(int c, int code) { *eu++ = make_int2(c, code); }
    __device__ void v(int c, int code) { table[(int64_t)slot_of_code[code] * ld + col] = c; }
    __device__ void w(int c, int code) { *ew++ = make_int2(c, code); }
    __device__ void x(int c, int code) { *ex++ = make_int2(c, code); }
};

// fill == false: per-box counts; true: entries at the box's offsets (M2L table for V)
template <bool FILL>
__global__ void eval_warp_kernel(TreeView T, Params P, int64_t *cu, int64_t *cv, int64_t *cw, int64_t *cx,
                                 const int64_t *ou, const int64_t *ow, const int64_t *ox, int2 *eu, int2 *ew, int2 *ex,
                                 int *table, int64_t ld, const int *col_of_box, const int *slot_of_code) {
    const int b = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (b >= T.nboxes) return; // whole warps exit together
    const int4 bc = T.cell[b];
    const int l = bc.w;
    bool skip = P.eval_mode != 0 && T.trng[b].y == T.trng[b].x;
    if (P.mask && !P.mask[b]) skip = true;
    LaneCount c;
    int2 *pu = nullptr, *pw = nullptr, *px = nullptr;
    if (FILL && !skip) pu = eu + ou[b], pw = ew + ow[b], px = ex + ox[b];
    // ---- U / W ----
    if (!skip && T.isleaf[b]) {
        int k = 0, scode = 0;
        const bool valid = lane_neighbour(T, P, bc, l, lane, k, scode);
        const bool coarse = valid && T.cell[k].w < l;
        const bool dup = lane_dup(coarse, k, scode, lane);
        LaneCount n;
        lane_uw(T, P, b, bc, lane, dup, k, scode, valid, n);
        if (FILL) {
            const int offu = warp_excl_scan(n.nu, lane), offw = warp_excl_scan(n.nw, lane);
            LaneFill f{pu + offu, pw + offw, nullptr, nullptr, 0, 0, nullptr};
            lane_uw(T, P, b, bc, lane, dup, k, scode, valid, f);
        }
        c.nu = n.nu, c.nw = n.nw;
    }
    // ---- V / X ----
    if (!skip && l > 0) {
        const int pb = T.parent[b];
        const int4 pc = T.cell[pb];
        int k = 0, scode = 0;
        const bool valid = lane_neighbour(T, P, pc, l - 1, lane, k, scode);
        const bool leafk = valid && T.isleaf[k];
        const bool dup = lane_dup(leafk, k, scode, lane);
        LaneCount n;
        lane_vx(T, P, bc, dup, k, scode, valid, n);
        if (FILL) {
            const int offx = warp_excl_scan(n.nx, lane);
            LaneFill f{nullptr, nullptr, px + offx, table, ld, col_of_box[b], slot_of_code};
            lane_vx(T, P, bc, dup, k, scode, valid, f);
        }
        c.nv = n.nv, c.nx = n.nx;
    }
    if (!FILL) {
        const int nu = warp_sum(c.nu), nv = warp_sum(c.nv), nw = warp_sum(c.nw), nx = warp_sum(c.nx);
        if (lane == 0) cu[b] = nu, cv[b] = nv, cw[b] = nw, cx[b] = nx;
    }
}

struct CountSink {
    int nu = 0, nv = 0, nw = 0, nx = 0;
    __device__ void u(int, int) { nu++; }
    __device__ void v(int, int) { nv++; }
    __device__ void w(int, int) { nw++; }
    __device__ void x(int, int) { nx++; }
};

struct FillSink {
    int2 *eu, *ev, *ew, *ex; // already offset to this box
    int nu = 0, nv = 0, nw = 0, nx = 0;
    __device__ void u(int c, int code) { eu[nu++] = make_int2(c, code); }
    __device__ void v(int c, int code) { ev[nv++] = make_int2(c, code); }
    __device__ void w(int c, int code) { ew[nw++] = make_int2(c, code); }
    __device__ void x(int c, int code) { ex[nx++] = make_int2(c, code); }
};

struct EvalFillSink {
    int2 *eu, *ew, *ex;
    int *table;
    int64_t ld;
    int col;
    const int *slot_of_code;
    int nu = 0, nw = 0, nx = 0;
    __device__ void u(int c, int code) { eu[nu++] = make_int2(c, code); }
    __device__ void v(int c, int code) { table[(int64_t)slot_of_code[code] * ld + col] = c; }
    __device__ void w(int c, int code) { ew[nw++] = make_int2(c, code); }
    __device__ void x(int c, int code) { ex[nx++] = make_int2(c, code); }
};

// which ranks need a box's equivalent density (partitioned runs): every target box c with
// V or W entries marks its sources with the ranks whose leaf ranges c meets
struct NeedSink {
    unsigned long long *need;
    unsigned long long m;
    bool skip_v;
    __device__ void u(int, int) {}
    __device__ void v(int c, int) {
        if (!skip_v) atomicOr(need + c, m);
    }
    __device__ void w(int c, int) { atomicOr(need + c, m); }
    __device__ void x(int, int) {}
};

__global__ void need_kernel(TreeView T, Params P, const int *__restrict__ rlo, const int *__restrict__ rhi,
                            unsigned long long *need, unsigned skip_v_levels) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    const int lo = rlo[b], hi = rhi[b];
    NeedSink s{need, ((hi >= 63 ? ~0ull : ((1ull << (hi + 1)) - 1ull)) >> lo) << lo,
               ((skip_v_levels >> T.cell[b].w) & 1u) != 0};
    enumerate_box(T, P, b, s);
}

__global__ void count_kernel(TreeView T, Params P, int64_t *cu, int64_t *cv, int64_t *cw, int64_t *cx) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    CountSink s;
    enumerate_box(T, P, b, s);
    cu[b] = s.nu;
    cv[b] = s.nv;
    cw[b] = s.nw;
    cx[b] = s.nx;
}

__global__ void fill_kernel(TreeView T, Params P, const int64_t *ou, const int64_t *ov, const int64_t *ow,
                            const int64_t *ox, int2 *eu, int2 *ev, int2 *ew, int2 *ex) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    FillSink s{eu + ou[b], ev + ov[b], ew + ow[b], ex + ox[b]};
    enumerate_box(T, P, b, s);
}

__global__ void eval_fill_kernel(TreeView T, Params P, const int64_t *ou, const int64_t *ow, const int64_t *ox,
                                 int2 *eu, int2 *ew, int2 *ex, int *table, int64_t ld, const int *col_of_box,
                                 const int *slot_of_code) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T.nboxes) return;
    EvalFillSink s{eu + ou[b], ew + ow[b], ex + ox[b], table, ld, col_of_box[b], slot_of_code};
    enumerate_box(T, P, b, s);
}

void scan_counts(Workspace &ws, int64_t *cnt, int64_t *off, int n, cudaStream_t st, int64_t &total) {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, n + 1, st);
    void *tmp = ws.get<char>("lscan_temp", tb);
    PK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, n + 1, st));
    PK_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
}

Params make_params(const ListSetup &S, int eval) {
    Params P{};
    for (int a = 0; a < 3; a++) P.per[a] = S.periodic[a];
    P.eval_mode = eval;
    P.mask = nullptr;
    return P;
}

} // namespace

void build_lists_csr(const DeviceTree &T, const ListSetup &S, DeviceLists &L, cudaStream_t st, int64_t *launches) {
    const int nb = (int)T.nboxes;
    const TreeView tv = T.view();
    const Params P = make_params(S, 0);
    Workspace &ws = L.ws;
    int64_t *cnt[4], *off[4];
    const char *names[4] = {"u", "v", "w", "x"};
    for (int i = 0; i < 4; i++) {
        cnt[i] = ws.get<int64_t>(std::string("cnt_") + names[i], nb + 1);
        off[i] = ws.get<int64_t>(std::string("off_") + names[i], nb + 1);
        PK_CUDA(cudaMemsetAsync(cnt[i] + nb, 0, sizeof(int64_t), st));
    }
    count_kernel<<<blocks_for(nb, 64), 64, 0, st>>>(tv, P, cnt[0], cnt[1], cnt[2], cnt[3]);
    int64_t tot[4];
    for (int i = 0; i < 4; i++) scan_counts(ws, cnt[i], off[i], nb, st, tot[i]);
    PK_CUDA(cudaStreamSynchronize(st));
    CsrList *lists[4] = {&L.u, &L.v, &L.w, &L.x};
    for (int i = 0; i < 4; i++) {
        lists[i]->off = off[i];
        lists[i]->count = tot[i];
        lists[i]->ent = ws.get<int2>(std::string("ent_") + names[i], tot[i] + 1);
    }
    fill_kernel<<<blocks_for(nb, 64), 64, 0, st>>>(tv, P, off[0], off[1], off[2], off[3], L.u.ent, L.v.ent, L.w.ent,
                                                   L.x.ent);
    PK_CUDA(cudaStreamSynchronize(st));
    *launches += 6;
}

void need_masks(const DeviceTree &T, const ListSetup &S, const int *rlo, const int *rhi, unsigned long long *need,
                cudaStream_t st, unsigned skip_v_levels) {
    const int nb = (int)T.nboxes;
    PK_CUDA(cudaMemsetAsync(need, 0, nb * sizeof(unsigned long long), st));
    need_kernel<<<blocks_for(nb, 64), 64, 0, st>>>(T.view(), make_params(S, 1), rlo, rhi, need, skip_v_levels);
    PK_CUDA(cudaGetLastError());
}

void build_lists_eval(const DeviceTree &T, const ListSetup &S, DeviceLists &L, int *m2l_table, int64_t ld,
                      const int *col_of_box, const int *slot_of_code, cudaStream_t st, int64_t *launches,
                      const int *mask) {
    const int nb = (int)T.nboxes;
    const TreeView tv = T.view();
    Params P = make_params(S, 1);
    P.mask = mask;
    Workspace &ws = L.ws;
    int64_t *cnt[4], *off[4];
    const char *names[4] = {"u", "v", "w", "x"};
    for (int i = 0; i < 4; i++) {
        cnt[i] = ws.get<int64_t>(std::string("cnt_") + names[i], nb + 1);
        off[i] = ws.get<int64_t>(std::string("off_") + names[i], nb + 1);
        PK_CUDA(cudaMemsetAsync(cnt[i] + nb, 0, sizeof(int64_t), st));
    }
    // warp per box where boxes are few (latency-bound single threads); thread per box on big
    // trees, which already fill the GPU (PKGPU_LIST_WARP_MAX boxes, default 50k)
    const int64_t warp_max = tuning().list_warp_max;
    const bool warp_lists = nb <= warp_max;
    if (warp_lists)
        eval_warp_kernel<false><<<blocks_for(32 * (size_t)nb, 128), 128, 0, st>>>(
            tv, P, cnt[0], cnt[1], cnt[2], cnt[3], nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
            nullptr, nullptr);
    else
        count_kernel<<<blocks_for(nb, 64), 64, 0, st>>>(tv, P, cnt[0], cnt[1], cnt[2], cnt[3]);
    int64_t tot[4];
    for (int i = 0; i < 4; i++) scan_counts(ws, cnt[i], off[i], nb, st, tot[i]);
    PK_CUDA(cudaStreamSynchronize(st));
    L.v_total = tot[1];
    L.v.off = off[1]; // per-box V counts as offsets (entries live in the M2L table)
    L.v.count = tot[1];
    L.v.ent = nullptr;
    CsrList *lists[4] = {&L.u, &L.v, &L.w, &L.x};
    for (int i : {0, 2, 3}) {
        lists[i]->off = off[i];
        lists[i]->count = tot[i];
        lists[i]->ent = ws.get<int2>(std::string("ent_") + names[i], tot[i] + 1);
    }
    if (warp_lists)
        eval_warp_kernel<true><<<blocks_for(32 * (size_t)nb, 128), 128, 0, st>>>(
            tv, P, nullptr, nullptr, nullptr, nullptr, off[0], off[2], off[3], L.u.ent, L.w.ent, L.x.ent, m2l_table,
            ld, col_of_box, slot_of_code);
    else
        eval_fill_kernel<<<blocks_for(nb, 64), 64, 0, st>>>(tv, P, off[0], off[2], off[3], L.u.ent, L.w.ent, L.x.ent,
                                                            m2l_table, ld, col_of_box, slot_of_code);
    *launches += 5;
}

} // namespace pkgpu
