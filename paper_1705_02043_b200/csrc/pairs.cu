// Pair-sum kernels (FP64 vector pipe). Sources are staged in shared memory in
// batches of segments (one segment = one source leaf / surface with its image shift);
// each target is owned by G consecutive lanes that split the sources and combine with
// warp shuffles, so each output is written once (no atomics, deterministic).
// The shift is applied to the target, r = (t - shift) - s, as in src/kernel.cpp:90-95.
#include <algorithm>

#include "kernels.cuh"
#include "pairs.h"
#include "tuning.h"

namespace pkgpu {

namespace {

constexpr int NT = 128;
#ifndef LEAF_NS
#define LEAF_NS 2
#endif
#ifndef LEAF_MINB
#define LEAF_MINB 5
#endif
constexpr int SB = 512;
constexpr int MAXU = 128;     // U entries per batch: one per thread of the leaf pass (NT)
constexpr int MAXSEG = MAXU;  // segments per stage: every entry of a batch may fall in one stage

template <int KERNEL> struct Stage {
    static constexpr int KS = KERNEL == 0 ? 1 : 3;
    // a staged source is two (Laplace) or three (Stokes) 16-byte words: (x, y), (z, d0), (d1, d2) --
    // one LDS.128 each in the pair loops instead of 4 / 6 LDS.64 with separate index arithmetic
    double2 xy[SB], zd[SB];
    double2 dd[KERNEL == 0 ? 1 : SB];
    __device__ __forceinline__ void put(int q, double x, double y, double z, const double (&d)[KS]) {
        xy[q] = make_double2(x, y);
        zd[q] = make_double2(z, d[0]);
        if (KERNEL != 0) dd[q] = make_double2(d[1], d[2]);
    }
    double sx[MAXSEG], sy[MAXSEG], sz[MAXSEG];
    int begin[MAXSEG + 1];
    int cnt[MAXSEG]; // count coincidences in this segment
    int nseg;
};

template <int KERNEL>
__device__ __forceinline__ void accumulate(const Stage<KERNEL> &S, double tx, double ty, double tz, int j, int G,
                                           double (&acc)[3], int *coincident) {
    constexpr int NS = 4; // sources per step: four interleaved pair chains (kernels.cuh, pair_tile)
    double a1[1][3] = {{acc[0], acc[1], acc[2]}};
    for (int s = 0; s < S.nseg; s++) {
        const double ux[1] = {tx - S.sx[s]}, uy[1] = {ty - S.sy[s]}, uz[1] = {tz - S.sz[s]};
        const int end = S.begin[s + 1];
        int q = S.begin[s] + j;
        for (; q + (NS - 1) * G < end; q += NS * G) {
            double2 a[NS], b[NS], c[NS];
#pragma unroll
            for (int u = 0; u < NS; u++) {
                a[u] = S.xy[q + u * G], b[u] = S.zd[q + u * G];
                c[u] = KERNEL != 0 ? S.dd[q + u * G] : make_double2(0.0, 0.0);
            }
            pair_tile<KERNEL, 1, NS>(ux, uy, uz, a, b, c, a1);
        }
        for (; q < end; q += G) {
            const double2 a[1] = {S.xy[q]}, b[1] = {S.zd[q]};
            const double2 c[1] = {KERNEL != 0 ? S.dd[q] : make_double2(0.0, 0.0)};
            pair_tile<KERNEL, 1, 1>(ux, uy, uz, a, b, c, a1);
        }
        if (S.cnt[s]) { // count coincidences in this segment (direct mode; src/kernel.cpp:97-98)
            int ncoin = 0;
            for (int p = S.begin[s] + j; p < end; p += G) {
                const double rx = ux[0] - S.xy[p].x, ry = uy[0] - S.xy[p].y, rz = uz[0] - S.zd[p].x;
                ncoin += (rx * rx + ry * ry + rz * rz) == 0.0;
            }
            if (ncoin) atomicAdd(coincident, ncoin);
        }
    }
    acc[0] = a1[0][0], acc[1] = a1[0][1], acc[2] = a1[0][2];
}

// one-segment surface stage: points fma(half, t_i, c), density phi[i*ks + a]
template <int KERNEL>
__device__ void stage_surface(Stage<KERNEL> &S, const double *__restrict__ tmpl, int i0, int cnt, double cx, double cy,
                              double cz, double half, const double *__restrict__ phi, double shx, double shy,
                              double shz) {
    constexpr int KS = Stage<KERNEL>::KS;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        const int i = i0 + q;
        double d[KS];
#pragma unroll
        for (int a = 0; a < KS; a++) d[a] = phi[KS * i + a];
        S.put(q, surf_coord(half, tmpl[3 * i], cx), surf_coord(half, tmpl[3 * i + 1], cy),
              surf_coord(half, tmpl[3 * i + 2], cz), d);
    }
    if (threadIdx.x == 0) {
        S.nseg = 1;
        S.begin[0] = 0;
        S.begin[1] = cnt;
        S.sx[0] = shx, S.sy[0] = shy, S.sz[0] = shz;
        S.cnt[0] = 0;
    }
}

template <int KERNEL>
__device__ __forceinline__ void stage_point(Stage<KERNEL> &S, int q, const double4 *__restrict__ pos,
                                            const double4 *__restrict__ f, int64_t k) {
    const double4 p = pos[k];
    S.xy[q] = make_double2(p.x, p.y);
    if (KERNEL == 0) {
        S.zd[q] = make_double2(p.z, p.w);
    } else {
        const double4 v = f[k];
        S.zd[q] = make_double2(p.z, v.x);
        S.dd[q] = make_double2(v.y, v.z);
    }
}

__device__ __forceinline__ void box_center(int4 c, double &cx, double &cy, double &cz) {
    const double h = ldexp(1.0, -c.w);
    cx = (c.x + 0.5) * h, cy = (c.y + 0.5) * h, cz = (c.z + 0.5) * h;
}

__device__ __forceinline__ int lanes_per_target(int ntg) {
    int G = 1;
    while (G < 32 && ntg * G * 2 <= NT) G *= 2;
    return G;
}

__device__ __forceinline__ void shift_of(int code, double &x, double &y, double &z) {
    int a, b, c;
    shift_decode(code, a, b, c);
    x = a, y = b, z = c;
}

struct LeafParams {
    TreeView T;
    int n, Kp;
    const double *tmpl;
    const double4 *src_pos, *src_f, *trg_pos;
    const int *trg_perm, *leaves;
    const int64_t *u_off, *w_off;
    const int2 *u_ent, *w_ent;
    const double *phi_dn, *phi_up, *phi_far;
    double *out;
};

// TT targets per thread (register tile: one shared-memory source read feeds TT independent
// pair chains); the lane takes sources j, j + G, ... of every staged segment
template <int KERNEL, int TT>
__device__ __forceinline__ void accumulate_tt(const Stage<KERNEL> &S, const double (&tx)[TT], const double (&ty)[TT],
                                              const double (&tz)[TT], int j, int G, double (&acc)[TT][3]) {
    for (int s = 0; s < S.nseg; s++) {
        double ux[TT], uy[TT], uz[TT];
#pragma unroll
        for (int k = 0; k < TT; k++) ux[k] = tx[k] - S.sx[s], uy[k] = ty[k] - S.sy[s], uz[k] = tz[k] - S.sz[s];
        const int end = S.begin[s + 1];
        int q = S.begin[s] + j;
        // LEAF_NS sources per step: LEAF_NS x TT interleaved pair chains (kernels.cuh, pair_tile)
        for (; q + (LEAF_NS - 1) * G < end; q += LEAF_NS * G) {
            double2 a[LEAF_NS], b[LEAF_NS], c[LEAF_NS];
#pragma unroll
            for (int u = 0; u < LEAF_NS; u++) {
                a[u] = S.xy[q + u * G], b[u] = S.zd[q + u * G];
                c[u] = KERNEL != 0 ? S.dd[q + u * G] : make_double2(0.0, 0.0);
            }
            pair_tile<KERNEL, TT, LEAF_NS>(ux, uy, uz, a, b, c, acc);
        }
        for (; q < end; q += G) {
            const double2 a[1] = {S.xy[q]}, b[1] = {S.zd[q]};
            double2 c[1] = {make_double2(0.0, 0.0)};
            if (KERNEL != 0) c[0] = S.dd[q];
            pair_tile<KERNEL, TT, 1>(ux, uy, uz, a, b, c, acc);
        }
    }
}

// Leaf pass: one CTA per target leaf; targets in groups of TT, G = NT / groups lanes per
// group (any G, so no lane idles for want of a power of two); sources staged in shared
// memory per batch of segments; the G partial sums of a group are reduced in a fixed order
// through shared memory (deterministic, each target written once).
template <int KERNEL, int TT> __global__ void __launch_bounds__(NT, LEAF_MINB) leaf_kernel(LeafParams P) {
    constexpr int KS = Stage<KERNEL>::KS;
    __shared__ union {
        Stage<KERNEL> S;
        double red[NT][TT][KS];
    } sm;
    Stage<KERNEL> &S = sm.S;
    __shared__ int s_ucode[MAXU], s_ub[MAXU];
    __shared__ int s_pre[MAXU + 1]; // exclusive prefix of the batch's entry sizes (flat source index)
    __shared__ int s_wtot[NT / 32], s_whead[NT / 32];
    // runs of consecutive entries with the same image shift are one segment of the pair loops
    // (an interior leaf's 27 neighbours: one run, no per-leaf tail of idle lanes)
    __shared__ int s_run[MAXU], s_runstart[MAXU], s_runcode[MAXU];
    const int b = P.leaves[blockIdx.x];
    const int2 tr = P.T.trng[b];
    const int ntg = tr.y - tr.x;
    if (ntg == 0) return;
    const int4 bc = P.T.cell[b];
    double cx, cy, cz;
    box_center(bc, cx, cy, cz);
    const double scale = ldexp(1.0, bc.w);
    const int ngroups = (ntg + TT - 1) / TT;
    const int G = max(1, min(32, NT / ngroups));
    const int gpc = NT / G; // groups per pass
    const int tid = threadIdx.x, j = tid % G;
    for (int g0 = 0; g0 < ngroups; g0 += gpc) {
        const int grp = g0 + tid / G;
        const bool active = tid / G < gpc && grp < ngroups;
        double tx[TT], ty[TT], tz[TT], acc[TT][3];
#pragma unroll
        for (int k = 0; k < TT; k++) {
            const int t = min(grp * TT + k, ntg - 1); // a missing target repeats the last one (not written)
            const double4 p = P.trg_pos[tr.x + (active ? t : 0)];
            tx[k] = p.x, ty[k] = p.y, tz[k] = p.z;
            acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
        }
        // L2T: outer (downward equivalent) surface of b, density phi_dn[b]
        {
            const double half = 0.5 * (kOuter / scale);
            for (int i0 = 0; i0 < P.n; i0 += SB) {
                __syncthreads();
                stage_surface<KERNEL>(S, P.tmpl, i0, min(SB, P.n - i0), cx, cy, cz, half,
                                      P.phi_dn + (int64_t)b * P.Kp, 0.0, 0.0, 0.0);
                __syncthreads();
                if (active) accumulate_tt<KERNEL, TT>(S, tx, ty, tz, j, G, acc);
            }
        }
        // W: inner (upward equivalent) surfaces of finer well-separated boxes
        for (int64_t e = P.w_off[b]; e < P.w_off[b + 1]; e++) {
            const int2 en = P.w_ent[e];
            const int4 cc = P.T.cell[en.x];
            double ccx, ccy, ccz, shx, shy, shz;
            box_center(cc, ccx, ccy, ccz);
            shift_of(en.y, shx, shy, shz);
            const double half = 0.5 * (kInner / ldexp(1.0, cc.w));
            for (int i0 = 0; i0 < P.n; i0 += SB) {
                __syncthreads();
                stage_surface<KERNEL>(S, P.tmpl, i0, min(SB, P.n - i0), ccx, ccy, ccz, half,
                                      P.phi_up + (int64_t)en.x * P.Kp, shx, shy, shz);
                __syncthreads();
                if (active) accumulate_tt<KERNEL, TT>(S, tx, ty, tz, j, G, acc);
            }
        }
        // U: adjacent source leaves. A batch of up to MAXU entries is one flat run of sources
        // (prefix sums of the entry sizes, a block scan); stages are SB-source windows of that
        // run. Every thread finds its sources' entries by binary search in the prefix, so the
        // segment table and all loads of a stage are issued in parallel (no serial
        // segmentation, no load chained per segment).
        const int64_t ub = P.u_off[b], ue = P.u_off[b + 1];
        for (int64_t e0 = ub; e0 < ue; e0 += MAXU) {
            const int ne = (int)(int64_t)::min((int64_t)MAXU, ue - e0);
            __syncthreads(); // the previous stage's sums are done with S and the tables
            int len = 0;
            if (tid < ne) {
                const int2 en = P.u_ent[e0 + tid];
                const int2 r = P.T.srng[en.x];
                s_ucode[tid] = en.y, s_ub[tid] = r.x;
                len = r.y - r.x;
            }
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if ((tid & 31) >= o) inc += v;
            }
            if ((tid & 31) == 31) s_wtot[tid >> 5] = inc;
            __syncthreads();
            int woff = 0;
            for (int w = 0; w < (tid >> 5); w++) woff += s_wtot[w];
            s_pre[tid] = woff + inc - len;
            if (tid == NT - 1) s_pre[NT] = woff + inc;
            const bool head = tid < ne && (tid == 0 || s_ucode[tid] != s_ucode[tid - 1]);
            const unsigned hb = __ballot_sync(0xffffffffu, head);
            if ((tid & 31) == 0) s_whead[tid >> 5] = __popc(hb);
            __syncthreads();
            if (tid < ne) {
                int rid = __popc(hb & (0xffffffffu >> (31 - (tid & 31)))) - 1;
                for (int w = 0; w < (tid >> 5); w++) rid += s_whead[w];
                s_run[tid] = rid;
                if (head) s_runstart[rid] = s_pre[tid], s_runcode[rid] = s_ucode[tid];
            }
            __syncthreads();
            const int total = s_pre[ne == NT ? NT : ne]; // entries past ne have length 0: s_pre[ne] is the total
            // largest k in [lo, hi] with s_pre[k] <= p
            auto entry_of = [&](int p, int lo, int hi) {
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_pre[mid] <= p) lo = mid;
                    else hi = mid - 1;
                }
                return lo;
            };
            for (int t0 = 0; t0 < total; t0 += SB) {
                const int t1 = min(total, t0 + SB);
                const int k0 = entry_of(t0, 0, ne - 1), k1 = entry_of(t1 - 1, k0, ne - 1);
                const int r0 = s_run[k0], nseg = s_run[k1] - r0 + 1;
                if (t0 > 0) __syncthreads(); // the previous stage's sums are done with S
                for (int i = tid; i <= nseg; i += NT) {
                    S.begin[i] = i < nseg ? max(s_runstart[r0 + i], t0) - t0 : t1 - t0;
                    if (i < nseg) {
                        double a, bb, c;
                        shift_of(s_runcode[r0 + i], a, bb, c);
                        S.sx[i] = a, S.sy[i] = bb, S.sz[i] = c;
                        S.cnt[i] = 0;
                    }
                }
                if (tid == 0) S.nseg = nseg;
#pragma unroll 4
                for (int p = t0 + tid; p < t1; p += NT) {
                    const int k = entry_of(p, k0, k1);
                    stage_point<KERNEL>(S, p - t0, P.src_pos, P.src_f, s_ub[k] + (p - s_pre[k]));
                }
                __syncthreads();
                if (active) accumulate_tt<KERNEL, TT>(S, tx, ty, tz, j, G, acc);
            }
        }
        // far field: root outer surface with the periodizing density (image layers
        // 2..ell + T_M2L, summed: both live on the same surface)
        if (P.phi_far) {
            const double half = 0.5 * kOuter;
            for (int i0 = 0; i0 < P.n; i0 += SB) {
                __syncthreads();
                stage_surface<KERNEL>(S, P.tmpl, i0, min(SB, P.n - i0), 0.5, 0.5, 0.5, half, P.phi_far, 0.0, 0.0,
                                      0.0);
                __syncthreads();
                if (active) accumulate_tt<KERNEL, TT>(S, tx, ty, tz, j, G, acc);
            }
        }
        // combine the G lanes of each group in a fixed order
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TT; k++)
#pragma unroll
            for (int a = 0; a < KS; a++) sm.red[tid][k][a] = acc[k][a];
        __syncthreads();
        if (active && j == 0) {
#pragma unroll
            for (int k = 0; k < TT; k++) {
                const int t = grp * TT + k;
                if (t >= ntg) continue;
                const int64_t orig = P.trg_perm[tr.x + t];
#pragma unroll
                for (int a = 0; a < KS; a++) {
                    double v = 0.0;
                    for (int l = 0; l < G; l++) v += sm.red[tid + l][k][a];
                    P.out[orig * KS + a] = KERNEL == 0 ? v : kOneOver8Pi * v;
                }
            }
        }
    }
}

struct CheckParams {
    TreeView T;
    int n, Kp;
    const double *tmpl;
    const double4 *src_pos, *src_f;
    const int *boxes; // leaves (s2m) or null (x: all boxes)
    const int64_t *x_off;
    const int2 *x_ent;
    double *q;
};

// S2M (upward check = outer surface) or X/S2L (downward check = inner surface)
template <int KERNEL, bool XLIST> __global__ void __launch_bounds__(NT) check_kernel(CheckParams P) {
    constexpr int KS = Stage<KERNEL>::KS;
    __shared__ Stage<KERNEL> S;
    const int b = XLIST ? blockIdx.x : P.boxes[blockIdx.x];
    int64_t e0 = 0, e1 = 1;
    if (XLIST) {
        e0 = P.x_off[b], e1 = P.x_off[b + 1];
        if (e0 == e1) return;
    } else {
        const int2 r = P.T.srng[b];
        if (r.y == r.x) return;
    }
    const int4 bc = P.T.cell[b];
    double cx, cy, cz;
    box_center(bc, cx, cy, cz);
    const double scale = ldexp(1.0, bc.w);
    const double half = 0.5 * ((XLIST ? kInner : kOuter) / scale);
    const int tid = threadIdx.x;
    for (int i0 = 0; i0 < P.n; i0 += NT) {
        const int i = i0 + tid;
        const bool active = i < P.n;
        double tx = 0, ty = 0, tz = 0;
        if (active) {
            tx = surf_coord(half, P.tmpl[3 * i], cx);
            ty = surf_coord(half, P.tmpl[3 * i + 1], cy);
            tz = surf_coord(half, P.tmpl[3 * i + 2], cz);
        }
        double acc[3] = {0.0, 0.0, 0.0};
        for (int64_t e = e0; e < e1; e++) {
            int c = b, code = shift_code(0, 0, 0);
            if (XLIST) {
                const int2 en = P.x_ent[e];
                c = en.x, code = en.y;
            }
            const int2 r = P.T.srng[c];
            double shx, shy, shz;
            shift_of(code, shx, shy, shz);
            for (int s0 = r.x; s0 < r.y; s0 += SB) {
                const int cnt = min(SB, r.y - s0);
                __syncthreads();
                for (int q = tid; q < cnt; q += NT) stage_point<KERNEL>(S, q, P.src_pos, P.src_f, s0 + q);
                if (tid == 0) {
                    S.nseg = 1, S.begin[0] = 0, S.begin[1] = cnt, S.cnt[0] = 0;
                    S.sx[0] = shx, S.sy[0] = shy, S.sz[0] = shz;
                }
                __syncthreads();
                if (active) accumulate<KERNEL>(S, tx, ty, tz, 0, 1, acc, nullptr);
            }
        }
        if (active) {
            double *q = P.q + (int64_t)b * P.Kp + KS * i;
#pragma unroll
            for (int a = 0; a < KS; a++) {
                const double v = KERNEL == 0 ? acc[a] : kOneOver8Pi * acc[a];
                if (XLIST)
                    q[a] += v;
                else
                    q[a] = v;
            }
        }
    }
}

struct DirectParams {
    const double *trg, *src, *den;
    int64_t nt, ns;
    const double *offs; // noff x 3
    int noff, skip_zero;
    int n;              // far surface points (0 = none)
    const double *tmpl, *phi_far;
    double *out;
    int accumulate;
    int *coincident;
};

template <int KERNEL> __global__ void __launch_bounds__(NT) direct_kernel(DirectParams P) {
    constexpr int KS = Stage<KERNEL>::KS;
    __shared__ Stage<KERNEL> S;
    const int tid = threadIdx.x;
    const int64_t t = blockIdx.x * (int64_t)NT + tid;
    const bool active = t < P.nt;
    double tx = 0, ty = 0, tz = 0;
    if (active) tx = P.trg[3 * t], ty = P.trg[3 * t + 1], tz = P.trg[3 * t + 2];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int o = 0; o < P.noff; o++) {
        const double ox = P.offs[3 * o], oy = P.offs[3 * o + 1], oz = P.offs[3 * o + 2];
        const bool zero = ox == 0.0 && oy == 0.0 && oz == 0.0;
        for (int64_t s0 = 0; s0 < P.ns; s0 += SB) {
            const int cnt = (int)(int64_t)::min((int64_t)SB, P.ns - s0);
            __syncthreads();
            for (int q = tid; q < cnt; q += NT) {
                const int64_t k = s0 + q;
                double d[KS];
#pragma unroll
                for (int a = 0; a < KS; a++) d[a] = P.den[KS * k + a];
                S.put(q, P.src[3 * k], P.src[3 * k + 1], P.src[3 * k + 2], d);
            }
            if (tid == 0) {
                S.nseg = 1, S.begin[0] = 0, S.begin[1] = cnt;
                S.sx[0] = ox, S.sy[0] = oy, S.sz[0] = oz;
                S.cnt[0] = (zero && P.skip_zero) ? 0 : 1;
            }
            __syncthreads();
            if (active) accumulate<KERNEL>(S, tx, ty, tz, 0, 1, acc, P.coincident);
        }
    }
    if (P.n > 0) {
        for (int i0 = 0; i0 < P.n; i0 += SB) {
            __syncthreads();
            stage_surface<KERNEL>(S, P.tmpl, i0, min(SB, P.n - i0), 0.5, 0.5, 0.5, 0.5 * kOuter, P.phi_far, 0.0, 0.0,
                                  0.0);
            __syncthreads();
            if (active) accumulate<KERNEL>(S, tx, ty, tz, 0, 1, acc, nullptr);
        }
    }
    if (active) {
#pragma unroll
        for (int a = 0; a < KS; a++) {
            const double v = KERNEL == 0 ? acc[a] : kOneOver8Pi * acc[a];
            if (P.accumulate)
                P.out[KS * t + a] += v;
            else
                P.out[KS * t + a] = v;
        }
    }
}

struct RootParams {
    int n;
    const double *tmpl, *src, *den;
    int64_t ns;
    int nsplit;
    double *part; // nsplit x (ks n)
};

template <int KERNEL> __global__ void __launch_bounds__(NT) root_check_kernel(RootParams P) {
    constexpr int KS = Stage<KERNEL>::KS;
    __shared__ Stage<KERNEL> S;
    const int tid = threadIdx.x;
    const int i = blockIdx.x * NT + tid;
    const bool active = i < P.n;
    const int64_t sb = P.ns * blockIdx.y / P.nsplit, se = P.ns * (blockIdx.y + 1) / P.nsplit;
    double tx = 0, ty = 0, tz = 0;
    const double half = 0.5 * kOuter;
    if (active) {
        tx = surf_coord(half, P.tmpl[3 * i], 0.5);
        ty = surf_coord(half, P.tmpl[3 * i + 1], 0.5);
        tz = surf_coord(half, P.tmpl[3 * i + 2], 0.5);
    }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t s0 = sb; s0 < se; s0 += SB) {
        const int cnt = (int)(int64_t)::min((int64_t)SB, se - s0);
        __syncthreads();
        for (int q = tid; q < cnt; q += NT) {
            const int64_t k = s0 + q;
            double d[KS];
#pragma unroll
            for (int a = 0; a < KS; a++) d[a] = P.den[KS * k + a];
            S.put(q, P.src[3 * k], P.src[3 * k + 1], P.src[3 * k + 2], d);
        }
        if (tid == 0) {
            S.nseg = 1, S.begin[0] = 0, S.begin[1] = cnt, S.cnt[0] = 0;
            S.sx[0] = 0.0, S.sy[0] = 0.0, S.sz[0] = 0.0;
        }
        __syncthreads();
        if (active) accumulate<KERNEL>(S, tx, ty, tz, 0, 1, acc, nullptr);
    }
    if (active)
#pragma unroll
        for (int a = 0; a < KS; a++)
            P.part[(int64_t)blockIdx.y * KS * P.n + KS * i + a] = KERNEL == 0 ? acc[a] : kOneOver8Pi * acc[a];
}

__global__ void split_sum_kernel(const double *part, int nsplit, int len, double *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    double v = 0.0;
    for (int s = 0; s < nsplit; s++) v += part[(int64_t)s * len + i];
    out[i] = v;
}

} // namespace

void leaf_pass(const PairGeom &g, const DeviceTree &T, const DeviceLists &L, const double *phi_dn,
               const double *phi_up, const double *phi_far, double *out, cudaStream_t st, const int *leaves,
               int nleaves) {
    if (!leaves) leaves = T.leaves, nleaves = (int)T.nleaves;
    if (nleaves == 0) return;
    LeafParams P{T.view(), g.n,         g.Kp,       g.tmpl,   T.src_pos, T.src_f, T.trg_pos, T.trg_perm, leaves,
                 L.u.off,  L.w.off,     L.u.ent,    L.w.ent,  phi_dn,    phi_up,  phi_far,   out};
    // targets per thread (register tile): PKGPU_LEAF_TT = 1 | 2 | 4, default 2
    const int tt = tuning().leaf_tt;
    if (g.kernel == 0) {
        if (tt == 1) leaf_kernel<0, 1><<<(unsigned)nleaves, NT, 0, st>>>(P);
        else if (tt == 4) leaf_kernel<0, 4><<<(unsigned)nleaves, NT, 0, st>>>(P);
        else leaf_kernel<0, 2><<<(unsigned)nleaves, NT, 0, st>>>(P);
    } else {
        if (tt == 1) leaf_kernel<1, 1><<<(unsigned)nleaves, NT, 0, st>>>(P);
        else if (tt == 4) leaf_kernel<1, 4><<<(unsigned)nleaves, NT, 0, st>>>(P);
        else leaf_kernel<1, 2><<<(unsigned)nleaves, NT, 0, st>>>(P);
    }
    PK_CUDA(cudaGetLastError());
}

void s2m_pass(const PairGeom &g, const DeviceTree &T, double *q, cudaStream_t st, const int *leaves, int nleaves) {
    if (!leaves) leaves = T.leaves, nleaves = (int)T.nleaves;
    if (nleaves == 0) return;
    CheckParams P{T.view(), g.n, g.Kp, g.tmpl, T.src_pos, T.src_f, leaves, nullptr, nullptr, q};
    if (g.kernel == 0)
        check_kernel<0, false><<<(unsigned)nleaves, NT, 0, st>>>(P);
    else
        check_kernel<1, false><<<(unsigned)nleaves, NT, 0, st>>>(P);
    PK_CUDA(cudaGetLastError());
}

void x_pass(const PairGeom &g, const DeviceTree &T, const DeviceLists &L, double *q, cudaStream_t st) {
    if (L.x.count == 0) return;
    CheckParams P{T.view(), g.n, g.Kp, g.tmpl, T.src_pos, T.src_f, nullptr, L.x.off, L.x.ent, q};
    if (g.kernel == 0)
        check_kernel<0, true><<<(unsigned)T.nboxes, NT, 0, st>>>(P);
    else
        check_kernel<1, true><<<(unsigned)T.nboxes, NT, 0, st>>>(P);
    PK_CUDA(cudaGetLastError());
}

void direct_pairs(int kernel, const double *d_trg, int64_t nt, const double *d_src, const double *d_den, int64_t ns,
                  const double *d_offsets, int noff, int skip_zero, const PairGeom *far_geom, const double *phi_far,
                  double *d_out, int accumulate, int *d_coincident, Workspace &, cudaStream_t st) {
    if (nt == 0) return;
    DirectParams P{d_trg,    d_src,
                   d_den,    nt,
                   ns,       d_offsets,
                   noff,     skip_zero,
                   far_geom && phi_far ? far_geom->n : 0,
                   far_geom ? far_geom->tmpl : nullptr,
                   phi_far,  d_out,
                   accumulate, d_coincident};
    const unsigned grid = (unsigned)((nt + NT - 1) / NT);
    if (kernel == 0)
        direct_kernel<0><<<grid, NT, 0, st>>>(P);
    else
        direct_kernel<1><<<grid, NT, 0, st>>>(P);
    PK_CUDA(cudaGetLastError());
}

void root_check_potential(const PairGeom &g, const double *d_src, const double *d_den, int64_t ns, double *d_q,
                          Workspace &ws, cudaStream_t st) {
    const int ks = g.kernel == 0 ? 1 : 3;
    const int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(256, ns / 1024));
    const int len = ks * g.n;
    double *part = ws.get<double>("root_part", (size_t)nsplit * len);
    RootParams P{g.n, g.tmpl, d_src, d_den, ns, nsplit, part};
    dim3 grid((g.n + NT - 1) / NT, nsplit);
    if (g.kernel == 0)
        root_check_kernel<0><<<grid, NT, 0, st>>>(P);
    else
        root_check_kernel<1><<<grid, NT, 0, st>>>(P);
    split_sum_kernel<<<(len + 255) / 256, 256, 0, st>>>(part, nsplit, len, d_q);
    PK_CUDA(cudaGetLastError());
}

} // namespace pkgpu
