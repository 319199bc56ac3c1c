"""CPU oracle: a numpy restatement of the reference's periodic-KIFMM evaluate path.

TEST INFRASTRUCTURE ONLY. Nothing in the product (`paper_1705_02043_b200`, libpkgpu.so)
imports, links or calls this module; only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` leg of `bench.py` may use it, and only as the checker.

Pinning: every function here is checked against golden vectors produced by the UNMODIFIED
reference (compiled into `oracle/_ref/refdump` by `oracle/refbuild/Makefile`) — see
`tests/golden/make_golden.py` and `tests/test_oracle_golden.py`.

Each function cites the reference file:line it restates (paths relative to
/root/reference/proj).
"""
from __future__ import annotations

import ctypes
import ctypes.util
import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

INNER = 1.05  # include/pkifmm/geometry.hpp:17
OUTER = 2.95  # include/pkifmm/geometry.hpp:18
ONE_OVER_8PI = 1.0 / (8.0 * math.pi)  # src/kernel.cpp:10

LAPLACE, STOKESLET = 0, 1
NONE, SP, DP, TP = 0, 1, 2, 3
PER_NAMES = ["none", "sp", "dp", "tp"]
KERNEL_NAMES = ["laplace", "stokeslet"]


def kdims(kernel):
    return (1, 1) if kernel == LAPLACE else (3, 3)


def default_axes(per):
    """PeriodicSetup::make defaults (src/geometry.cpp:27-39): SP=z, DP=xy, TP=xyz."""
    return {NONE: (False, False, False), SP: (False, False, True), DP: (True, True, False),
            TP: (True, True, True)}[per]


# ---------------------------------------------------------------------------
# geometry (src/geometry.cpp:41-87)

def surface_point_count(p):
    return 6 * (p - 1) * (p - 1) + 2  # src/geometry.cpp:41


def surface_grid_indices(p):
    """Fixed ordering of src/geometry.cpp:43-58."""
    idx = [(0, 0, 0)]
    for i in range(p - 1):
        for j in range(p - 1):
            idx.append((0, i + 1, j))
    for i in range(p - 1):
        for j in range(p - 1):
            idx.append((i, 0, j + 1))
    for i in range(p - 1):
        for j in range(p - 1):
            idx.append((i + 1, j, 0))
    half = len(idx)
    for i in range(half):
        a = idx[i]
        idx.append((p - 1 - a[0], p - 1 - a[1], p - 1 - a[2]))
    return np.array(idx, dtype=np.int64)


_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
_vfma = np.frompyfunc(_libm.fma, 3, 1)


def fma(a, b, c):
    """Correctly rounded a*b+c (libm fma), elementwise."""
    a, b, c = np.broadcast_arrays(np.asarray(a, np.float64), np.asarray(b, np.float64), np.asarray(c, np.float64))
    return _vfma(a, b, c).astype(np.float64)


_TEMPLATE = {}


def surface_template(p):
    """t = g*2/(p-1) - 1 per coordinate. The reference is built with FMA contraction
    (-O3 -march=..., GNU mode), so this is fma(g, scale, -1) (src/geometry.cpp:66)."""
    if p not in _TEMPLATE:
        g = surface_grid_indices(p).astype(np.float64)
        _TEMPLATE[p] = fma(g, 2.0 / (p - 1), -1.0)
    return _TEMPLATE[p]


def surface_points(p, center, edge):
    """src/geometry.cpp:60-71: center + (0.5*edge)*t, contracted to fma(half, t, center)
    exactly as the compiled reference evaluates it (pinned bit-exact by tests)."""
    t = surface_template(p)
    half = 0.5 * edge
    c = np.asarray(center, dtype=np.float64)
    return fma(half, t, c[None, :])


def image_offsets(axes, min_norm, max_norm):
    """src/geometry.cpp:73-87 (lexicographic ox, oy, oz)."""
    lx, ly, lz = (max_norm if a else 0 for a in axes)
    out = []
    for ox in range(-lx, lx + 1):
        for oy in range(-ly, ly + 1):
            for oz in range(-lz, lz + 1):
                n = max(abs(ox), abs(oy), abs(oz))
                if min_norm <= n <= max_norm:
                    out.append((ox, oy, oz))
    return out


# ---------------------------------------------------------------------------
# kernels (src/kernel.cpp:29-129)

def kernel_block(kernel, targets, sources):
    """Dense (kt*T) x (ks*S) matrix, src/kernel.cpp:29-78 (coincident pairs raise)."""
    t = np.asarray(targets, dtype=np.float64)
    s = np.asarray(sources, dtype=np.float64)
    r = t[:, None, :] - s[None, :, :]
    r2 = r[..., 0] * r[..., 0] + r[..., 1] * r[..., 1] + r[..., 2] * r[..., 2]
    if np.any(r2 == 0.0) and np.any((t[:, None, :] == s[None, :, :]).all(-1)):
        raise ValueError("kernel evaluation at zero separation")
    if kernel == LAPLACE:
        return 1.0 / np.sqrt(r2)
    rinv = 1.0 / np.sqrt(r2)
    rinv3 = rinv / r2
    nt, ns = r2.shape
    m = np.empty((nt, 3, ns, 3))
    for a in range(3):
        for b in range(3):
            v = r[..., a] * r[..., b] * rinv3
            if a == b:
                v = rinv + v
            m[:, a, :, b] = ONE_OVER_8PI * v
    return m.reshape(3 * nt, 3 * ns)


class CoincidentError(ValueError):
    pass


def kernel_block_apply(kernel, targets, sources, shift, density, out, skip_coincident=False):
    """out[kt*i+a] += sum_j K((t_i - shift) - s_j) rho_j, src/kernel.cpp:80-129.

    rinv = r2 > 0 ? 1/sqrt(r2) : 0; coincident pairs raise unless skip_coincident.
    """
    t = np.asarray(targets, dtype=np.float64).reshape(-1, 3)
    s = np.asarray(sources, dtype=np.float64).reshape(-1, 3)
    if len(t) == 0 or len(s) == 0:
        return out
    sh = np.asarray(shift, dtype=np.float64)
    tt = t - sh[None, :]
    rx = tt[:, 0:1] - s[None, :, 0]
    ry = tt[:, 1:2] - s[None, :, 1]
    rz = tt[:, 2:3] - s[None, :, 2]
    r2 = rx * rx + ry * ry + rz * rz
    zero = r2 == 0.0
    with np.errstate(divide="ignore"):
        rinv = np.where(zero, 0.0, 1.0 / np.sqrt(np.where(zero, 1.0, r2)))
    ncoin = int(zero.sum())
    if ncoin and not skip_coincident:
        raise CoincidentError(f"kernel_block_apply: {ncoin} coincident target/source pairs")
    d = np.asarray(density, dtype=np.float64)
    if kernel == LAPLACE:
        out[: len(t)] += rinv @ d
        return out
    f = d.reshape(-1, 3)
    rdotf = (rx * f[None, :, 0] + ry * f[None, :, 1] + rz * f[None, :, 2]) * rinv * rinv
    o = out.reshape(-1, 3)
    o[:, 0] += ONE_OVER_8PI * ((f[None, :, 0] + rx * rdotf) * rinv).sum(1)
    o[:, 1] += ONE_OVER_8PI * ((f[None, :, 1] + ry * rdotf) * rinv).sum(1)
    o[:, 2] += ONE_OVER_8PI * ((f[None, :, 2] + rz * rdotf) * rinv).sum(1)
    return out


# ---------------------------------------------------------------------------
# linear algebra (src/linalg.cpp:44-104)

@dataclass
class SvdFactors:
    u: np.ndarray
    sigma: np.ndarray
    vt: np.ndarray

    @property
    def eps_svd(self):
        return np.finfo(np.float64).eps * (self.sigma[0] if len(self.sigma) else 0.0)  # :64-66

    def sinv(self):
        s = self.sigma
        return np.where(s > self.eps_svd, 1.0 / np.where(s > 0, s, 1.0), 0.0)


def svd(a):
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    return SvdFactors(u, s, vt)


def pinv_apply(f: SvdFactors, b):
    """x = V (S+ (U^T b)) in nested order, src/linalg.cpp:78-87."""
    t = f.u.T @ b
    t = np.where(f.sigma[:, None] > f.eps_svd if t.ndim == 2 else f.sigma > f.eps_svd,
                 t / (f.sigma[:, None] if t.ndim == 2 else f.sigma), 0.0)
    return f.vt.T @ t


# ---------------------------------------------------------------------------
# tree (src/fmm.cpp:301-413), restated through 36-bit Morton keys

def morton_keys(points):
    """36-bit key, x = least significant bit of each (x,y,z) triple; floor(x*4096) is exact."""
    q = np.floor(np.asarray(points, dtype=np.float64) * 4096.0).astype(np.int64)
    key = np.zeros(len(q), dtype=np.int64)
    for bit in range(12):
        for a in range(3):
            key |= ((q[:, a] >> bit) & 1) << (3 * bit + a)
    return key


@dataclass
class Tree:
    level: np.ndarray
    cell: np.ndarray      # (nb, 3)
    parent: np.ndarray
    child: np.ndarray     # (nb, 8)
    leaf: np.ndarray
    src: list             # per box, increasing original indices (leaves only)
    trg: list
    src_subtree: np.ndarray
    trg_subtree: np.ndarray
    depth: int

    @property
    def nboxes(self):
        return len(self.level)

    def table(self):
        """Same layout as refdump's .boxes.i32 dump."""
        nb = self.nboxes
        t = np.zeros((nb, 18), dtype=np.int32)
        t[:, 0] = self.level
        t[:, 1:4] = self.cell
        t[:, 4] = self.parent
        t[:, 5] = self.leaf
        t[:, 6] = [len(x) for x in self.src]
        t[:, 7] = [len(x) for x in self.trg]
        t[:, 8] = self.src_subtree
        t[:, 9] = self.trg_subtree
        t[:, 10:18] = self.child
        return t

    def center(self, b):
        h = 2.0 ** (-int(self.level[b]))
        c = self.cell[b]
        return np.array([(c[0] + 0.5) * h, (c[1] + 0.5) * h, (c[2] + 0.5) * h])


class TreeError(RuntimeError):
    pass


def check_points(src, trg):
    """src/fmm.cpp:305-323 — message lists the first 8 offenders."""
    bad = 0
    msg = ""
    for what, pts in (("source", src), ("target", trg)):
        pts = np.asarray(pts).reshape(-1, 3)
        m = ~((pts >= 0) & (pts < 1)).all(1)
        for i in np.nonzero(m)[0]:
            if bad < 8:
                x = pts[i]
                msg += f" {what}[{i}]=({_g6(x[0])},{_g6(x[1])},{_g6(x[2])})"
            bad += 1
    if bad:
        raise ValueError(f"FmmTree: {bad} points outside [0,1)^3:{msg}")


def _g6(v):
    """std::ostream default formatting (%g, 6 significant digits)."""
    return "%g" % v


def build_tree(src, trg, leaf_capacity=1000, max_depth=12):
    """BFS adaptive octree, src/fmm.cpp:301-389, via the Morton-key recipe of SURVEY §8a."""
    if leaf_capacity < 1:
        raise ValueError("FmmTree: leaf capacity must be positive")
    src = np.asarray(src, dtype=np.float64).reshape(-1, 3)
    trg = np.asarray(trg, dtype=np.float64).reshape(-1, 3)
    check_points(src, trg)
    ks_, kt_ = morton_keys(src), morton_keys(trg)
    so = np.argsort(ks_, kind="stable")
    to = np.argsort(kt_, kind="stable")
    sk, tk = ks_[so], kt_[to]
    level, cell, parent, child, leaf = [0], [(0, 0, 0)], [-1], [[-1] * 8], [True]
    srng, trng = [(0, len(sk))], [(0, len(tk))]
    bi = 0
    while bi < len(level):
        ns = srng[bi][1] - srng[bi][0]
        nt = trng[bi][1] - trng[bi][0]
        if ns > leaf_capacity or nt > leaf_capacity:
            l = level[bi]
            if l >= max_depth:
                raise TreeError(f"FmmTree: leaf over capacity at maximum depth {max_depth} "
                                "(duplicate point pathology)")
            leaf[bi] = False
            shift = 3 * (11 - l)
            for o in range(8):
                # child range: keys whose octant digit at level l+1 equals o
                def sub(keys, rng):
                    lo, hi = rng
                    seg = (keys[lo:hi] >> shift) & 7
                    a = lo + int(np.searchsorted(seg, o, "left"))
                    b = lo + int(np.searchsorted(seg, o, "right"))
                    return a, b
                cs, ct = sub(sk, srng[bi]), sub(tk, trng[bi])
                if cs[1] == cs[0] and ct[1] == ct[0]:
                    continue
                c = cell[bi]
                level.append(l + 1)
                cell.append((2 * c[0] + (o & 1), 2 * c[1] + ((o >> 1) & 1), 2 * c[2] + ((o >> 2) & 1)))
                parent.append(bi)
                child.append([-1] * 8)
                leaf.append(True)
                srng.append(cs)
                trng.append(ct)
                child[bi][o] = len(level) - 1
        bi += 1
    nb = len(level)
    srcl = [np.sort(so[a:b]) if leaf[i] else np.zeros(0, np.int64) for i, (a, b) in enumerate(srng)]
    trgl = [np.sort(to[a:b]) if leaf[i] else np.zeros(0, np.int64) for i, (a, b) in enumerate(trng)]
    return Tree(np.array(level), np.array(cell, dtype=np.int64), np.array(parent), np.array(child),
                np.array(leaf, dtype=bool), srcl, trgl,
                np.array([b - a for a, b in srng]), np.array([b - a for a, b in trng]), max(level))


def structure_hash(tree: Tree):
    """FNV-1a style mix, src/fmm.cpp:397-413."""
    M = (1 << 64) - 1
    h = 1469598103934665603
    prime = 1099511628211

    def mix(v):
        nonlocal h
        h = ((h ^ (v & M)) * prime) & M

    for b in range(tree.nboxes):
        mix(int(tree.level[b]))
        for a in range(3):
            mix(int(tree.cell[b][a]))
        mix(1 if tree.leaf[b] else 0)
        for i in tree.src[b]:
            mix(int(i) + 0x9E3779B97F4A7C15)
        for i in tree.trg[b]:
            mix(int(i) + 0x517CC1B727220A95)
    return h


# ---------------------------------------------------------------------------
# interaction lists: closed forms of the dual traversal (src/fmm.cpp:422-503)

def boxes_adjacent(bc, bl, cc, cl, shift):
    """src/fmm.cpp:422-433 (closed boxes touch or overlap under the image shift)."""
    lf = max(bl, cl)
    for a in range(3):
        lob = bc[a] << (lf - bl)
        hib = ((bc[a] + 1) << (lf - bl)) - 1
        sc = cc[a] + (shift[a] << cl)
        loc = sc << (lf - cl)
        hic = ((sc + 1) << (lf - cl)) - 1
        if loc > hib + 1 or lob > hic + 1:
            return False
    return True


def wraps_for(per, axes, ell):
    if per == NONE or ell < 1:
        return []
    return image_offsets(axes, 1, 1)


def build_lists(tree: Tree, wraps):
    """Returns dict u/v/w/x: per box list of (c, (sx,sy,sz)) — V stores the cell offset d.

    Restates the recursive traversal (src/fmm.cpp:436-486) as a direct recursion, which
    yields the same multisets (order may differ; callers compare sorted multisets).
    """
    nb = tree.nboxes
    L = {k: [[] for _ in range(nb)] for k in "uvwx"}
    lv, cl, lf, ch = tree.level, tree.cell, tree.leaf, tree.child

    def adj(b, c, s):
        return boxes_adjacent(tuple(cl[b]), int(lv[b]), tuple(cl[c]), int(lv[c]), s)

    def trav(b, c, s):
        if lf[b] and lf[c]:
            L["u"][b].append((c, s))
            return
        if lf[b]:
            for o in range(8):
                cc = ch[c][o]
                if cc < 0:
                    continue
                if adj(b, cc, s):
                    trav(b, cc, s)
                else:
                    L["w"][b].append((cc, s))
            return
        if lf[c]:
            for o in range(8):
                bb = ch[b][o]
                if bb < 0:
                    continue
                if adj(bb, c, s):
                    trav(bb, c, s)
                else:
                    L["x"][bb].append((c, s))
            return
        for ob in range(8):
            bb = ch[b][ob]
            if bb < 0:
                continue
            for oc in range(8):
                cc = ch[c][oc]
                if cc < 0:
                    continue
                if adj(bb, cc, s):
                    trav(bb, cc, s)
                else:
                    lvl = int(lv[bb])
                    d = tuple(int(cl[cc][a] + (s[a] << lvl) - cl[bb][a]) for a in range(3))
                    L["v"][bb].append((cc, d))

    import sys
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10000))
    try:
        trav(0, 0, (0, 0, 0))
        for s in wraps:
            trav(0, 0, tuple(s))
    finally:
        sys.setrecursionlimit(old)
    return L


def lists_to_csr(L):
    out = {}
    for k, lst in L.items():
        off = [0]
        ent = []
        for v in lst:
            for c, s in v:
                ent.append((c, s[0], s[1], s[2]))
            off.append(len(ent))
        out[k] = (np.array(off, dtype=np.int64), np.array(ent, dtype=np.int64).reshape(-1, 4))
    return out


def sorted_multiset(off, ent):
    """Canonical per-box sorted entry list for multiset comparison."""
    res = []
    for b in range(len(off) - 1):
        seg = ent[off[b]:off[b + 1]]
        res.append(sorted(map(tuple, seg.tolist())))
    return res


# ---------------------------------------------------------------------------
# KIFMM operators (src/fmm.cpp:180-236, 262-283) and evaluation (src/fmm.cpp:508-742)

ROOT = np.array([0.5, 0.5, 0.5])


@dataclass
class Operators:
    kernel: int
    p: int
    n: int
    inner: np.ndarray
    outer: np.ndarray
    a_up: SvdFactors
    a_dn: SvdFactors
    _m2l: dict = field(default_factory=dict)
    _m2m: dict = field(default_factory=dict)
    _l2l: dict = field(default_factory=dict)

    def child_inner(self, o):
        c = ROOT + np.array([0.25 if o & 1 else -0.25, 0.25 if o & 2 else -0.25, 0.25 if o & 4 else -0.25])
        return surface_points(self.p, c, 0.5 * INNER)

    def m2l(self, d):
        """K(inner, inner + d) — equal to the reference's class matrix under the signed
        permutation up to rounding (src/fmm.cpp:82-91, 111-130)."""
        d = tuple(d)
        if d not in self._m2l:
            self._m2l[d] = kernel_block(self.kernel, self.inner, self.inner + np.array(d, dtype=np.float64))
        return self._m2l[d]

    def m2m(self, o):  # src/fmm.cpp:93-99
        if o not in self._m2m:
            self._m2m[o] = kernel_block(self.kernel, self.outer, self.child_inner(o))
        return self._m2m[o]

    def l2l(self, o):  # src/fmm.cpp:101-107
        if o not in self._l2l:
            self._l2l[o] = kernel_block(self.kernel, self.child_inner(o), self.outer)
        return self._l2l[o]


def make_operators(kernel, p, factors=None):
    inner = surface_points(p, ROOT, INNER)
    outer = surface_points(p, ROOT, OUTER)
    if factors is None:
        a_up = svd(kernel_block(kernel, outer, inner))  # src/fmm.cpp:187
        a_dn = svd(kernel_block(kernel, inner, outer))  # src/fmm.cpp:188
    else:
        a_up, a_dn = factors
    return Operators(kernel, p, surface_point_count(p), inner, outer, a_up, a_dn)


def root_image_operator(ops: Operators, axes, ell):
    """M_img = sum_{2<=|d|<=ell} K(inner, inner+d), src/fmm.cpp:262-283."""
    kt, ks = kdims(ops.kernel)
    m = np.zeros((kt * ops.n, ks * ops.n))
    for d in image_offsets(axes, 2, ell):
        m += ops.m2l(d)
    return m


def check_compatibility(kernel, per, strengths):
    """src/refsum.cpp:733-756."""
    if per == NONE or (kernel == STOKESLET and per == TP):
        return True, "", 0.0
    ks = kdims(kernel)[0]
    s = np.asarray(strengths, dtype=np.float64).reshape(-1, ks)
    abs_total = float(np.abs(s).sum())
    worst = float(np.abs(s.sum(0)).max()) if len(s) else 0.0
    if worst > 1e-12 * abs_total:
        return False, ("neutrality: net charge must vanish" if kernel == LAPLACE
                       else "neutrality: net force must vanish"), worst
    return True, "", 0.0


def fmm_near(tree: Tree, lists, ops: Operators, src, strengths, trg, per, axes, ell, stages=None):
    """FmmTree::run, src/fmm.cpp:508-653. Returns (potentials, phi_up[0])."""
    kernel, p, n = ops.kernel, ops.p, ops.n
    kt, ks = kdims(kernel)
    src = np.asarray(src, dtype=np.float64).reshape(-1, 3)
    trg = np.asarray(trg, dtype=np.float64).reshape(-1, 3)
    rho = np.asarray(strengths, dtype=np.float64)
    nb = tree.nboxes
    phi_up = [None] * nb
    phi_dn = [None] * nb
    levels = [np.nonzero(tree.level == l)[0] for l in range(tree.depth + 1)]
    U, V, W, X = lists["u"], lists["v"], lists["w"], lists["x"]

    def gather(b):
        idx = tree.src[b]
        return src[idx], rho.reshape(-1, ks)[idx].reshape(-1)

    # upward pass src/fmm.cpp:532-553
    for l in range(tree.depth, -1, -1):
        scale = 2.0 ** l
        for b in levels[l]:
            if tree.src_subtree[b] == 0:
                continue
            q = np.zeros(kt * n)
            if tree.leaf[b]:
                pts, den = gather(b)
                check = surface_points(p, tree.center(b), OUTER / scale)
                kernel_block_apply(kernel, check, pts, (0, 0, 0), den, q)
            else:
                for o in range(8):
                    c = tree.child[b][o]
                    if c < 0 or tree.src_subtree[c] == 0:
                        continue
                    q += scale * (ops.m2m(o) @ phi_up[c])
            phi_up[b] = pinv_apply(ops.a_up, q) / scale
    if stages is not None:
        stages["phi_up"] = phi_up
    out = np.zeros(kt * len(trg))
    # downward pass src/fmm.cpp:557-601
    for l in range(tree.depth + 1):
        scale = 2.0 ** l
        for b in levels[l]:
            if tree.trg_subtree[b] == 0:
                continue
            q = np.zeros(kt * n)
            anyc = False
            for c, d in V[b]:
                if tree.src_subtree[c] == 0:
                    continue
                q += scale * (ops.m2l(d) @ phi_up[c])
                anyc = True
            if X[b]:
                chk = surface_points(p, tree.center(b), INNER / scale)
                for c, s in X[b]:
                    if tree.src_subtree[c] == 0:
                        continue
                    pts, den = gather(c)
                    kernel_block_apply(kernel, chk, pts, s, den, q)
                    anyc = True
            par = tree.parent[b]
            if par >= 0 and phi_dn[par] is not None:
                c3 = tree.cell[b]
                o = (c3[0] & 1) | ((c3[1] & 1) << 1) | ((c3[2] & 1) << 2)
                q += (scale * 0.5) * (ops.l2l(o) @ phi_dn[par])
                anyc = True
            if anyc:
                phi_dn[b] = pinv_apply(ops.a_dn, q) / scale
    if stages is not None:
        stages["phi_dn"] = phi_dn
    # leaves src/fmm.cpp:603-633
    for b in range(nb):
        if not tree.leaf[b] or len(tree.trg[b]) == 0:
            continue
        scale = 2.0 ** int(tree.level[b])
        tb = trg[tree.trg[b]]
        lo = np.zeros(kt * len(tb))
        if phi_dn[b] is not None:
            eq = surface_points(p, tree.center(b), OUTER / scale)
            kernel_block_apply(kernel, tb, eq, (0, 0, 0), phi_dn[b], lo)
        for c, s in W[b]:
            if tree.src_subtree[c] == 0:
                continue
            eq = surface_points(p, tree.center(c), INNER / 2.0 ** int(tree.level[c]))
            kernel_block_apply(kernel, tb, eq, s, phi_up[c], lo)
        for c, s in U[b]:
            if len(tree.src[c]) == 0:
                continue
            pts, den = gather(c)
            kernel_block_apply(kernel, tb, pts, s, den, lo, skip_coincident=(tuple(s) == (0, 0, 0)))
        o2 = out.reshape(-1, kt)
        o2[tree.trg[b]] += lo.reshape(-1, kt)
    # image layers src/fmm.cpp:635-645
    if per != NONE and ell >= 2 and tree.src_subtree[0] > 0:
        m_img = root_image_operator(ops, axes, ell)
        dn = pinv_apply(ops.a_dn, m_img @ phi_up[0])
        far_field_eval(kernel, p, dn, trg, out)
    return out, phi_up[0]


def far_field_eval(kernel, p, density, targets, out):
    """src/periodize.cpp:173-187: targets x outer root surface."""
    eq = surface_points(p, ROOT, OUTER)
    kernel_block_apply(kernel, targets, eq, (0, 0, 0), density, out)
    return out


def direct_root_upward_density(ops: Operators, src, strengths):
    """src/fmm.cpp:676-686."""
    kt = kdims(ops.kernel)[0]
    q = np.zeros(kt * ops.n)
    kernel_block_apply(ops.kernel, ops.outer, src, (0, 0, 0), strengths, q)
    return pinv_apply(ops.a_up, q)


class ConfigError(RuntimeError):
    pass


def evaluate(kernel, src, strengths, trg, per=NONE, axes=None, ell=2, p=8, op=None, mode="fmm",
             leaf_capacity=1000, force=False, factors=None, ops=None):
    """pkifmm::evaluate, src/fmm.cpp:690-742. `op` is a PeriodizingOperator dict
    (load_operator) or None."""
    axes = tuple(axes) if axes is not None else default_axes(per)
    kt, ks = kdims(kernel)
    src = np.asarray(src, dtype=np.float64).reshape(-1, 3)
    trg = np.asarray(trg, dtype=np.float64).reshape(-1, 3)
    rho = np.asarray(strengths, dtype=np.float64)
    if rho.size != ks * len(src):
        raise ValueError("evaluate: strengths length does not match sources")
    periodic = per != NONE
    if periodic and op is None:
        raise ConfigError("evaluate: a periodizing operator is required for periodic runs")
    ok, viol, res = check_compatibility(kernel, per, rho)
    if not ok and not force:
        raise ConfigError(f"evaluate: compatibility violation ({viol})")
    ops = ops or make_operators(kernel, p, factors)
    if mode == "direct":
        pot = np.zeros(kt * len(trg))
        offs = image_offsets(axes, 0, ell) if periodic else [(0, 0, 0)]
        for d in offs:
            kernel_block_apply(kernel, trg, src, d, rho, pot, skip_coincident=(tuple(d) == (0, 0, 0)))
        up = direct_root_upward_density(ops, src, rho)
    else:
        tree = build_tree(src, trg, leaf_capacity)
        lists = build_lists(tree, wraps_for(per, axes, ell) if periodic else [])
        pot, up = fmm_near(tree, lists, ops, src, rho, trg, per if periodic else NONE, axes, ell)
        if up is None:
            up = np.zeros(ks * ops.n)
    if periodic:
        dn = op["matrix"] @ up  # apply_m2l, src/periodize.cpp:160-171
        far_field_eval(kernel, p, dn, trg, pot)
    return pot


# ---------------------------------------------------------------------------
# PKM2L operator files (src/periodize.cpp:40-55, 189-278)

_CRC_TABLE = None


def crc64(data: bytes) -> int:
    """CRC-64/XZ, src/periodize.cpp:40-55."""
    global _CRC_TABLE
    if _CRC_TABLE is None:
        t = np.zeros(256, dtype=np.uint64)
        for i in range(256):
            c = i
            for _ in range(8):
                c = (c >> 1) ^ 0xC96C5795D7870F42 if c & 1 else c >> 1
            t[i] = c
        _CRC_TABLE = [int(x) for x in t]
    crc = 0xFFFFFFFFFFFFFFFF
    tab = _CRC_TABLE
    for b in data:
        crc = tab[(crc ^ b) & 0xFF] ^ (crc >> 8)
    return crc ^ 0xFFFFFFFFFFFFFFFF


def load_operator(path):
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:6] != b"PKM2L\x01":
        raise RuntimeError(f"load_operator: bad magic in {path}")
    (hlen,) = struct.unpack("<Q", raw[6:14])
    hdr = json.loads(raw[14:14 + hlen].decode())
    n = surface_point_count(hdr["p"])
    ks = 1 if hdr["kernel"] == "laplace" else 3
    rows, cols = hdr["rows"], hdr["cols"]
    if rows != ks * n or cols != ks * n or hdr["n"] != n:
        raise RuntimeError(f"load_operator: inconsistent dimensions in {path}")
    payload = raw[14 + hlen:14 + hlen + rows * cols * 8]
    if len(payload) != rows * cols * 8:
        raise RuntimeError(f"load_operator: truncated payload in {path}")
    m = np.frombuffer(payload, dtype="<f8").reshape(rows, cols).copy()
    hdr["matrix"] = m
    return hdr
