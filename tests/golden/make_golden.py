"""Generates the committed golden fixtures under tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/refdump, built by oracle/refbuild/Makefile from /root/reference).

Run in the build container (needs /root/reference only to BUILD refdump):
    make -C oracle/refbuild && python tests/golden/make_golden.py

Fixtures (npz) hold inputs + reference outputs: kernel_block_apply pair sums, surfaces,
trees (box tables, leaf index lists, structure_hash), U/V/W/X lists, evaluate potentials
and root upward densities, error messages; PKM2L operator files go to tests/golden/ops/.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REFDUMP = os.path.join(REPO, "oracle", "_ref", "refdump")
OPS = os.path.join(HERE, "ops")


def run(*args, ok_codes=(0,)):
    r = subprocess.run([REFDUMP, *map(str, args)], capture_output=True, text=True)
    if r.returncode not in ok_codes:
        raise RuntimeError(f"refdump {args} failed rc={r.returncode}: {r.stdout} {r.stderr}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def f64(path):
    return np.fromfile(path, dtype="<f8")


def i32(path):
    return np.fromfile(path, dtype="<i4")


def gen(tmp, name, n, kind="uniform", ks=1, seed=12345, **kw):
    args = ["gen", "--n", n, "--kind", kind, "--ks", ks, "--seed", seed, "--out", os.path.join(tmp, name)]
    for k, v in kw.items():
        args += ["--" + k, v]
    run(*args)
    return f64(os.path.join(tmp, name + ".src.f64")).reshape(-1, 3), f64(os.path.join(tmp, name + ".str.f64"))


def save_pts(tmp, name, arr):
    p = os.path.join(tmp, name)
    np.ascontiguousarray(arr, dtype="<f8").tofile(p)
    return p


def golden_pairs(tmp):
    rng = np.random.default_rng(7)
    out = {}
    for kernel, ks in (("laplace", 1), ("stokeslet", 3)):
        trg = rng.random((37, 3))
        src = rng.random((53, 3))
        src[5] = trg[3]  # one exact coincidence
        den = rng.standard_normal(53 * ks)
        for tag, shift, skip in (("s0_skip", (0, 0, 0), True), ("s0_noskip", (0, 0, 0), False),
                                 ("shift", (1.0, 0.0, -1.0), False)):
            pt, ps = save_pts(tmp, "pt", trg), save_pts(tmp, "ps", src)
            pd, psh = save_pts(tmp, "pd", den), save_pts(tmp, "psh", np.array(shift, dtype=float))
            args = ["pairs", "--kernel", kernel, "--trg", pt, "--src", ps, "--den", pd, "--shift", psh,
                    "--out", os.path.join(tmp, "pr")]
            if skip:
                args.append("--skip")
            r = run(*args)
            key = f"{kernel}_{tag}"
            out[key + "_trg"] = trg
            out[key + "_src"] = src
            out[key + "_den"] = den
            out[key + "_shift"] = np.array(shift, dtype=float)
            out[key + "_skip"] = np.array(skip)
            out[key + "_pot"] = f64(os.path.join(tmp, "pr.pot.f64"))
            out[key + "_error"] = np.array(r["error"])
    np.savez_compressed(os.path.join(HERE, "pairs.npz"), **out)


def golden_surfaces(tmp):
    out = {}
    for p in (2, 4, 6, 8, 10):
        for (cx, cy, cz, edge) in ((0.5, 0.5, 0.5, 1.05), (0.5, 0.5, 0.5, 2.95), (0.3125, 0.8125, 0.0625, 2.95 / 8)):
            r = run("surface", "--p", p, "--cx", cx, "--cy", cy, "--cz", cz, "--edge", edge,
                    "--out", os.path.join(tmp, "s"))
            out[f"p{p}_{cx}_{cy}_{cz}_{edge}"] = f64(os.path.join(tmp, "s.surf.f64")).reshape(-1, 3)
            assert r["n"] == 6 * (p - 1) ** 2 + 2
    np.savez_compressed(os.path.join(HERE, "surfaces.npz"), **out)


TREE_CASES = {
    # name: (leaf capacity, list variants)
    "uniform3k": 40,
    "adaptive": 30,
    "cfg1": 50,
}
LIST_VARIANTS = {"none": ("none", ""), "sp": ("sp", ""), "dp": ("dp", ""), "tp": ("tp", ""), "spx": ("sp", "x")}


def tree_inputs(tmp):
    cases = {}
    src, _ = gen(tmp, "t_u", 3000, seed=11)
    cases["uniform3k"] = (src, src)
    # adaptive: clustered sources + points on dyadic split planes + separate targets
    src, _ = gen(tmp, "t_c", 4000, kind="clusters", nclusters=4, sigma=0.02, axes="xyz", seed=21)
    rng = np.random.default_rng(5)
    plane = rng.integers(0, 64, size=(200, 3)) / 64.0
    src = np.concatenate([src, plane])
    trg, _ = gen(tmp, "t_t", 1500, seed=22)
    trg = np.concatenate([trg, plane[:50]])
    cases["adaptive"] = (src, trg)
    src, _ = gen(tmp, "c1", 20000, seed=12345)
    cases["cfg1"] = (src, src)
    return cases


def golden_trees(tmp):
    cases = tree_inputs(tmp)
    for name, (src, trg) in cases.items():
        leaf = TREE_CASES[name]
        ps, pt = save_pts(tmp, "ts", src), save_pts(tmp, "tt", trg)
        out = {"src": src, "trg": trg, "leaf": np.array(leaf)}
        base = os.path.join(tmp, "tr")
        for vname, (per, axes) in LIST_VARIANTS.items():
            if name == "cfg1" and vname not in ("spx", "none"):
                continue
            args = ["tree", "--src", ps, "--trg", pt, "--leaf", leaf, "--out", base, "--lists", "--per", per,
                    "--ell", 2]
            if axes:
                args += ["--axes", axes]
            r = run(*args)
            out["hash"] = np.array(r["hash"], dtype=np.uint64)
            out["boxes"] = i32(base + ".boxes.i32").reshape(-1, 18)
            out["srcidx"] = i32(base + ".srcidx.i32")
            out["trgidx"] = i32(base + ".trgidx.i32")
            for lst in "uvwx":
                out[f"{vname}_{lst}_off"] = i32(f"{base}.{lst}.off.i32")
                out[f"{vname}_{lst}_ent"] = i32(f"{base}.{lst}.ent.i32").reshape(-1, 4)
        np.savez_compressed(os.path.join(HERE, f"tree_{name}.npz"), **out)
        print(name, hex(int(out["hash"])), out["boxes"].shape[0])


# evaluate cases: (name, kernel, per, axes, ell, p, leaf, n, op-spec)
EVAL_CASES = [
    ("lap_none_p6", "laplace", "none", "", 2, 6, 40, 2000, None),
    ("lap_sp_p8", "laplace", "sp", "", 2, 8, 40, 2000, "gated"),
    ("lap_spx_p8", "laplace", "sp", "x", 2, 8, 40, 2000, "spx"),
    ("lap_dp_p6", "laplace", "dp", "", 2, 6, 40, 2000, "gated"),
    ("lap_tp_p8", "laplace", "tp", "", 2, 8, 40, 2000, "ungated"),
    ("lap_tp_p6_ell1", "laplace", "tp", "", 1, 6, 40, 2000, "ungated"),
    ("sto_none_p6", "stokeslet", "none", "", 2, 6, 40, 2000, None),
    ("sto_tp_p6", "stokeslet", "tp", "", 2, 6, 40, 2000, "gated"),
    ("sto_tp_p8", "stokeslet", "tp", "", 2, 8, 40, 2000, "gated"),
    ("sto_dp_p6", "stokeslet", "dp", "", 2, 6, 40, 2000, "standin"),
    ("cfg1", "laplace", "sp", "x", 2, 8, 50, 20000, "spx"),
]


# adaptive evaluate cases: clustered sources (deep, graded octrees with W and X lists),
# (name, kernel, per, axes, ell, p, leaf, n, op-spec, nclusters, sigma)
EVAL_ADAPTIVE = [
    ("lap_none_p6_clu", "laplace", "none", "", 2, 6, 30, 4000, None, 4, 0.02),
    ("lap_sp_p8_clu", "laplace", "sp", "", 2, 8, 30, 4000, "gated", 4, 0.02),
    ("lap_dp_p6_clu", "laplace", "dp", "", 2, 6, 30, 4000, "gated", 3, 0.03),
    ("sto_tp_p6_clu", "stokeslet", "tp", "", 2, 6, 30, 4000, "gated", 4, 0.02),
]


# p = 10 (K = 1464 for Stokes: BASELINE cfg3 / cfg5's order), ~4k points each
EVAL_P10 = [
    ("sto_tp_p10", "stokeslet", "tp", "", 2, 10, 40, 4000, "gated"),
    ("sto_tp_p10_clu", "stokeslet", "tp", "", 2, 10, 30, 4000, "gated", 4, 0.02),
    ("sto_dp_p10_clu", "stokeslet", "dp", "", 2, 10, 30, 4000, "standin", 8, 0.04),
]


def op_path(kernel, per, axes, ell, p, kind):
    tag = f"{kernel}_{per}{axes}_ell{ell}_p{p}_{kind}.pkm2l"
    return os.path.join(OPS, tag)


def make_op(kernel, per, axes, ell, p, kind):
    os.makedirs(OPS, exist_ok=True)
    path = op_path(kernel, per, axes, ell, p, kind)
    if os.path.exists(path):
        return path
    if kind == "standin":  # DP Stokes has no K^P: relabelled TP operator (SURVEY §8c cfg 3)
        return make_op(kernel, "tp", "", ell, p, "gated")
    args = ["precompute", "--kernel", kernel, "--per", per, "--ell", ell, "--p", p, "--out", path]
    if kind == "ungated":
        args.append("--ungated")
    if kind == "spx":
        args.append("--spx")
    r = run(*args)
    print("operator", os.path.basename(path), r)
    return path


def golden_eval(tmp, cases=None, transform=None):
    for case in cases or EVAL_CASES:
        (name, kernel, per, axes, ell, p, leaf, n, opk), extra = case[:9], case[9:11]
        ks = 1 if kernel == "laplace" else 3
        gaxes = {"none": "xyz", "sp": axes or "z", "dp": "xy", "tp": "xyz"}[per]
        if extra:
            src, rho = gen(tmp, "e", n, kind="clusters", ks=ks, seed=2000 + n + len(name), axes=gaxes,
                           nclusters=extra[0], sigma=extra[1])
        else:
            src, rho = gen(tmp, "e", n, kind="uniform", ks=ks, seed=1000 + n + len(name), axes=gaxes)
        if transform:
            rho = transform(case, rho)
        ps, pr = save_pts(tmp, "es", src), save_pts(tmp, "er", rho)
        args = ["eval", "--kernel", kernel, "--per", per, "--ell", ell, "--p", p, "--leaf", leaf, "--src", ps,
                "--str", pr, "--out", os.path.join(tmp, "ev")]
        if axes:
            args += ["--axes", axes]
        op = None
        if opk:
            op = make_op(kernel, per, axes, ell, p, opk)
            args += ["--op", op]
            if opk in ("standin", "spx"):
                args.append("--relabel")
        out = {"src": src, "str": rho}
        res = {}
        for th in (1, 8):
            r = run(*args, "--threads", th)
            res[th] = (f64(os.path.join(tmp, "ev.pot.f64")), f64(os.path.join(tmp, "ev.phiup0.f64")))
        out["pot"], out["phiup0"] = res[8]
        out["pot_1thread"] = res[1][0]
        d = res[8][0] - res[1][0]
        spread = float(np.linalg.norm(d) / np.linalg.norm(res[8][0]))
        out["self_spread"] = np.array(spread)
        meta = dict(kernel=kernel, per=per, axes=axes, ell=ell, p=p, leaf=leaf,
                    op=os.path.basename(op) if op else "", relabel=opk in ("standin", "spx"))
        out["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(os.path.join(HERE, f"eval_{name}.npz"), **out)
        print(name, "spread", spread)


def golden_eval_adaptive(tmp):
    golden_eval(tmp, EVAL_ADAPTIVE)


# dynamic range of the strengths (the int8 M2L's fixed point is relative to each level's
# max |phi|): two clusters, each made neutral on its own, cluster 0 scaled down by `scale`
# (name, kernel, per, axes, ell, p, leaf, n, op-spec, nclusters, sigma, scale)
EVAL_DYN = [
    ("lap_sp_p8_dyn", "laplace", "sp", "", 2, 8, 30, 4000, "gated", 2, 0.03, 1e-6),
    ("sto_tp_p8_dyn", "stokeslet", "tp", "", 2, 8, 30, 4000, "gated", 2, 0.03, 1e-8),
]


def dyn_strengths(case, rho):
    ks = 1 if case[1] == "laplace" else 3
    ncl, scale = case[9], case[11]
    r = rho.reshape(-1, ks).copy()
    member = np.arange(r.shape[0]) % ncl  # point i belongs to cluster i mod K
    for k in range(ncl):
        r[member == k] -= r[member == k].mean(axis=0)
    r[member == 0] *= scale
    return r.reshape(-1)


def golden_eval_dyn(tmp):
    golden_eval(tmp, [c[:11] + (c[11],) for c in EVAL_DYN], transform=dyn_strengths)


def golden_eval_p10(tmp):
    golden_eval(tmp, EVAL_P10)


def golden_direct(tmp):
    """Direct mode (madelung configuration, src/experiments.cpp:461-465) + error paths."""
    src = np.array([[0.5, 0.5, 0.125], [0.5, 0.5, 0.375], [0.5, 0.5, 0.625], [0.5, 0.5, 0.875]])
    q = np.array([1.0, -1.0, 1.0, -1.0])
    trg = src[[0, 2]]
    op = make_op("laplace", "sp", "", 2, 8, "gated")
    ps, pr, pt = save_pts(tmp, "ds", src), save_pts(tmp, "dq", q), save_pts(tmp, "dt", trg)
    out = {}
    for mode in ("direct", "fmm"):
        run("eval", "--kernel", "laplace", "--per", "sp", "--ell", 2, "--p", 8, "--leaf", 1000, "--src", ps,
            "--str", pr, "--trg", pt, "--op", op, "--mode", mode, "--out", os.path.join(tmp, "dv"))
        out[f"{mode}_pot"] = f64(os.path.join(tmp, "dv.pot.f64"))
    out["src"], out["str"], out["trg"] = src, q, trg
    # error paths
    errs = {}
    bad = src.copy()
    bad[1] = [1.0, 0.5, 0.5]
    bad[2] = [-0.25, 0.5, 2.5]
    errs["outside"] = run("eval", "--kernel", "laplace", "--per", "sp", "--p", 8, "--src", save_pts(tmp, "b1", bad),
                          "--str", pr, "--op", op, ok_codes=(3,))
    errs["compat"] = run("eval", "--kernel", "laplace", "--per", "sp", "--p", 8, "--src", ps,
                         "--str", save_pts(tmp, "b2", np.array([1.0, 1.0, 1.0, -1.0])), "--op", op, ok_codes=(3,))
    errs["strlen"] = run("eval", "--kernel", "laplace", "--per", "sp", "--p", 8, "--src", ps,
                         "--str", save_pts(tmp, "b3", np.array([1.0, -1.0])), "--op", op, ok_codes=(3,))
    errs["provenance"] = run("eval", "--kernel", "laplace", "--per", "sp", "--p", 6, "--src", ps, "--str", pr,
                             "--op", op, ok_codes=(3,))
    errs["noop"] = run("eval", "--kernel", "laplace", "--per", "sp", "--p", 8, "--src", ps, "--str", pr,
                       ok_codes=(3,))
    out["errors"] = np.array(json.dumps(errs))
    np.savez_compressed(os.path.join(HERE, "direct_and_errors.npz"), **out)


def golden_kblock(tmp):
    """kernel_block (src/kernel.cpp:54-78) on the KIFMM surfaces: a_up, a_dn, canonical
    M2L class matrices and image-offset blocks, for bit-exact operator assembly checks."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pkifmm_oracle as O
    out = {}
    for kernel, plist in (("laplace", (4, 6)), ("stokeslet", (4,))):
        for p in plist:
            inner = O.surface_points(p, (0.5, 0.5, 0.5), 1.05)
            outer = O.surface_points(p, (0.5, 0.5, 0.5), 2.95)
            pairs = {"a_up": (outer, inner), "a_dn": (inner, outer)}
            for d in ((3, 1, 0), (2, 2, 2), (3, 3, 1), (2, 0, 0)):
                pairs["cls_%d%d%d" % d] = (inner, inner + np.array(d, dtype=float))
            for o in (0, 5):
                c = np.array([0.5 + (0.25 if o & 1 else -0.25), 0.5 + (0.25 if o & 2 else -0.25),
                              0.5 + (0.25 if o & 4 else -0.25)])
                ci = O.surface_points(p, c, 0.5 * 1.05)
                pairs[f"m2m_{o}"] = (outer, ci)
                pairs[f"l2l_{o}"] = (ci, outer)
            for tag, (trg, src) in pairs.items():
                pt, ps = save_pts(tmp, "kt", trg), save_pts(tmp, "ks", src)
                r = run("kblock", "--kernel", kernel, "--trg", pt, "--src", ps, "--out", os.path.join(tmp, "kb"))
                out[f"{kernel}_p{p}_{tag}"] = f64(os.path.join(tmp, "kb.kb.f64")).reshape(r["rows"], r["cols"])
    np.savez_compressed(os.path.join(HERE, "kblock.npz"), **out)


def main():
    if not os.path.exists(REFDUMP):
        sys.exit("build oracle/_ref first: make -C oracle/refbuild")
    only = sys.argv[1:]
    with tempfile.TemporaryDirectory() as tmp:
        if only:
            for name in only:
                globals()["golden_" + name](tmp)
            return
        golden_kblock(tmp)
        golden_pairs(tmp)
        golden_surfaces(tmp)
        golden_trees(tmp)
        golden_direct(tmp)
        golden_eval(tmp)
        golden_eval_adaptive(tmp)
        golden_eval_p10(tmp)
        golden_eval_dyn(tmp)


if __name__ == "__main__":
    main()
