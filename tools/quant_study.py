"""M2L arithmetic study: evaluate the golden cases and full-size cfg2 under several M2L
paths and report rel-L2 against the reference next to each case's tolerance.

Specs (';'-separated):
  dmma              FP64 DMMA everywhere
  i8:NM,BA,BB       int8 residue path (NM moduli) on levels >= 2048 boxes (the default)
  i8all:NM,BA,BB    int8 residue path on every level >= 1

    python tools/quant_study.py --specs "dmma;i8:17,56,56;i8all:16,52,52"   (GPU box; oracle/_ref prebuilt)
"""
import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, os.path.join(REPO, "oracle"))


def child(spec):
    import numpy as np

    import paper_1705_02043_b200 as pk
    from test_gpu_parity import EVAL_ALL, golden_request, load

    ctx = pk.Context(0)
    kind, _, args = spec.partition(":")
    if kind == "dmma":
        ctx.set_m2l("dmma")
    elif kind in ("i8", "i8all"):
        nm, ba, bb = (int(v) for v in args.split(","))
        ctx.set_m2l("int8", min_boxes=1 if kind == "i8all" else 2048, nmod=nm, beta_a=ba, beta_b=bb)
    out = {}
    for name in EVAL_ALL:
        g = load(f"eval_{name}.npz")
        req, meta = golden_request(g)
        res = pk.evaluate(req, context=ctx)
        rel = float(np.linalg.norm(res.potentials - g["pot"]) / np.linalg.norm(g["pot"]))
        out[name] = (rel, max(1e-10, 10 * float(g["self_spread"])))
    ref = np.load("/tmp/quant_c2.npz")
    req = pk.EvalRequest(kernel=pk.KernelSpec.stokeslet(), sources=ref["pts"], strengths=ref["f"], targets=ref["pts"],
                         setup=pk.PeriodicSetup.make(pk.Periodicity.tp), p=8,
                         op=pk.load_operator(os.path.join(REPO, "tests", "golden", "ops",
                                                          "stokeslet_tp_ell2_p8_gated.pkm2l")), leaf_capacity=50)
    res = pk.evaluate(req, context=ctx)
    out["cfg2_full"] = (float(np.linalg.norm(res.potentials - ref["pot"]) / np.linalg.norm(ref["pot"])), 1.4e-7)
    worst = max(v[0] / v[1] for v in out.values())
    print(json.dumps({"spec": spec, "worst_frac_of_tol": worst, "cases": out}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--specs", default="dmma;i8:17,56,56")
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child is not None:
        return child(a.child)
    import numpy as np

    refdump = os.path.join(REPO, "oracle", "_ref", "refdump")
    base = "/tmp/quant_c2"
    subprocess.run([refdump, "gen", "--n", "100000", "--kind", "uniform", "--ks", "3", "--seed", "12345", "--out", base],
                   check=True, capture_output=True)
    subprocess.run([refdump, "eval", "--kernel", "stokeslet", "--per", "tp", "--ell", "2", "--p", "8", "--leaf", "50",
                    "--src", base + ".src.f64", "--str", base + ".str.f64", "--op",
                    os.path.join(REPO, "tests", "golden", "ops", "stokeslet_tp_ell2_p8_gated.pkm2l"), "--out", base],
                   check=True, capture_output=True)
    np.savez("/tmp/quant_c2.npz", pts=np.fromfile(base + ".src.f64").reshape(-1, 3), f=np.fromfile(base + ".str.f64"),
             pot=np.fromfile(base + ".pot.f64"))
    for spec in a.specs.split(";"):
        env = dict(os.environ)
        r = subprocess.run([sys.executable, __file__, "--child", spec], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or (spec + " FAILED: " + r.stderr[-3000:]), flush=True)


if __name__ == "__main__":
    main()
