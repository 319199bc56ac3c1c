"""Run a BASELINE.json config through the GPU evaluate path (device-resident inputs).

    python tools/run_config.py --cfg {1..5} [--n N] [--evals E] [--stats] [--save out.npz]

Inputs follow the SURVEY §8(d) protocol (pk.generate, mt19937_64 seed 12345). Operators:
  cfg1 Laplace SP-x p8  tests/golden/ops/laplace_spx_ell2_p8_spx.pkm2l (permuted SP-z, §8c)
  cfg2 Stokes TP p8     tests/golden/ops/stokeslet_tp_ell2_p8_gated.pkm2l
  cfg3 Stokes DP p10    tests/golden/ops/stokeslet_tp_ell2_p10_gated.pkm2l relabelled DP (stand-in, §8c)
  cfg4 Laplace TP p8    tests/golden/ops/laplace_tp_ell2_p8_ungated.pkm2l (ungated, §8c)
  cfg5 Stokes TP p10    tests/golden/ops/stokeslet_tp_ell2_p10_gated.pkm2l
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import paper_1705_02043_b200 as pk  # noqa: E402

G = os.path.join(REPO, "tests", "golden", "ops")
O = os.path.join(REPO, "operators")
CONFIGS = {
    1: dict(kernel="laplace", per="sp", axes=(True, False, False), n=20000, p=8, leaf=50, kind="uniform",
            op=os.path.join(G, "laplace_spx_ell2_p8_spx.pkm2l"), relabel=True),
    2: dict(kernel="stokeslet", per="tp", axes=None, n=100000, p=8, leaf=50, kind="uniform",
            op=os.path.join(G, "stokeslet_tp_ell2_p8_gated.pkm2l"), relabel=False),
    3: dict(kernel="stokeslet", per="dp", axes=None, n=1000000, p=10, leaf=64, kind="clusters", nclusters=8,
            sigma=0.04, op=os.path.join(G, "stokeslet_tp_ell2_p10_gated.pkm2l"), relabel=True),
    4: dict(kernel="laplace", per="tp", axes=None, n=8000000, p=8, leaf=64, kind="uniform",
            op=os.path.join(G, "laplace_tp_ell2_p8_ungated.pkm2l"), relabel=False),
    5: dict(kernel="stokeslet", per="tp", axes=None, n=32000000, p=10, leaf=64, kind="mixed", nclusters=64,
            sigma=0.02, op=os.path.join(G, "stokeslet_tp_ell2_p10_gated.pkm2l"), relabel=False),
}


def request_for(cfg, n=None, seed=12345, device=True):
    import torch

    c = dict(CONFIGS[cfg])
    n = n or c["n"]
    k = pk.KernelSpec.from_name(c["kernel"])
    setup = pk.PeriodicSetup.make(pk.Periodicity.from_name(c["per"]))
    if c["axes"]:
        setup.axes = c["axes"]
    pts, q = pk.generate(c["kind"], n, k.ks, seed=seed, nclusters=c.get("nclusters", 8), sigma=c.get("sigma", 0.04),
                         periodic_axes=setup.axes)
    op = pk.load_operator(c["op"])
    if c["relabel"]:
        op.relabel(k, setup)
    if device:
        dev = torch.device("cuda", 0)
        src = torch.from_numpy(pts).to(dev).reshape(-1).contiguous()
        qq = torch.from_numpy(q).to(dev)
    else:
        src, qq = pts, q
    req = pk.EvalRequest(kernel=k, sources=src, strengths=qq, targets=src, setup=setup, p=c["p"], op=op,
                         leaf_capacity=c["leaf"])
    return req, pts, q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, required=True)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--evals", type=int, default=1)
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--save", default=None)
    a = ap.parse_args()
    import torch

    ctx = pk.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    t0 = time.time()
    req, pts, q = request_for(a.cfg, a.n)
    t_gen = time.time() - t0
    tree = pk.FmmTree(pts, pts, req.leaf_capacity, context=ctx)
    info = dict(cfg=a.cfg, n=len(pts), boxes=tree.box_count(), leaves=tree.leaf_count(), depth=tree.depth(),
                hash=hex(tree.structure_hash()), gen_s=t_gen)
    del tree
    out = torch.empty(req.kernel.kt * len(pts), dtype=torch.float64, device="cuda")
    r = pk.evaluate(req, context=ctx, out=out)  # warm-up (operators, workspaces)
    torch.cuda.synchronize()
    ctx.set_profiling(a.stats)
    ctx.reset_stats()
    ev = []
    torch.cuda.cudart().cudaProfilerStart()  # `ncu --profile-from-start off` captures the timed evaluates
    for _ in range(a.evals):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = pk.evaluate(req, context=ctx, out=out)
        e.record()
        torch.cuda.synchronize()
        ev.append(s.elapsed_time(e))
    torch.cuda.cudart().cudaProfilerStop()
    info.update(ms_per_eval=float(np.mean(ev)), evals_per_s=len(pts) / (np.mean(ev) * 1e-3),
                timings=r.timings.__dict__, free_gb=torch.cuda.mem_get_info()[0] / 1e9,
                peak_alloc_gb=torch.cuda.max_memory_allocated() / 1e9)
    if a.stats:
        info["stages"] = {k: dict(ms=1e3 * v["seconds"] / a.evals,
                                  tflops=(v["flops"] / v["seconds"] / 1e12) if v["seconds"] and v["flops"] else None,
                                  units=v["units"] / a.evals)
                          for k, v in ctx.stage_stats().items()}
    print(json.dumps(info))
    if a.save:
        np.savez_compressed(a.save, pot=out.cpu().numpy(), pts=pts, q=q)


if __name__ == "__main__":
    main()
