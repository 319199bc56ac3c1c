"""Evaluate one BASELINE config with several M2L paths (device-resident, warm) and print
the per-evaluate and M2L-stage times, plus each path's difference from the first.

    python tools/m2l_compare.py --cfg 3 --paths int8 fft [--evals 2] [--profile-one PATH]

--profile-one PATH: one extra evaluate of PATH between cudaProfilerStart / Stop (for
`ncu --profile-from-start off`)."""
import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import torch  # noqa: E402

import paper_1705_02043_b200 as pk  # noqa: E402
from run_config import request_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, required=True)
    ap.add_argument("--paths", nargs="+", default=["int8", "fft"])
    ap.add_argument("--evals", type=int, default=2)
    ap.add_argument("--profile-one", default=None)
    a = ap.parse_args()
    req, pts, _ = request_for(a.cfg)
    ref = None
    for path in a.paths:
        ctx = pk.Context(0)
        ctx.set_m2l(path)
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        out = torch.empty(req.kernel.kt * len(pts), dtype=torch.float64, device="cuda")
        pk.evaluate(req, context=ctx, out=out)
        torch.cuda.synchronize()
        if a.profile_one == path:
            torch.cuda.cudart().cudaProfilerStart()
            pk.evaluate(req, context=ctx, out=out)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            continue
        ctx.set_profiling(True)
        ctx.reset_stats()
        t0 = time.time()
        for _ in range(a.evals):
            pk.evaluate(req, context=ctx, out=out)
        torch.cuda.synchronize()
        dt = (time.time() - t0) / a.evals
        st = ctx.stage_stats()
        line = f"cfg{a.cfg} {path}: {dt * 1e3:.1f} ms/eval, M2L {1e3 * st['m2l']['seconds'] / a.evals:.1f} ms"
        if ref is None:
            ref = out.clone()
        else:
            line += f", rel-L2 vs {a.paths[0]} {float(torch.linalg.norm(out - ref) / torch.linalg.norm(ref)):.2e}"
        print(line, flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
