"""GPU timeline of one evaluate (CUPTI through torch.profiler): every kernel / memcpy /
memset of the library with its start and end, and the idle gaps between them, attributed
to the operation that follows the gap. Shows where host synchronisation leaves the GPU
idle inside a step.

    python tools/timeline.py --cfg 2 [--evals 3] [--top 30] [--json out.json]
"""
import argparse
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from run_config import request_for  # noqa: E402

import paper_1705_02043_b200 as pk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--evals", type=int, default=3)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--json", default=None)
    ap.add_argument("--profiling", action="store_true", help="stage profiler on (everything on the work stream)")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    ctx = pk.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    req, pts, q = request_for(a.cfg)
    out = torch.empty(req.kernel.kt * len(pts), dtype=torch.float64, device="cuda")
    ctx.set_profiling(a.profiling)
    for _ in range(3):
        pk.evaluate(req, context=ctx, out=out)
    torch.cuda.synchronize()
    marks = []
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(a.evals):
            torch.cuda.synchronize()
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            pk.evaluate(req, context=ctx, out=out)
            e.record()
            torch.cuda.synchronize()
            marks.append(s.elapsed_time(e))
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    tr = json.load(open(path))
    evs = tr["traceEvents"] if isinstance(tr, dict) else tr
    gpu = [e for e in evs if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    gpu.sort(key=lambda e: e["ts"])
    cpu_sync = [e for e in evs if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"
                and "Synchronize" in e.get("name", "")]
    # split into evaluates at gaps > 1 ms (the host synchronize between evaluates)
    steps, cur = [], []
    for e in gpu:
        if cur and e["ts"] - (cur[-1]["ts"] + cur[-1]["dur"]) > 1000:
            steps.append(cur)
            cur = []
        cur.append(e)
    if cur:
        steps.append(cur)
    step = steps[-1]
    t0 = step[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in step)
    busy = 0.0
    last_end = t0
    gaps = []
    for e in step:
        if e["ts"] > last_end:
            gaps.append((e["ts"] - last_end, e["name"][:70], e["ts"] - t0))
        busy += max(0.0, e["ts"] + e["dur"] - max(e["ts"], last_end))
        last_end = max(last_end, e["ts"] + e["dur"])
    span = t1 - t0
    nsync = sum(1 for c in cpu_sync if t0 <= c["ts"] <= t1)
    gaps.sort(reverse=True)
    res = dict(cfg=a.cfg, event_ms=marks, span_us=span, busy_us=busy, idle_us=span - busy, ops=len(step),
               host_syncs=nsync, gaps_over_2us=sum(1 for g in gaps if g[0] > 2),
               top_gaps=[dict(us=round(g[0], 1), before=g[1], at_us=round(g[2], 1)) for g in gaps[:a.top]])
    print(json.dumps(res, indent=1))
    if a.json:
        json.dump(dict(res, ops_list=[dict(name=e["name"][:80], ts=e["ts"] - t0, dur=e["dur"]) for e in step]),
                  open(a.json, "w"))


if __name__ == "__main__":
    main()
