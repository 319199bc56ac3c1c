"""Print one evaluate of a tools/timeline.py --json dump as a launch sequence
(start, duration, name, idle gap before it): python tools/timeline_seq.py dump.json [index]"""
import json
import re
import sys

d = json.load(open(sys.argv[1]))
which = int(sys.argv[2]) if len(sys.argv) > 2 else -1
ops = d["ops_list"]
steps, cur, end = [], [], None
for o in ops:
    if cur and o["ts"] - end > 100:
        steps.append(cur)
        cur = []
    cur.append(o)
    end = max(end or 0, o["ts"] + o["dur"])
steps.append(cur)
ev = steps[which]
t0, end, tot = ev[0]["ts"], 0, 0
for o in ev:
    gap = o["ts"] - end if end else 0
    nm = re.sub(r"pkgpu::\(anonymous namespace\)::|pkgpu::|void |cub::CUB_\d+_SM_\d+::", "", o["name"])[:48]
    if gap > 0:
        tot += gap
    print(f"{o['ts'] - t0:8.1f} {o['dur']:7.1f} {nm}" + (f"  <-- idle {gap:.1f}" if gap > 1.5 else ""))
    end = max(end, o["ts"] + o["dur"])
print(f"span {end - t0:.1f} us, idle {tot:.1f} us")
