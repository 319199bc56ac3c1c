"""Print the per-launch sequence (name, grid, duration) of an ncu --csv launch list,
last N launches (one evaluate), for comparing schedules launch by launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 140
hdr, out = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        out.append(dict(zip(hdr, r)))
for d in out[-n:]:
    print(f"{d['ID']:>5} {d['Kernel Name'][:44]:44} {d['Grid Size']:>14} {float(d['Metric Value'])/1000:9.1f} us")
