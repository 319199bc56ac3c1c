"""Print per-launch durations (ms) from an `ncu --metrics gpu__time_duration.sum --csv` log."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
if not rows:
    print("no launches")
    sys.exit(0)
h = rows[0]
vi, ki = h.index("Metric Value"), h.index("Kernel Name")
short = len(sys.argv) > 2
for r in rows[1:]:
    ms = float(r[vi].replace(",", "")) / 1e6
    print(f"{ms:.3f}" if not short else f"{r[ki][:40]} {ms:.3f}", end="\n" if short else " ")
print()
