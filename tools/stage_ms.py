"""Per-evaluate stage milliseconds from a run_cfg2.py --stats log: stage_ms.py LOG EVALS STAGE..."""
import ast
import sys

d = {}
for line in open(sys.argv[1]):
    k, _, v = line.partition(" ")
    if k in sys.argv[3:]:
        d[k] = round(ast.literal_eval(v)["seconds"] / int(sys.argv[2]) * 1e3, 3)
print(sys.argv[1], d, round(sum(d.values()), 3))
