"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel name.

    python tools/launch_agg.py LOG.csv [--seq]   (--seq: also print the launch sequence)
"""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    out = []
    for x in csv.DictReader(lines):
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(x["Metric Value"].replace(",", ""))
        u = x["Metric Unit"]
        v = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
        out.append((x["Kernel Name"].split("(")[0].replace("pkgpu::<unnamed>::", "").replace("void ", "")[:70], v))
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    agg = collections.OrderedDict()
    for n, v in seq:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v for _, v in seq)
    print(f"| kernel | launches | ms | share |\n|---|---|---|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{n}` | {c} | {t:.3f} | {100 * t / tot:.1f}% |")
    print(f"| total | {len(seq)} | {tot:.3f} | |")
    if "--seq" in sys.argv:
        for n, v in seq:
            print(f"{v:8.4f}  {n}")
