"""M2L tile over-issue under column orderings (analysis tool, runs where a GPU builds the tree).

For one BASELINE config, exports the V lists and counts, per level, the MMA rows the int8
pair-dual kernel issues (512-box quads, per slot: MMA half h = 256 columns issued when either
of its 128-column quarters has a source) against the V-list applications, for
  morton : octant groups in Morton order (the current layout)
  count  : within each octant group, boxes sorted by V-list size (descending), then Morton
  lex    : within each octant group, boxes sorted by the V-slot bitmask (lexicographic)

    python tools/sim_m2l_layout.py --cfg 3
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import paper_1705_02043_b200 as pk  # noqa: E402
from run_config import CONFIGS  # noqa: E402


def slot_of(d):
    return (d[:, 0] + 3) * 49 + (d[:, 1] + 3) * 7 + (d[:, 2] + 3)


def issued_rows(order, S):
    """S: [nbox, 343] bool slot masks in column order `order` (octant groups padded to 64)."""
    cols = S[order]
    n = len(order)
    pad = (-n) % 512
    cols = np.concatenate([cols, np.zeros((pad, S.shape[1]), dtype=bool)])
    q = cols.reshape(-1, 4, 128, S.shape[1]).any(axis=2)  # [quad, quarter, slot]
    halves = q[:, 0::2] | q[:, 1::2]  # MMA h covers quarters 2h, 2h + 1
    return int(halves.sum()) * 256


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=3)
    a = ap.parse_args()
    c = CONFIGS[a.cfg]
    k = pk.KernelSpec.from_name(c["kernel"])
    setup = pk.PeriodicSetup.make(pk.Periodicity.from_name(c["per"]))
    if c["axes"]:
        setup.axes = c["axes"]
    pts, _ = pk.generate(c["kind"], c["n"], k.ks, seed=12345, nclusters=c.get("nclusters", 8),
                         sigma=c.get("sigma", 0.04), periodic_axes=setup.axes)
    t = pk.FmmTree(pts, pts, c["leaf"])
    table, _, _ = t.boxes()
    off, ent = t.lists(setup, "v")
    lev = table[:, 0]
    oct_ = (table[:, 1] & 1) | ((table[:, 2] & 1) << 1) | ((table[:, 3] & 1) << 2)
    nb = len(table)
    tgt = np.repeat(np.arange(nb), np.diff(off))
    out = {}
    tot = {"apps": 0, "morton": 0, "count": 0, "lex": 0}
    for l in range(1, lev.max() + 1):
        bl = np.nonzero(lev == l)[0]
        if len(bl) < 1024:
            continue
        sel = (tgt >= bl[0]) & (tgt <= bl[-1])
        S = np.zeros((len(bl), 343), dtype=bool)
        S[tgt[sel] - bl[0], slot_of(ent[sel, 1:4])] = True
        apps = int(sel.sum())
        res = {"boxes": len(bl), "apps": apps}
        for name in ("morton", "count", "lex"):
            order = []
            for o in range(8):
                g = np.nonzero(oct_[bl] == o)[0]
                if name == "count":
                    g = g[np.argsort(-S[g].sum(axis=1), kind="stable")]
                elif name == "lex":
                    packed = np.packbits(S[g], axis=1)
                    keys = [packed[:, i] for i in range(packed.shape[1] - 1, -1, -1)]
                    g = g[np.lexsort(keys)[::-1]]
                order.extend(g.tolist())
                order.extend([-1] * ((-len(g)) % 64))
            order = np.array(order)
            Sx = np.vstack([S, np.zeros((1, 343), dtype=bool)])
            rows = issued_rows(np.where(order >= 0, order, len(bl)), Sx)
            res[name] = rows / apps
            tot[name] += rows
        tot["apps"] += apps
        out[l] = res
        print(l, json.dumps(res), flush=True)
    print("total", {k: (v / tot["apps"] if k != "apps" else v) for k, v in tot.items()})


if __name__ == "__main__":
    main()
