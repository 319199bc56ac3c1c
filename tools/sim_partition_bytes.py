"""Bytes moved per rank by the partitioned evaluate, from the real trees and
lists of the BASELINE configs (analysis tool; runs where a GPU builds the tree).

Ranks own contiguous Morton (DFS) ranges of leaves, equal leaf counts (as
pkgpu_evaluate_partitioned). Per rank and evaluate:
  v1   : one allreduce of every box's equivalent density (nb x Kp doubles; ring allreduce
         moves 2 (N - 1) / N of the buffer per rank) -- round 1's scheme
  strad: allreduce of the straddling boxes only (boxes whose leaves span several ranks)
  halo : equivalent densities the rank RECEIVES point to point -- V / W sources of its
         target boxes owned by another rank (alltoallv)
  out  : the final potentials (every rank returns all of them: ring allreduce of kt x nt)
  small: the small-level int8 run split by modulus (each rank 16 / N moduli), residue sums
         exchanged by allgather (int32)

    python tools/sim_partition_bytes.py --cfg 2 4 5
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

KP = {(0, 8): 320, (1, 8): 896, (1, 10): 1472}
KI = {(0, 8): 384, (1, 8): 896, (1, 10): 1536}


def morton(cx, cy, cz, level):
    key = np.zeros(len(cx), dtype=np.uint64)
    for b in range(12):
        for a, c in enumerate((cx, cy, cz)):
            key |= (((c.astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a))
    return key << (np.uint64(3) * (np.uint64(12) - level.astype(np.uint64)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="+", default=[2, 4, 5])
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    a = ap.parse_args()
    for cfg in a.cfg:
        c = CONFIGS[cfg]
        k = pk.KernelSpec.from_name(c["kernel"])
        setup = pk.PeriodicSetup.make(pk.Periodicity.from_name(c["per"]))
        if c["axes"]:
            setup.axes = c["axes"]
        pts, _ = pk.generate(c["kind"], c["n"], k.ks, seed=12345, nclusters=c.get("nclusters", 8),
                             sigma=c.get("sigma", 0.04), periodic_axes=setup.axes)
        t = pk.FmmTree(pts, pts, c["leaf"])
        table, _, _ = t.boxes()
        nb = len(table)
        lev, cx, cy, cz, leaf = (table[:, i] for i in (0, 1, 2, 3, 5))
        kp, ki = KP[(int(k.type), c["p"])], KI[(int(k.type), c["p"])]
        key0 = morton(cx, cy, cz, lev)
        key1 = key0 + (np.uint64(1) << (np.uint64(3) * (np.uint64(12) - lev.astype(np.uint64))))
        lk = np.sort(key0[leaf == 1])
        nl = len(lk)
        la, lc = np.searchsorted(lk, key0), np.searchsorted(lk, key1)  # leaf interval of each box
        src, tgt = [], []
        for lst in "vw":
            off, ent = t.lists(setup, lst)
            tgt.append(np.repeat(np.arange(nb, dtype=np.int64), np.diff(off)))
            src.append(ent[:, 0].astype(np.int64))
        src, tgt = np.concatenate(src), np.concatenate(tgt)
        small = [l for l in range(1, lev.max() + 1) if (lev == l).sum() <= 1024]
        small_cols = sum(((lev == l).sum() + 255) // 256 * 256 for l in small)
        res = {"cfg": cfg, "boxes": nb, "leaves": nl, "Kp": kp, "vw_entries": int(len(src))}
        for n in a.ranks:
            lo = (np.arange(n + 1) * nl) // n
            rank_of_leaf = lambda i: np.searchsorted(lo, i, side="right") - 1  # noqa: E731
            rlo, rhi = rank_of_leaf(la), rank_of_leaf(lc - 1)
            strad = rlo != rhi
            halo = []
            for r in range(n):
                m = (rlo[tgt] <= r) & (rhi[tgt] >= r) & ~strad[src] & (rlo[src] != r)
                halo.append(len(np.unique(src[m])))
            row = 8 * kp
            res[f"N{n}"] = {
                "v1_allreduce_MB": 2 * (n - 1) / n * nb * row / 1e6,
                "straddlers": int(strad.sum()),
                "strad_allreduce_MB": 2 * (n - 1) / n * int(strad.sum()) * row / 1e6,
                "halo_recv_boxes_max": int(max(halo)),
                "halo_recv_MB_max": max(halo) * row / 1e6,
                "out_allreduce_MB": 2 * (n - 1) / n * c["n"] * k.kt * 8 / 1e6,
                "small_run_cols": int(small_cols),
                "small_allgather_MB": (n - 1) / n * 16 * small_cols * ki * 4 / 1e6,
            }
        print(json.dumps(res), flush=True)
        del t


if __name__ == "__main__":
    main()
