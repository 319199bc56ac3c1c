"""Full-size parity fixtures for BASELINE cfg3 and cfg4 (SURVEY §8c protocol), made by
running the UNMODIFIED reference (oracle/_ref/refdump, built from /root/reference) once at
full size in the build container and keeping a strided sample of its output.

    python tests/golden/make_fullsize.py [cfg3] [cfg4]

Inputs are the seeded SURVEY §8(d) workloads (refdump gen == pk.generate bit for bit;
the GPU test regenerates them and checks a fingerprint). Each fixture
tests/golden/full_<cfg>.npz holds
  idx      65,536 strided target indices (stride N / 65,536)
  pot      the reference's potentials at those targets (kt per target), 8 threads
  spread   rel-L2 between the 8-thread and 4-thread reference runs on the sample (the
           reference's own reduction-order spread; the bar is 10 x spread)
  phiup0   the reference's root upward density
  hash     the reference's structure_hash of the tree
  fp       fingerprint of the inputs (sum of coordinates and strengths)
  meta     the configuration (json)
cfg3 (Stokes DP p = 10) runs with the stand-in operator (the TP Stokes p = 10 operator
relabelled DP); cfg4 (Laplace TP p = 8) with the ungated operator.
"""
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REFDUMP = os.path.join(REPO, "oracle", "_ref", "refdump")
OPS = os.path.join(HERE, "ops")
NSAMPLE = 65536

CFGS = {
    "cfg3": dict(kernel="stokeslet", per="dp", n=1_000_000, p=10, leaf=64, kind="clusters", nclusters=8, sigma=0.04,
                 ks=3, axes="xy", op="stokeslet_tp_ell2_p10_gated.pkm2l", relabel=True),
    "cfg4": dict(kernel="laplace", per="tp", n=8_000_000, p=8, leaf=64, kind="uniform", nclusters=8, sigma=0.04,
                 ks=1, axes="xyz", op="laplace_tp_ell2_p8_ungated.pkm2l", relabel=False),
}


def refdump(*args, threads=8):
    env = dict(os.environ, OMP_NUM_THREADS=str(threads), OPENBLAS_NUM_THREADS=str(threads))
    r = subprocess.run([REFDUMP, *map(str, args)], capture_output=True, text=True, env=env)
    if r.returncode != 0:
        raise RuntimeError(f"refdump {args} failed: {r.stdout} {r.stderr}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def make(name):
    c = CFGS[name]
    kt = c["ks"]
    with tempfile.TemporaryDirectory() as tmp:
        base = os.path.join(tmp, name)
        refdump("gen", "--n", c["n"], "--kind", c["kind"], "--ks", c["ks"], "--seed", 12345, "--nclusters",
                c["nclusters"], "--sigma", c["sigma"], "--axes", c["axes"], "--out", base)
        pts = np.fromfile(base + ".src.f64")
        q = np.fromfile(base + ".str.f64")
        tree = refdump("tree", "--src", base + ".src.f64", "--leaf", c["leaf"])
        stride = c["n"] // NSAMPLE
        idx = np.arange(NSAMPLE, dtype=np.int64) * stride
        pots, walls = {}, {}
        for th in (8, 4):
            args = ["eval", "--kernel", c["kernel"], "--per", c["per"], "--ell", 2, "--p", c["p"], "--leaf", c["leaf"],
                    "--src", base + ".src.f64", "--str", base + ".str.f64", "--op", os.path.join(OPS, c["op"]),
                    "--threads", th, "--out", base]
            if c["relabel"]:
                args.append("--relabel")
            t0 = time.time()
            r = refdump(*args, threads=th)
            walls[th] = time.time() - t0
            pot = np.fromfile(base + ".pot.f64").reshape(-1, kt)
            pots[th] = pot[idx].reshape(-1)
            if th == 8:
                phiup0 = np.fromfile(base + ".phiup0.f64")
            print(name, th, "threads", r["runs"][0], f"wall {walls[th]:.1f} s", file=sys.stderr, flush=True)
        spread = float(np.linalg.norm(pots[8] - pots[4]) / np.linalg.norm(pots[8]))
    out = dict(idx=idx, pot=pots[8], spread=np.array(spread), phiup0=phiup0, hash=np.array(int(tree["hash"]),
               dtype=np.uint64), fp=np.array([pts.sum(), q.sum()]), meta=np.array(json.dumps(
                   dict(c, boxes=tree["boxes"], leaves=tree["leaves"], depth=tree["depth"], wall_s=walls))))
    np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), **out)
    print(name, "spread", spread, "hash", hex(int(tree["hash"])), file=sys.stderr)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CFGS):
        make(nm)
