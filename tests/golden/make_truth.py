"""Ground-truth fixtures for the SURVEY §8(c)(iii) accuracy check (run in the build
container, where /root/reference and oracle/_ref exist; the GPU box only reads the
committed npz).

For each golden evaluate case whose periodicity has a reference truth evaluator, the
reference's own `oracle_system_eval` (pairwise Ewald / direct sums, include/pkifmm/
refsum.hpp:88) is run through oracle/_ref/refdump at a stride sample of 64 targets and
stored with the sample stride:  tests/golden/truth_<case>.npz {truth, stride}.

    python tests/golden/make_truth.py
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REFDUMP = os.path.join(HERE, "..", "..", "oracle", "_ref", "refdump")
# cases with a periodic truth evaluator: Laplace SP/DP/TP, Stokes TP
# (Stokes DP has no K^P in the reference, src/refsum.cpp:620-622; cfg1 is SP-x)
CASES = ["lap_sp_p8", "lap_dp_p6", "lap_tp_p8", "sto_tp_p6", "sto_tp_p8", "lap_sp_p8_clu", "lap_dp_p6_clu",
         "sto_tp_p6_clu", "sto_tp_p10", "sto_tp_p10_clu"]


def main():
    for case in sys.argv[1:] or CASES:
        g = np.load(os.path.join(HERE, f"eval_{case}.npz"))
        meta = json.loads(str(g["meta"]))
        with tempfile.TemporaryDirectory() as tmp:
            base = os.path.join(tmp, "c")
            g["src"].astype(np.float64).tofile(base + ".src.f64")
            g["str"].astype(np.float64).tofile(base + ".str.f64")
            args = [REFDUMP, "truth", "--kernel", meta["kernel"], "--per", meta["per"], "--ell", str(meta["ell"]),
                    "--src", base + ".src.f64", "--str", base + ".str.f64", "--ntrg", "64", "--out", base]
            if meta["axes"]:
                args += ["--axes", meta["axes"]]
            r = subprocess.run(args, check=True, capture_output=True, text=True)
            info = json.loads(r.stdout.strip().splitlines()[-1])
            truth = np.fromfile(base + ".truth.f64")
        np.savez(os.path.join(HERE, f"truth_{case}.npz"), truth=truth, stride=info["stride"])
        print(case, info, file=sys.stderr)


if __name__ == "__main__":
    main()
