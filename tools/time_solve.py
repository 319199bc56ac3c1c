"""Time the GPU periodizing-operator precompute (solve_m2l) per configuration.

    python tools/time_solve.py
"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1705_02043_b200 as pk  # noqa: E402

CASES = [("stokeslet", "tp", 8, True), ("stokeslet", "tp", 10, True), ("laplace", "tp", 8, False),
         ("laplace", "sp", 8, True), ("laplace", "dp", 8, True), ("stokeslet", "sp", 8, True)]

for kn, per, p, gated in CASES:
    k = pk.KernelSpec.from_name(kn)
    s = pk.PeriodicSetup.make(pk.Periodicity.from_name(per), 2)
    ctx = pk.Context(0)
    pk.kifmm_matrix(k, p, "a_dn", context=ctx)  # KIFMM factors built outside the timing
    t0 = time.perf_counter()
    try:
        op = pk.solve_m2l(k, s, p, gated=gated, context=ctx)
        res = op.residual_max
    except Exception as e:  # noqa: BLE001
        res = f"{type(e).__name__}: {e}"
    dt = time.perf_counter() - t0
    print(json.dumps({"kernel": kn, "per": per, "p": p, "gated": gated, "seconds": dt, "residual": res}))
    ctx.close()
