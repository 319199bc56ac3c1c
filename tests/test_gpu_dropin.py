"""The drop-in binary: the reference's own experiment harness (src/experiments.cpp,
unmodified objects) with pkifmm::evaluate / solve_m2l resolved to the C++ shim over
libpkgpu (shim/pkifmm_gpu_evaluate.cpp; built by oracle/refbuild/Makefile `dropin` in the
build container, where /root/reference's headers exist -- skipped where it is absent).
Exit code 0 = every check of the experiment passed (tools/pkifmm.cpp cmd_experiment
convention). Callers exercised: src/experiments.cpp:115, 183, 227 (madelung1d direct mode,
stokes-tp-force, laplace-dp-pair) -- the tools/pkifmm.cpp:95-133 call sites' path."""
import json
import os
import subprocess

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu
DROPIN = os.path.join(REPO, "oracle", "_ref", "pkifmm_dropin")


@pytest.mark.skipif(not os.path.exists(DROPIN), reason="oracle/_ref/pkifmm_dropin not built (build container builds it)")
@pytest.mark.parametrize("experiment,plist", [("madelung1d", "6,8"), ("laplace-dp-pair", "8"),
                                              ("stokes-tp-force", "8")])
def test_dropin_experiment(experiment, plist, tmp_path):
    r = subprocess.run([DROPIN, experiment, "--p-list", plist, "--operator-dir", str(tmp_path)], capture_output=True,
                       text=True, timeout=900, cwd=tmp_path)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    for x in lines:
        print(x)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    # rc 0 = the experiment's report passed; any checks it printed must pass too
    assert all(x.get("pass", False) for x in lines if "check" in x)
    assert not any("error" in x for x in lines)
