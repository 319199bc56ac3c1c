"""Full-size parity against the reference run on the GPU box's own host (oracle/_ref,
prebuilt in the build container; skipped where it is absent): BASELINE cfg2 (Stokes TP,
N = 100k, p = 8) through the reference's own evaluate vs the CUDA path, on the same
seeded inputs. Protocol: rel-L2 <= 10 x the reference's thread-count
self-spread for Stokes TP p = 8 (1.4e-8 measured on the golden case)."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import paper_1705_02043_b200 as pk
from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu
REFDUMP = os.path.join(REPO, "oracle", "_ref", "refdump")


@pytest.mark.skipif(not os.path.exists(REFDUMP), reason="oracle/_ref not built (build container builds it)")
def test_cfg2_full_size_vs_reference():
    op_path = os.path.join(GOLDEN, "ops", "stokeslet_tp_ell2_p8_gated.pkm2l")
    with tempfile.TemporaryDirectory() as tmp:
        base = os.path.join(tmp, "c2")
        subprocess.run([REFDUMP, "gen", "--n", "100000", "--kind", "uniform", "--ks", "3", "--seed", "12345",
                        "--out", base], check=True, capture_output=True)
        r = subprocess.run([REFDUMP, "eval", "--kernel", "stokeslet", "--per", "tp", "--ell", "2", "--p", "8",
                            "--leaf", "50", "--src", base + ".src.f64", "--str", base + ".str.f64", "--op", op_path,
                            "--out", base], check=True, capture_output=True, text=True)
        ref = np.fromfile(base + ".pot.f64")
        ref_up = np.fromfile(base + ".phiup0.f64")
        pts = np.fromfile(base + ".src.f64").reshape(-1, 3)
        f = np.fromfile(base + ".str.f64")
    gpts, gf = pk.generate("uniform", 100000, 3, seed=12345)
    assert np.array_equal(gpts, pts) and np.array_equal(gf, f)  # same inputs
    req = pk.EvalRequest(kernel=pk.KernelSpec.stokeslet(), sources=pts, strengths=f, targets=pts,
                         setup=pk.PeriodicSetup.make(pk.Periodicity.tp), p=8, op=pk.load_operator(op_path),
                         leaf_capacity=50)
    res = pk.evaluate(req)
    rel = float(np.linalg.norm(res.potentials - ref) / np.linalg.norm(ref))
    print(f"cfg2 full size: rel-L2 vs reference {rel:.3e}; ref wall {json.loads(r.stdout)['runs'][0]['wall']:.2f} s")
    assert rel <= 1.4e-7
    assert ref_up.shape == (3 * 296,)


def _fixture_request(name):
    import torch

    f = np.load(os.path.join(GOLDEN, f"full_{name}.npz"))
    c = json.loads(str(f["meta"]))
    k = pk.KernelSpec.from_name(c["kernel"])
    setup = pk.PeriodicSetup.make(pk.Periodicity.from_name(c["per"]))
    axes = tuple(a in c["axes"] for a in "xyz")
    pts, q = pk.generate(c["kind"], c["n"], c["ks"], seed=12345, nclusters=c["nclusters"], sigma=c["sigma"],
                         periodic_axes=axes)
    assert np.array_equal(np.array([pts.sum(), q.sum()]), f["fp"])  # the reference's inputs, bit for bit
    op = pk.load_operator(os.path.join(GOLDEN, "ops", c["op"]))
    if c["relabel"]:
        op.relabel(k, setup)
    dev = torch.device("cuda", 0)
    d_pts = torch.from_numpy(pts).to(dev).reshape(-1).contiguous()
    req = pk.EvalRequest(kernel=k, sources=d_pts, strengths=torch.from_numpy(q).to(dev), targets=d_pts, setup=setup,
                         p=c["p"], op=op, leaf_capacity=c["leaf"])
    return f, c, k, pts, req


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_full_size_vs_reference_fixture(name):
    if not os.path.exists(os.path.join(GOLDEN, f"full_{name}.npz")):
        pytest.skip(f"tests/golden/full_{name}.npz not generated")
    """BASELINE cfg3 (Stokes DP p = 10, 1M clustered, stand-in operator) and cfg4 (Laplace TP
    p = 8, 8M uniform, ungated operator) at full size against the unmodified reference run
    once in the build container (tests/golden/make_fullsize.py: 65,536 strided targets).
    Bar (SURVEY §8c): rel-L2 <= max(1e-10, 10 x the reference's 8-vs-4-thread spread)."""
    f, c, k, pts, req = _fixture_request(name)
    t = pk.FmmTree(pts, pts, c["leaf"])
    assert t.structure_hash() == int(f["hash"])
    del t
    res = pk.evaluate(req)
    got = res.potentials.cpu().numpy().reshape(-1, k.kt)[f["idx"]].reshape(-1)
    ref = f["pot"]
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    tol = max(1e-10, 10 * float(f["spread"]))
    print(f"{name} full size ({c['n']} points): rel-L2 vs reference {rel:.3e} on {len(f['idx'])} targets "
          f"(reference spread {float(f['spread']):.1e}, tol {tol:.1e}); reference wall {c['wall_s']}")
    assert rel <= tol
