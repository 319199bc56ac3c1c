"""M2L on the int8 tensor pipe (tcgen05.mma kind::i8, csrc/m2l_i8.cu).

(1) The integer gather-GEMM is exact: R mod m_t equals the int64 product computed on the
    host (float64 BLAS is exact here: |products| <= 2^14, sums < 2^53).
(2) End to end, the residue path (fixed-point operands, CRT rebuild in FP64) meets the
    same tolerances against the reference as the FP64 DMMA path, with every level >= 1
    forced onto it.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1705_02043_b200 as pk
from test_gpu_parity import EVAL_ALL, golden_request, load, rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def host_residue_gemm(A, B, src, box0, zero_row):
    nmod, nslots, Ki, _ = A.shape
    ncols = src.shape[1]
    rows = np.where(src >= 0, src - box0, zero_row)
    R = np.zeros((nmod, ncols, Ki), dtype=np.float64)
    for t in range(nmod):
        for s in range(nslots):
            R[t] += B[t][rows[s]].astype(np.float64) @ A[t][s].astype(np.float64).T
    return R.astype(np.int64)


# ncols >= 2048 runs the big-level kernel (pair-dual: cta_group::2, 512-column quads); the
# other variants are covered by test_gather_gemm_exact_other_variants
@pytest.mark.parametrize("Ki,nslots,ncols,nmod", [(128, 3, 256, 2), (384, 7, 512, 3), (896, 12, 256, 2),
                                                  (1536, 5, 512, 1), (896, 9, 2048, 1), (384, 4, 2560, 2)])
def test_i8_gather_gemm_exact(Ki, nslots, ncols, nmod):
    rng = np.random.default_rng(Ki * 31 + nslots)
    mods = pk.i8_moduli()[:nmod]
    nrows, box0 = 300, 1000
    zero_row = nrows - 1
    A = rng.integers(-128, 128, size=(nmod, nslots, Ki, Ki), dtype=np.int8)
    B = rng.integers(-128, 128, size=(nmod, nrows, Ki), dtype=np.int8)
    B[:, zero_row] = 0
    src = rng.integers(box0, box0 + nrows - 1, size=(nslots, ncols)).astype(np.int32)
    src[rng.random(src.shape) < 0.3] = -1
    src[1, :256] = -1  # a slot with no source in the first column tile (skipped by the prepass)
    dev = torch.device("cuda", 0)
    R = torch.zeros((nmod, ncols, Ki), dtype=torch.int32, device=dev)
    pk.i8_gather_gemm(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), nrows, zero_row,
                      torch.from_numpy(src).to(dev), box0, R)
    got = R.cpu().numpy().astype(np.int64)  # [t][c][r]
    ref = host_residue_gemm(A, B, src, box0, zero_row)
    for t, m in enumerate(mods):
        bad = np.count_nonzero((got[t] - ref[t]) % m)
        assert bad == 0, f"modulus {m}: {bad} of {got[t].size} entries wrong"
        assert np.abs(got[t]).max() <= 128 * nslots  # reduced per unit before the atomics


@pytest.mark.parametrize("kernel", ["dual", "pairdual"])
def test_gather_gemm_exact_other_variants(kernel):
    """The exactness cases with every launch forced onto another kernel variant
    (PKGPU_I8_KERNEL: the dual-tile kernel; the pair-dual kernel wherever the columns form
    whole 512-column quads); the variant is read once per process."""
    env = dict(os.environ, PKGPU_I8_KERNEL=kernel)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__, "-k",
                        "test_i8_gather_gemm_exact"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_int8_all_levels_on_the_pair_dual_kernel():
    """End to end with every level >= 1 laid out as its own big run (PKGPU_I8_SMALL=0): the
    pair-dual kernel then serves levels of 8-4096 boxes on the adaptive golden cases too --
    quads with empty quarters and partial offset masks."""
    env = dict(os.environ, PKGPU_I8_SMALL="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__, "-k",
                        "test_evaluate_int8_all_levels_vs_reference"], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.fixture(scope="module")
def i8_everywhere():
    ctx = pk.Context(0)
    ctx.set_m2l("int8", min_boxes=1)
    yield ctx
    ctx.close()


@pytest.mark.parametrize("name", EVAL_ALL)
def test_evaluate_int8_all_levels_vs_reference(name, i8_everywhere):
    """Same bar as test_evaluate_vs_reference, with M2L on the int8 pipe at every level."""
    g = load(f"eval_{name}.npz")
    req, meta = golden_request(g)
    res = pk.evaluate(req, context=i8_everywhere)
    rel = rel_l2(res.potentials, g["pot"])
    tol = max(1e-10, 10 * float(g["self_spread"]))
    print(f"{name} [int8 M2L]: rel-L2 {rel:.3e} (tol {tol:.1e})")
    assert rel <= tol


def test_int8_and_dmma_paths_agree_and_are_deterministic():
    g = load("eval_sto_tp_p8.npz")
    req, _ = golden_request(g)
    a, b = pk.Context(0), pk.Context(0)
    a.set_m2l("int8", min_boxes=1)
    b.set_m2l("dmma")
    r1 = pk.evaluate(req, context=a).potentials
    r2 = pk.evaluate(req, context=a).potentials
    r3 = pk.evaluate(req, context=b).potentials
    assert np.array_equal(r1, r2)  # integer atomics + fixed-order rebuild: bitwise reproducible
    assert rel_l2(r1, r3) <= 10 * float(g["self_spread"])
    with pytest.raises(ValueError):
        a.set_m2l("int8", nmod=14, beta_a=60, beta_b=60)  # range of the moduli exceeded


@pytest.fixture(scope="module")
def i8_all():
    ctx = pk.Context(0)
    ctx.set_m2l("int8_all", min_boxes=1)
    yield ctx
    ctx.close()


@pytest.mark.parametrize("name", EVAL_ALL)
def test_evaluate_int8_translations_vs_reference(name, i8_all):
    """M2M / L2L / pseudo-inverses on the int8 pipe too (i8_translate): same bar."""
    g = load(f"eval_{name}.npz")
    req, meta = golden_request(g)
    res = pk.evaluate(req, context=i8_all)
    rel = rel_l2(res.potentials, g["pot"])
    tol = max(1e-10, 10 * float(g["self_spread"]))
    print(f"{name} [int8 M2L + translations]: rel-L2 {rel:.3e} (tol {tol:.1e})")
    assert rel <= tol
