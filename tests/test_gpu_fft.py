"""FFT-accelerated M2L (csrc/m2l_fft.cu): the V-list translations as
lattice convolutions (cuFFT batched transforms, own frequency-domain accumulation), FP64
throughout. Same parity bar as the dense paths on every golden case, Laplace / Stokes,
every periodicity, p = 6 / 8 / 10, uniform and adaptive trees; and agreement with the
dense FP64 (DMMA) path to rounding."""
import numpy as np
import pytest

import paper_1705_02043_b200 as pk
from test_gpu_parity import EVAL_ALL, golden_request, load, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fft_ctx():
    ctx = pk.Context(0)
    ctx.set_m2l("fft")
    yield ctx
    ctx.close()


@pytest.fixture(scope="module")
def dmma_ctx():
    ctx = pk.Context(0)
    ctx.set_m2l("dmma")
    yield ctx
    ctx.close()


@pytest.mark.parametrize("name", EVAL_ALL)
def test_evaluate_fft_m2l_vs_reference(name, fft_ctx, dmma_ctx):
    g = load(f"eval_{name}.npz")
    req, meta = golden_request(g)
    res = pk.evaluate(req, context=fft_ctx).potentials
    rel = rel_l2(res, g["pot"])
    tol = max(1e-10, 10 * float(g["self_spread"]))
    dm = pk.evaluate(req, context=dmma_ctx).potentials
    d = rel_l2(res, dm)
    print(f"{name} [fft M2L]: rel-L2 vs reference {rel:.3e} (tol {tol:.1e}); vs DMMA path {d:.3e}")
    assert rel <= tol
    assert d <= max(1e-11, 3 * float(g["self_spread"]))
