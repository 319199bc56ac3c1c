"""Out-of-bounds write checks with guard zones (compute-sanitizer is closed on this GPU pool:
"runs under it have left GPUs needing a reset" -- profiles/r02_sanitizers.md). Every output
buffer is a view into a larger device allocation whose margins hold a sentinel pattern; the
kernels must compute the same result and leave the margins untouched.
  * the int8 tensor-pipe gather-GEMM (all three kernel variants' shapes): residue sums R
  * evaluate, device-resident, Laplace / Stokes, uniform / adaptive: the potentials
"""
import numpy as np
import pytest

import paper_1705_02043_b200 as pk
from test_gpu_i8 import host_residue_gemm
from test_gpu_parity import golden_request, load

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GUARD = 1 << 16


@pytest.mark.parametrize("Ki,nslots,ncols,nmod", [(128, 3, 256, 2), (896, 9, 2048, 1), (384, 4, 2560, 2)])
def test_i8_gather_gemm_guard_zones(Ki, nslots, ncols, nmod):
    rng = np.random.default_rng(Ki + nslots)
    nrows, box0 = 300, 1000
    zero_row = nrows - 1
    A = rng.integers(-128, 128, size=(nmod, nslots, Ki, Ki), dtype=np.int8)
    B = rng.integers(-128, 128, size=(nmod, nrows, Ki), dtype=np.int8)
    B[:, zero_row] = 0
    src = rng.integers(box0, box0 + nrows - 1, size=(nslots, ncols)).astype(np.int32)
    src[rng.random(src.shape) < 0.3] = -1
    dev = torch.device("cuda", 0)
    n = nmod * ncols * Ki
    big = torch.full((n + 2 * GUARD,), 0x5A5A5A5A, dtype=torch.int32, device=dev)
    R = big[GUARD:GUARD + n]
    R.zero_()
    pk.i8_gather_gemm(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), nrows, zero_row,
                      torch.from_numpy(src).to(dev), box0, R.view(nmod, ncols, Ki))
    h = big.cpu().numpy()
    assert np.all(h[:GUARD] == 0x5A5A5A5A) and np.all(h[GUARD + n:] == 0x5A5A5A5A)
    got = h[GUARD:GUARD + n].reshape(nmod, ncols, Ki).astype(np.int64)
    ref = host_residue_gemm(A, B, src, box0, zero_row)
    for t, m in enumerate(pk.i8_moduli()[:nmod]):
        assert np.count_nonzero((got[t] - ref[t]) % m) == 0


@pytest.mark.parametrize("name", ["lap_sp_p8_clu", "sto_tp_p6_clu", "sto_tp_p10_clu"])
def test_evaluate_guard_zones(name):
    g = load(f"eval_{name}.npz")
    req, meta = golden_request(g)
    host = pk.evaluate(req).potentials
    dev = torch.device("cuda", 0)
    sentinel = float(np.frombuffer(np.uint64(0x7FF4DEADBEEF0001).tobytes(), dtype=np.float64)[0])  # a NaN payload
    src = torch.from_numpy(np.ascontiguousarray(req.sources, dtype=np.float64)).to(dev).reshape(-1)
    q = torch.from_numpy(np.ascontiguousarray(req.strengths, dtype=np.float64)).to(dev)
    n = host.size
    big = torch.full((n + 2 * GUARD,), sentinel, dtype=torch.float64, device=dev)
    out = big[GUARD:GUARD + n]
    dreq = pk.EvalRequest(kernel=req.kernel, sources=src, strengths=q, targets=src, setup=req.setup, p=req.p, op=req.op,
                          leaf_capacity=req.leaf_capacity)
    pk.evaluate(dreq, out=out)
    h = big.cpu().numpy().view(np.uint64)
    assert np.all(h[:GUARD] == np.uint64(0x7FF4DEADBEEF0001)) and np.all(h[GUARD + n:] == np.uint64(0x7FF4DEADBEEF0001))
    assert np.array_equal(out.cpu().numpy(), host)  # device-resident == host path, bit for bit
