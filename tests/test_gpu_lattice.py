"""Lattice M2L (csrc/m2l_fft.cu, m2l_lattice_level; the default for filled levels): the
V-list sum of a whole level (src/fmm.cpp:560-574) as ONE convolution over the level's box
lattice -- pruned surface DFTs, a 3D FFT over the parent lattice, pointwise products with
precomputed stencil spectra. FP64 throughout.

* every golden case (Laplace / Stokes; none / SP / SP-x / DP / TP; p = 6 / 8 / 10; uniform
  and adaptive trees): the default path against the reference, and against the dense FP64
  (DMMA) products of the same V lists, with the levels that ran on the lattice reported;
* free and mixed periodic axes (zero-padded lattice edges), partially filled levels (absent
  boxes are zero densities; the V lists are checked against the stencil on the device before
  the lattice is used, a mismatch falls back to the dense products);
* a level's lattice sum equals the dense sum to rounding on a uniform tree deep enough for a
  32^3 lattice (the separable axis-FFT path rather than the shared-memory transform)."""
import numpy as np
import pytest

import paper_1705_02043_b200 as pk
from test_gpu_parity import EVAL_ALL, golden_request, load, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lat_ctx():
    ctx = pk.Context(0)  # default: int8 dense products + lattice M2L on filled levels
    ctx.set_profiling(True)
    yield ctx
    ctx.close()


@pytest.fixture(scope="module")
def dmma_ctx():
    ctx = pk.Context(0)
    ctx.set_m2l("dmma")  # dense FP64 products everywhere, no lattice
    yield ctx
    ctx.close()


def standin_operator(kernel, setup, p):
    """A periodizing operator of the right shape and provenance with arbitrary small entries:
    the lattice / dense comparison does not depend on what the far-field operator is."""
    k = surface_k(kernel, p)
    rng = np.random.default_rng(p)
    return pk.PeriodizingOperator.create(kernel, setup, p, 1e-3 * rng.standard_normal((k, k)))


def surface_k(kernel, p):
    return pk.surface_point_count(p) * kernel.ks


def lattice_applications(ctx, req, **kw):
    """evaluate with profiling on; returns (potentials, V applications served by the lattice,
    all V applications)."""
    ctx.reset_stats()
    res = pk.evaluate(req, context=ctx, **kw).potentials
    st = ctx.stage_stats()
    return res, st.get("m2l_lattice", {}).get("units", 0.0), st["m2l"]["units"]


@pytest.mark.parametrize("name", EVAL_ALL)
def test_lattice_vs_reference_and_dense(name, lat_ctx, dmma_ctx):
    g = load(f"eval_{name}.npz")
    req, meta = golden_request(g)
    res, v_lat, v_all = lattice_applications(lat_ctx, req)
    dm = pk.evaluate(req, context=dmma_ctx).potentials
    rel, d = rel_l2(res, g["pot"]), rel_l2(res, dm)
    spread = float(g["self_spread"])
    print(f"{name}: {v_lat:.0f} of {v_all:.0f} V applications on the lattice; rel-L2 vs reference {rel:.3e} "
          f"(tol {max(1e-10, 10 * spread):.1e}); vs dense FP64 products {d:.3e}")
    assert rel <= max(1e-10, 10 * spread)
    assert d <= max(1e-11, 3 * spread)
    if "clu" not in name:  # uniform golden trees have filled levels
        assert v_lat > 0


@pytest.mark.parametrize("kernel,per,axes", [
    ("laplace", "none", None), ("laplace", "sp", (False, True, False)), ("laplace", "dp", (True, False, True)),
    ("stokeslet", "none", None), ("stokeslet", "dp", None)])
def test_lattice_free_and_mixed_axes_deep(kernel, per, axes, lat_ctx, dmma_ctx):
    """Uniform tree to level 4 (free axes: zero-padded lattice edges of 16; periodic axes wrap,
    edge 8) with a stand-in far-field operator: lattice vs dense FP64 products."""
    k = pk.KernelSpec.laplace() if kernel == "laplace" else pk.KernelSpec.stokeslet()
    ks = 1 if kernel == "laplace" else 3
    pts, f = pk.generate("uniform", 60000, ks, seed=7)
    periodicity = pk.Periodicity.from_name(per)
    setup = pk.PeriodicSetup.make(periodicity, 2)
    if axes is not None:
        setup.axes = axes
    op = standin_operator(k, setup, 6) if per != "none" else None
    req = pk.EvalRequest(kernel=k, sources=pts, strengths=f, targets=pts, setup=setup, p=6, op=op,
                         leaf_capacity=40)
    res, v_lat, v_all = lattice_applications(lat_ctx, req)
    dm = pk.evaluate(req, context=dmma_ctx).potentials
    d = rel_l2(res, dm)
    print(f"{kernel} {per} {axes}: {v_lat:.0f} of {v_all:.0f} V applications on the lattice; vs dense {d:.3e}")
    assert v_lat == v_all > 0  # every level of a uniform tree is filled
    assert d <= (1e-12 if kernel == "laplace" else 1e-9)


def test_lattice_partially_filled_level(lat_ctx, dmma_ctx):
    """A cloud with an empty octant-sized hole and a dense blob: the coarse levels are filled,
    the deeper ones partly (absent boxes) or hardly (dense products): same potentials."""
    rng = np.random.default_rng(11)
    pts = rng.random((40000, 3))
    pts = pts[~((pts[:, 0] < 0.25) & (pts[:, 1] < 0.25) & (pts[:, 2] < 0.5))]
    blob = 0.7 + 0.02 * rng.standard_normal((6000, 3))
    pts = np.ascontiguousarray(np.vstack([pts, blob[(blob > 0).all(1) & (blob < 1).all(1)]]))
    q = rng.uniform(-1, 1, len(pts))
    q -= q.mean()
    setup = pk.PeriodicSetup.make(pk.Periodicity.tp, 2)
    req = pk.EvalRequest(kernel=pk.KernelSpec.laplace(), sources=pts, strengths=q, targets=pts, setup=setup, p=6,
                         op=standin_operator(pk.KernelSpec.laplace(), setup, 6), leaf_capacity=40)
    res, v_lat, v_all = lattice_applications(lat_ctx, req)
    dm = pk.evaluate(req, context=dmma_ctx).potentials
    d = rel_l2(res, dm)
    print(f"holey cloud: {v_lat:.0f} of {v_all:.0f} V applications on the lattice; vs dense {d:.3e}")
    assert 0 < v_lat < v_all
    assert d <= 1e-12


def test_lattice_axis_fft_path(lat_ctx, dmma_ctx):
    """Level 6 of a uniform TP tree: a 32^3 parent lattice, transformed axis by axis in
    registers (levels <= 4 use the shared-memory 3D transform)."""
    pts, q = pk.generate("uniform", 2_000_000, 1, seed=5)
    setup = pk.PeriodicSetup.make(pk.Periodicity.tp, 2)
    req = pk.EvalRequest(kernel=pk.KernelSpec.laplace(), sources=pts, strengths=q, targets=pts, setup=setup, p=4,
                         op=standin_operator(pk.KernelSpec.laplace(), setup, 4), leaf_capacity=32)
    res, v_lat, v_all = lattice_applications(lat_ctx, req)
    dm = pk.evaluate(req, context=dmma_ctx).potentials
    d = rel_l2(res, dm)
    print(f"2M uniform p=4: {v_lat:.0f} of {v_all:.0f} V applications on the lattice; vs dense {d:.3e}")
    assert v_lat == v_all > 0  # levels 1-6 all filled at 7.6 points per level-6 box
    assert d <= 1e-12


def test_lattice_separate_targets(lat_ctx, dmma_ctx):
    """Targets that are not the sources (src/fmm.cpp:301-389 builds one tree over both): target
    boxes without sources carry zero densities on the lattice, source boxes without targets
    get results nobody reads; the evaluate lists leave both out and the check accepts that."""
    rng = np.random.default_rng(3)
    src, f = pk.generate("uniform", 50000, 3, seed=9)
    trg = np.ascontiguousarray(np.vstack([0.5 * rng.random((8000, 3)), rng.random((2000, 3))]))
    setup = pk.PeriodicSetup.make(pk.Periodicity.tp, 2)
    k = pk.KernelSpec.stokeslet()
    req = pk.EvalRequest(kernel=k, sources=src, strengths=f, targets=trg, setup=setup, p=6,
                         op=standin_operator(k, setup, 6), leaf_capacity=40)
    res, v_lat, v_all = lattice_applications(lat_ctx, req)
    dm = pk.evaluate(req, context=dmma_ctx).potentials
    d = rel_l2(res, dm)
    print(f"separate targets: {v_lat:.0f} of {v_all:.0f} V applications on the lattice; vs dense {d:.3e}")
    assert v_lat > 0.9 * v_all
    assert d <= 1e-9
