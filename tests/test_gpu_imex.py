"""IMEX Cahn-Hilliard on the device: the reference's own
CH path, CahnHilliardStepper (cahn_hilliard.cpp:121-189), against the oracle
restatement and the reference's golden runs (tests/golden/imex_*.npz).

Bars: L, B and the implicit matrix bit-exact (GPU assembly +
identity_plus_scaled); the state after N steps within 1e-9 relative L2 (the
CG solves to rel_tol 1e-12 with a different reduction order than the
reference's OpenMP dots); drivers reproduce the reference's invariants."""
from pathlib import Path

import numpy as np
import pytest

from paper_2205_03354_b200.cahn_hilliard import (CahnHilliardParams, CahnHilliardState, CahnHilliardStepper,
                                                 ch_init, imex_step)
from paper_2205_03354_b200.errors import StencilkitError
from paper_2205_03354_b200.experiments import ChBenchmarkOptions, ch_benchmark, ch_temporal_convergence
from paper_2205_03354_b200.grid import BoundaryKind, make_grid, make_periodic_grid
from paper_2205_03354_b200.stencil import compose, laplacian

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("path", sorted(GOLD.glob("imex_*.npz")), ids=lambda p: p.stem)
def test_imex_vs_reference_golden(path):
    d = np.load(path)
    dim, n = (int(x) for x in d["meta"])
    h = float(d["h"])
    g = make_periodic_grid(dim, n, h)
    st = ch_init(g)
    assert np.array_equal(st.c, d["c0"])  # ch_init is bit-identical
    stepper = CahnHilliardStepper(g, CahnHilliardParams())
    for dt, order, steps in d["seq"]:
        stepper.step(st, float(dt), int(order), int(steps))
    assert rel_l2(st.c, d["c"]) <= 1e-9


@pytest.mark.parametrize("dim,n,order,steps", [(2, 48, 1, 8), (2, 40, 2, 10), (3, 12, 1, 4), (3, 14, 2, 5)])
def test_imex_vs_oracle(orc, dim, n, order, steps):
    p = CahnHilliardParams()
    h = 0.75
    g = make_periodic_grid(dim, n, h)
    st = ch_init(g)
    st.c = st.c + 0.01 * np.sin(np.arange(st.c.size) * 0.37)  # break the IC's symmetry
    c0 = st.c.copy()
    stepper = CahnHilliardStepper(g, p)
    for _ in range(steps):  # one call per step: the AB2 history lives in the stepper
        imex_step(stepper, st, 0.04, order)
    ref = orc.ch_imex(dim, n, h, p, 0.04, order, steps, c0)
    assert rel_l2(st.c, ref) <= 1e-9
    assert abs(st.t - 0.04 * steps) < 1e-15


def test_imex_matrices_bit_exact(orc):
    # L and B from the GPU assembly, the implicit matrix from identity_plus_scaled
    # on the GPU, cached per (factor, order) like ensure_implicit_matrix
    p = CahnHilliardParams()
    same = lambda a, b: all(np.array_equal(x, y) for x, y in zip(a, b))  # noqa: E731
    for dim, n, h in [(2, 17, 0.5), (3, 7, 1.0)]:
        g = make_periodic_grid(dim, n, h)
        stepper = CahnHilliardStepper(g, p)
        st = ch_init(g)
        lap = laplacian(dim, 2)
        assert same(stepper.matrix("laplacian"), orc.assemble(lap, g))
        rb = orc.assemble(compose(lap, lap), g)
        assert same(stepper.matrix("bilaplacian"), rb)
        be = orc.identity_plus_scaled(*rb, 0.05 * p.mobility * p.kappa * 1.0)   # backward Euler
        cn = orc.identity_plus_scaled(*rb, 0.05 * p.mobility * p.kappa * 0.5)   # Crank-Nicolson
        stepper.step(st, 0.05, 1)
        assert same(stepper.matrix("implicit"), be)
        stepper.step(st, 0.05, 2)  # no history after an order-1 step: bootstrap (order 1)
        assert same(stepper.matrix("implicit"), be)
        stepper.step(st, 0.05, 2)  # history at the same dt: CN/AB2
        assert same(stepper.matrix("implicit"), cn)


def test_imex_errors():
    g = make_grid(2, 16, 1.0 / 15, BoundaryKind.simply_supported)
    with pytest.raises(StencilkitError) as e:
        CahnHilliardStepper(g, CahnHilliardParams())
    assert e.value.code.name == "non_periodic"
    g = make_periodic_grid(2, 16, 1.0)
    s = CahnHilliardStepper(g, CahnHilliardParams())
    st = ch_init(g)
    with pytest.raises(StencilkitError):
        s.step(st, 0.1, 3)
    with pytest.raises(StencilkitError):
        s.step(st, 0.0, 1)
    with pytest.raises(StencilkitError):
        s.step(CahnHilliardState(g, np.zeros(10)), 0.1, 1)


def test_ch_benchmark_invariants(orc):
    # ch_benchmark (experiments.cpp:145-184) on a small grid: mass conserved,
    # energy non-increasing after step 1, the final state equals the oracle run
    opts = ChBenchmarkOptions(dim=2, n=32, h=1.0, dt=0.05, t_end=1.5, order=2, energy_every=1)
    res = ch_benchmark(opts)
    assert res.mass_rel_drift_max < 1e-12
    assert res.energy_monotone_after_first
    assert len(res.state.energy_history) == 31
    g = make_periodic_grid(2, 32, 1.0)
    ref = orc.ch_imex(2, 32, 1.0, CahnHilliardParams(), 0.05, 2, 30, ch_init(g).c)
    assert rel_l2(res.state.c, ref) <= 1e-9
    assert res.c_min <= ref.min() + 1e-12 and res.c_max >= ref.max() - 1e-12


def test_temporal_convergence_orders():
    # ch_temporal_convergence (experiments.cpp:186-218), small: order 1 and 2 slopes
    fits = ch_temporal_convergence(2, (1, 2), n=16, t_end=1.0, dt_ladder=[1 / 4, 1 / 8, 1 / 16, 1 / 32],
                                   ref_dt=1 / 512)
    slopes = {f.order: f.fit.slope for f in fits}
    assert 0.8 <= slopes[1] <= 1.3, slopes
    assert 1.7 <= slopes[2] <= 2.5, slopes


def test_biharmonic_solve_driver_vs_reference(ref):
    # experiments.cpp:99-143 (the reference's own BVP driver): same fit and residual bar
    import ctypes

    from paper_2205_03354_b200.experiments import biharmonic_solve

    ladder = [8, 16, 32, 64]
    lad = np.ascontiguousarray(ladder, np.int32)
    slope, coeff = ctypes.c_double(), ctypes.c_double()
    res = np.empty(len(ladder))
    assert ref.L.skref_biharmonic_solve(len(ladder), lad.ctypes.data, 1e-10, ctypes.byref(slope),
                                        ctypes.byref(coeff), res.ctypes.data) == 0
    for mf in (False, True):
        r = biharmonic_solve(ladder, 1e-10, matrix_free=mf)
        assert r.fit.slope == pytest.approx(slope.value, rel=1e-6)
        assert r.fit.coefficient == pytest.approx(coeff.value, rel=1e-5)
        assert max(r.residuals) <= 1e-10 and max(res) <= 1e-10
