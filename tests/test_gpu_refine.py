"""Exact-operator iterative refinement (configs 2 / 5; sk_refine.cu).

The composed 73-point weights are non-dyadic rationals (compose(laplacian(3,4),
itself), stencil.cpp:75-87); their doubles (Rational::to_double, grid.cpp:77-81)
sum to -2.6e-15, a zeroth-order perturbation of the assembled operator. The
refined residual evaluates b - A x with the EXACT weights in double-double;
checked here against exact rational arithmetic, and the refined solve against
the plain device CG and the manufactured solution (experiments.cpp:99-143).
"""
from fractions import Fraction

import numpy as np
import pytest

from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, make_grid, residual_refined
from paper_2205_03354_b200.linalg import (RefineReport, SolveOptions, SolveReport, cg_solve_stencil,
                                          cg_solve_stencil_refined)
from paper_2205_03354_b200.stencil import bilaplacian, to_double


def test_weight_corrections_are_exact_to_double_double():
    # CPU: hi + lo reproduces every 73-point coefficient to ~2^-106 relative,
    # and the doubles alone do not sum to zero (the perturbation refinement removes)
    s = bilaplacian(3, 4)
    tot_hi = Fraction(0)
    for q in s.entries.values():
        hi = to_double(q)
        lo = float(q - Fraction(hi))
        assert abs(Fraction(hi) + Fraction(lo) - q) <= abs(q) * Fraction(1, 2 ** 104)
        tot_hi += Fraction(hi)
    assert sum(s.entries.values()) == 0
    assert abs(float(tot_hi)) > 1e-16


def exact_residual(s, dims_unknowns, n_pts, h, b, x):
    """b - A x in exact rationals: clamped even reflection / boundary drop (the
    refined kernel's mapping; grid.cpp:104-122 without the sign flip)."""
    dim = len(dims_unknowns)
    scale = Fraction(1) / Fraction(h) ** (-s.h_power)
    w = [(off, q * scale) for off, q in s.entries.items()]
    un = dims_unknowns
    out = np.empty(len(b))
    for row in range(len(b)):
        idx, rem = [], row
        for d in range(dim):
            idx.append(rem % un[d])
            rem //= un[d]
        acc = Fraction(0)
        for off, q in w:
            col, stride, drop = 0, 1, False
            for d in range(dim):
                gi = idx[d] + 1 + off[d]
                if gi < 0:
                    gi = -gi
                elif gi > n_pts - 1:
                    gi = 2 * (n_pts - 1) - gi
                if gi == 0 or gi == n_pts - 1:
                    drop = True
                    break
                col += stride * (gi - 1)
                stride *= un[d]
            if not drop:
                acc += q * Fraction(float(x[col]))
        out[row] = float(Fraction(float(b[row])) - acc)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("dim,acc,intervals", [(3, 4, 16), (2, 2, 32)])  # dyadic h: h^-4 exact in fp64
def test_refined_residual_matches_exact_rationals(dim, acc, intervals):
    s = bilaplacian(dim, acc)
    g = make_grid(dim, intervals + 1, 1.0 / intervals, BoundaryKind.clamped)
    rows = g.unknown_count()
    rng = np.random.default_rng(intervals)
    x = rng.uniform(-1, 1, rows)
    # b close to A x, so the residual cancels heavily (the refinement regime)
    from paper_2205_03354_b200.grid import composed_apply

    b = composed_apply(s, g, x) * (1 + 1e-12 * rng.uniform(-1, 1, rows))
    r = residual_refined(DeviceStencil(s), g, b, x)
    ref = exact_residual(s, [intervals - 1] * dim, intervals + 1, 1.0 / intervals, b, x)
    scale = float(np.abs(b).max())
    assert np.abs(r - ref).max() <= 1e-26 * scale + 4e-16 * np.abs(ref).max()


@pytest.mark.gpu
def test_refined_solve_config5_small(orc):
    # 73-point clamped at 32 intervals: the refined iterate's exact-operator
    # residual drops far below the fp64 floor of the plain CG, and the
    # solution moves by the (tiny at this size) weight perturbation only
    N = 32
    s = DeviceStencil(bilaplacian(3, 4))
    g = make_grid(3, N + 1, 1.0 / N, BoundaryKind.clamped)
    f, u = orc.biharmonic_clamped(3, N)  # analytic Delta^2 of prod sin^2 (oracle extension)
    o = SolveOptions(rel_tol=1e-10, accept_recurrence=True)
    rep0 = SolveReport()
    x0 = cg_solve_stencil(s, g, f, o, rep0)
    rep = RefineReport()
    x = cg_solve_stencil_refined(s, g, f, o, 1e-6, 4, rep)
    assert rep.refinements >= 1
    assert rep.last_correction_rel <= 1e-13  # converged to fp64 resolution of x
    # the exact-operator residual sits at the representation floor of an fp64
    # x: |b - A x| <= c eps (|A| |x|) componentwise (|A| from the weight magnitudes)
    r = residual_refined(s, g, f, x)
    wabs = sum(abs(float(q)) for q in bilaplacian(3, 4).entries.values()) * N ** 4
    assert np.abs(r).max() <= 64 * 2.2e-16 * wabs * np.abs(x).max()
    assert rep.refined_rel_residual <= 2 * rep.initial_true_rel_residual
    e0, e1 = np.abs(x0 - u).max(), np.abs(x - u).max()
    assert abs(e1 - e0) <= 1e-3 * e0  # discretisation error dominates at N = 32
    assert np.linalg.norm(x - x0) <= 1e-8 * np.linalg.norm(x0)


@pytest.mark.gpu
def test_config5_fourth_order_at_256(orc):
    """Config 5 at its own sizes (128^3 and 256^3 intervals): with the exact-operator
    refinement the pairwise observed order (experiments.cpp:128-141) is ~4 and the
    256^3 error is the 4th-order prediction (128^3 error / 16)."""
    import math

    s = DeviceStencil(bilaplacian(3, 4))
    o = SolveOptions(rel_tol=1e-10, accept_recurrence=True, check_every=256)
    errs = {}
    for N in (128, 256):
        g = make_grid(3, N + 1, 1.0 / N, BoundaryKind.clamped)
        f, u = orc.biharmonic_clamped(3, N)
        rep = RefineReport()
        x = cg_solve_stencil_refined(s, g, f, o, 1e-6, 4, rep)
        assert rep.last_correction_rel <= 1e-13
        errs[N] = float(np.abs(x - u).max())
    order = math.log(errs[128] / errs[256]) / math.log(2.0)
    assert order >= 3.9, (errs, order)
    assert errs[256] <= 1.05 * errs[128] / 16
