"""Factored 73-point apply (sk_fac73.cuh, default on periodic 16-byte grids; SK_OPT_APPLY73_FACTORED): B = compose(L4, L4)
as two fused fourth-order Laplacian passes.

The operator is the reference's composed stencil (stencil.cpp:75-87 applied to
laplacian(3, 4), generators.cpp:94-108); only the rounding differs from the
literal 73-weight kernel, so both are checked against the oracle's
csr_matvec-equivalent apply at the north-star bar (<= 1e-12 relative max
error) and against each other.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2205_03354_b200.grid import BoundaryKind, GridSpec, composed_apply  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402


def rel_max(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("dims", [(64, 64, 64), (128, 96, 40), (72, 48, 9), (66, 34, 11), (130, 50, 20),
                                  (192, 160, 33), (64, 32, 9), (64, 32, 10), (256, 64, 17), (128, 128, 12)])
def test_fac73_vs_literal_and_oracle(orc, dims, sk_option):
    # whole and partial tiles, z extents down to 9, odd widths (8-byte loader)
    h = 1.0 / max(dims)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    s = bilaplacian(3, 4)
    rng = np.random.default_rng(sum(dims))
    u = rng.uniform(-1, 1, g.unknown_count())
    out = {}
    for flag in ("1", "0"):
        sk_option("apply73_factored", int(flag))
        out[flag] = composed_apply(s, g, u)
    ref = orc.apply_direct(s, g, u)
    for flag in ("1", "0"):
        assert rel_max(out[flag], ref) <= 1e-12, flag
    assert rel_max(out["1"], out["0"]) <= 1e-12


def test_fac73_smooth_input(orc, sk_option):
    # smooth field (large cancellation in B u): still within the bar
    n = 96
    h = 1.0 / n
    g = GridSpec(dim=3, n=[n, n, n], h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    x = np.arange(n) * h
    u = (np.sin(2 * np.pi * x)[None, None, :] * np.sin(2 * np.pi * x)[None, :, None] *
         np.cos(4 * np.pi * x)[:, None, None]).ravel() + 1e-3 * np.random.default_rng(1).uniform(-1, 1, n ** 3)
    s = bilaplacian(3, 4)
    sk_option("apply73_factored", 1)
    v = composed_apply(s, g, u)
    assert rel_max(v, orc.apply_direct(s, g, u)) <= 1e-12


def test_fac73_not_used_off_periodic(orc, sk_option):
    # clamped grids keep the literal kernel (the factorisation does not hold at
    # reflected boundaries): SK_OPT_APPLY73_FACTORED has no effect there
    g = GridSpec(dim=3, n=[41, 41, 41], h=1.0 / 40, origin=[0.0] * 3, bc=[BoundaryKind.clamped] * 3)
    s = bilaplacian(3, 4)
    u = np.random.default_rng(3).uniform(-1, 1, g.unknown_count())
    out = {}
    for flag in ("1", "0"):
        sk_option("apply73_factored", int(flag))
        out[flag] = composed_apply(s, g, u)
    assert np.array_equal(out["1"], out["0"])
    assert rel_max(out["1"], orc.apply_direct(s, g, u)) <= 1e-12
