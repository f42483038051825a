"""Two fused CH steps per launch (sk_chf3d2.cuh, temporal blocking; opt-in
with SK_CH_2STEP=1, measured slower than single steps on B200).

Inside a 100-step graph chunk of the 3D factored path, 49 launches each
advance the ghost-padded field by two steps. Every point is computed with the
single-step kernel's operation order, so the result must be BIT-identical to
the single-step padded path (SK_CH_2STEP=0) and to the plain cp.async path,
and match the oracle (<= 1e-9 relative L2, the north-star bar).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams, CahnHilliardState  # noqa: E402
from paper_2205_03354_b200.grid import BoundaryKind, GridSpec  # noqa: E402


def uniform(seed, n, lo=-1.0, hi=1.0):
    from paper_2205_03354_b200._lib import load

    out = np.empty(n)
    load().sk_fill_uniform_host(seed, n, lo, hi, out.ctypes.data)
    return out


def run(dims, steps, env, monkeypatch, seed=11):
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    c0 = 0.05 * uniform(seed, g.unknown_count())
    out = {}
    for name, kv in env.items():
        for k, v in kv.items():
            monkeypatch.setenv(k, v)
        st = CahnHilliardState(g, c0.copy())
        CahnHilliardExplicit(g, p).step(st, dt, steps)
        out[name] = st.c.copy()
    return out, (p, h, dt, c0)


MODES = {"two": {"SK_CH_PADDED": "1", "SK_CH_2STEP": "1"},
         "one": {"SK_CH_PADDED": "1", "SK_CH_2STEP": "0"},
         "plain": {"SK_CH_PADDED": "0", "SK_CH_2STEP": "1"}}


# partial x tiles (56-wide cores: 64 -> 56 + 8, 128 -> 3 tiles, 192 -> 4 tiles),
# y tiles of 24 rows (32 -> 24 + 8), z extents from the minimum (9) up,
# chunks + remainders
@pytest.mark.parametrize("dims,steps", [((64, 64, 64), 100), ((128, 32, 9), 100), ((192, 96, 17), 230),
                                        ((64, 32, 40), 300), ((128, 128, 128), 100)])
def test_two_step_bit_identical(orc, dims, steps, monkeypatch):
    out, (p, h, dt, c0) = run(dims, steps, MODES, monkeypatch)
    assert np.array_equal(out["two"], out["one"])
    assert np.array_equal(out["two"], out["plain"])
    ref = orc.ch_explicit_dims(dims, h, p, dt, steps, c0)
    assert np.linalg.norm(out["two"] - ref) / np.linalg.norm(ref) <= 1e-9


def test_two_step_config4_grid(monkeypatch):
    # config 4's 256^3 grid, 200 steps (2 chunks): bit-identical to the
    # single-step kernels (which the oracle tests pin at 128^3 and below)
    out, _ = run((256, 256, 256), 200, {k: MODES[k] for k in ("two", "one")}, monkeypatch, seed=2)
    assert np.array_equal(out["two"], out["one"])
    assert np.isfinite(out["two"]).all()


@pytest.mark.parametrize("dims,steps", [((384, 384, 384), 100), ((512, 256, 64), 100)])
def test_padded_large_grids(dims, steps, monkeypatch):
    # the ghost-padded TMA path at any size (rotated-column schedule, 64x16
    # tiles): bit-identical to the plain cp.async path
    out, _ = run(dims, steps, {k: MODES[k] for k in ("one", "plain")}, monkeypatch, seed=5)
    assert np.array_equal(out["one"], out["plain"])
    assert np.isfinite(out["one"]).all()
