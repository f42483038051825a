"""Randomised parity sweep: random stencils (the reference's own generator
shape, test_util.hpp:17-33) on random grids, every boundary kind per axis,
dims 1-3 — GPU assembly bit-exact (int64 and int32 columns) against the
oracle's restatement of assemble (grid.cpp:62-158), the GPU SpMV bit-exact
against its csr_matvec (kernels.cpp:8-17), and the matrix-free apply
(classified symmetric kernels or the generic one) within the north-star
1e-12 relative bar. Seeded: the same cases every run."""
import random
from fractions import Fraction

import numpy as np
import pytest

from paper_2205_03354_b200.grid import BoundaryKind, GridSpec, apply, assemble, composed_apply
from paper_2205_03354_b200.stencil import compose, from_entries, laplacian

pytestmark = pytest.mark.gpu

KINDS = [BoundaryKind.periodic, BoundaryKind.simply_supported, BoundaryKind.clamped]


def random_stencil(rng, dim, support):
    entries = {}
    for _ in range(rng.randint(1, 5)):
        off = tuple(rng.randint(-support, support) for _ in range(dim))
        entries[off] = Fraction(rng.randint(-6, 6) or 1, rng.randint(1, 4))
    return from_entries(dim, rng.randint(-2, 0), entries.items())


def case(seed):
    rng = random.Random(seed)
    dim = 1 + seed % 3
    support = rng.randint(1, 3 if dim < 3 else 2)
    if seed % 4 == 3:  # symmetric compositions too: the classified streaming kernels
        s = compose(laplacian(dim, 2), laplacian(dim, 2 if dim == 1 else rng.choice([2, 4])))
        support = max(max(abs(c) for c in o) for o in s.entries)
    else:
        s = random_stencil(rng, dim, support)
    bc = [rng.choice(KINDS) for _ in range(dim)]
    top = {1: 40, 2: 24, 3: 13}[dim]
    n = [rng.randint(2 * support + 3, max(2 * support + 3, top)) for _ in range(dim)]
    h = rng.choice([1.0, 0.5, 0.25, 1.0 / 7])
    return s, GridSpec(dim=dim, n=n, h=h, origin=[0.0] * dim, bc=bc)


@pytest.mark.parametrize("seed", range(48))
def test_random_stencil_parity(orc, seed):
    s, g = case(seed)
    orp, oci, ov = orc.assemble(s, g)
    for bits in (64, 32):
        m = assemble(s, g, index_bits=bits)
        rp, ci, v = m.to_host()
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci) and np.array_equal(v, ov), (seed, bits)
    u = np.random.default_rng(seed).uniform(-1, 1, g.unknown_count())
    want = orc.csr_matvec(orp, oci, ov, u)
    assert np.array_equal(apply(m, u), want), seed  # SpMV: the reference's summation order
    got = composed_apply(s, g, u)
    scale = max(float(np.abs(want).max()), 1e-300)
    assert float(np.abs(got - want).max()) <= 1e-12 * scale, seed


def ch_case(seed):
    rng = random.Random(1000 + seed)
    dim = 2 + seed % 2
    if dim == 2:
        dims = [rng.choice([rng.randint(5, 40), rng.randint(64, 140)]) for _ in range(2)]
    else:
        dims = [rng.choice([rng.randint(5, 20), 64, rng.randint(65, 90)]), rng.choice([rng.randint(5, 20), 16, 32, 48]),
                rng.randint(5, 24)]
    steps = rng.choice([1, 2, 3, rng.randint(4, 30), 101, 102])
    form = rng.choice(["factored", "composed"])
    return dims, steps, form


@pytest.mark.parametrize("seed", range(20))
def test_random_ch_parity(orc, seed):
    # explicit CH on random periodic grids (partial and whole tiles, z extents
    # down to 5, chunk boundaries at 101 / 102 steps), both formulations, vs the
    # oracle's restated step (cahn_hilliard.cpp:146-152) at the 1e-9 bar
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams, CahnHilliardState

    dims, steps, form = ch_case(seed)
    dim = len(dims)
    p = CahnHilliardParams.from_epsilon(0.02, form)
    h = 1.0 / max(dims)
    dt = (0.2 * h ** 4 / (144 * p.kappa)) if dim == 3 else (0.25 * h ** 4 / (64 * p.kappa))
    g = GridSpec(dim=dim, n=dims, h=h, origin=[0.0] * dim, bc=[BoundaryKind.periodic] * dim)
    c0 = 0.05 * np.random.default_rng(seed).uniform(-1, 1, g.unknown_count())
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, steps)
    ref = orc.ch_explicit_dims(dims, h, p, dt, steps, c0)
    assert np.linalg.norm(st.c - ref) / np.linalg.norm(ref) <= 1e-9, (dims, steps, form)
