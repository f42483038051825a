"""The slab step (sk_ch_explicit_slab: z wrap replaced by ghost planes) on one
GPU: with a single rank the halo exchange is the periodic self-copy, and the
result is bit-identical to the single-domain kernel (same loads, same order)."""
import numpy as np
import pytest

from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams, CahnHilliardState
from paper_2205_03354_b200.grid import BoundaryKind, GridSpec
from paper_2205_03354_b200.slab import SlabCahnHilliard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,formulation", [((64, 64, 32), "factored"), ((70, 40, 12), "factored"),
                                              ((64, 32, 16), "composed")])
def test_slab_single_rank_equals_single_domain(dims, formulation):
    p = CahnHilliardParams.from_epsilon(0.02, formulation)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    c0 = 0.05 * np.random.default_rng(11).uniform(-1, 1, g.unknown_count())
    s = SlabCahnHilliard(g, p)
    s.scatter(c0)
    s.step(dt, 20)
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, 20)
    assert np.array_equal(s.local_field(), st.c)
