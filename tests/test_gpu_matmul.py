"""csr_matmul on the device (linalg.cpp:253-283): bit-exact
against the oracle restatement (pinned to the reference in test_oracle.py),
and the compose-vs-product identity (test_grid.cpp:133-143) at scale."""
import numpy as np
import pytest

from paper_2205_03354_b200.errors import StencilkitError
from paper_2205_03354_b200.grid import (BoundaryKind, DeviceStencil, assemble, csr_matmul, make_grid,
                                        make_periodic_grid)
from paper_2205_03354_b200.stencil import compose, laplacian, make, StencilSpec

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,n,bc,acc", [(2, 23, BoundaryKind.periodic, 2), (2, 19, BoundaryKind.simply_supported, 4),
                                          (3, 9, BoundaryKind.periodic, 2), (1, 40, BoundaryKind.clamped, 4)])
def test_matmul_bit_exact_vs_oracle(orc, dim, n, bc, acc):
    g = make_grid(dim, n, 1.0 / (n - 1), bc)
    sa, sb = laplacian(dim, acc), compose(laplacian(dim, 2), laplacian(dim, 2))
    a, b = assemble(DeviceStencil(sa), g), assemble(DeviceStencil(sb), g)
    got = csr_matmul(b, a).to_host()
    want = orc.csr_matmul(orc.assemble(sb, g), orc.assemble(sa, g))
    assert all(np.array_equal(x, y) for x, y in zip(got, want))


@pytest.mark.parametrize("dim,n", [(2, 1024), (3, 96)])
def test_compose_matches_product_at_scale(dim, n):
    # assemble(compose(a, b)) == csr_matmul(assemble(b), assemble(a)) (periodic)
    g = make_periodic_grid(dim, n, 0.5)
    a, b = laplacian(dim, 2), make(StencilSpec(2, 2)) if dim == 1 else laplacian(dim, 2)
    direct = assemble(DeviceStencil(compose(a, b)), g).to_host()
    prod = csr_matmul(assemble(DeviceStencil(b), g), assemble(DeviceStencil(a), g)).to_host()
    assert np.array_equal(direct[0], prod[0]) and np.array_equal(direct[1], prod[1])
    assert np.max(np.abs(direct[2] - prod[2])) <= 1e-13 * np.max(np.abs(direct[2]))


def test_matmul_shape_errors():
    g1, g2 = make_periodic_grid(2, 8, 1.0), make_periodic_grid(2, 9, 1.0)
    a = assemble(DeviceStencil(laplacian(2, 2)), g1)
    b = assemble(DeviceStencil(laplacian(2, 2)), g2)
    with pytest.raises(StencilkitError):
        csr_matmul(b, a)
