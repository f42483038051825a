"""Out-of-bounds write detection without compute-sanitizer (closed on this pool).

Every device entry point is run on fields that live in the middle of a larger
allocation whose head and tail guard regions hold a sentinel bit pattern (a
signalling-NaN payload no kernel produces). After each call the guards must
be bit-identical: any write outside the caller's buffers (a tile loader or
store past the last row / plane, a ghost frame written into the wrong buffer,
a reduction partial written past its slot) changes them. The guard is 64 KB
on each side, more than one plane of the test grids, so a stray plane or row
lands inside it. Results are checked against the oracle at the same time, so
a read of guard memory (the sentinel is a NaN) shows up as a wrong result.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200 import kernels as K  # noqa: E402
from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams, free_energy  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.grid import (BoundaryKind, DeviceStencil, assemble, composed_apply,  # noqa: E402
                                        composed_apply_repeat, make_grid, make_periodic_grid)
from paper_2205_03354_b200.linalg import SolveOptions, cg_solve, cg_solve_stencil  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402

GUARD = 8192  # doubles (64 KB) on each side
SENTINEL = np.frombuffer(np.uint64(0x7FF4DEADBEEF1234).tobytes(), dtype=np.float64)[0]


class Guarded(DeviceArray):
    """A DeviceArray whose ptr points GUARD doubles into a larger allocation."""

    def __init__(self, count: int):
        super().__init__(count + 2 * GUARD)
        self.inner = int(count)
        self.base = self._ptr
        host = np.full(self.count, SENTINEL)
        _lib.check(self.lib.sk_memcpy_h2d(self.base, host.ctypes.data, host.nbytes, None))
        _lib.check(self.lib.sk_stream_sync(None))
        self.count = self.inner
        self.nbytes = 8 * self.inner

    @property
    def ptr(self) -> int:
        return self.base + 8 * GUARD

    @classmethod
    def of(cls, a: np.ndarray) -> "Guarded":
        g = cls(a.size)
        g.upload(np.ascontiguousarray(a, np.float64))
        return g

    def guards_intact(self) -> bool:
        n = self.inner + 2 * GUARD
        host = np.empty(n)
        _lib.check(self.lib.sk_stream_sync(None))
        _lib.check(self.lib.sk_memcpy_d2h(host.ctypes.data, self.base, 8 * n, None))
        want = SENTINEL.view(np.uint64)
        return bool((host[:GUARD].view(np.uint64) == want).all() and (host[-GUARD:].view(np.uint64) == want).all())


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dims,steps,form", [((64, 64, 64), 5, "factored"), ((64, 64, 64), 1, "factored"),
                                             ((64, 32, 9), 4, "factored"), ((67, 36, 9), 3, "factored"),
                                             ((64, 64, 64), 3, "composed"), ((128, 96), 4, "factored")])
def test_ch_stays_inside_its_buffers(orc, dims, steps, form):
    from paper_2205_03354_b200.grid import GridSpec

    dim = len(dims)
    p = CahnHilliardParams.from_epsilon(0.02, form)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=dim, n=list(dims), h=h, origin=[0.0] * dim, bc=[BoundaryKind.periodic] * dim)
    c0 = 0.05 * np.random.default_rng(1).uniform(-1, 1, g.unknown_count())
    c, s = Guarded.of(c0), Guarded(g.unknown_count())
    out = CahnHilliardExplicit(g, p).run_device(c, s, dt, steps)
    assert c.guards_intact() and s.guards_intact()
    ref = orc.ch_explicit_dims(dims, h, p, dt, steps, c0)
    assert rel(out.to_host(), ref) <= 1e-9
    e = free_energy(out, p, g)
    assert np.isfinite(e) and c.guards_intact() and s.guards_intact()


@pytest.mark.parametrize("dim,acc,n,bc", [(2, 2, 130, BoundaryKind.periodic), (2, 2, 67, BoundaryKind.clamped),
                                          (3, 2, 37, BoundaryKind.periodic), (3, 2, 21, BoundaryKind.simply_supported),
                                          (3, 4, 40, BoundaryKind.periodic), (3, 4, 19, BoundaryKind.clamped)])
def test_apply_stays_inside_its_buffers(orc, dim, acc, n, bc):
    g = make_grid(dim, n, 1.0 / (n - 1), bc)
    s = bilaplacian(dim, acc)
    x = np.random.default_rng(n).uniform(-1, 1, g.unknown_count())
    u, v = Guarded.of(x), Guarded(g.unknown_count())
    composed_apply(s, g, u, out=v)
    assert u.guards_intact() and v.guards_intact()
    ref = orc.apply_direct(s, g, x)
    assert np.abs(v.to_host() - ref).max() <= 1e-12 * np.abs(ref).max()
    if dim == 2:
        v1 = Guarded(g.unknown_count())
        composed_apply_repeat(DeviceStencil(s), g, u, v, v1, 3)
        assert u.guards_intact() and v.guards_intact() and v1.guards_intact()


@pytest.mark.parametrize("dim,acc,N", [(2, 2, 40), (3, 4, 12), (3, 2, 14)])
def test_spmv_cg_and_blas_stay_inside_their_buffers(orc, dim, acc, N):
    g = make_grid(dim, N + 1, 1.0 / N, BoundaryKind.clamped)
    s = bilaplacian(dim, acc)
    m = assemble(s, g)
    f = np.sin(np.arange(m.rows) * 0.01) + 1.0
    b, x, y = Guarded.of(f), Guarded(m.rows), Guarded(m.rows)
    K.csr_matvec(m, b, y)
    assert b.guards_intact() and y.guards_intact()
    cg_solve(m, b, SolveOptions(rel_tol=1e-9), x_out=x)
    assert b.guards_intact() and x.guards_intact()
    cg_solve_stencil(s, g, b, SolveOptions(rel_tol=1e-9), x_out=y)
    assert b.guards_intact() and y.guards_intact()
    assert rel(y.to_host(), x.to_host()) <= 1e-6
    K.axpy(0.5, x, y)
    K.xpby(x, 0.25, y)
    for fn in (lambda: K.dot(x, y), lambda: K.sum(x), lambda: K.nrm2(y), lambda: K.minmax(x)):
        fn()
    assert x.guards_intact() and y.guards_intact()
