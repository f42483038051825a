#!/usr/bin/env python3
"""Small invocations of every device path, each checked against the oracle —
for tools that wrap a whole program (compute-sanitizer where it is available;
it is closed on this GPU pool, see profiles/r2_race_and_guards.md):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/device_cases.py

Covers: the ghost-padded TMA chunk of the 3D CH step (mbarrier ring, PDL
chain), the plain cp.async CH kernels (2D and 3D, composed and factored), the
2D apply graph with programmatic launch, the 3D 25/73-point streaming apply on
every boundary kind, the last-CTA reductions (dot / nrm2 / sum / minmax / free
energy), CSR assembly + SELL SpMV, the device CG loop (CSR, matrix-free 2D
fused + cooperative, 3D with p.q in the apply epilogue), an IMEX step, and
power iteration. Each case also checks its result against the oracle, so a
wrapped run is also a parity run. Sizes are tiny (sanitizers slow kernels
down by 10-100x).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.ffi import Oracle  # noqa: E402  (checker only)
from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200 import kernels as K  # noqa: E402
from paper_2205_03354_b200.cahn_hilliard import (CahnHilliardExplicit, CahnHilliardParams,  # noqa: E402
                                                 CahnHilliardState, CahnHilliardStepper, ch_init, free_energy)
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.grid import (BoundaryKind, DeviceStencil, assemble, composed_apply,  # noqa: E402
                                        composed_apply_repeat, make_grid, make_periodic_grid)
from paper_2205_03354_b200.linalg import SolveOptions, cg_solve, cg_solve_stencil, power_iteration  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main() -> int:
    lib = _lib.ensure_device(0)
    orc = Oracle()
    rng = np.random.default_rng(0)
    done = []

    # 3D CH: padded TMA chunk (>= 2 steps), plain kernel (1 step), composed
    n = 64
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g3 = make_periodic_grid(3, n, h)
    c0 = 0.05 * rng.uniform(-1, 1, g3.unknown_count())
    for steps, form in ((6, "factored"), (1, "factored"), (3, "composed")):
        p.formulation = form
        st = CahnHilliardState(g3, c0.copy())
        CahnHilliardExplicit(g3, p).step(st, dt, steps)
        assert rel(st.c, orc.ch_explicit(3, n, h, p, dt, steps, c0)) <= 1e-9, (steps, form)
        e = free_energy(st, p)
        assert abs(e - orc.free_energy(3, n, h, p, st.c)) <= 1e-12 * abs(e)
    done.append("ch3d")

    # 2D CH and the 2D apply graph (programmatic dependent launch)
    g2 = make_periodic_grid(2, 128, 1.0 / 128)
    p2 = CahnHilliardParams.from_epsilon(0.01)
    dt2 = 0.25 * (1.0 / 128) ** 4 / (64 * p2.kappa)
    c2 = 0.05 * rng.uniform(-1, 1, g2.unknown_count())
    st = CahnHilliardState(g2, c2.copy())
    CahnHilliardExplicit(g2, p2).step(st, dt2, 4)
    assert rel(st.c, orc.ch_explicit(2, 128, 1.0 / 128, p2, dt2, 4, c2)) <= 1e-9
    s2 = DeviceStencil(bilaplacian(2))
    u = DeviceArray.from_host(rng.uniform(-1, 1, g2.unknown_count()))
    v0, v1 = DeviceArray(g2.unknown_count()), DeviceArray(g2.unknown_count())
    composed_apply_repeat(s2, g2, u, v0, v1, 4)
    ref = orc.apply_direct(bilaplacian(2), g2, u.to_host())
    assert np.abs(v1.to_host() - ref).max() <= 1e-12 * np.abs(ref).max()
    done.append("ch2d+apply2d")

    # 3D streaming apply, every boundary kind, radius 2 and 4
    for bc in (BoundaryKind.periodic, BoundaryKind.clamped, BoundaryKind.simply_supported):
        for acc, m in ((2, 21), (4, 19)):
            g = make_grid(3, m, 1.0 / (m - 1), bc)
            s = bilaplacian(3, acc)
            x = rng.uniform(-1, 1, g.unknown_count())
            v = composed_apply(s, g, x)
            ref = orc.apply_direct(s, g, x)
            assert np.abs(v - ref).max() <= 1e-12 * np.abs(ref).max(), (bc, acc)
    done.append("apply3d")

    # reductions (last-CTA pattern) and BLAS-1
    a = rng.uniform(-1, 1, 100_003)
    b = rng.uniform(-1, 1, 100_003)
    da, db = DeviceArray.from_host(a), DeviceArray.from_host(b)
    assert abs(K.dot(da, db) - a @ b) <= 1e-12 * np.abs(a * b).sum()
    assert abs(K.sum(da) - a.sum()) <= 1e-12 * np.abs(a).sum()
    assert abs(K.nrm2(da) - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)
    assert K.minmax(da) == (a.min(), a.max())
    K.axpy(0.5, da, db)
    assert np.array_equal(db.to_host(), b + 0.5 * a)
    done.append("blas1")

    # CSR assembly + SpMV + CG (device while loop), clamped 2D and 3D
    for dim, acc, N in ((2, 2, 32), (3, 4, 12)):
        g = make_grid(dim, N + 1, 1.0 / N, BoundaryKind.clamped)
        s = bilaplacian(dim, acc)
        mat = assemble(s, g)
        rp, ci, vv = mat.to_host()
        orp, oci, ov = orc.assemble(s, g)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci) and np.array_equal(vv, ov)
        f, _ = orc.biharmonic_clamped(dim, N)
        x = cg_solve(mat, f, SolveOptions(rel_tol=1e-10))
        xo, status, _, _ = orc.cg_solve(orp, oci, ov, f, 1e-10)
        assert status == 0 and rel(x, xo) <= 1e-8
        xm = cg_solve_stencil(s, g, f, SolveOptions(rel_tol=1e-10))  # 2D: fused / cooperative; 3D: 4-kernel
        assert rel(xm, xo) <= 1e-7
    g = make_grid(3, 17, 1.0 / 16, BoundaryKind.clamped)  # 3D radius 2: p.q in the apply epilogue
    f = np.sin(np.arange(g.unknown_count()) * 0.01) + 1.0
    s = bilaplacian(3)
    x = cg_solve_stencil(s, g, f, SolveOptions(rel_tol=1e-10))
    rp, ci, vv = orc.assemble(s, g)
    xo, status, _, _ = orc.cg_solve(rp, ci, vv, f, 1e-10)
    assert status == 0 and rel(x, xo) <= 1e-7
    with _lib.options(cg_coop=0):  # the two-kernel 2D graph
        g = make_grid(2, 33, 1.0 / 32, BoundaryKind.clamped)
        f, _ = orc.biharmonic_clamped(2, 32)
        cg_solve_stencil(DeviceStencil(bilaplacian(2)), g, f, SolveOptions(rel_tol=1e-10))
    done.append("csr+cg")

    # IMEX step (the reference's own CH path) and power iteration
    gi = make_periodic_grid(2, 32, 1.0)
    pi = CahnHilliardParams()
    st = ch_init(gi)
    CahnHilliardStepper(gi, pi).step(st, 0.05, 2)
    assert np.isfinite(st.c).all()
    gp = make_periodic_grid(2, 16, 1.0)
    lam = power_iteration(assemble(bilaplacian(2), gp), 1e-10)
    assert abs(lam - 64.0) <= 1e-6 * 64.0  # 13-point symbol max (4 + 4)^2 at h = 1
    done.append("imex+power")

    print("device cases ok:", ", ".join(done), f"({lib.sk_launch_count()} kernel launches)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
