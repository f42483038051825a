#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists and `make -C oracle` has built
oracle/_ref/libstencilkit_ref.so from the unmodified reference sources):

    python tests/golden/make_golden.py

Every array comes from a reference API call (oracle/ref_capi.cpp is a thin
C-ABI over them): laplacian/compose weights, assemble (periodic and simply
supported from the reference's own grid.cpp; clamped from the restated
even-reflection extension), kernels::serial::csr_matvec, cg_solve,
free_energy, the restated explicit Cahn-Hilliard step built from the
stepper's matrices, std::mt19937_64 uniform draws, fit_loglog. The fixtures
travel with the repo so GPU-box tests never need /root/reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.ffi import Reference  # noqa: E402

OUT = Path(__file__).resolve().parent


class P:  # CahnHilliardParams subset
    def __init__(self, kappa, mobility, rho_w, c_alpha, c_beta):
        self.kappa, self.mobility, self.rho_w, self.c_alpha, self.c_beta = kappa, mobility, rho_w, c_alpha, c_beta


def main() -> None:
    ref = Reference()
    ref.L.skref_set_threads(1)  # serial-order reductions in cg_solve / free_energy for reproducibility
    out = {}

    # stencils: laplacian(d, acc) and compose(lap, lap)
    for dim, acc in [(1, 2), (2, 2), (3, 2), (1, 4), (3, 4)]:
        for kind, name in [(1, "lap"), (2, "bilap")]:
            off, cd, num, den, hp = ref.stencil(dim, acc, kind)
            key = f"st_{name}{dim}d_a{acc}"
            out[key + "_off"] = off
            out[key + "_coeff"] = cd
            out[key + "_num"] = num
            out[key + "_den"] = den
            out[key + "_hp"] = np.int64(hp)
    np.savez_compressed(OUT / "stencils.npz", **out)

    # assembly: (name, dim, acc, kind, n, h, bc)
    cases = [
        ("bilap2d_per37", 2, 2, 2, 37, 1.0, 0),      # test_kernels.cpp:26-35
        ("lap2d_per25", 2, 2, 1, 25, 8.0, 0),        # test_grid.cpp:60-74
        ("bilap2d_ss17", 2, 2, 2, 17, 1.0 / 16, 1),  # test_grid.cpp:165-172
        ("bilap2d_cl17", 2, 2, 2, 17, 1.0 / 16, 2),
        ("bilap2d_ss6", 2, 2, 2, 6, 0.2, 1),         # merged columns near both walls
        ("bilap3d_per9", 3, 2, 2, 9, 0.125, 0),
        ("bilap3d_cl10", 3, 2, 2, 10, 1.0 / 9, 2),
        ("bilap3d4_cl12", 3, 4, 2, 12, 1.0 / 11, 2),  # 73-point, config 5 family
        ("bilap3d4_ss12", 3, 4, 2, 12, 1.0 / 11, 1),
        ("bilap3d4_per10", 3, 4, 2, 10, 0.1, 0),
        ("lap3d4_cl11", 3, 4, 1, 11, 0.1, 2),
    ]
    for name, dim, acc, kind, n, h, bc in cases:
        rp, ci, v = ref.assemble(dim, acc, kind, [n] * dim, h, [bc] * dim)
        x = ref.uniform(99, rp.size - 1)
        from oracle.ffi import RefCsr

        m = RefCsr(ref, dim, acc, kind, [n] * dim, h, [bc] * dim)
        y = np.empty(rp.size - 1)
        m.matvec(x, y, serial=True)
        arrays = dict(row_ptr=rp, col_idx=ci, values=v, x=x, y=y,
                      meta=np.array([dim, acc, kind, n, bc], np.int64), h=np.float64(h))
        if bc == 2 and kind == 2 and dim == 2:
            # CG on the clamped biharmonic with a seeded rhs (reference cg_solve)
            b = ref.uniform(3, rp.size - 1)
            xs = np.empty_like(b)
            st = m.cg_solve(b, xs, 1e-9)
            arrays.update(cg_b=b, cg_x=xs, cg_status=np.int64(st))
        np.savez_compressed(OUT / f"csr_{name}.npz", **arrays)

    # explicit Cahn-Hilliard (restated from the stepper's matrices) + free energy
    for dim, n, eps, frac, lw, steps, seed in [(2, 32, 0.01, 0.25, 64.0, 50, 1), (3, 16, 0.02, 0.2, 144.0, 20, 2)]:
        h = 1.0 / n
        p = P(eps * eps, 1.0, 0.25, -1.0, 1.0)
        dt = frac * h ** 4 / (lw * eps * eps)
        c0 = 0.05 * ref.uniform(seed, n ** dim)
        c = c0.copy()
        hd = ref.ch_create(dim, n, h, p)
        ref.ch_steps(hd, dt, steps, c)
        ref.ch_free(hd)
        e0 = ref.free_energy(dim, n, h, p, c0, serial=True)
        e1 = ref.free_energy(dim, n, h, p, c, serial=True)
        np.savez_compressed(OUT / f"ch_{dim}d.npz", c0=c0, c=c, dt=np.float64(dt), h=np.float64(h),
                            meta=np.array([dim, n, steps, seed], np.int64), params=np.array([eps * eps, 1.0, 0.25, -1.0, 1.0]),
                            energy0=np.float64(e0), energy=np.float64(e1))

    # the reference's IMEX stepper (cahn_hilliard.cpp:121-189) with its benchmark
    # parameters, from ch_init (:20-63); "seq" = (dt, order, steps) legs on ONE
    # stepper, so the AB2 history and its re-bootstrap on a dt change are pinned
    pd = P(2.0, 5.0, 5.0, 0.3, 0.7)
    for name, dim, n, h, seq in [("imex_2d_o1", 2, 24, 1.0, [(0.05, 1, 5)]),
                                 ("imex_2d_o2", 2, 24, 1.0, [(0.05, 2, 6)]),
                                 ("imex_3d_o2", 3, 10, 1.0, [(0.05, 2, 4)]),
                                 ("imex_2d_dtchange", 2, 20, 0.5, [(0.02, 2, 3), (0.01, 2, 3), (0.01, 1, 1), (0.01, 2, 2)])]:
        c0 = ref.ch_init(dim, n, h, 0.5, 0.01)
        c = c0.copy()
        hd = ref.imex_create(dim, n, h, pd, 1e-12)
        for dt, order, steps in seq:
            ref.imex_steps(hd, dt, order, steps, c)
        ref.imex_free(hd)
        np.savez_compressed(OUT / f"{name}.npz", c0=c0, c=c, h=np.float64(h), meta=np.array([dim, n], np.int64),
                            seq=np.array(seq, np.float64), params=np.array([2.0, 5.0, 5.0, 0.3, 0.7]))

    # the reference's benchmark chemistry (cahn_hilliard.hpp:14-22) on a few values
    cs = np.linspace(-1.5, 1.5, 31)
    fp = np.array([ref.L.skref_f_chem_prime(float(x), 5.0, 0.3, 0.7) for x in cs])
    np.savez_compressed(OUT / "chem.npz", c=cs, fprime_default=fp)

    # generator: std::mt19937_64 + uniform_real_distribution<double>(-1, 1)
    np.savez_compressed(OUT / "uniform.npz", **{f"seed{s}": ref.uniform(s, 2000) for s in (0, 1, 2, 3, 99)})
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
