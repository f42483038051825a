#!/usr/bin/env python3
"""Race amplification check (compute-sanitizer is closed on this pool).

    python tools/ab_build.py jitter -DSK_RACE_JITTER      # test build: random sleeps at every sync point
    python tools/race_jitter.py run --out gpurun_out/rj_ref.npz
    python tools/race_jitter.py run --lib _ab/jitter.so --out gpurun_out/rj_jit1.npz
    python tools/race_jitter.py compare gpurun_out/rj_ref.npz gpurun_out/rj_jit1.npz

Every device path (mbarrier/TMA CH chunks, split step barriers, cp.async
rings, programmatic-launch chains, last-CTA reductions, the cooperative CG
grid barrier, the CG device loop) runs on fixed inputs; all of them are
deterministic by construction (fixed reduction orders), so the jittered
build must reproduce the product build BIT FOR BIT. A missing barrier, fence
or mbarrier wait lets a warp read a stage or mu slot before it is written (or
after it is overwritten) once its neighbours are delayed by up to ~1 us, and
the outputs differ.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def run(lib_path: str | None, out: str) -> int:
    from paper_2205_03354_b200 import _lib

    if lib_path:
        _lib.load(Path(lib_path))
    _lib.ensure_device(0)
    from paper_2205_03354_b200 import kernels as K
    from paper_2205_03354_b200.cahn_hilliard import (CahnHilliardExplicit, CahnHilliardParams, CahnHilliardState,
                                                     CahnHilliardStepper, ch_init, free_energy)
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import (BoundaryKind, DeviceStencil, GridSpec, assemble, composed_apply,
                                            composed_apply_repeat, make_grid, make_periodic_grid, residual_refined)
    from paper_2205_03354_b200.linalg import SolveOptions, cg_solve, cg_solve_stencil
    from paper_2205_03354_b200.stencil import bilaplacian

    rng = np.random.default_rng(7)
    res = {}
    # 3D CH: TMA chunk (>= 2 steps), single plain step, composed, fallback loader, 2D
    for name, dims, steps, form in (("ch3d_tma", (64, 64, 64), 12, "factored"), ("ch3d_one", (64, 64, 64), 1, "factored"),
                                    ("ch3d_comp", (64, 64, 64), 3, "composed"), ("ch3d_odd", (67, 36, 9), 5, "factored"),
                                    ("ch2d", (128, 96), 6, "factored")):
        dim = len(dims)
        p = CahnHilliardParams.from_epsilon(0.02, form)
        h = 1.0 / max(dims)
        g = GridSpec(dim=dim, n=list(dims), h=h, origin=[0.0] * dim, bc=[BoundaryKind.periodic] * dim)
        st = CahnHilliardState(g, 0.05 * rng.uniform(-1, 1, g.unknown_count()))
        CahnHilliardExplicit(g, p).step(st, 0.2 * h ** 4 / (144 * p.kappa), steps)
        res[name] = st.c
        res[name + "_energy"] = np.array([free_energy(st, p)])
    # applies, every boundary kind; the 2D programmatic-launch graph
    for dim, acc, n, bc in ((2, 2, 130, BoundaryKind.periodic), (2, 2, 67, BoundaryKind.clamped),
                            (3, 2, 37, BoundaryKind.periodic), (3, 2, 21, BoundaryKind.simply_supported),
                            (3, 4, 40, BoundaryKind.periodic), (3, 4, 19, BoundaryKind.clamped)):
        g = make_grid(dim, n, 1.0 / (n - 1), bc)
        res[f"apply_{dim}_{acc}_{n}_{int(bc)}"] = composed_apply(bilaplacian(dim, acc), g,
                                                                 rng.uniform(-1, 1, g.unknown_count()))
    g = make_periodic_grid(2, 256, 1.0 / 256)
    u = DeviceArray.from_host(rng.uniform(-1, 1, g.unknown_count()))
    v0, v1 = DeviceArray(g.unknown_count()), DeviceArray(g.unknown_count())
    composed_apply_repeat(DeviceStencil(bilaplacian(2)), g, u, v0, v1, 5)
    res["apply_repeat"] = v0.to_host()
    # SpMV, CG (CSR device loop; matrix-free 2D fused + cooperative, 3D with p.q epilogue), refined residual
    for dim, acc, N in ((2, 2, 48), (3, 4, 12), (3, 2, 16)):
        g = make_grid(dim, N + 1, 1.0 / N, BoundaryKind.clamped)
        s = bilaplacian(dim, acc)
        m = assemble(s, g)
        f = np.sin(np.arange(m.rows) * 0.01) + 1.0
        res[f"spmv_{dim}_{acc}"] = K_apply(m, f)
        res[f"cg_{dim}_{acc}"] = cg_solve(m, f, SolveOptions(rel_tol=1e-9))
        res[f"cgmf_{dim}_{acc}"] = cg_solve_stencil(s, g, f, SolveOptions(rel_tol=1e-9))
        res[f"resid_{dim}_{acc}"] = residual_refined(DeviceStencil(s), g, f, res[f"cg_{dim}_{acc}"])
    from paper_2205_03354_b200 import _lib as L
    with L.options(cg_coop=0):
        g = make_grid(2, 49, 1.0 / 48, BoundaryKind.clamped)
        f = np.cos(np.arange(g.unknown_count()) * 0.02) + 1.0
        res["cgmf_2d_twokernel"] = cg_solve_stencil(DeviceStencil(bilaplacian(2)), g, f, SolveOptions(rel_tol=1e-9))
    # reductions
    a = DeviceArray.from_host(rng.uniform(-1, 1, 1_000_003))
    b = DeviceArray.from_host(rng.uniform(-1, 1, 1_000_003))
    res["blas"] = np.array([K.dot(a, b), K.sum(a), K.nrm2(b), *K.minmax(a)])
    # IMEX (the reference's CH path: CG per step)
    gi = make_periodic_grid(2, 64, 1.0)
    st = ch_init(gi)
    CahnHilliardStepper(gi, CahnHilliardParams()).step(st, 0.05, 2, 3)
    res["imex"] = st.c
    np.savez(out, **res)
    print(f"{len(res)} outputs -> {out}")
    return 0


def K_apply(m, f):
    from paper_2205_03354_b200.grid import apply

    return apply(m, f)


def compare(a: str, b: str) -> int:
    za, zb = np.load(a), np.load(b)
    bad = [k for k in za.files if k not in zb.files or not np.array_equal(za[k], zb[k], equal_nan=True)]
    for k in bad:
        d = np.abs(za[k] - zb[k]).max() if k in zb.files and za[k].shape == zb[k].shape else "missing/shape"
        print(f"DIFFERS: {k} (max |diff| {d})")
    print(f"{len(za.files) - len(bad)}/{len(za.files)} outputs bit-identical")
    return 1 if bad else 0


def main() -> int:
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--lib", default=None)
    r.add_argument("--out", required=True)
    c = sub.add_parser("compare")
    c.add_argument("a")
    c.add_argument("b")
    args = ap.parse_args()
    return run(args.lib, args.out) if args.cmd == "run" else compare(args.a, args.b)


if __name__ == "__main__":
    sys.exit(main())
