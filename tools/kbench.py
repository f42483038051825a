#!/usr/bin/env python3
"""Kernel micro-benchmarks for profiling one hot kernel at a time (ncu-friendly).

    python tools/kbench.py <case> [--reps N]

cases: ch3d, ch2d, apply2d, apply3d25, apply3d73, spmv73, spmv73_32, asm73, cg2d
Prints one line per case: ms per launch and achieved GB/s (algorithmic bytes).
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.grid import (BoundaryKind, DeviceStencil, assemble, composed_apply,  # noqa: E402
                                        make_grid, make_periodic_grid)
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402


def timer(lib, fn, reps):
    a, b = C.c_void_p(), C.c_void_p()
    lib.sk_event_create(C.byref(a))
    lib.sk_event_create(C.byref(b))
    for _ in range(3):
        fn()
    lib.sk_event_record(a, None)
    for _ in range(reps):
        fn()
    lib.sk_event_record(b, None)
    ms = C.c_float()
    lib.sk_event_elapsed_ms(a, b, C.byref(ms))
    return ms.value / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2, help="CH steps per timed call (>= 100: graph chunks)")
    ap.add_argument("--lib", default=None, help="alternative build (tools/ab_build.py)")
    ap.add_argument("--opt", action="append", default=[], help="sk_set_option name=value (repeatable)")
    args = ap.parse_args()
    if args.lib:
        _lib.load(Path(args.lib))
    lib = _lib.ensure_device(0)
    for o in args.opt:
        k, v = o.split("=")
        _lib.set_option(k, int(v))
    rng = np.random.default_rng(0)
    case = args.case
    if case.startswith("ch"):
        from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams

        dim = 3 if case.startswith("ch3d") else 2
        n = args.n or (256 if dim == 3 else 2048)
        eps = 0.02 if dim == 3 else 0.01
        form = "composed" if case.endswith("c") else "factored"
        p = CahnHilliardParams.from_epsilon(eps, form)
        h = 1.0 / n
        dt = (0.2 * h ** 4 / (144 * eps * eps)) if dim == 3 else (0.25 * h ** 4 / (64 * eps * eps))
        g = make_periodic_grid(dim, n, h)
        st = CahnHilliardExplicit(g, p)
        c = DeviceArray.from_host(0.05 * rng.uniform(-1, 1, g.unknown_count()))
        s = DeviceArray(g.unknown_count())
        ms = timer(lib, lambda: st.run_device(c, s, dt, args.steps), args.reps) / args.steps
        byts = 16.0 * g.unknown_count()
    elif case.startswith("apply"):
        dim = 2 if case == "apply2d" else 3
        acc = 4 if case.endswith("73") else 2
        n = args.n or (1024 if dim == 2 else 256)
        g = make_periodic_grid(dim, n, 1.0 / n)
        s = DeviceStencil(bilaplacian(dim, acc))
        u = DeviceArray.from_host(rng.uniform(-1, 1, g.unknown_count()))
        v = DeviceArray(g.unknown_count())
        ms = timer(lib, lambda: composed_apply(s, g, u, out=v), args.reps)
        byts = 16.0 * g.unknown_count()
    elif case.startswith("spmv") or case.startswith("asm73"):
        from paper_2205_03354_b200.kernels import csr_matvec

        bits = 32 if case.endswith("_32") else 64
        N = args.n or 256
        g = make_grid(3, N + 1, 1.0 / N, BoundaryKind.clamped)
        s = DeviceStencil(bilaplacian(3, 4))
        if case.startswith("asm73"):
            from paper_2205_03354_b200.grid import assemble_into

            m = assemble(s, g, index_bits=bits)
            ms = timer(lib, lambda: assemble_into(s, g, m), max(2, args.reps // 5))
            byts = (8 + bits // 8) * m.nnz() + 8.0 * (m.rows + 1)
        else:
            m = assemble(s, g, index_bits=bits)
            x = DeviceArray.from_host(rng.uniform(-1, 1, m.rows))
            y = DeviceArray(m.rows)
            ms = timer(lib, lambda: csr_matvec(m, x, y), args.reps)
            byts = (8 + bits // 8) * m.nnz() + 8.0 * (m.rows + 1) + 16.0 * m.rows
    elif case.startswith("imex"):  # imex2d / imex3d: IMEX CH steps (reference's own CH path), order 2
        from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams, CahnHilliardStepper, ch_init

        dim = 3 if case == "imex3d" else 2
        n = args.n or (1024 if dim == 2 else 128)
        g = make_periodic_grid(dim, n, 1.0)
        st = CahnHilliardStepper(g, CahnHilliardParams())
        c = DeviceArray.from_host(ch_init(g).c)
        st.step_device(c, 0.05, 2, 2)  # bootstrap + build both implicit matrices
        its = []

        def one():
            st.step_device(c, 0.05, 2, 1)
            its.append(st.last_cg_iterations)

        ms = timer(lib, one, args.reps)
        print(f"{case}: n={n}^{dim} CG iterations/step {np.mean(its):.1f}")
        byts = 16.0 * g.unknown_count()
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"{case}: {ms * 1e3:.2f} us/launch, {byts / (ms * 1e-3) / 1e9:.1f} GB/s algorithmic")


if __name__ == "__main__":
    main()
