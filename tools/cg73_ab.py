#!/usr/bin/env python3
"""Config 5 matrix-free CG iteration time, literal vs factored 73-point apply on the padded p (tools only).

    python tools/cg73_ab.py [N]
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.errors import StencilkitError  # noqa: E402
from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, make_grid  # noqa: E402
from paper_2205_03354_b200.linalg import SolveOptions, SolveReport, cg_solve_stencil  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402


def main():
    _lib.ensure_device(0)
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    g = make_grid(3, N + 1, 1.0 / N, BoundaryKind.clamped)
    b = np.sin(np.arange(g.unknown_count()) * 0.01) + 1.0
    o = SolveOptions(rel_tol=1e-30, max_iter=200)
    s = DeviceStencil(bilaplacian(3, 4))
    for fac in (0, 1, 0, 1):
        _lib.set_option("apply73_factored", fac)
        best = 1e30
        for k in range(3):
            rep = SolveReport()
            t = time.perf_counter()
            try:
                cg_solve_stencil(s, g, b, o, rep)
            except StencilkitError:
                pass
            if k:
                best = min(best, (time.perf_counter() - t) / max(rep.iterations, 1) * 1e6)
        print(f"N={N} factored={fac} cg {best:.2f} us/it", flush=True)


if __name__ == "__main__":
    main()
