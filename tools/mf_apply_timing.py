"""Matrix-free apply and CG timing on the clamped BVP operators (configs 2, 5):
device time per apply (CUDA events over a repeated-apply graph) and per CG
iteration, best of a few repetitions.

    python tools/mf_apply_timing.py
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
    for dim, acc, N in [(2, 2, 1024), (3, 2, 256), (3, 4, 128), (3, 4, 256)]:
        g = make_grid(dim, N + 1, 1.0 / N, BoundaryKind.clamped)
        b = np.sin(np.arange(g.unknown_count()) * 0.01) + 1.0
        its = 200 if dim == 3 else 1000
        o = SolveOptions(rel_tol=1e-30, max_iter=its)
        s = DeviceStencil(bilaplacian(dim, acc))
        best = 1e30
        for k in range(4):
            rep = SolveReport()
            t = time.perf_counter()
            try:
                cg_solve_stencil(s, g, b, o, rep)
            except StencilkitError:
                pass
            if k:
                best = min(best, (time.perf_counter() - t) / max(rep.iterations, 1) * 1e6)
        print(f"dim={dim} acc={acc} N={N} unknowns={g.unknown_count()} cg {best:.2f} us/it", flush=True)


if __name__ == "__main__":
    main()
