"""Matrix-free CG per-iteration time on config 2's clamped biharmonic: the
cooperative kernel, the two-kernel and the four-kernel 2D iteration graphs. Each variant is timed `reps` times,
alternating, and the best is reported (GPU clocks vary run to run).

    python tools/cg_fused_timing.py [N ...]
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
    sizes = [int(a) for a in sys.argv[1:]] or [256, 1024, 2048]
    reps, iters = 5, 1000
    for N in sizes:
        g = make_grid(2, N + 1, 1.0 / N, BoundaryKind.clamped)
        b = np.sin(np.arange(g.unknown_count()) * 0.01) + 1.0
        o = SolveOptions(rel_tol=1e-30, max_iter=iters)
        best = {}
        variants = {"coop": ("1", "1"), "2k": ("1", "0"), "4k": ("0", "0")}
        for _ in range(reps):
            for name, (fused, coop) in variants.items():
                _lib.set_option("cg_fused", int(fused))
                _lib.set_option("cg_coop", int(coop))
                s = DeviceStencil(bilaplacian(2))  # a new plan with this setting (one cached plan per thread)
                try:
                    cg_solve_stencil(s, g, b, o)  # untimed: plan, graph
                except StencilkitError:
                    pass
                rep = SolveReport()
                t = time.perf_counter()
                try:
                    cg_solve_stencil(s, g, b, o, rep)
                except StencilkitError:
                    pass
                us = (time.perf_counter() - t) / max(rep.iterations, 1) * 1e6
                best[name] = min(best.get(name, 1e30), us)
        print(f"N={N} unknowns={g.unknown_count()} cooperative {best['coop']:.2f} us/it  two-kernel {best['2k']:.2f}"
              f"  four-kernel {best['4k']:.2f}", flush=True)


if __name__ == "__main__":
    main()
