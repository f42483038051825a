"""One matrix-free CG solve on config 2's operator with the cooperative
iteration kernel forced on (profiling case; tools only).

    python tools/cg2d_coop_case.py [N] [iters] [graph]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.errors import StencilkitError  # noqa: E402
from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, make_grid  # noqa: E402
from paper_2205_03354_b200.linalg import SolveOptions, cg_solve_stencil  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402

_lib.ensure_device(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
its = int(sys.argv[2]) if len(sys.argv) > 2 else 200
_lib.set_option("cg_coop", 0 if "graph" in sys.argv else 1)
if "graph" in sys.argv:  # the two-kernel iteration graphs, unrolled (ncu profiles no kernels under conditional nodes)
    _lib.set_option("cg_device_loop", 0)
g = make_grid(2, N + 1, 1.0 / N, BoundaryKind.clamped)
b = np.sin(np.arange(g.unknown_count()) * 0.01) + 1.0
try:
    cg_solve_stencil(DeviceStencil(bilaplacian(2)), g, b, SolveOptions(rel_tol=1e-30, max_iter=its))
except StencilkitError:
    pass
