import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2205_03354_b200 import _lib
from paper_2205_03354_b200.device import DeviceArray
from paper_2205_03354_b200.errors import StencilkitError
from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, make_grid
from paper_2205_03354_b200.linalg import SolveOptions, cg_solve_stencil
from paper_2205_03354_b200.stencil import bilaplacian
if "--lib" in sys.argv:  # an A/B build (tools/ab_build.py)
    from pathlib import Path

    _lib.load(Path(sys.argv[sys.argv.index("--lib") + 1]))
lib = _lib.ensure_device(0)
if "unrolled" in sys.argv:  # unrolled iteration graphs: ncu cannot profile kernel nodes under conditional nodes
    _lib.set_option("cg_device_loop", 0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 2
acc = 2 if dim == 2 else 4
g = make_grid(dim, N + 1, 1.0 / N, BoundaryKind.clamped)
s = DeviceStencil(bilaplacian(dim, acc))
b = DeviceArray.from_host(np.random.default_rng(0).uniform(-1, 1, g.unknown_count()))
x = DeviceArray(g.unknown_count())
try:
    cg_solve_stencil(s, g, b, SolveOptions(rel_tol=1e-30, max_iter=64), x_out=x)
except StencilkitError:
    pass
