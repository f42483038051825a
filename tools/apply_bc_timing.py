"""Composed 2D / 3D apply per boundary kind (device time per application from a
repeated-apply graph, CUDA events): how much the boundary-mapped loaders cost
against the periodic 16-byte path.

    python tools/apply_bc_timing.py
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, composed_apply_repeat, make_grid  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402


def main():
    _lib.ensure_device(0)
    s2 = DeviceStencil(bilaplacian(2, 2))
    for bc, n in [(BoundaryKind.periodic, 1024), (BoundaryKind.clamped, 1025), (BoundaryKind.clamped, 1026),
                  (BoundaryKind.simply_supported, 1025), (BoundaryKind.periodic, 4096), (BoundaryKind.clamped, 4097)]:
        time_case(s2, 2, 2, bc, n)
    for acc in (2, 4):
        s = DeviceStencil(bilaplacian(3, acc))
        for bc, n in [(BoundaryKind.periodic, 256), (BoundaryKind.clamped, 257), (BoundaryKind.clamped, 258),
                      (BoundaryKind.simply_supported, 257)]:
            time_case(s, 3, acc, bc, n)


def time_case(s, dim, acc, bc, n):
    g = make_grid(dim, n, 1.0 / (n - 1), bc)
    m = g.unknown_count()
    u = DeviceArray.from_host(np.random.default_rng(0).uniform(-1, 1, m))
    v0, v1 = DeviceArray(m), DeviceArray(m)
    reps = 20
    composed_apply_repeat(s, g, u, v0, v1, reps)
    best = 1e30
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        composed_apply_repeat(s, g, u, v0, v1, reps)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    print(f"dim={dim} acc={acc} {bc.name:17s} n={n} unknowns/axis={g.unknowns_per_axis(0)} {best:8.2f} us/apply "
          f"{m * 16 / best / 1e3:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
