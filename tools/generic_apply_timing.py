#!/usr/bin/env python3
"""Generic-kernel apply throughput (stencils outside the symmetric classes:
mixed derivatives, non-symmetric compositions), device time per apply.

    python tools/generic_apply_timing.py [--lib _ab/x.so]
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2205_03354_b200 import _lib  # noqa: E402


def main():
    if "--lib" in sys.argv:
        _lib.load(Path(sys.argv[sys.argv.index("--lib") + 1]))
    lib = _lib.ensure_device(0)
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, composed_apply, make_grid
    from paper_2205_03354_b200.stencil import StencilSpec, compose, make, outer_product

    d1, d2 = make(StencilSpec(1, 2)), make(StencilSpec(2, 2))
    cases = [("2D f_(3,2) mixed, 2048^2 periodic", outer_product(compose(d1, d2), d2), 2, 2048, BoundaryKind.periodic),
             ("2D f_(3,2) mixed, 2048^2 clamped", outer_product(compose(d1, d2), d2), 2, 2050, BoundaryKind.clamped),
             ("3D d1 x d2 x d1, 256^3 periodic", outer_product(outer_product(d1, d2), d1), 3, 256,
              BoundaryKind.periodic)]
    a, b = C.c_void_p(), C.c_void_p()
    lib.sk_event_create(C.byref(a))
    lib.sk_event_create(C.byref(b))
    for name, s, dim, n, bc in cases:
        g = make_grid(dim, n, 1.0 / n, bc)
        ds = DeviceStencil(s)
        u = DeviceArray.from_host(np.random.default_rng(0).uniform(-1, 1, g.unknown_count()))
        v = DeviceArray(g.unknown_count())
        for _ in range(3):
            composed_apply(ds, g, u, out=v)
        reps = 20
        lib.sk_event_record(a, None)
        for _ in range(reps):
            composed_apply(ds, g, u, out=v)
        lib.sk_event_record(b, None)
        ms = C.c_float()
        lib.sk_event_elapsed_ms(a, b, C.byref(ms))
        us = ms.value / reps * 1e3
        print(f"{name}: {len(s.entries)} entries, kernel class {ds.kernel_class}, {us:.1f} us/apply, "
              f"{16.0 * g.unknown_count() / (us * 1e-6) / 1e9:.0f} GB/s algorithmic", flush=True)


if __name__ == "__main__":
    main()
