#!/usr/bin/env python3
"""Large-grid sanity check of the 3D CH paths (int64 addressing, 100-step graph
chunks through the ghost-padded TMA kernel): mass conservation and agreement
of the padded and plain paths after N steps at n^3 (default 768^3 = 3.6 GB
per field).

    python tools/large_grid_check.py [--n 768] [--steps 100]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.grid import make_periodic_grid  # noqa: E402
from paper_2205_03354_b200.kernels import sum as dsum  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=768)
    ap.add_argument("--steps", type=int, default=100)
    args = ap.parse_args()
    lib = _lib.ensure_device(0)
    n = args.n
    h = 1.0 / n
    p = CahnHilliardParams.from_epsilon(0.02)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = make_periodic_grid(3, n, h)
    rng = np.random.default_rng(7)
    c0 = 0.05 * rng.uniform(-1, 1, g.unknown_count())
    out = {}
    for flag in ("1", "0"):
        _lib.set_option("ch_padded", int(flag))
        st = CahnHilliardExplicit(g, p)
        c, s = DeviceArray.from_host(c0), DeviceArray(g.unknown_count())
        m0 = dsum(c)
        st.run_device(c, s, dt, args.steps)  # graph capture + padded buffers (not timed)
        lib.sk_stream_sync(None)
        c.upload(c0)
        t0 = time.perf_counter()
        res = st.run_device(c, s, dt, args.steps)
        lib.sk_stream_sync(None)
        el = time.perf_counter() - t0
        out[flag] = (res.to_host(), m0, dsum(res), el)
        del c, s
    a, b = out["1"][0], out["0"][0]
    print(json.dumps({"n": n, "steps": args.steps, "bytes_per_field": 8 * n ** 3,
                      "padded_equals_plain": bool(np.array_equal(a, b)),
                      "mass_rel_drift": abs(out["1"][2] - out["1"][1]) / abs(out["1"][1]),
                      "seconds_padded": out["1"][3], "seconds_plain": out["0"][3],
                      "ms_per_step_padded": 1e3 * out["1"][3] / args.steps}))


if __name__ == "__main__":
    main()
