#!/usr/bin/env python3
"""Where the time of a K-step 3D CH call goes (config 4, 256^3).

For each K: `single` = one call timed alone between syncs (what bench.py
measures), `pipelined` = the same call replayed back to back (launch latency
hidden). The slope of pipelined time over K is the mid-chunk kernel; the
intercept is the first/last steps; single - pipelined is the exposed launch
latency of one call.

    python tools/ch_overhead.py [--n 256] [--ks 1,2,3,20,52,102]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.grid import make_periodic_grid  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--ks", default="1,2,3,20,52,102")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--lib", default=None, help="alternative build (tools/ab_build.py)")
    args = ap.parse_args()
    if args.lib:
        _lib.load(Path(args.lib))
    lib = _lib.ensure_device(0)
    n = args.n
    eps = 0.02
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * eps * eps)
    p = CahnHilliardParams.from_epsilon(eps)
    g = make_periodic_grid(3, n, h)
    st = CahnHilliardExplicit(g, p)
    c = DeviceArray.from_host(0.05 * np.random.default_rng(0).uniform(-1, 1, g.unknown_count()))
    s = DeviceArray(g.unknown_count())
    a, b = C.c_void_p(), C.c_void_p()
    lib.sk_event_create(C.byref(a))
    lib.sk_event_create(C.byref(b))
    ms = C.c_float()
    out = {}
    for k in [int(x) for x in args.ks.split(",")]:
        for _ in range(3):
            st.run_device(c, s, dt, k)
        lib.sk_stream_sync(None)
        singles = []
        for _ in range(args.reps):
            lib.sk_stream_sync(None)
            lib.sk_event_record(a, None)
            st.run_device(c, s, dt, k)
            lib.sk_event_record(b, None)
            lib.sk_event_elapsed_ms(a, b, C.byref(ms))
            singles.append(ms.value * 1e3)
        lib.sk_stream_sync(None)
        lib.sk_event_record(a, None)
        for _ in range(args.reps):
            st.run_device(c, s, dt, k)
        lib.sk_event_record(b, None)
        lib.sk_event_elapsed_ms(a, b, C.byref(ms))
        pipe = ms.value * 1e3 / args.reps
        out[k] = {"single_us": float(np.median(singles)), "single_min_us": float(np.min(singles)),
                  "pipelined_us": pipe, "per_step_single_us": float(np.median(singles)) / k,
                  "per_step_pipelined_us": pipe / k}
        print(json.dumps({"k": k, **out[k]}))
    ks = sorted(out)
    if len(ks) >= 2:
        k0, k1 = ks[-2], ks[-1]
        slope = (out[k1]["pipelined_us"] - out[k0]["pipelined_us"]) / (k1 - k0)
        print(json.dumps({"mid_step_us": slope, "alg_gbs": 16.0 * n ** 3 / (slope * 1e-6) / 1e9}))


if __name__ == "__main__":
    main()
