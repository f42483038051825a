#!/usr/bin/env python3
"""Timeline of the overlapped host CH call (tools only).

    python tools/ab_build.py trace -DSK_PIPE_TRACE
    python tools/host_pipeline_trace.py _ab/trace.so [--n 256] [--steps 20] [--calls 4]

Runs CahnHilliardExplicit.run_host on one registered (pinned) field; the trace
build prints, per call, the CUDA-event time of every upload chunk, every round
of step fronts and every download (ms from the call's first event) to stderr.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2205_03354_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--calls", type=int, default=4)
    args = ap.parse_args()
    _lib.load(Path(args.lib))
    _lib.ensure_device(0)
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams
    from paper_2205_03354_b200.device import pinned
    from paper_2205_03354_b200.grid import make_periodic_grid

    n = args.n
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    st = CahnHilliardExplicit(make_periodic_grid(3, n, h), p)
    c0 = 0.05 * np.random.default_rng(2).uniform(-1, 1, n ** 3)
    host = c0.copy()
    with pinned(host):
        for i in range(args.calls):
            host[:] = c0
            t0 = time.perf_counter()
            st.run_host(host, dt, args.steps)
            print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr)


if __name__ == "__main__":
    main()
