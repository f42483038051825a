"""sk_ch_explicit_host with a pinned 3D field: upload, z-wavefront stepping
and download overlapped on three streams (sk_ch.cu, ch_host_pipelined).

Every plane is produced by the same kernel arithmetic as the serial path, so
the result must be bit-identical to run_device and to the serial host path
(SK_OPT_CH_HOST_PIPELINE off), for both formulations, odd extents (the
8-byte loader), step counts at the eligibility edge (nz = 4K + 8) and the
config-4 size; and the overlapped call must not be slower than the serial one.
"""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray, pinned  # noqa: E402
from paper_2205_03354_b200.grid import BoundaryKind, GridSpec  # noqa: E402


def setup(dims, form, seed=3):
    p = CahnHilliardParams.from_epsilon(0.02, form)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=3, n=list(dims), h=h, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
    c0 = 0.05 * np.random.default_rng(seed).uniform(-1, 1, int(np.prod(dims)))
    return g, p, dt, c0


def device_result(st, g, c0, dt, steps):
    c, s = DeviceArray.from_host(c0), DeviceArray(g.unknown_count())
    return st.run_device(c, s, dt, steps).to_host()


@pytest.mark.parametrize("dims,steps,form", [((64, 64, 64), 5, "factored"), ((64, 64, 64), 4, "composed"),
                                             ((64, 32, 48), 10, "factored"), ((70, 40, 40), 3, "factored"),
                                             ((64, 64, 100), 1, "factored"), ((64, 48, 72), 16, "factored"),
                                             ((64, 64, 37), 7, "composed")])
def test_pipelined_host_equals_device(dims, steps, form, sk_option):
    g, p, dt, c0 = setup(dims, form)
    st = CahnHilliardExplicit(g, p)
    ref = device_result(st, g, c0, dt, steps)
    out = {}
    for flag in (1, 0):
        sk_option("ch_host_pipeline", flag)
        host = c0.copy()
        with pinned(host):
            st.run_host(host, dt, steps)
        out[flag] = host
    assert np.array_equal(out[0], ref)
    assert np.array_equal(out[1], ref), float(np.abs(out[1] - ref).max())


def test_pipelined_host_config4_and_faster(sk_option):
    # config 4 (256^3, 20 steps): bit-identical, and the overlapped call beats the serial one
    g, p, dt, c0 = setup((256, 256, 256), "factored", seed=2)
    st = CahnHilliardExplicit(g, p)
    ref = device_result(st, g, c0, dt, 20)
    times = {}
    for flag in (1, 0):
        sk_option("ch_host_pipeline", flag)
        host = c0.copy()
        with pinned(host):
            st.run_host(host, dt, 20)  # warm (buffers, streams)
            assert np.array_equal(host, ref)
            best = 1e9
            for _ in range(3):
                host[:] = c0
                t0 = time.perf_counter()
                st.run_host(host, dt, 20)
                best = min(best, time.perf_counter() - t0)
            assert np.array_equal(host, ref)
        times[flag] = best
    print(f"host call 256^3 x 20: overlapped {times[1] * 1e3:.2f} ms, serial {times[0] * 1e3:.2f} ms")
    assert times[1] < times[0]


def test_pageable_host_field_takes_the_serial_path(sk_option):
    sk_option("ch_host_pipeline", 1)
    g, p, dt, c0 = setup((64, 64, 64), "factored")
    st = CahnHilliardExplicit(g, p)
    host = c0.copy()  # not registered: the serial path (same result)
    st.run_host(host, dt, 6)
    assert np.array_equal(host, device_result(st, g, c0, dt, 6))
