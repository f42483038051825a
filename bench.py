#!/usr/bin/env python3
"""Benchmark of the B200 stencil-composition hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

Headline workload (default `ch3d`, BASELINE config 4): the fused explicit
Cahn-Hilliard step on a periodic 256^3 fp64 grid (7-point Laplacian on
f'(u) + composed 25-point biharmonic), one step = one pass over the grid,
metric "CH steps/s". The working set (2 x 134 MB) is larger than the 126 MB
L2, so every step streams from HBM. `extra` carries the other configs' hot
paths (config 1 composed apply Gpts/s, config 3 2D CH steps/s, the 73-point
apply, config 5 CSR assembly + SpMV, config 2 CG iteration rate), each with
its roofline.

value  : device throughput with the field resident in HBM, CUDA events on
         the launching stream, K steps between a barrier + sync on both sides,
         max over ranks (N > 1 runs N independent replicas: "replicas only").
e2e    : the same K steps through the reference-facing host call
         (sk_ch_explicit_host on a pinned field: H2D of the field, K steps,
         D2H of the result; in 3D overlapped plane chunk by plane chunk),
         wall clock around the synchronous call, median of three calls.
roofline: algorithmic bytes per launch (16 B per grid point: read c, write c')
         / average launch duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline / --impl reference: the reference library itself
         (oracle/_ref/libstencilkit_ref.so: unmodified reference sources) on
         the host cores, the restated explicit step (2 csr_matvec + 2 OpenMP
         loops).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FALLBACK_HBM_GBS = 6650.0


# ------------------------------------------------------------------ helpers --
def peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if not self.path or not os.path.exists(self.path):
            return out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(smax), reasons=sorted(reasons), samples=len(sm))
        return out


class Dist:
    """One process per GPU (torchrun); N > 1 is replicas only (no data-path collective)."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = None
        self.device = "cpu"
        if self.world > 1:
            import torch
            import torch.distributed as dist

            if torch.cuda.is_available():  # one rank per GPU over NCCL (plumbing only)
                torch.cuda.set_device(self.local)
                self.device = f"cuda:{self.local}"
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:  # CPU test path (tests/test_dist.py)
                dist.init_process_group("gloo")
            self.dist = dist
            self.torch = torch

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        """Max over ranks (the timing rule: the slowest rank defines the step time)."""
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


class Events:
    def __init__(self, lib):
        self.lib = lib
        self.a, self.b = C.c_void_p(), C.c_void_p()
        lib.sk_event_create(C.byref(self.a))
        lib.sk_event_create(C.byref(self.b))

    def start(self, stream=None):
        self.lib.sk_event_record(self.a, stream)

    def stop_ms(self, stream=None) -> float:
        self.lib.sk_event_record(self.b, stream)
        ms = C.c_float()
        self.lib.sk_event_elapsed_ms(self.a, self.b, C.byref(ms))
        return float(ms.value)


def ncu_traffic(kernel_key: str, steady: bool = False):
    """dram bytes per launch from the committed ncu summary, if any: the one
    `--set full` launch (cold L2: writes still dirty in L2 at the end are not
    counted), or with steady=True consecutive launches under
    `--cache-control none` (the L2 state a step really starts from)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text()).get(kernel_key, {})
        if steady:
            ss = d.get("steady_state", {})
            v = ss.get("dram_read_bytes", 0) + ss.get("dram_write_bytes", 0)
        else:
            v = d.get("dram_bytes_per_launch")
        return float(v) if v else None
    except Exception:
        return None


# -------------------------------------------------------------- workloads --
def ch_setup(dim: int):
    """Configs 3 (2D, 2048^2, eps 0.01, seed 1) and 4 (3D, 256^3, eps 0.02, seed 2)."""
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams

    if dim == 2:
        n, eps, seed, frac, lap_w = 2048, 0.01, 1, 0.25, 64.0
    else:
        n, eps, seed, frac, lap_w = 256, 0.02, 2, 0.2, 144.0
    h = 1.0 / n
    p = CahnHilliardParams.from_epsilon(eps)
    dt = frac * h ** 4 / (lap_w * eps * eps)
    return n, h, p, dt, seed


def field(seed: int, count: int, amp: float = 0.05) -> np.ndarray:
    from paper_2205_03354_b200._lib import load

    out = np.empty(count)
    load().sk_fill_uniform_host(seed, count, -1.0, 1.0, out.ctypes.data)
    return amp * out


def run_ch(lib, dim: int, steps: int, warmup: int, d: Dist, e2e: bool = True, formulation: str = "factored"):
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import make_periodic_grid

    n, h, p, dt, seed = ch_setup(dim)
    p.formulation = formulation
    g = make_periodic_grid(dim, n, h)
    points = g.unknown_count()
    c0 = field(seed, points)
    stepper = CahnHilliardExplicit(g, p)
    c, s = DeviceArray.from_host(c0), DeviceArray(points)
    ev = Events(lib)
    # the clock sampler starts first (its start-up idles the GPU), then the
    # untimed warm-up runs right before the timed region: W single steps and
    # one K-step call (builds / caches the chunk graph)
    with ClockSampler(d.local) as clk:
        for _ in range(max(1, warmup)):
            stepper.run_device(c, s, dt, 1)
        stepper.run_device(c, s, dt, steps)
        lib.sk_stream_sync(None)
        d.barrier()
        lib.sk_stream_sync(None)
        l0 = lib.sk_launch_count()
        ev.start()
        stepper.run_device(c, s, dt, steps)
        ms = ev.stop_ms()
        launches = lib.sk_launch_count() - l0
    lib.sk_stream_sync(None)
    d.barrier()
    ms = d.max(ms)
    res = {"points": points, "ms": ms, "launches": launches, "clocks": clk.summary(), "n": n, "dt": dt}
    if e2e:
        # the reference-facing host call on a pinned field (sk_ch_explicit_host;
        # 3D: upload, steps and download overlapped), warmed once on the same
        # buffer (device buffers, streams, events), then timed from c0
        from paper_2205_03354_b200.device import pinned

        host = np.ascontiguousarray(c0.copy())
        with pinned(host):
            stepper.run_host(host, dt, steps)
            calls = []
            for _ in range(3):  # the median of three calls, each from c0
                host[:] = c0
                d.barrier()
                t0 = time.perf_counter()
                stepper.run_host(host, dt, steps)
                calls.append(d.max(time.perf_counter() - t0))
            e2e_s = sorted(calls)[1]
        res["e2e_s"] = e2e_s
        res["e2e_bytes"] = host.nbytes
    return res


def _ref_csr_timing(dim: int, acc: int, kind: int, n: int, h: float, bc: int, matvecs: int = 5, cg_iters: int = 0):
    """The reference's own CPU path on the host cores: assemble (timed) + csr_matvec
    (+ a bounded cg_solve) on the same operator. Returns a dict for 'reference_cpu'."""
    try:
        from oracle.ffi import RefCsr, Reference

        ref = Reference()
        t0 = time.perf_counter()
        m = RefCsr(ref, dim, acc, kind, [n] * dim, h, [bc] * dim)
        asm_s = time.perf_counter() - t0
        x, y = field(13, m.rows, 1.0), np.empty(m.rows)
        m.matvec(x, y)
        t0 = time.perf_counter()
        for _ in range(matvecs):
            m.matvec(x, y)
        mv_s = (time.perf_counter() - t0) / matvecs
        out = {"cores": ref.threads(), "assembly_ms": asm_s * 1e3, "matvec_ms": mv_s * 1e3, "rows": m.rows,
               "nnz": m.nnz, "rows_per_s": m.rows / mv_s}
        if cg_iters:
            xs = np.zeros(m.rows)
            t0 = time.perf_counter()
            m.cg_solve(x, xs, 1e-30, cg_iters)  # runs out of budget by design: a timed iteration sample
            out["cg_ms_per_iteration"] = (time.perf_counter() - t0) * 1e3 / cg_iters
        m.close()
        return out
    except Exception as ex:  # the reference library only exists where it was built
        return {"unavailable": repr(ex)}


def extra_apply2d(lib):
    """Config 1: 13-point composed biharmonic, 1024^2 periodic, 100 applications (one CUDA graph)."""
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import DeviceStencil, composed_apply_repeat, make_periodic_grid
    from paper_2205_03354_b200.stencil import bilaplacian

    n, reps = 1024, 100
    g = make_periodic_grid(2, n, 1.0 / n)
    s = DeviceStencil(bilaplacian(2))
    x = np.arange(n) / n
    u0 = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x)).ravel() + 1e-3 * field(0, n * n, 1.0)
    u, v0, v1 = DeviceArray.from_host(u0), DeviceArray(n * n), DeviceArray(n * n)
    for _ in range(3):
        composed_apply_repeat(s, g, u, v0, v1, reps)
    ev = Events(lib)
    times = []
    for _ in range(5):
        lib.sk_l2_flush(None)
        ev.start()
        composed_apply_repeat(s, g, u, v0, v1, reps)
        times.append(ev.stop_ms())
    ms = statistics.median(times)
    pts = reps * n * n
    gbs = 16.0 * pts / (ms * 1e-3) / 1e9
    rc = _ref_csr_timing(2, 2, 2, n, 1.0 / n, 0, matvecs=10)
    if "matvec_ms" in rc:
        rc.update(value=n * n / (rc["matvec_ms"] * 1e-3) / 1e9, unit="Gpts/s",
                  sample="10 csr_matvec of the reference-assembled 13-pt matrix (the reference has no matrix-free "
                         "apply); assembly timed separately")
    return {"config": "1: 13-pt apply 1024^2 x100 (graph)", "value": pts / (ms * 1e-3) / 1e9, "unit": "Gpts/s",
            "ms_per_100": ms, "achieved_gbs": gbs, "note": "8.4 MB field: L2-resident across the 100 applications; "
            "L2 flushed before each timed batch", "reference_cpu": rc}


def extra_apply2d_hbm(lib, n: int = 8192, reps: int = 20):
    """Config 1's 13-point apply on a grid far larger than L2 (2 x 537 MB at 8192^2): HBM-bound."""
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import DeviceStencil, composed_apply, make_periodic_grid
    from paper_2205_03354_b200.stencil import bilaplacian

    g = make_periodic_grid(2, n, 1.0 / n)
    s = DeviceStencil(bilaplacian(2))
    u, v = DeviceArray.from_host(field(0, n * n, 1.0)), DeviceArray(n * n)
    for _ in range(3):
        composed_apply(s, g, u, out=v)
    ev = Events(lib)
    lib.sk_stream_sync(None)
    ev.start()
    for _ in range(reps):
        composed_apply(s, g, u, out=v)
    ms = ev.stop_ms() / reps
    pts = n * n
    return {"config": f"1 (HBM size): 13-pt apply {n}^2 periodic", "value": pts / (ms * 1e-3) / 1e9, "unit": "Gpts/s",
            "ms_per_apply": ms, "achieved_gbs": 16.0 * pts / (ms * 1e-3) / 1e9,
            "note": f"2 x {8 * pts / 1e6:.0f} MB fields, larger than the 126 MB L2: every apply streams from HBM"}


def extra_ch2d_hbm(lib, n: int = 8192, steps: int = 20):
    """Config 3's fused CH step on a grid far larger than L2 (8192^2, eps and dt rule of config 3)."""
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import make_periodic_grid

    h = 1.0 / n
    p = CahnHilliardParams.from_epsilon(0.01)
    dt = 0.25 * h ** 4 / (64 * p.kappa)
    g = make_periodic_grid(2, n, h)
    st = CahnHilliardExplicit(g, p)
    c, s = DeviceArray.from_host(field(1, n * n)), DeviceArray(n * n)
    st.run_device(c, s, dt, steps)
    lib.sk_stream_sync(None)
    ev = Events(lib)
    ev.start()
    st.run_device(c, s, dt, steps)
    ms = ev.stop_ms() / steps
    pts = n * n
    return {"config": f"3 (HBM size): CH {n}^2 periodic, composed 13-pt B + 5-pt L kernel", "value": 1e3 / ms,
            "unit": "steps/s", "ms_per_step": ms, "achieved_gbs": 16.0 * pts / (ms * 1e-3) / 1e9,
            "note": f"2 x {8 * pts / 1e6:.0f} MB fields, larger than L2; {steps} steps in one call"}


def extra_apply3d(lib, which: str):
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import DeviceStencil, composed_apply, make_periodic_grid
    from paper_2205_03354_b200.stencil import bilaplacian

    n = 256
    acc = 4 if which == "73" else 2
    g = make_periodic_grid(3, n, 1.0 / n)
    s = DeviceStencil(bilaplacian(3, acc))
    u, v = DeviceArray.from_host(field(5, n ** 3, 1.0)), DeviceArray(n ** 3)
    for _ in range(3):
        composed_apply(s, g, u, out=v)
    ev = Events(lib)
    reps = 20
    lib.sk_stream_sync(None)
    ev.start()
    for _ in range(reps):
        composed_apply(s, g, u, out=v)
    ms = ev.stop_ms() / reps
    pts = n ** 3
    rc = _ref_csr_timing(3, acc, 2, 128, 1.0 / 128, 0, matvecs=3)
    if "matvec_ms" in rc:
        rc.update(value=128 ** 3 / (rc["matvec_ms"] * 1e-3) / 1e9, unit="Gpts/s",
                  sample="3 csr_matvec of the reference-assembled matrix at 128^3 (256^3 assembly alone needs "
                         "~20 GB and 20+ s on the host)")
    return {"config": f"{which}-pt composed apply 256^3 periodic", "value": pts / (ms * 1e-3) / 1e9,
            "unit": "Gpts/s", "ms_per_apply": ms, "achieved_gbs": 16.0 * pts / (ms * 1e-3) / 1e9,
            "reference_cpu": rc}


def extra_csr73(lib, bits: int):
    """Config 5 at 256 intervals (255^3 rows, 73-point clamped): GPU assembly + SpMV."""
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, assemble, make_grid
    from paper_2205_03354_b200.kernels import csr_matvec
    from paper_2205_03354_b200.stencil import bilaplacian

    N = 256
    from paper_2205_03354_b200.grid import assemble_into

    g = make_grid(3, N + 1, 1.0 / N, BoundaryKind.clamped)
    s = DeviceStencil(bilaplacian(3, 4))
    ev = Events(lib)
    ev.start()
    m = assemble(s, g, index_bits=bits)
    first_ms = ev.stop_ms()  # includes the 14-19 GB cudaMalloc
    assemble_into(s, g, m)  # warm
    lib.sk_stream_sync(None)
    reps = 3
    ev.start()
    for _ in range(reps):  # the assembly kernel alone: same matrix, no allocation
        assemble_into(s, g, m)
    asm_ms = ev.stop_ms() / reps
    rows, nnz = m.rows, m.nnz()
    x, y = DeviceArray.from_host(field(11, rows, 1.0)), DeviceArray(rows)
    for _ in range(3):
        csr_matvec(m, x, y)
    reps = 10
    lib.sk_stream_sync(None)
    ev.start()
    for _ in range(reps):
        csr_matvec(m, x, y)
    ms = ev.stop_ms() / reps
    idx = bits // 8
    spmv_bytes = (8 + idx) * nnz + 8 * (rows + 1) + 16 * rows
    asm_bytes = (8 + idx) * nnz + 8 * (rows + 1)
    del m
    out = {"config": f"5: 73-pt clamped CSR 255^3 (int{bits} cols)", "rows": rows, "nnz": nnz,
           "assembly_ms": asm_ms, "assembly_first_call_ms": first_ms,
           "assembly_gbs_written": asm_bytes / (asm_ms * 1e-3) / 1e9,
           "assembly_note": "assembly_ms: sk_csr_assemble_into on the allocated matrix (kernel + host class "
                            "templates, back to back); first call includes the allocation",
           "spmv_ms": ms, "spmv_grows_per_s": rows / (ms * 1e-3) / 1e9,
           "spmv_achieved_gbs": spmv_bytes / (ms * 1e-3) / 1e9}
    if bits == 64:
        rc = _ref_csr_timing(3, 4, 2, 128, 1.0 / 128, 2, matvecs=3)
        if "matvec_ms" in rc:
            rc.update(sample="reference assemble + 3 csr_matvec at 128 intervals (127^3 rows; 255^3 needs 38 GB "
                             "RSS and 22 s for the assembly alone)",
                      assembly_rows_per_s=rc["rows"] / (rc["assembly_ms"] * 1e-3))
        out["reference_cpu"] = rc
    return out


def extra_cg(lib, N: int = 1024, iters: int = 256):
    """Config 2 at N=1024: time a fixed number of device CG iterations (13-pt clamped)."""
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.errors import StencilkitError
    from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, assemble, make_grid
    from paper_2205_03354_b200.linalg import SolveOptions, SolveReport, cg_solve
    from paper_2205_03354_b200.stencil import bilaplacian

    g = make_grid(2, N + 1, 1.0 / N, BoundaryKind.clamped)
    m = assemble(DeviceStencil(bilaplacian(2)), g)
    b = DeviceArray.from_host(field(3, m.rows, 1.0))
    x = DeviceArray(m.rows)
    opts = SolveOptions(rel_tol=1e-30, max_iter=iters, check_every=64)
    for _ in range(1):
        try:
            cg_solve(m, b, opts, x_out=x)
        except StencilkitError:
            pass
    ev = Events(lib)
    rep = SolveReport()
    ev.start()
    try:
        cg_solve(m, b, opts, rep, x_out=x)
    except StencilkitError:
        pass
    ms = ev.stop_ms()
    per = ms / max(rep.iterations, 1)
    bytes_it = 16 * m.nnz() + 8 * (m.rows + 1) + 16 * m.rows + 48 * m.rows + 24 * m.rows
    rc = _ref_csr_timing(2, 2, 2, N + 1, 1.0 / N, 2, matvecs=3, cg_iters=20)
    if "cg_ms_per_iteration" in rc:
        rc.update(sample="20 cg_solve iterations of the reference on its own assembled matrix")
    return {"config": f"2: CG 13-pt clamped N={N} ({m.rows} rows)", "iterations": rep.iterations,
            "ms_per_iteration": per, "achieved_gbs": bytes_it / (per * 1e-3) / 1e9, "reference_cpu": rc}


def extra_cg_matrix_free(lib, dim: int, acc: int, N: int, iters: int):
    """Configs 2 / 5 CG with the matrix-free operator (stencil apply on the clamped grid,
    no matrix stream): a fixed number of device iterations."""
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.errors import StencilkitError
    from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, make_grid
    from paper_2205_03354_b200.linalg import SolveOptions, SolveReport, cg_solve_stencil
    from paper_2205_03354_b200.stencil import bilaplacian

    g = make_grid(dim, N + 1, 1.0 / N, BoundaryKind.clamped)
    s = DeviceStencil(bilaplacian(dim, acc))
    rows = g.unknown_count()
    b = DeviceArray.from_host(field(3, rows, 1.0))
    x = DeviceArray(rows)
    opts = SolveOptions(rel_tol=1e-30, max_iter=iters)
    for _ in range(2):
        try:
            cg_solve_stencil(s, g, b, opts, x_out=x)
        except StencilkitError:
            pass
    ev = Events(lib)
    rep = SolveReport()
    ev.start()
    try:
        cg_solve_stencil(s, g, b, opts, rep, x_out=x)
    except StencilkitError:
        pass
    per = ev.stop_ms() / max(rep.iterations, 1)
    # vectors only: 2D two-kernel iteration = apply (r, p in; q out) 24 + p, x, r update 56 B/row;
    # 3D radius 4 (config 5), three kernels: apply of the ghost-padded p with p.q in its epilogue 16 +
    # x, r update 48 + p update 24 B/row + 8 B/row writing the ghost-padded copy of p
    # (SK_OPT_CG_PADDED, SK_OPT_CG_PQ); 3D radius 2 (not run here): apply 16 + p.q 16 + 48 + 24
    per_row = 80 if dim == 2 else (96 if acc == 4 else 104)
    bytes_it = per_row * rows
    npts = 13 if dim == 2 else 73
    return {"config": f"{2 if dim == 2 else 5}: matrix-free CG {npts}-pt clamped N={N} ({rows} rows)",
            "iterations": rep.iterations, "ms_per_iteration": per, "achieved_gbs": bytes_it / (per * 1e-3) / 1e9,
            "note": "sk_cg_solve_stencil: operator = composed stencil on the clamped grid (no matrix stream); "
                    f"roofline bytes = vectors only ({per_row} B/row/iteration"
                    + (", two kernels per iteration)" if dim == 2 else
                       ", three kernels per iteration: the factored 73-point apply reads the ghost-padded p "
                       "and reduces p.q in its epilogue)")}


def extra_imex(lib, dim: int = 2, n: int = 1024, steps: int = 10, ref_steps: int = 2):
    """The reference's own CH path (IMEX, CahnHilliardStepper, order 2 = CN/AB2) on
    the device vs the compiled reference on the host cores; reference benchmark
    parameters, ch_init field, dt = 0.05, h = 1."""
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams, CahnHilliardStepper, ch_init
    from paper_2205_03354_b200.device import DeviceArray
    from paper_2205_03354_b200.grid import make_periodic_grid

    p = CahnHilliardParams()
    g = make_periodic_grid(dim, n, 1.0)
    c0 = ch_init(g).c
    st = CahnHilliardStepper(g, p)
    c = DeviceArray.from_host(c0)
    st.step_device(c, 0.05, 2, 2)  # bootstrap + both implicit matrices (not timed)
    ev = Events(lib)
    its = 0
    ev.start()
    for _ in range(steps):
        st.step_device(c, 0.05, 2, 1)
        its += st.last_cg_iterations
    ms = ev.stop_ms() / steps
    out = {"config": f"IMEX CH (reference CahnHilliardStepper, order 2) {n}^{dim}, dt 0.05",
           "value": 1e3 / ms, "unit": "steps/s", "ms_per_step": ms, "cg_iterations_per_step": its / steps,
           "note": "matrix-free implicit operator in a device-side CG while loop"}
    try:
        from oracle.ffi import Reference

        ref = Reference()
        hd = ref.imex_create(dim, n, 1.0, p)
        cr = c0.copy()
        ref.imex_steps(hd, 0.05, 2, 2, cr)
        t0 = time.perf_counter()
        ref.imex_steps(hd, 0.05, 2, ref_steps, cr)
        el = (time.perf_counter() - t0) / ref_steps
        ref.imex_free(hd)
        out["reference_cpu"] = {"ms_per_step": el * 1e3, "cores": ref.threads(),
                                "sample": f"{ref_steps} order-2 steps after a 2-step bootstrap"}
    except Exception as ex:  # the reference library only exists where it was built
        out["reference_cpu"] = {"unavailable": repr(ex)}
    return out


# ----------------------------------------------------------- CPU reference --
def ref_ch_steps_per_s(dim: int, steps: int, warmup: int):
    """The reference library on the host cores: restated explicit CH step."""
    from oracle.ffi import Reference

    n, h, p, dt, seed = ch_setup(dim)
    ref = Reference()
    t0 = time.perf_counter()
    handle = ref.ch_create(dim, n, h, p)
    setup_s = time.perf_counter() - t0
    c = ref.uniform(seed, n ** dim) * 0.05
    ref.ch_steps(handle, dt, warmup, c)
    t0 = time.perf_counter()
    ref.ch_steps(handle, dt, steps, c)
    el = time.perf_counter() - t0
    ref.ch_free(handle)
    return steps / el, el, setup_s, ref.threads()


# ------------------------------------------------------------------- main --
def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["ch3d", "ch2d"], default="ch3d")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=10, help="CPU-baseline sample (steps)")
    args = ap.parse_args()
    dim = 3 if args.workload == "ch3d" else 2
    n, h, p, dt, seed = ch_setup(dim)
    kb, kl = (25, 7) if dim == 3 else (13, 5)
    if dim == 3:
        form = (f"u' = u + dt L(f'(u) - eps^2 L u) with the {kl}-pt L, i.e. the {kb}-pt composed B = compose(L, L) "
                f"applied as two fused {kl}-pt passes (the literal {kb}-pt-weights kernel is the 'composed' extra line)")
    else:  # 2D: one kernel for both formulations (sk_ch.cu: the factored 2D tile kernel measured slower)
        form = (f"u' = u + dt (L f'(u) - eps^2 B u) with the {kl}-pt L and the literal {kb}-pt composed "
                f"B = compose(L, L) in one fused kernel")
    workload = (f"config {4 if dim == 3 else 3}: fused explicit Cahn-Hilliard step, periodic fp64 {n}^{dim}, "
                f"eps={0.02 if dim == 3 else 0.01}, dt={dt:.4e}; {form}")
    config = {"workload": workload, "grid": [n] * dim, "points_per_step": n ** dim, "dtype": "fp64",
              "l2": "inputs larger than L2 (2 x 134 MB fields)" if dim == 3 else
              "2 x 33.5 MB fields fit in the 126 MB L2", "parallelism": f"replicas x{args.gpus}"}

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return 0
        sps, el, setup_s, threads = ref_ch_steps_per_s(dim, args.steps, args.warmup)
        line = {"metric": "CH steps/s", "value": sps, "unit": "steps/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 / sps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded mt19937_64 uniform noise, as the configs specify)",
                "config": config,
                "cpu_baseline": {"value": sps, "unit": "steps/s", "cores": threads, "kind": "reference",
                                 "sample": f"{args.steps} timed steps after {args.warmup} warm-up on the full "
                                           f"{n}^{dim} grid (L, B assembly {setup_s:.1f}s excluded)"},
                "e2e": {"value": sps, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    d = Dist()
    from paper_2205_03354_b200 import _lib

    lib = _lib.ensure_device(d.local)
    r = run_ch(lib, dim, args.steps, args.warmup, d)
    ms_step = r["ms"] / args.steps
    steps_per_s = args.steps / (r["ms"] * 1e-3)
    value = steps_per_s * d.world  # whole job: replicas
    peak, peak_kind = peak_hbm()
    bytes_step = 16.0 * r["points"]
    achieved = bytes_step / (ms_step * 1e-3) / 1e9
    if dim == 3 and args.steps >= 2:  # one chunk graph: first step (cp.async) + TMA steps on ghost-padded buffers
        kernel = "chf3d_kernel<Cfg3<2,64,16,2,2,7,2>,0,1,1,0> (TMA, ghost-padded mid-chunk step)"
        ncu_key = "chf3d_kernel TMA mid-chunk (r2)"
        launch_mix = {"first (cp.async, plain -> padded)": 1, "mid (TMA, padded -> padded)": max(args.steps - 2, 0),
                      "last (TMA, padded -> plain)": 1}
    elif dim == 3:
        kernel, ncu_key, launch_mix = "chf3d_kernel (cp.async, plain field)", "chf3d_kernel (r1)", {"single": 1}
    else:
        kernel, ncu_key, launch_mix = "stencil2d_kernel<CahnHilliard>", "stencil2d_kernel_ch", {"2D step": args.steps}
    line = {
        "metric": "CH steps/s",
        "value": value,
        "unit": "steps/s",
        "n_gpus": d.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded mt19937_64 uniform noise, as the configs specify)",
        "config": config,
        "gpoints_per_s": r["points"] / (ms_step * 1e-3) / 1e9 * d.world,
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy read+write)", "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(ncu_key),
                     "traffic_source": f"profiles/ncu_summary.json[{ncu_key!r}] (dram read + write per launch)",
                     "algorithmic_bytes_per_launch": bytes_step, "launch_mix": launch_mix,
                     "achieved_note": "algorithmic bytes / CUDA-event step time averaged over the timed K-step "
                                      "call (all launch kinds of the chunk)"},
    }
    if "e2e_s" in r:
        line["e2e"] = {"value": args.steps / r["e2e_s"] * d.world, "unit": "steps/s",
                       "h2d_bytes_per_step": r["e2e_bytes"] / args.steps,
                       "d2h_bytes_per_step": r["e2e_bytes"] / args.steps,
                       "note": f"sk_ch_explicit_host on a pinned field: the {r['e2e_bytes']} B field up, "
                               f"{args.steps} steps, the field down (3D: in plane chunks, overlapped "
                               f"with the steps); wall clock of the call; bytes per step amortised"}
    if d.rank == 0 and not args.no_extra and d.world == 1:
        extra = []
        for fn in (lambda: extra_apply2d(lib), lambda: extra_apply2d_hbm(lib), lambda: extra_ch2d_hbm(lib),
                   lambda: run_ch_2d_extra(lib, dim, args),
                   lambda: run_ch_2d_extra(lib, dim, args, "composed", same=True),
                   lambda: extra_apply3d(lib, "25"), lambda: extra_apply3d(lib, "73"),
                   lambda: extra_csr73(lib, 64), lambda: extra_csr73(lib, 32), lambda: extra_cg(lib),
                   lambda: extra_cg_matrix_free(lib, 2, 2, 1024, 256), lambda: extra_cg_matrix_free(lib, 3, 4, 256, 64),
                   lambda: extra_imex(lib, 2, 1024), lambda: extra_imex(lib, 3, 128, ref_steps=1)):
            try:
                e = fn()
                if e:
                    if "achieved_gbs" in e:
                        e["frac_of_peak"] = e["achieved_gbs"] / peak
                    if "spmv_achieved_gbs" in e:
                        e["spmv_frac_of_peak"] = e["spmv_achieved_gbs"] / peak
                    if "assembly_gbs_written" in e:
                        e["assembly_frac_of_peak"] = e["assembly_gbs_written"] / peak
                    extra.append(e)
            except Exception as ex:  # keep the headline line even if an extra fails
                extra.append({"error": repr(ex)})
        line["extra"] = extra
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        try:
            sps, el, setup_s, threads = ref_ch_steps_per_s(dim, args.cpu_steps, 1)
            line["cpu_baseline"] = {"value": sps, "unit": "steps/s", "cores": threads, "kind": "reference",
                                    "sample": f"{args.cpu_steps} steps of the full {n}^{dim} grid "
                                              f"({el:.1f}s; L,B assembly {setup_s:.1f}s excluded)"}
        except Exception as ex:
            line["cpu_baseline"] = {"error": repr(ex)}
    if d.rank == 0:
        print(json.dumps(line))
    d.close()
    return 0


def run_ch_2d_extra(lib, dim, args, formulation="factored", same=False):
    """The other CH config (config 3 when the headline is config 4), or the
    headline config with the other kernel formulation (same=True)."""
    other = dim if same else (2 if dim == 3 else 3)
    r = run_ch(lib, other, 200, 5, _NoDist(), e2e=False, formulation=formulation)
    ms = r["ms"] / 200
    kname = ("composed 13-pt B + 5-pt L kernel (2D uses it for both formulations: a factored 2D kernel measured "
             "14.8 vs 13.2 us)") if other == 2 else f"{formulation} kernel"
    out = {"config": f"{3 if other == 2 else 4}: CH {r['n']}^{other} ({kname})", "value": 1e3 / ms,
           "unit": "steps/s", "ms_per_step": ms, "achieved_gbs": 16.0 * r["points"] / (ms * 1e-3) / 1e9,
           "note": "2 x 33.5 MB fields stay L2-resident" if other == 2 else ""}
    if not same:
        try:
            sps, el, setup_s, threads = ref_ch_steps_per_s(other, 3, 1)
            out["reference_cpu"] = {"value": sps, "unit": "steps/s", "cores": threads,
                                    "sample": "3 explicit steps from the reference's own L, B matrices"}
        except Exception as ex:
            out["reference_cpu"] = {"unavailable": repr(ex)}
    return out


class _NoDist:
    world, rank, local = 1, 0, 0

    def barrier(self):
        pass

    def max(self, x):
        return x


if __name__ == "__main__":
    sys.exit(main())
