#!/usr/bin/env python3
"""Clamped biharmonic BVP convergence study on the device (BASELINE configs 2 and 5).

    python tools/bvp_convergence.py --dim 2 --ladder 64 128 256 512 [--rtol 1e-10] [--nested]
    python tools/bvp_convergence.py --dim 3 --acc 4 --ladder 16 32 64 128

The driver of experiments.cpp:99-143 (biharmonic_solve) on the GPU path:
composed stencil (13-point for --acc 2, 73-point for --dim 3 --acc 4) ->
GPU CSR assembly with clamped (even-reflection) ghosts -> analytic f = Delta^2 u
for u = prod sin^2(pi x_i) -> device CG -> max-norm error vs u -> fit_loglog
(experiments.cpp:16-42) slope = observed order. One JSON line per grid plus a
summary line.

CG stopping: the reference accepts only on the TRUE residual (linalg.cpp:31-66),
which has an fp64 floor above 1e-10 at these sizes; with
--accept-recurrence (default) the solve stops on the recurrence residual and
reports the attained true residual. --nested starts each grid from the
4th-order interpolation of the previous grid's solution (an extension; the
reference starts from x0 = 0).
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2205_03354_b200 import _lib  # noqa: E402
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.errors import StencilkitError  # noqa: E402
from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, assemble, make_grid  # noqa: E402
from paper_2205_03354_b200.experiments import fit_loglog  # noqa: E402
from paper_2205_03354_b200.linalg import (RefineReport, SolveOptions, SolveReport, cg_solve,  # noqa: E402
                                          cg_solve_stencil, cg_solve_stencil_refined)
from paper_2205_03354_b200.stencil import bilaplacian  # noqa: E402


def manufactured(dim: int, intervals: int):
    """u = prod a(x_i), a = sin^2(pi x); f = Delta^2 u (a'' = 2 pi^2 cos 2 pi x, a'''' = -8 pi^4 cos 2 pi x)."""
    h = 1.0 / intervals
    x = (np.arange(intervals - 1) + 1) * h
    a = np.sin(np.pi * x) ** 2
    a2 = 2 * np.pi ** 2 * np.cos(2 * np.pi * x)
    a4 = -8 * np.pi ** 4 * np.cos(2 * np.pi * x)
    if dim == 2:  # arrays indexed [y, x] (x fastest in memory)
        u = np.multiply.outer(a, a)
        f = np.multiply.outer(a, a4) + 2 * np.multiply.outer(a2, a2) + np.multiply.outer(a4, a)
    else:  # [z, y, x]
        o = np.multiply.outer
        u = o(o(a, a), a)
        f = o(o(a4, a), a) + o(o(a, a4), a) + o(o(a, a), a4) + 2 * (o(o(a2, a2), a) + o(o(a2, a), a2) + o(o(a, a2), a2))
    return f.ravel(), u.ravel()


def refine_axis(v: np.ndarray, axis: int) -> np.ndarray:
    """Coarse interior values (nc-1 per axis) -> fine interior (2nc-1): 4-point Lagrange
    at midpoints, zero boundary values and even (clamped) ghost reflection."""
    v = np.moveaxis(v, axis, 0)
    m = v.shape[0]
    pad = np.zeros((m + 4,) + v.shape[1:])
    pad[2:m + 2] = v
    pad[1] = 0.0          # boundary node (u = 0)
    pad[0] = v[0]         # ghost u_{-1} = u_{1}
    pad[m + 2] = 0.0
    pad[m + 3] = v[m - 1]
    out = np.empty((2 * m + 1,) + v.shape[1:])
    out[1::2] = v
    # midpoints between coarse nodes k and k+1, k = 0..m (node 0 and m+1 are boundaries)
    c = np.arange(m + 1)
    out[0::2] = (-pad[c] + 9 * pad[c + 1] + 9 * pad[c + 2] - pad[c + 3]) / 16.0
    return np.moveaxis(out, 0, axis)


def refine(x_coarse: np.ndarray, dim: int, nc: int) -> np.ndarray:
    v = x_coarse.reshape((nc - 1,) * dim)
    for ax in range(dim):
        v = refine_axis(v, ax)
    return v.ravel()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--acc", type=int, default=2)
    ap.add_argument("--ladder", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--reference-criterion", action="store_true", help="require the true residual (reference)")
    ap.add_argument("--nested", action="store_true")
    ap.add_argument("--max-iter", type=int, default=0)
    ap.add_argument("--index-bits", type=int, default=64)
    ap.add_argument("--matrix-free", action="store_true",
                    help="CG on the stencil operator (sk_cg_solve_stencil) instead of the assembled CSR")
    ap.add_argument("--refine", type=int, default=0,
                    help="iterative refinement steps against the exact composed operator (matrix-free; "
                         "sk_cg_solve_stencil_refined)")
    ap.add_argument("--inner-rtol", type=float, default=1e-6, help="CG tolerance of each refinement correction")
    args = ap.parse_args()
    lib = _lib.ensure_device(0)
    s = DeviceStencil(bilaplacian(args.dim, args.acc))
    samples, prev = [], None
    for N in args.ladder:
        g = make_grid(args.dim, N + 1, 1.0 / N, BoundaryKind.clamped)
        t0 = time.perf_counter()
        m = None if (args.matrix_free or args.refine) else assemble(s, g, index_bits=args.index_bits)
        t_asm = time.perf_counter() - t0
        rows = g.unknown_count()
        f, u = manufactured(args.dim, N)
        b = DeviceArray.from_host(f)
        x = DeviceArray(rows)
        use_x0 = args.nested and prev is not None and prev[0] * 2 == N
        if use_x0:
            x.upload(refine(prev[1], args.dim, prev[0]))
        opts = SolveOptions(rel_tol=args.rtol, max_iter=args.max_iter, check_every=256,
                            accept_recurrence=not args.reference_criterion, use_initial_guess=use_x0)
        rep = SolveReport()
        rrep = RefineReport()
        status = "ok"
        t0 = time.perf_counter()
        try:
            if args.refine:
                cg_solve_stencil_refined(s, g, b, opts, args.inner_rtol, args.refine, rrep, x_out=x)
                rep.iterations = rrep.iterations
                rep.true_rel_residual = rrep.initial_true_rel_residual
            elif m is None:
                cg_solve_stencil(s, g, b, opts, rep, x_out=x)
            else:
                cg_solve(m, b, opts, rep, x_out=x)
        except StencilkitError as e:
            status = str(e)
        t_cg = time.perf_counter() - t0
        xh = x.to_host()
        err = float(np.abs(xh - u).max())
        samples.append((1.0 / N, err))
        prev = (N, xh)
        print(json.dumps({"dim": args.dim, "acc": args.acc, "N": N, "rows": rows, "nnz": m.nnz() if m else None,
                          "matrix_free": m is None,
                          "assembly_s": round(t_asm, 4), "cg_s": round(t_cg, 3), "iterations": rep.iterations,
                          "ms_per_iteration": round(1e3 * t_cg / max(rep.iterations, 1), 4),
                          "true_rel_residual": rep.true_rel_residual,
                          "recurrence_rel_residual": rep.recurrence_rel_residual, "max_error": err,
                          "nested_x0": use_x0, "status": status,
                          **({"refinements": rrep.refinements, "refined_rel_residual": rrep.refined_rel_residual,
                              "last_correction_rel": rrep.last_correction_rel} if args.refine else {})}),
              flush=True)
        del m, b, x
    if len(samples) >= 3:
        fit = fit_loglog(samples)
        pairs = [math.log(samples[i][1] / samples[i + 1][1]) / math.log(samples[i][0] / samples[i + 1][0])
                 for i in range(len(samples) - 1)]
        print(json.dumps({"fit": {"slope": fit.slope, "coefficient": fit.coefficient, "fit_residual": fit.fit_residual},
                          "pairwise_orders": pairs, "samples": samples}), flush=True)


if __name__ == "__main__":
    main()
