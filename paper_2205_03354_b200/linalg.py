"""Device CG with the reference's contract (linalg.hpp:13-23, linalg.cpp:15-72)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import SolveOptionsC, SolveReportC, check
from .device import DeviceArray
from .errors import Errc, StencilkitError
from .grid import CsrMatrix


@dataclass
class SolveOptions:
    rel_tol: float = 1e-10
    max_iter: int = 0          # 0: 10 * unknown count
    deflate_mean: bool = False
    check_every: int = 64      # device iterations per host status poll
    # extensions (off = reference semantics, linalg.cpp:15-72)
    accept_recurrence: bool = False  # stop on sqrt(r.r) <= tol ||b||, report the true residual
    use_initial_guess: bool = False  # start from x_out's contents instead of x0 = 0


@dataclass
class SolveReport:
    iterations: int = 0
    restarts: int = 0
    true_rel_residual: float = 0.0
    recurrence_rel_residual: float = 0.0


def _opts(o: SolveOptions) -> SolveOptionsC:
    c = SolveOptionsC()
    c.rel_tol = o.rel_tol
    c.max_iter = o.max_iter
    c.deflate_mean = 1 if o.deflate_mean else 0
    c.check_every = o.check_every
    c.accept_recurrence = 1 if o.accept_recurrence else 0
    c.use_initial_guess = 1 if o.use_initial_guess else 0
    return c


def cg_solve(m: CsrMatrix, b, opts: SolveOptions | None = None, report: SolveReport | None = None,
             x_out: DeviceArray | None = None, stream=None):
    """Solve M x = b. Host b -> host x (numpy); DeviceArray b -> DeviceArray x.

    Raises StencilkitError(no_convergence) exactly when the reference throws
    (non-PD Krylov space, or true residual above tol after the budget)."""
    opts = opts or SolveOptions()
    if m.rows != m.cols:
        raise StencilkitError(Errc.shape_mismatch, "cg_solve needs a square matrix")
    rep = SolveReportC()
    o = _opts(opts)
    try:
        if isinstance(b, DeviceArray):
            if b.count != m.rows:
                raise StencilkitError(Errc.shape_mismatch, "rhs length does not match matrix")
            x = x_out if x_out is not None else DeviceArray(m.rows)
            check(m.lib.sk_cg_solve(m.handle, b.ptr, x.ptr, C.byref(o), C.byref(rep), stream))
            return x
        bs = np.ascontiguousarray(np.asarray(b, dtype=np.float64).ravel())
        if bs.size != m.rows:
            raise StencilkitError(Errc.shape_mismatch, "rhs length does not match matrix")
        x = np.empty_like(bs)
        check(m.lib.sk_cg_solve_host(m.handle, bs.ctypes.data, x.ctypes.data, C.byref(o), C.byref(rep)))
        return x
    finally:
        if report is not None:
            report.iterations = rep.iterations
            report.restarts = rep.restarts
            report.true_rel_residual = rep.true_rel_residual
            report.recurrence_rel_residual = rep.recurrence_rel_residual


def cg_solve_stencil(stencil, grid, b, opts: SolveOptions | None = None, report: SolveReport | None = None,
                     x_out: DeviceArray | None = None, stream=None):
    """Matrix-free CG on the composed stencil's operator over `grid` (assemble(s, g)
    without the matrix); same contract as cg_solve. Host b -> host x; DeviceArray b
    -> DeviceArray x."""
    from .grid import as_device_stencil

    opts = opts or SolveOptions()
    ds = as_device_stencil(stencil)
    d = grid.desc()
    rows = grid.unknown_count()
    rep = SolveReportC()
    o = _opts(opts)
    host = not isinstance(b, DeviceArray)
    bd = DeviceArray.from_host(np.ascontiguousarray(np.asarray(b, np.float64).ravel())) if host else b
    if bd.count != rows:
        raise StencilkitError(Errc.shape_mismatch, "rhs length does not match the grid")
    x = x_out if x_out is not None else DeviceArray(rows)
    try:
        check(ds.lib.sk_cg_solve_stencil(ds.handle, C.byref(d), bd.ptr, x.ptr, C.byref(o), C.byref(rep), stream))
    finally:
        if report is not None:
            report.iterations, report.restarts = rep.iterations, rep.restarts
            report.true_rel_residual, report.recurrence_rel_residual = rep.true_rel_residual, rep.recurrence_rel_residual
    return x.to_host() if host else x


# ------------------------------------------------------------ spectral --
def power_iteration(m: CsrMatrix, tol: float, seed: int = 20240801, max_iter: int = 2_000_000,
                    stream=None) -> float:
    """power_iteration (linalg.cpp:74-106): |Rayleigh quotient| from a seeded
    mt19937_64 start, geometric-tail stopping rule, the loop on the device."""
    if m.rows != m.cols:
        raise StencilkitError(Errc.shape_mismatch, "power iteration needs a square matrix")
    out, its = C.c_double(), C.c_int64()
    check(m.lib.sk_power_iteration(m.handle, tol, seed, max_iter, C.byref(out), C.byref(its), stream))
    power_iteration.last_iterations = its.value
    return out.value


@dataclass
class SpectrumReport:
    """linalg.hpp SpectrumReport"""
    eigenvalues: np.ndarray = None  # complex128, one per Fourier mode (x fastest)
    spectral_radius: float = 0.0
    symbol_radius: float = 0.0
    condition_estimate: float = 0.0  # max|lambda| / min nonzero |lambda|


def periodic_spectrum(stencil, grid, affine_shift: float = 0.0, affine_scale: float = 1.0) -> SpectrumReport:
    """periodic_spectrum (linalg.cpp:149-222) on the device."""
    from .grid import DeviceStencil

    ds = stencil if isinstance(stencil, DeviceStencil) else DeviceStencil(stencil)
    grid.validate()
    d = grid.desc()
    ev = np.empty(2 * grid.unknown_count())
    rho, sym, cond = C.c_double(), C.c_double(), C.c_double()
    check(ds.lib.sk_periodic_spectrum(ds.handle, C.byref(d), affine_shift, affine_scale, ev.ctypes.data,
                                      C.byref(rho), C.byref(sym), C.byref(cond)))
    return SpectrumReport(ev.view(np.complex128), rho.value, sym.value, cond.value)


@dataclass
class RefineReport:
    """sk_refine_report: CG iterations over all solves, refinement steps, the
    first solve's fp64 true residual, the exact-operator residual at return and
    the last correction's relative size."""
    iterations: int = 0
    refinements: int = 0
    initial_true_rel_residual: float = float("nan")
    refined_rel_residual: float = float("nan")
    last_correction_rel: float = float("nan")


def cg_solve_stencil_refined(stencil, grid, b, opts: SolveOptions | None = None, inner_rel_tol: float = 1e-6,
                             max_refinements: int = 4, report: RefineReport | None = None,
                             x_out: DeviceArray | None = None, stream=None):
    """Matrix-free CG, then iterative refinement against the exact composed
    operator (double-double residual): x converges to the solution of the
    exact-rational system instead of the fp64-weight one (sk_cg_solve_stencil_refined)."""
    from ._lib import RefineReportC
    from .grid import as_device_stencil

    opts = opts or SolveOptions()
    ds = as_device_stencil(stencil)
    d = grid.desc()
    rows = grid.unknown_count()
    rep = RefineReportC()
    o = _opts(opts)
    host = not isinstance(b, DeviceArray)
    db = DeviceArray.from_host(np.ascontiguousarray(b, np.float64)) if host else b
    x = x_out if x_out is not None else DeviceArray(rows)
    check(ds.lib.sk_cg_solve_stencil_refined(ds.handle, C.byref(d), db.ptr, x.ptr, C.byref(o), inner_rel_tol,
                                             max_refinements, C.byref(rep), stream))
    if report is not None:
        report.iterations, report.refinements = rep.iterations, rep.refinements
        report.initial_true_rel_residual = rep.initial_true_rel_residual
        report.refined_rel_residual, report.last_correction_rel = rep.refined_rel_residual, rep.last_correction_rel
    return x.to_host() if host else x
