"""Experiment drivers over the device path (experiments.hpp / experiments.cpp).

fit_loglog (experiments.cpp:16-42), ch_benchmark (:145-184) and
ch_temporal_convergence (:186-218). The CH drivers run the IMEX stepper
(cahn_hilliard.CahnHilliardStepper) with the field resident on the device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from .cahn_hilliard import CahnHilliardParams, CahnHilliardState, CahnHilliardStepper, ch_init, free_energy
from .device import DeviceArray
from .errors import Errc, StencilkitError


@dataclass
class ConvergenceFit:
    """experiments.hpp ConvergenceFit: err ~ coefficient * h^slope."""
    slope: float = 0.0
    coefficient: float = 0.0
    fit_residual: float = 0.0
    samples: List[Tuple[float, float]] = field(default_factory=list)


def fit_loglog(samples: Sequence[Tuple[float, float]]) -> ConvergenceFit:
    """Least squares of log(err) against log(h) (experiments.cpp:16-42), same sums."""
    samples = list(samples)
    if len(samples) < 3:
        raise StencilkitError(Errc.invalid_argument, "a convergence fit needs at least 3 samples")
    sx = sy = sxx = sxy = 0.0
    n = float(len(samples))
    for h, err in samples:
        if not (h > 0) or not (err > 0):
            raise StencilkitError(Errc.invalid_argument, "convergence samples must be positive")
        lx, ly = math.log(h), math.log(err)
        sx += lx
        sy += ly
        sxx += lx * lx
        sxy += lx * ly
    slope = (n * sxy - sx * sy) / (n * sxx - sx * sx)
    intercept = (sy - slope * sx) / n
    rss = 0.0
    for h, err in samples:
        r = math.log(err) - (slope * math.log(h) + intercept)
        rss += r * r
    return ConvergenceFit(slope, math.exp(intercept), math.sqrt(rss / n), samples)


@dataclass
class ChBenchmarkOptions:
    """experiments.hpp:44-54"""
    dim: int = 2
    n: int = 100
    h: float = 1.0
    dt: float = 0.05
    t_end: float = 100.0
    order: int = 1
    energy_every: int = 1
    snapshot_hook: object = None
    snapshot_every: int = 0


@dataclass
class ChBenchmarkResult:
    """experiments.hpp:56-63"""
    state: CahnHilliardState = None
    mass_initial: float = 0.0
    mass_final: float = 0.0
    mass_rel_drift_max: float = 0.0
    c_min: float = 0.0
    c_max: float = 0.0
    energy_monotone_after_first: bool = True
    max_energy_uptick: float = 0.0
    cg_iterations: int = 0


def ch_benchmark(opts: ChBenchmarkOptions, params: CahnHilliardParams | None = None) -> ChBenchmarkResult:
    """ch_benchmark (experiments.cpp:145-184): the field stays on the device;
    mass, extrema and free energy are device reductions per step."""
    from .grid import make_periodic_grid
    from .kernels import minmax
    from .kernels import sum as sum_

    params = params or CahnHilliardParams()
    grid = make_periodic_grid(opts.dim, opts.n, opts.h)
    state = ch_init(grid)
    stepper = CahnHilliardStepper(grid, params)
    dev = DeviceArray.from_host(state.c)
    res = ChBenchmarkResult()
    res.mass_initial = sum_(dev)
    state.energy_history.append((0.0, free_energy(dev, params, grid)))
    res.c_min, res.c_max = minmax(dev)
    steps = int(round(opts.t_end / opts.dt))
    prev_energy = state.energy_history[-1][1]
    for k in range(1, steps + 1):
        stepper.step_device(dev, opts.dt, opts.order)
        res.cg_iterations += stepper.last_cg_iterations
        state.t += opts.dt
        mass = sum_(dev)
        res.mass_rel_drift_max = max(res.mass_rel_drift_max, abs(mass - res.mass_initial) / abs(res.mass_initial))
        lo, hi = minmax(dev)
        res.c_min, res.c_max = min(res.c_min, lo), max(res.c_max, hi)
        if opts.energy_every > 0 and (k % opts.energy_every == 0 or k == steps):
            energy = free_energy(dev, params, grid)
            state.energy_history.append((state.t, energy))
            if k > 1 and energy > prev_energy:
                res.energy_monotone_after_first = False
                res.max_energy_uptick = max(res.max_energy_uptick, energy - prev_energy)
            prev_energy = energy
        if opts.snapshot_every > 0 and opts.snapshot_hook and k % opts.snapshot_every == 0:
            state.c = dev.to_host()
            opts.snapshot_hook(state, k)
    state.c = dev.to_host()
    res.mass_final = sum_(dev)
    res.state = state
    return res


@dataclass
class TemporalFit:
    """experiments.hpp TemporalFit"""
    order: int = 0
    fit: ConvergenceFit = None


def ch_temporal_convergence(dim: int, orders=(1, 2), n: int = 32, t_end: float = 10.0, dt_ladder=None,
                            ref_dt: float = 1.0 / 1024.0, params: CahnHilliardParams | None = None):
    """ch_temporal_convergence (experiments.cpp:186-218): errors at t_end against
    one fine-step order-2 reference, one log-log fit per scheme order."""
    from .grid import make_periodic_grid

    params = params or CahnHilliardParams()
    dt_ladder = list(dt_ladder or [1 / 2, 1 / 4, 1 / 8, 1 / 16, 1 / 32])
    grid = make_periodic_grid(dim, n, 1.0)
    initial = ch_init(grid).c

    def run(dt, order):
        stepper = CahnHilliardStepper(grid, params)
        dev = DeviceArray.from_host(initial)
        stepper.step_device(dev, dt, order, int(round(t_end / dt)))
        return dev.to_host()

    reference = run(ref_dt, 2)
    ref_norm = float(np.sqrt(np.sum(reference * reference)))
    fits = []
    for order in orders:
        samples = []
        for dt in dt_ladder:
            c = run(dt, order)
            samples.append((dt, float(np.sqrt(np.sum((c - reference) ** 2)) / ref_norm)))
        fits.append(TemporalFit(order, fit_loglog(samples)))
    return fits


@dataclass
class BiharmonicResult:
    """experiments.hpp BiharmonicResult"""
    fit: ConvergenceFit = None
    residuals: List[float] = field(default_factory=list)  # relative solver residual per ladder point


def biharmonic_solve(interval_ladder: Sequence[int] = (8, 16, 32, 64), rel_tol: float = 1e-10,
                     matrix_free: bool = False) -> BiharmonicResult:
    """biharmonic_solve (experiments.cpp:99-143) on the device: the simply-supported
    plate Delta^2 u = 4 pi^4 sin(pi x) sin(pi y) on the unit square, GPU assembly of
    compose(laplacian(2, 2), itself), device CG (CSR, or the matrix-free operator),
    max-norm error fit and relative residuals ||b - M x|| / ||b||."""
    from .grid import BoundaryKind, DeviceStencil, GridSpec, assemble
    from .kernels import csr_matvec
    from .linalg import SolveOptions, cg_solve, cg_solve_stencil
    from .stencil import compose, laplacian

    lap = laplacian(2, 2)
    bilap = DeviceStencil(compose(lap, lap))
    result = BiharmonicResult()
    samples = []
    for intervals in interval_ladder:
        h = 1.0 / intervals
        g = GridSpec(dim=2, n=[intervals + 1] * 2, h=h, origin=[0.0, 0.0],
                     bc=[BoundaryKind.simply_supported] * 2)
        m = assemble(bilap, g)
        nu = intervals - 1
        coord = (np.arange(nu) + 1) * h  # GridSpec::coordinate (grid.cpp:37-40), simply supported
        sxy = np.outer(np.sin(math.pi * coord), np.sin(math.pi * coord)).ravel()  # row = j * nu + i
        b = 4.0 * math.pow(math.pi, 4) * sxy
        opts = SolveOptions(rel_tol=rel_tol)
        x = cg_solve_stencil(bilap, g, b, opts) if matrix_free else cg_solve(m, b, opts)
        samples.append((h, float(np.max(np.abs(x - sxy)))))
        xd = DeviceArray.from_host(x)
        mx = DeviceArray(m.rows)
        csr_matvec(m, xd, mx)
        r = b - mx.to_host()
        result.residuals.append(math.sqrt(float(np.dot(r, r)) / float(np.dot(b, b))))
    result.fit = fit_loglog(samples)
    return result
