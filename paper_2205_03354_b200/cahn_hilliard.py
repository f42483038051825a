"""Fused explicit Cahn-Hilliard stepping and the free energy on the device.

Mirrors the reference's CahnHilliardParams / CahnHilliardState / free_energy
(cahn_hilliard.hpp:14-44) with the EXPLICIT forward-Euler step the BASELINE
configs specify (the reference's stepper is IMEX, cahn_hilliard.cpp:139-189;
SURVEY.md Appendix A restates the explicit step from its pieces):
    c <- c + dt M (L f'(c) - kappa B c),  L = laplacian(d, 2), B = compose(L, L)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from ._lib import ChParams, check, ensure_device
from .device import DeviceArray
from .errors import Errc, StencilkitError
from .grid import BoundaryKind, DeviceStencil, GridSpec
from .stencil import compose, laplacian


@dataclass
class CahnHilliardParams:
    """cahn_hilliard.hpp:14-22 (defaults are the reference's benchmark values)."""
    kappa: float = 2.0
    mobility: float = 5.0
    rho_w: float = 5.0
    c_alpha: float = 0.3
    c_beta: float = 0.7
    # device kernel: "factored" c + dt M L(f'(c) - kappa L c) or the literal
    # "composed" B = compose(L, L); identical in exact arithmetic
    formulation: str = "factored"

    @staticmethod
    def from_epsilon(eps: float, formulation: str = "factored") -> "CahnHilliardParams":
        """u_t = Delta(u^3 - u - eps^2 Delta u): f'(u) = u^3 - u <=> rho_w = 1/4, c_alpha = -1, c_beta = 1."""
        return CahnHilliardParams(kappa=eps * eps, mobility=1.0, rho_w=0.25, c_alpha=-1.0, c_beta=1.0,
                                  formulation=formulation)

    def c_struct(self) -> ChParams:
        p = ChParams()
        p.kappa, p.mobility, p.rho_w, p.c_alpha, p.c_beta = (self.kappa, self.mobility, self.rho_w, self.c_alpha,
                                                              self.c_beta)
        codes = {"factored": 0, "composed": 1}
        if self.formulation not in codes:
            raise StencilkitError(Errc.invalid_argument, f"unknown CH formulation '{self.formulation}'")
        p.formulation = codes[self.formulation]
        return p


@dataclass
class CahnHilliardState:
    grid: GridSpec
    c: np.ndarray
    t: float = 0.0
    energy_history: List[Tuple[float, float]] = field(default_factory=list)


class CahnHilliardExplicit:
    """Device stepper: L and B composed on the host, one fused kernel per step."""

    def __init__(self, grid: GridSpec, params: CahnHilliardParams):
        grid.validate()
        if any(b != BoundaryKind.periodic for b in grid.bc):
            raise StencilkitError(Errc.non_periodic, "Cahn-Hilliard runs on periodic grids")
        self.lib = ensure_device()
        self.grid = grid
        self.params = params
        lap = laplacian(grid.dim, 2)
        self.lap = DeviceStencil(lap)
        self.bilap = DeviceStencil(compose(lap, lap))
        self._desc = grid.desc()
        self._p = params.c_struct()

    def run_device(self, c: DeviceArray, scratch: DeviceArray, dt: float, nsteps: int, stream=None) -> DeviceArray:
        """nsteps fused steps ping-ponging c <-> scratch; returns the buffer holding the result."""
        which = C.c_int()
        check(self.lib.sk_ch_explicit(self.lap.handle, self.bilap.handle, C.byref(self._desc), C.byref(self._p),
                                      dt, nsteps, c.ptr, scratch.ptr, C.byref(which), stream))
        return scratch if which.value else c

    def run_host(self, c: np.ndarray, dt: float, nsteps: int) -> None:
        """nsteps steps on a contiguous float64 host field, in place. A pinned or
        registered field (kernels.host_register) of a 3D grid with nz >= 4 nsteps + 8
        overlaps the upload, the steps and the download (sk_ch_explicit_host)."""
        if c.dtype != np.float64 or not c.flags.c_contiguous or c.size != self.grid.unknown_count():
            raise StencilkitError(Errc.shape_mismatch, "host field must be contiguous float64 of the grid's size")
        check(self.lib.sk_ch_explicit_host(self.lap.handle, self.bilap.handle, C.byref(self._desc),
                                           C.byref(self._p), dt, nsteps, c.ctypes.data))

    def step(self, state: CahnHilliardState, dt: float, nsteps: int = 1) -> None:
        """Host state in/out (the reference-facing call): copies in, steps, copies out."""
        if not dt > 0:
            raise StencilkitError(Errc.invalid_argument, "dt must be positive")
        c = np.ascontiguousarray(state.c, dtype=np.float64).ravel().copy()
        if c.size != self.grid.unknown_count():
            raise StencilkitError(Errc.shape_mismatch, "state does not match the stepper grid")
        check(self.lib.sk_ch_explicit_host(self.lap.handle, self.bilap.handle, C.byref(self._desc),
                                           C.byref(self._p), dt, nsteps, c.ctypes.data))
        state.c = c
        state.t += dt * nsteps


def free_energy(state_or_field, params: CahnHilliardParams, grid: GridSpec | None = None, stream=None) -> float:
    """h^d sum [f_chem(c) + kappa/2 |central grad c|^2] (cahn_hilliard.cpp:77-114)."""
    lib = ensure_device()
    if isinstance(state_or_field, CahnHilliardState):
        grid = state_or_field.grid
        dev = DeviceArray.from_host(np.asarray(state_or_field.c, dtype=np.float64).ravel())
    elif isinstance(state_or_field, DeviceArray):
        dev = state_or_field
    else:
        dev = DeviceArray.from_host(np.asarray(state_or_field, dtype=np.float64).ravel())
    assert grid is not None
    d = grid.desc()
    p = params.c_struct()
    out = C.c_double()
    check(lib.sk_free_energy(C.byref(d), C.byref(p), dev.ptr, C.byref(out), stream))
    return out.value


# ------------------------------------------------------------------ IMEX ----
# The reference's own CH path (cahn_hilliard.cpp:121-189) on the device.

def ch_init(grid: GridSpec, c0: float = 0.5, eps_ic: float = 0.01) -> CahnHilliardState:
    """ch_init (cahn_hilliard.cpp:20-63): trigonometric initial condition, bit-identical."""
    grid.validate()
    if any(b != BoundaryKind.periodic for b in grid.bc):
        raise StencilkitError(Errc.non_periodic, "Cahn-Hilliard runs on periodic grids")
    lib = ensure_device()
    out = np.empty(grid.unknown_count())
    d = grid.desc()
    check(lib.sk_ch_init_host(C.byref(d), c0, eps_ic, out.ctypes.data))
    return CahnHilliardState(grid, out)


class CahnHilliardStepper:
    """IMEX stepper (cahn_hilliard.hpp:47-68): bi-Laplacian implicit (CG on the
    device), chemistry explicit; order 1 (backward/forward Euler) or 2
    (Crank-Nicolson + Adams-Bashforth 2, bootstrapped by one order-1 step and
    again whenever dt changes). The AB2 history and the implicit matrix cache
    live in the device stepper between calls, as in the reference."""

    def __init__(self, grid: GridSpec, params: CahnHilliardParams, solve=None):
        from .linalg import SolveOptions, _opts

        grid.validate()
        if any(b != BoundaryKind.periodic for b in grid.bc):
            raise StencilkitError(Errc.non_periodic, "Cahn-Hilliard runs on periodic grids")
        self.lib = ensure_device()
        self.grid = grid
        self.params = params
        self.solve = solve if solve is not None else SolveOptions(rel_tol=1e-12)
        self._desc = grid.desc()
        self._p = params.c_struct()
        self._o = _opts(self.solve)
        h = C.c_void_p()
        check(self.lib.sk_ch_imex_create(C.byref(self._desc), C.byref(self._p), C.byref(self._o), C.byref(h)))
        self.handle = h
        self.last_cg_iterations = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.sk_ch_imex_destroy(h)
            self.handle = None

    def step_device(self, c: DeviceArray, dt: float, order: int = 1, nsteps: int = 1, stream=None):
        """nsteps IMEX steps of the device field c in place; returns the last CG report."""
        from ._lib import SolveReportC
        from .linalg import SolveReport

        rep, its = SolveReportC(), C.c_int64()
        check(self.lib.sk_ch_imex_step(self.handle, c.ptr, dt, order, nsteps, C.byref(rep), C.byref(its), stream))
        self.last_cg_iterations = its.value
        return SolveReport(rep.iterations, rep.restarts, rep.true_rel_residual, rep.recurrence_rel_residual)

    def step(self, state: CahnHilliardState, dt: float, order: int = 1, nsteps: int = 1) -> None:
        """Host state in/out (CahnHilliardStepper::step, :139-189)."""
        c = np.ascontiguousarray(state.c, dtype=np.float64).ravel()
        if c.size != self.grid.unknown_count():
            raise StencilkitError(Errc.shape_mismatch, "state does not match the stepper grid")
        dev = DeviceArray.from_host(c)
        self.step_device(dev, dt, order, nsteps)
        state.c = dev.to_host()
        state.t += dt * nsteps

    def reset_history(self) -> None:
        check(self.lib.sk_ch_imex_reset_history(self.handle))

    def matrix(self, which: str = "implicit"):
        """(row_ptr, col_idx, values) of L ('laplacian'), B ('bilaplacian') or the cached implicit matrix."""
        code = {"laplacian": 0, "bilaplacian": 1, "implicit": 2}[which]
        m = C.c_void_p()
        check(self.lib.sk_ch_imex_matrix(self.handle, code, C.byref(m)))
        rows, cols, nnz, bits = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        check(self.lib.sk_csr_info(m, C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(bits)))
        rp = np.empty(rows.value + 1, np.int64)
        ci = np.empty(max(nnz.value, 1), np.int64)
        v = np.empty(max(nnz.value, 1))
        check(self.lib.sk_csr_download(m, rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
        return rp, ci[: nnz.value], v[: nnz.value]


def imex_step(stepper: CahnHilliardStepper, state: CahnHilliardState, dt: float, order: int) -> None:
    """imex_step (cahn_hilliard.cpp:191-193)."""
    stepper.step(state, dt, order)
