"""Grids, device stencils, CSR assembly and the composed apply.

Python mirror of the reference's L2 interface (grid.hpp:15-56) over the
C-ABI: `GridSpec`, `BoundaryKind`, `make_periodic_grid`, `assemble`,
`sparsity_report`, `apply`; plus the matrix-free `composed_apply` that the
reference lacks (its apply is always assemble + csr_matvec, grid.cpp:166-172).
"""
from __future__ import annotations

import ctypes as C
from fractions import Fraction
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from ._lib import GridDesc, check, ensure_device
from .device import DeviceArray
from .errors import Errc, StencilkitError
from .stencil import Stencil


class BoundaryKind(enum.IntEnum):
    periodic = 0
    simply_supported = 1  # odd reflection (grid.cpp:108-122)
    clamped = 2           # even reflection: u = du/dn = 0 (BASELINE configs 2, 5)


@dataclass
class GridSpec:
    """grid.hpp:22-34: n = points per axis INCLUDING boundary points."""
    dim: int = 1
    n: List[int] = field(default_factory=lambda: [3])
    h: float = 1.0
    origin: List[float] = field(default_factory=lambda: [0.0])
    bc: List[BoundaryKind] = field(default_factory=lambda: [BoundaryKind.periodic])

    def validate(self) -> None:  # grid.cpp:17-25
        if self.dim < 1:
            raise StencilkitError(Errc.invalid_argument, "grid dimension must be >= 1")
        if len(self.n) != self.dim or len(self.origin) != self.dim or len(self.bc) != self.dim:
            raise StencilkitError(Errc.dim_mismatch, "grid axis arrays do not match dimension")
        if any(v < 3 for v in self.n):
            raise StencilkitError(Errc.invalid_argument, "grid needs at least 3 points per axis")
        if not self.h > 0:
            raise StencilkitError(Errc.invalid_argument, "grid spacing must be positive")

    def unknowns_per_axis(self, axis: int) -> int:
        return self.n[axis] if self.bc[axis] == BoundaryKind.periodic else self.n[axis] - 2

    def unknown_count(self) -> int:
        total = 1
        for a in range(self.dim):
            total *= self.unknowns_per_axis(a)
        return total

    def coordinate(self, axis: int, unknown_index) -> np.ndarray:
        gi = unknown_index if self.bc[axis] == BoundaryKind.periodic else np.asarray(unknown_index) + 1
        return self.origin[axis] + np.asarray(gi) * self.h

    def shape(self) -> Tuple[int, ...]:
        """numpy shape of a field (slowest axis first; x fastest)."""
        return tuple(self.unknowns_per_axis(a) for a in reversed(range(self.dim)))

    def desc(self) -> GridDesc:
        self.validate()
        d = GridDesc()
        d.dim = self.dim
        d.h = self.h
        for a in range(3):
            d.n[a] = self.n[a] if a < self.dim else 1
            d.bc[a] = int(self.bc[a]) if a < self.dim else 0
        return d


def make_periodic_grid(dim: int, n_per_axis: int, h: float, origin: float = 0.0) -> GridSpec:
    g = GridSpec(dim, [n_per_axis] * dim, h, [origin] * dim, [BoundaryKind.periodic] * dim)
    g.validate()
    return g


def make_grid(dim: int, n_per_axis: int, h: float, bc: BoundaryKind) -> GridSpec:
    g = GridSpec(dim, [n_per_axis] * dim, h, [0.0] * dim, [bc] * dim)
    g.validate()
    return g


class DeviceStencil:
    """A composed stencil uploaded for the device kernels (sk_stencil_create)."""

    def __init__(self, s: Stencil):
        self.lib = ensure_device()
        self.stencil = s
        offs, coeffs = s.flat()
        # exact-weight corrections (only the refined residual uses them):
        # coefficient - to_double(coefficient), exactly, rounded once
        lows = [float(q - Fraction(d)) for q, d in zip(s.entries.values(), coeffs)]
        o = (C.c_int32 * len(offs))(*offs)
        c = (C.c_double * len(coeffs))(*coeffs)
        lo = (C.c_double * len(lows))(*lows)
        h = C.c_void_p()
        check(self.lib.sk_stencil_create_exact(s.dim, len(coeffs), o, c, lo, s.h_power, C.byref(h)))
        self.handle = h.value

    @property
    def kernel_class(self) -> int:
        return self.lib.sk_stencil_kernel_class(self.handle)

    def __del__(self):
        try:
            if self.handle:
                self.lib.sk_stencil_destroy(self.handle)
        except Exception:
            pass


def as_device_stencil(s) -> DeviceStencil:
    return s if isinstance(s, DeviceStencil) else DeviceStencil(s)


class CsrMatrix:
    """Device-resident CSR (grid.hpp:39-46). Download with to_host()."""

    def __init__(self, handle: int):
        self.lib = ensure_device()
        self.handle = handle
        rows, cols, nnz, bits = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        check(self.lib.sk_csr_info(handle, C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(bits)))
        self.rows, self.cols, self._nnz, self.index_bits = rows.value, cols.value, nnz.value, bits.value

    def nnz(self) -> int:
        return self._nnz

    @classmethod
    def upload(cls, row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, cols: Optional[int] = None,
               index_bits: int = 64) -> "CsrMatrix":
        lib = ensure_device()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        rows = rp.size - 1
        h = C.c_void_p()
        check(lib.sk_csr_upload(rows, rows if cols is None else cols, v.size, rp.ctypes.data, ci.ctypes.data,
                                v.ctypes.data, index_bits, C.byref(h)))
        return cls(h.value)

    def to_host(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        rp = np.empty(self.rows + 1, np.int64)
        ci = np.empty(max(self._nnz, 1), np.int64)
        v = np.empty(max(self._nnz, 1), np.float64)
        check(self.lib.sk_csr_download(self.handle, rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
        return rp, ci[: self._nnz], v[: self._nnz]

    def __del__(self):
        try:
            if self.handle:
                self.lib.sk_csr_destroy(self.handle)
        except Exception:
            pass


def assemble(s, g: GridSpec, index_bits: int = 64, stream=None) -> CsrMatrix:
    """GPU assembly, same rows/columns/values as assemble (grid.cpp:62-158)."""
    ds = as_device_stencil(s)
    d = g.desc()
    h = C.c_void_p()
    check(ds.lib.sk_csr_assemble(ds.handle, C.byref(d), index_bits, C.byref(h), stream))
    check(ds.lib.sk_stream_sync(stream))
    return CsrMatrix(h.value)


def assemble_into(s, g: GridSpec, m: "CsrMatrix", stream=None) -> "CsrMatrix":
    """Re-assemble the operator into an existing matrix of the same shape (sk_csr_assemble_into)."""
    ds = as_device_stencil(s)
    d = g.desc()
    check(ds.lib.sk_csr_assemble_into(ds.handle, C.byref(d), m.handle, stream))
    return m


def csr_matmul(b: CsrMatrix, a: CsrMatrix, stream=None) -> CsrMatrix:
    """b * a on the device (linalg.cpp:253-283), bit-identical values."""
    if b.cols != a.rows:
        raise StencilkitError(Errc.shape_mismatch, "inner dimensions do not match")
    h = C.c_void_p()
    check(b.lib.sk_csr_matmul(b.handle, a.handle, C.byref(h), stream))
    return CsrMatrix(h.value)


def sparsity_report(m: CsrMatrix) -> Tuple[int, float]:
    """(nnz, fill percentage), grid.cpp:160-164."""
    return m.nnz(), 100.0 * float(m.nnz()) / (float(m.rows) * float(m.cols))


def _as_device(x) -> Tuple[DeviceArray, bool]:
    if isinstance(x, DeviceArray):
        return x, False
    return DeviceArray.from_host(np.asarray(x, dtype=np.float64).ravel()), True


def apply(m: CsrMatrix, x) -> np.ndarray:
    """grid.cpp:166-172: y = M x with a shape check; host in, host out."""
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    if xs.size != m.cols:
        raise StencilkitError(Errc.shape_mismatch, "vector length does not match matrix columns")
    y = np.empty(m.rows, np.float64)
    check(m.lib.sk_csr_matvec_host(m.handle, xs.ctypes.data, y.ctypes.data))
    return y


def composed_apply(s, g: GridSpec, u, out: Optional[DeviceArray] = None, stream=None):
    """Matrix-free v = S u. Host array in -> host array out; DeviceArray in -> DeviceArray out."""
    ds = as_device_stencil(s)
    d = g.desc()
    if isinstance(u, DeviceArray):
        if u.count != g.unknown_count():
            raise StencilkitError(Errc.shape_mismatch, "field length does not match the grid")
        v = out if out is not None else DeviceArray(u.count)
        check(ds.lib.sk_composed_apply(ds.handle, C.byref(d), u.ptr, v.ptr, stream))
        return v
    us = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel())
    if us.size != g.unknown_count():
        raise StencilkitError(Errc.shape_mismatch, "field length does not match the grid")
    v = np.empty_like(us)
    check(ds.lib.sk_composed_apply_host(ds.handle, C.byref(d), us.ctypes.data, v.ctypes.data))
    return v


def composed_apply_repeat(s, g: GridSpec, u: DeviceArray, v0: DeviceArray, v1: DeviceArray, repeats: int,
                          stream=None) -> None:
    """`repeats` applications to the same u, outputs ping-ponging (BASELINE config 1), one CUDA graph."""
    ds = as_device_stencil(s)
    d = g.desc()
    check(ds.lib.sk_composed_apply_repeat(ds.handle, C.byref(d), u.ptr, v0.ptr, v1.ptr, repeats, stream))


def residual_refined(s, g: GridSpec, b, x) -> np.ndarray:
    """b - A x with the composed stencil's EXACT weights, in double-double (sk_residual_refined)."""
    ds = as_device_stencil(s)
    db, hb = _as_device(b)
    dx, _ = _as_device(x)
    r = DeviceArray(g.unknown_count())
    d = g.desc()
    check(ds.lib.sk_residual_refined(ds.handle, C.byref(d), db.ptr, dx.ptr, r.ptr, None))
    return r.to_host() if hb else r
