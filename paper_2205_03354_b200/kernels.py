"""Device BLAS-1 + SpMV mirroring `stencilkit::kernels` (kernels.hpp:14-20).

Arguments are DeviceArray (device) — host numpy arrays are copied in for the
reductions so the reference's test shapes read the same.
"""
from __future__ import annotations

import ctypes as C
from typing import Tuple

import numpy as np

from ._lib import check, ensure_device
from .device import DeviceArray
from .errors import Errc, StencilkitError
from .grid import CsrMatrix


def _dev(x) -> DeviceArray:
    return x if isinstance(x, DeviceArray) else DeviceArray.from_host(np.asarray(x, dtype=np.float64).ravel())


def csr_matvec(m: CsrMatrix, x: DeviceArray, y: DeviceArray, stream=None) -> None:
    """y = M x (kernels.cpp:8-17); no size checks, as the reference."""
    check(m.lib.sk_csr_matvec(m.handle, x.ptr, y.ptr, stream))


def dot(a, b, stream=None) -> float:
    lib = ensure_device()
    da, db = _dev(a), _dev(b)
    out = C.c_double()
    check(lib.sk_dot(da.count, da.ptr, db.ptr, C.byref(out), stream))
    return out.value


def nrm2(a, stream=None) -> float:
    lib = ensure_device()
    da = _dev(a)
    out = C.c_double()
    check(lib.sk_nrm2(da.count, da.ptr, C.byref(out), stream))
    return out.value


def sum(a, stream=None) -> float:  # noqa: A001 - mirrors kernels::sum
    lib = ensure_device()
    da = _dev(a)
    out = C.c_double()
    check(lib.sk_sum(da.count, da.ptr, C.byref(out), stream))
    return out.value


def minmax(a, stream=None) -> Tuple[float, float]:
    lib = ensure_device()
    da = _dev(a)
    lo, hi = C.c_double(), C.c_double()
    check(lib.sk_minmax(da.count, da.ptr, C.byref(lo), C.byref(hi), stream))
    return lo.value, hi.value


def axpy(a: float, x: DeviceArray, y: DeviceArray, stream=None) -> None:
    """y += a x (kernels.cpp:29-33)."""
    if x.count != y.count:
        raise StencilkitError(Errc.shape_mismatch, "axpy length mismatch")
    check(ensure_device().sk_axpy(x.count, a, x.ptr, y.ptr, stream))


def xpby(x: DeviceArray, b: float, y: DeviceArray, stream=None) -> None:
    """y = x + b y (kernels.cpp:35-40)."""
    if x.count != y.count:
        raise StencilkitError(Errc.shape_mismatch, "xpby length mismatch")
    check(ensure_device().sk_xpby(x.count, x.ptr, b, y.ptr, stream))
