"""Device-resident fp64 vectors allocated through the C-ABI (no torch needed)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, ensure_device


class DeviceArray:
    """A contiguous fp64 (or int64) buffer in HBM, owned by this object."""

    def __init__(self, count: int, dtype=np.float64):
        self.lib = ensure_device()
        self.count = int(count)
        self.dtype = np.dtype(dtype)
        self.nbytes = self.count * self.dtype.itemsize
        p = C.c_void_p()
        check(self.lib.sk_device_alloc(self.nbytes, C.byref(p)))
        self._ptr = p.value

    @property
    def ptr(self) -> int:
        return self._ptr or 0

    @classmethod
    def from_host(cls, a: np.ndarray, stream=None) -> "DeviceArray":
        a = np.ascontiguousarray(a)
        d = cls(a.size, a.dtype)
        d.upload(a, stream)
        return d

    def upload(self, a: np.ndarray, stream=None) -> None:
        a = np.ascontiguousarray(a, dtype=self.dtype)
        assert a.size == self.count
        check(self.lib.sk_memcpy_h2d(self.ptr, a.ctypes.data, self.nbytes, stream))
        check(self.lib.sk_stream_sync(stream))

    def to_host(self, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        if out is None:
            out = np.empty(self.count, dtype=self.dtype)
        check(self.lib.sk_memcpy_d2h(out.ctypes.data, self.ptr, self.nbytes, stream))
        return out

    def free(self) -> None:
        if self._ptr:
            self.lib.sk_device_free(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __len__(self) -> int:
        return self.count


class pinned:
    """Page-lock a contiguous numpy array for the duration of a `with` block
    (sk_host_register / sk_host_unregister), so host entry points can overlap
    their copies with device work."""

    def __init__(self, arr: np.ndarray):
        if not arr.flags.c_contiguous:
            raise ValueError("pinned() needs a contiguous array")
        self.arr = arr

    def __enter__(self) -> np.ndarray:
        check(ensure_device().sk_host_register(self.arr.ctypes.data, self.arr.nbytes))
        return self.arr

    def __exit__(self, *exc) -> None:
        check(ensure_device().sk_host_unregister(self.arr.ctypes.data))
