"""ORACLE TEST INFRASTRUCTURE — ctypes access to the CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module. Two checkers:
  * `Oracle`    — oracle/_ref/libsk_oracle.so, the plain-C restatement
                  (oracle/sk_oracle.c); builds anywhere gcc exists.
  * `Reference` — oracle/_ref/libstencilkit_ref.so, the UNMODIFIED reference
                  sources + oracle/ref_capi.cpp (built here from
                  /root/reference; the prebuilt .so travels to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_ref" / "libsk_oracle.so"
REF_SO = HERE / "_ref" / "libstencilkit_ref.so"

vp = C.c_void_p
i64 = C.c_int64
dbl = C.c_double


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "_ref/libsk_oracle.so"], check=True)


class SkoCsr(C.Structure):
    _fields_ = [("rows", i64), ("cols", i64), ("nnz", i64), ("row_ptr", C.POINTER(i64)),
                ("col_idx", C.POINTER(i64)), ("values", C.POINTER(dbl))]


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _flat(stencil):
    offs, coeffs = stencil.flat()
    return (np.ascontiguousarray(offs, dtype=np.int32), np.ascontiguousarray(coeffs, dtype=np.float64))


def _grid_arrays(grid):
    n = np.ones(3, np.int64)
    bc = np.zeros(3, np.int32)
    for a in range(grid.dim):
        n[a] = grid.n[a]
        bc[a] = int(grid.bc[a])
    return n, bc


class Oracle:
    def __init__(self):
        if not ORACLE_SO.exists():
            build_oracle()
        L = C.CDLL(str(ORACLE_SO))
        L.sko_assemble.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, dbl, vp, C.POINTER(SkoCsr)]
        L.sko_assemble_row.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, dbl, vp, i64, vp, vp]
        L.sko_csr_free.argtypes = [C.POINTER(SkoCsr)]
        L.sko_csr_matvec.argtypes = [C.POINTER(SkoCsr), vp, vp]
        for f in ("sko_dot",):
            getattr(L, f).argtypes = [i64, vp, vp]
            getattr(L, f).restype = dbl
        L.sko_nrm2.argtypes = [i64, vp]
        L.sko_nrm2.restype = dbl
        L.sko_sum.argtypes = [i64, vp]
        L.sko_sum.restype = dbl
        L.sko_minmax.argtypes = [i64, vp, C.POINTER(dbl), C.POINTER(dbl)]
        L.sko_axpy.argtypes = [i64, dbl, vp, vp]
        L.sko_xpby.argtypes = [i64, vp, dbl, vp]
        L.sko_cg_solve.argtypes = [C.POINTER(SkoCsr), vp, vp, dbl, i64, C.c_int, C.POINTER(i64), C.POINTER(dbl)]
        L.sko_apply_direct.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, dbl, vp, vp, vp]
        L.sko_ch_explicit.argtypes = [C.c_int, i64, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64, vp]
        L.sko_ch_explicit_dims.argtypes = [C.c_int, vp, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64, vp]
        L.sko_ch_imex.argtypes = [C.c_int, i64, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, C.c_int, i64, vp]
        L.sko_ch_init.argtypes = [C.c_int, i64, dbl, dbl, dbl, vp]
        L.sko_ch_imex_seq.argtypes = [C.c_int, i64, dbl, dbl, dbl, dbl, dbl, dbl, dbl, C.c_int, vp, vp, vp, vp]
        L.sko_identity_plus_scaled.argtypes = [C.POINTER(SkoCsr), dbl, C.POINTER(SkoCsr)]
        L.sko_csr_matmul.argtypes = [C.POINTER(SkoCsr), C.POINTER(SkoCsr), C.POINTER(SkoCsr)]
        L.sko_power_iteration.argtypes = [C.POINTER(SkoCsr), dbl, C.c_uint64, i64, C.POINTER(dbl), C.POINTER(i64)]
        L.sko_periodic_eigen.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, dbl, dbl, dbl, vp, C.POINTER(dbl),
                                         C.POINTER(dbl)]
        L.sko_free_energy.argtypes = [C.c_int, i64, dbl, dbl, dbl, dbl, dbl, vp]
        L.sko_free_energy.restype = dbl
        L.sko_biharmonic_clamped.argtypes = [C.c_int, i64, vp, vp]
        L.sko_fit_loglog.argtypes = [C.c_int, vp, vp, C.POINTER(dbl), C.POINTER(dbl), C.POINTER(dbl)]
        L.sko_uniform.argtypes = [C.c_uint64, i64, dbl, dbl, vp]
        L.sko_threads.restype = C.c_int
        self.L = L

    def threads(self) -> int:
        return self.L.sko_threads()

    def assemble(self, stencil, grid) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        off, co = _flat(stencil)
        n, bc = _grid_arrays(grid)
        m = SkoCsr()
        st = self.L.sko_assemble(stencil.dim, co.size, _p(off), _p(co), stencil.h_power, _p(n), grid.h, _p(bc),
                                 C.byref(m))
        if st:
            raise ValueError(f"oracle assemble failed with status {st}")
        rp = np.ctypeslib.as_array(m.row_ptr, shape=(m.rows + 1,)).copy()
        ci = np.ctypeslib.as_array(m.col_idx, shape=(max(m.nnz, 1),))[: m.nnz].copy()
        v = np.ctypeslib.as_array(m.values, shape=(max(m.nnz, 1),))[: m.nnz].copy()
        self.L.sko_csr_free(C.byref(m))
        return rp, ci, v

    def assemble_row(self, stencil, grid, row: int) -> Tuple[np.ndarray, np.ndarray]:
        off, co = _flat(stencil)
        n, bc = _grid_arrays(grid)
        cols = np.empty(co.size, np.int64)
        vals = np.empty(co.size, np.float64)
        cnt = self.L.sko_assemble_row(stencil.dim, co.size, _p(off), _p(co), stencil.h_power, _p(n), grid.h, _p(bc),
                                      row, _p(cols), _p(vals))
        if cnt < 0:
            raise ValueError(f"oracle assemble_row failed with status {-cnt}")
        return cols[:cnt], vals[:cnt]

    @staticmethod
    def _csr(rp, ci, v) -> SkoCsr:
        m = SkoCsr()
        m.rows = m.cols = rp.size - 1
        m.nnz = v.size
        m.row_ptr = rp.ctypes.data_as(C.POINTER(i64))
        m.col_idx = ci.ctypes.data_as(C.POINTER(i64))
        m.values = v.ctypes.data_as(C.POINTER(dbl))
        return m

    def csr_matvec(self, rp, ci, v, x) -> np.ndarray:
        rp, ci, v = (np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int64),
                     np.ascontiguousarray(v, np.float64))
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(rp.size - 1)
        m = self._csr(rp, ci, v)
        self.L.sko_csr_matvec(C.byref(m), _p(x), _p(y))
        return y

    def cg_solve(self, rp, ci, v, b, rel_tol=1e-10, max_iter=0, deflate_mean=False):
        rp, ci, v = (np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int64),
                     np.ascontiguousarray(v, np.float64))
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        it, tr = i64(), dbl()
        m = self._csr(rp, ci, v)
        st = self.L.sko_cg_solve(C.byref(m), _p(b), _p(x), rel_tol, max_iter, int(deflate_mean), C.byref(it),
                                 C.byref(tr))
        return x, st, it.value, tr.value

    def apply_direct(self, stencil, grid, u) -> np.ndarray:
        off, co = _flat(stencil)
        n, bc = _grid_arrays(grid)
        u = np.ascontiguousarray(u, np.float64).ravel()
        v = np.empty_like(u)
        self.L.sko_apply_direct(stencil.dim, co.size, _p(off), _p(co), stencil.h_power, _p(n), grid.h, _p(bc),
                                _p(u), _p(v))
        return v

    def ch_explicit(self, dim, n, h, params, dt, nsteps, c) -> np.ndarray:
        c = np.ascontiguousarray(c, np.float64).ravel().copy()
        st = self.L.sko_ch_explicit(dim, n, h, params.mobility, params.kappa, params.rho_w, params.c_alpha,
                                    params.c_beta, dt, nsteps, _p(c))
        if st:
            raise ValueError(f"oracle ch_explicit failed with status {st}")
        return c

    def ch_explicit_dims(self, dims, h, params, dt, nsteps, c) -> np.ndarray:
        """explicit CH on a non-cubic periodic grid (dims: points per axis)"""
        c = np.ascontiguousarray(c, np.float64).ravel().copy()
        nd = np.ascontiguousarray(list(dims) + [1] * (3 - len(dims)), np.int64)
        st = self.L.sko_ch_explicit_dims(len(dims), _p(nd), h, params.mobility, params.kappa, params.rho_w,
                                         params.c_alpha, params.c_beta, dt, nsteps, _p(c))
        if st:
            raise ValueError(f"oracle ch_explicit failed with status {st}")
        return c

    def ch_imex(self, dim, n, h, params, dt, order, nsteps, c, rel_tol=1e-12) -> np.ndarray:
        """IMEX steps from a fresh stepper (cahn_hilliard.cpp:121-189), serial CG."""
        c = np.ascontiguousarray(c, np.float64).ravel().copy()
        st = self.L.sko_ch_imex(dim, n, h, params.mobility, params.kappa, params.rho_w, params.c_alpha,
                                params.c_beta, rel_tol, dt, order, nsteps, _p(c))
        if st:
            raise ValueError(f"oracle ch_imex failed with status {st}")
        return c

    def ch_imex_seq(self, dim, n, h, params, seq, c, rel_tol=1e-12) -> np.ndarray:
        """IMEX legs [(dt, order, steps), ...] on one fresh stepper (AB2 history across legs)."""
        c = np.ascontiguousarray(c, np.float64).ravel().copy()
        dts = np.ascontiguousarray([float(s[0]) for s in seq], np.float64)
        orders = np.ascontiguousarray([int(s[1]) for s in seq], np.int32)
        steps = np.ascontiguousarray([int(s[2]) for s in seq], np.int64)
        st = self.L.sko_ch_imex_seq(dim, n, h, params.mobility, params.kappa, params.rho_w, params.c_alpha,
                                    params.c_beta, rel_tol, len(seq), _p(dts), _p(orders), _p(steps), _p(c))
        if st:
            raise ValueError(f"oracle ch_imex_seq failed with status {st}")
        return c

    def ch_init(self, dim, n, h, c0, eps) -> np.ndarray:
        out = np.empty(n ** dim)
        self.L.sko_ch_init(dim, n, h, c0, eps, _p(out))
        return out

    def csr_matmul(self, b, a):
        """b, a: (row_ptr, col_idx, values) triples -> the product triple (linalg.cpp:253-283)."""
        def mk(t, keep):
            m = SkoCsr()
            rp, ci, v = (np.ascontiguousarray(t[0], np.int64), np.ascontiguousarray(t[1], np.int64),
                         np.ascontiguousarray(t[2], np.float64))
            keep += [rp, ci, v]
            m.rows = rp.size - 1
            m.cols = int(ci.max()) + 1 if ci.size else 0
            m.nnz = ci.size
            m.row_ptr = rp.ctypes.data_as(C.POINTER(C.c_int64))
            m.col_idx = ci.ctypes.data_as(C.POINTER(C.c_int64))
            m.values = v.ctypes.data_as(C.POINTER(C.c_double))
            return m
        keep = []
        mb, ma, out = mk(b, keep), mk(a, keep), SkoCsr()
        ma.cols = max(ma.cols, ma.rows)
        self.L.sko_csr_matmul(C.byref(mb), C.byref(ma), C.byref(out))
        r = np.ctypeslib.as_array(out.row_ptr, shape=(out.rows + 1,)).copy()
        c = np.ctypeslib.as_array(out.col_idx, shape=(max(out.nnz, 1),))[: out.nnz].copy()
        v = np.ctypeslib.as_array(out.values, shape=(max(out.nnz, 1),))[: out.nnz].copy()
        self.L.sko_csr_free(C.byref(out))
        return r, c, v

    def power_iteration(self, rp, ci, vals, tol, seed=20240801, max_iter=2_000_000):
        m = SkoCsr()
        rp = np.ascontiguousarray(rp, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        m.rows = m.cols = rp.size - 1
        m.nnz = ci.size
        m.row_ptr = rp.ctypes.data_as(C.POINTER(C.c_int64))
        m.col_idx = ci.ctypes.data_as(C.POINTER(C.c_int64))
        m.values = vals.ctypes.data_as(C.POINTER(C.c_double))
        out, its = dbl(), i64()
        if self.L.sko_power_iteration(C.byref(m), tol, seed, max_iter, C.byref(out), C.byref(its)):
            raise ValueError("oracle power iteration did not settle")
        return out.value, its.value

    def periodic_eigen(self, stencil, grid, shift=0.0, scale=1.0):
        off, co = _flat(stencil)
        n, _ = _grid_arrays(grid)
        modes = int(np.prod(n[: stencil.dim]))
        eig = np.empty(2 * modes)
        rho, cond = dbl(), dbl()
        self.L.sko_periodic_eigen(stencil.dim, co.size, _p(off), _p(co), stencil.h_power, _p(n), grid.h, shift, scale,
                                  _p(eig), C.byref(rho), C.byref(cond))
        return eig.view(np.complex128), rho.value, cond.value

    def identity_plus_scaled(self, rp, ci, vals, alpha):
        m, out = SkoCsr(), SkoCsr()
        rp = np.ascontiguousarray(rp, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        m.rows = m.cols = rp.size - 1
        m.nnz = ci.size
        m.row_ptr = rp.ctypes.data_as(C.POINTER(C.c_int64))
        m.col_idx = ci.ctypes.data_as(C.POINTER(C.c_int64))
        m.values = vals.ctypes.data_as(C.POINTER(C.c_double))
        if self.L.sko_identity_plus_scaled(C.byref(m), alpha, C.byref(out)):
            raise MemoryError("identity_plus_scaled")
        r = np.ctypeslib.as_array(out.row_ptr, shape=(out.rows + 1,)).copy()
        c = np.ctypeslib.as_array(out.col_idx, shape=(max(out.nnz, 1),))[: out.nnz].copy()
        v = np.ctypeslib.as_array(out.values, shape=(max(out.nnz, 1),))[: out.nnz].copy()
        self.L.sko_csr_free(C.byref(out))
        return r, c, v

    def free_energy(self, dim, n, h, params, c) -> float:
        c = np.ascontiguousarray(c, np.float64).ravel()
        return self.L.sko_free_energy(dim, n, h, params.kappa, params.rho_w, params.c_alpha, params.c_beta, _p(c))

    def biharmonic_clamped(self, dim, intervals) -> Tuple[np.ndarray, np.ndarray]:
        count = (intervals - 1) ** dim
        f = np.empty(count)
        u = np.empty(count)
        self.L.sko_biharmonic_clamped(dim, intervals, _p(f), _p(u))
        return f, u

    def fit_loglog(self, hs: Sequence[float], errs: Sequence[float]):
        h = np.ascontiguousarray(hs, np.float64)
        e = np.ascontiguousarray(errs, np.float64)
        s, c, r = dbl(), dbl(), dbl()
        st = self.L.sko_fit_loglog(h.size, _p(h), _p(e), C.byref(s), C.byref(c), C.byref(r))
        if st:
            raise ValueError("fit_loglog needs >= 3 positive samples")
        return s.value, c.value, r.value

    def uniform(self, seed: int, count: int, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(count)
        self.L.sko_uniform(seed, count, lo, hi, _p(out))
        return out

    def dot(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.L.sko_dot(a.size, _p(a), _p(b))

    def sum(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return self.L.sko_sum(a.size, _p(a))

    def nrm2(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return self.L.sko_nrm2(a.size, _p(a))

    def minmax(self, a):
        a = np.ascontiguousarray(a, np.float64)
        lo, hi = dbl(), dbl()
        self.L.sko_minmax(a.size, _p(a), C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def axpy(self, alpha, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64).copy()
        self.L.sko_axpy(x.size, alpha, _p(x), _p(y))
        return y

    def xpby(self, x, beta, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64).copy()
        self.L.sko_xpby(x.size, _p(x), beta, _p(y))
        return y


class Reference:
    """The compiled reference library (optional: absent if never built here)."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self):
        L = C.CDLL(str(REF_SO))
        L.skref_last_error.restype = C.c_char_p
        L.skref_threads.restype = C.c_int
        L.skref_stencil.argtypes = [C.c_int] * 4 + [vp] * 6
        L.skref_assemble.argtypes = [C.c_int, C.c_int, C.c_int, vp, dbl, vp, C.POINTER(vp)]
        L.skref_assemble_entries.argtypes = [C.c_int, C.c_int, vp, vp, vp, C.c_int, vp, dbl, vp, C.POINTER(vp)]
        L.skref_csr_rows.argtypes = [vp]
        L.skref_csr_rows.restype = C.c_longlong
        L.skref_csr_nnz.argtypes = [vp]
        L.skref_csr_nnz.restype = C.c_longlong
        L.skref_csr_copy.argtypes = [vp, vp, vp, vp]
        L.skref_csr_free.argtypes = [vp]
        L.skref_csr_matvec.argtypes = [vp, vp, vp, C.c_int]
        L.skref_dot.argtypes = [C.c_longlong, vp, vp, C.c_int]
        L.skref_dot.restype = dbl
        L.skref_nrm2.argtypes = [C.c_longlong, vp, C.c_int]
        L.skref_nrm2.restype = dbl
        L.skref_sum.argtypes = [C.c_longlong, vp, C.c_int]
        L.skref_sum.restype = dbl
        L.skref_minmax.argtypes = [C.c_longlong, vp, C.POINTER(dbl), C.POINTER(dbl), C.c_int]
        L.skref_axpy.argtypes = [C.c_longlong, dbl, vp, vp, C.c_int]
        L.skref_xpby.argtypes = [C.c_longlong, vp, dbl, vp, C.c_int]
        L.skref_cg_solve.argtypes = [vp, vp, vp, dbl, C.c_longlong, C.c_int]
        L.skref_ch_create.argtypes = [C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, dbl, C.POINTER(vp)]
        L.skref_ch_steps.argtypes = [vp, dbl, C.c_longlong, vp]
        L.skref_ch_free.argtypes = [vp]
        L.skref_free_energy.argtypes = [C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, vp, C.c_int]
        L.skref_free_energy.restype = dbl
        L.skref_f_chem_prime.argtypes = [dbl, dbl, dbl, dbl]
        L.skref_f_chem_prime.restype = dbl
        L.skref_uniform.argtypes = [C.c_ulonglong, C.c_longlong, dbl, dbl, vp]
        L.skref_fit_loglog.argtypes = [C.c_int, vp, vp, C.POINTER(dbl), C.POINTER(dbl), C.POINTER(dbl)]
        L.skref_biharmonic_solve.argtypes = [C.c_int, vp, dbl, C.POINTER(dbl), C.POINTER(dbl), vp]
        L.skref_set_threads.argtypes = [C.c_int]
        L.skref_imex_create.argtypes = [C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, dbl, dbl, C.POINTER(vp)]
        L.skref_imex_steps.argtypes = [vp, dbl, C.c_int, C.c_longlong, vp]
        L.skref_imex_free.argtypes = [vp]
        L.skref_ch_init.argtypes = [C.c_int, C.c_int, dbl, dbl, dbl, vp]
        L.skref_power_iteration.argtypes = [vp, dbl, C.c_ulonglong, C.c_longlong, C.POINTER(dbl)]
        L.skref_periodic_spectrum.argtypes = [C.c_int, C.c_int, C.c_int, vp, dbl, dbl, dbl, vp, C.POINTER(dbl),
                                              C.POINTER(dbl), C.POINTER(dbl)]
        L.skref_csr_matmul.argtypes = [vp, vp]
        L.skref_csr_matmul.restype = vp
        L.skref_identity_plus_scaled.argtypes = [vp, dbl]
        L.skref_identity_plus_scaled.restype = vp
        self.L = L

    def err(self) -> str:
        return self.L.skref_last_error().decode()

    def threads(self) -> int:
        return self.L.skref_threads()

    def stencil(self, dim: int, acc: int, kind: int):
        """kind 0 identity, 1 laplacian(dim, acc), 2 compose(lap, lap). Returns
        (offsets[nent, dim], coeff_double[nent], num[nent], den[nent], h_power)."""
        cap = 512
        nent, hp = C.c_int(), C.c_int()
        off = np.zeros(cap * dim, np.int32)
        cd = np.zeros(cap)
        num = np.zeros(cap, np.int64)
        den = np.zeros(cap, np.int64)
        st = self.L.skref_stencil(dim, acc, kind, cap, C.byref(nent), _p(off), _p(cd), _p(num), _p(den), C.byref(hp))
        if st:
            raise ValueError(self.err())
        k = nent.value
        return off[: k * dim].reshape(k, dim), cd[:k], num[:k], den[:k], hp.value

    def _take(self, h) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        rows = self.L.skref_csr_rows(h)
        nnz = self.L.skref_csr_nnz(h)
        rp = np.empty(rows + 1, np.int64)
        ci = np.empty(max(nnz, 1), np.int64)
        v = np.empty(max(nnz, 1), np.float64)
        self.L.skref_csr_copy(h, _p(rp), _p(ci), _p(v))
        self.L.skref_csr_free(h)
        return rp, ci[:nnz], v[:nnz]

    def assemble(self, dim: int, acc: int, kind: int, n: Sequence[int], h: float, bc: Sequence[int]):
        na = np.ascontiguousarray(list(n) + [1] * (3 - len(n)), np.int32)
        ba = np.ascontiguousarray(list(bc) + [0] * (3 - len(bc)), np.int32)
        out = vp()
        st = self.L.skref_assemble(dim, acc, kind, _p(na), h, _p(ba), C.byref(out))
        if st:
            raise RuntimeError(f"reference assemble: status {st}: {self.err()}")
        return self._take(out)

    def assemble_entries(self, dim, offsets, num, den, h_power, n, h, bc):
        off = np.ascontiguousarray(np.asarray(offsets).ravel(), np.int32)
        nu = np.ascontiguousarray(num, np.int64)
        de = np.ascontiguousarray(den, np.int64)
        na = np.ascontiguousarray(list(n) + [1] * (3 - len(n)), np.int32)
        ba = np.ascontiguousarray(list(bc) + [0] * (3 - len(bc)), np.int32)
        out = vp()
        st = self.L.skref_assemble_entries(dim, nu.size, _p(off), _p(nu), _p(de), h_power, _p(na), h, _p(ba),
                                           C.byref(out))
        if st:
            raise RuntimeError(f"reference assemble: status {st}: {self.err()}")
        return self._take(out)

    def uniform(self, seed: int, count: int, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(count)
        self.L.skref_uniform(seed, count, lo, hi, _p(out))
        return out

    def ch_create(self, dim, n, h, params):
        out = vp()
        st = self.L.skref_ch_create(dim, n, h, params.mobility, params.kappa, params.rho_w, params.c_alpha,
                                    params.c_beta, C.byref(out))
        if st:
            raise RuntimeError(self.err())
        return out

    def ch_steps(self, handle, dt, nsteps, c: np.ndarray) -> None:
        self.L.skref_ch_steps(handle, dt, nsteps, _p(c))

    def ch_free(self, handle) -> None:
        self.L.skref_ch_free(handle)

    def imex_create(self, dim, n, h, params, rel_tol=1e-12):
        out = vp()
        st = self.L.skref_imex_create(dim, n, h, params.mobility, params.kappa, params.rho_w, params.c_alpha,
                                      params.c_beta, rel_tol, C.byref(out))
        if st:
            raise RuntimeError(self.err())
        return out

    def imex_steps(self, handle, dt, order, nsteps, c: np.ndarray) -> None:
        if self.L.skref_imex_steps(handle, dt, order, nsteps, _p(c)):
            raise RuntimeError(self.err())

    def imex_free(self, handle) -> None:
        self.L.skref_imex_free(handle)

    def periodic_spectrum(self, dim, acc, kind, n, h, shift=0.0, scale=1.0):
        na = np.ascontiguousarray(list(n) + [1] * (3 - len(n)), np.int32)
        eig = np.empty(2 * int(np.prod(n)))
        rho, sym, cond = dbl(), dbl(), dbl()
        if self.L.skref_periodic_spectrum(dim, acc, kind, _p(na), h, shift, scale, _p(eig), C.byref(rho),
                                          C.byref(sym), C.byref(cond)):
            raise RuntimeError(self.err())
        return eig.view(np.complex128), rho.value, sym.value, cond.value

    def ch_init(self, dim, n, h, c0, eps) -> np.ndarray:
        out = np.empty(n ** dim)
        if self.L.skref_ch_init(dim, n, h, c0, eps, _p(out)):
            raise RuntimeError(self.err())
        return out

    def free_energy(self, dim, n, h, params, c, serial=False) -> float:
        c = np.ascontiguousarray(c, np.float64)
        return self.L.skref_free_energy(dim, n, h, params.kappa, params.rho_w, params.c_alpha, params.c_beta, _p(c),
                                        int(serial))


class RefCsr:
    """A reference-owned CsrMatrix handle for timing loops (kept assembled)."""

    def __init__(self, ref: Reference, dim, acc, kind, n, h, bc):
        self.ref = ref
        na = np.ascontiguousarray(list(n) + [1] * (3 - len(n)), np.int32)
        ba = np.ascontiguousarray(list(bc) + [0] * (3 - len(bc)), np.int32)
        out = vp()
        st = ref.L.skref_assemble(dim, acc, kind, _p(na), h, _p(ba), C.byref(out))
        if st:
            raise RuntimeError(ref.err())
        self.h = out
        self.rows = ref.L.skref_csr_rows(out)
        self.nnz = ref.L.skref_csr_nnz(out)

    def arrays(self):
        rp = np.empty(self.rows + 1, np.int64)
        ci = np.empty(max(self.nnz, 1), np.int64)
        v = np.empty(max(self.nnz, 1))
        self.ref.L.skref_csr_copy(self.h, _p(rp), _p(ci), _p(v))
        return rp, ci[: self.nnz], v[: self.nnz]

    def matvec(self, x: np.ndarray, y: np.ndarray, serial: bool = False) -> None:
        self.ref.L.skref_csr_matvec(self.h, _p(x), _p(y), int(serial))

    def cg_solve(self, b: np.ndarray, x: np.ndarray, rel_tol: float, max_iter: int = 0, deflate: bool = False) -> int:
        return self.ref.L.skref_cg_solve(self.h, _p(b), _p(x), rel_tol, max_iter, int(deflate))

    def close(self) -> None:
        if self.h:
            self.ref.L.skref_csr_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_oracle: Optional[Oracle] = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle()
    return _oracle
