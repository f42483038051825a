"""ctypes binding of the C-ABI in include/sk_cuda.h (libsk_cuda.so, in-tree).

There is no CPU fallback: if the shared library is missing or cannot load,
every entry point raises. `load()` never builds; build() in
__graft_entry__.py / paper_2205_03354_b200.build_ext compiles it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Optional

from .errors import Errc, StencilkitError

LIB_PATH = Path(__file__).resolve().parent / "libsk_cuda.so"

c_i64 = C.c_int64
c_dbl = C.c_double
c_int = C.c_int
vp = C.c_void_p
pd = C.POINTER(C.c_double)


class GridDesc(C.Structure):
    _fields_ = [("dim", c_int), ("n", c_i64 * 3), ("h", c_dbl), ("bc", c_int * 3)]


class ChParams(C.Structure):
    _fields_ = [("kappa", c_dbl), ("mobility", c_dbl), ("rho_w", c_dbl), ("c_alpha", c_dbl), ("c_beta", c_dbl),
                ("formulation", c_int)]


CH_FACTORED, CH_COMPOSED = 0, 1


class SolveOptionsC(C.Structure):
    _fields_ = [("rel_tol", c_dbl), ("max_iter", c_i64), ("deflate_mean", c_int), ("check_every", c_int),
                ("accept_recurrence", c_int), ("use_initial_guess", c_int)]


class RefineReportC(C.Structure):
    _fields_ = [("iterations", c_i64), ("refinements", c_int), ("initial_true_rel_residual", c_dbl),
                ("refined_rel_residual", c_dbl), ("last_correction_rel", c_dbl)]


class SolveReportC(C.Structure):
    _fields_ = [("iterations", c_i64), ("restarts", c_i64), ("true_rel_residual", c_dbl),
                ("recurrence_rel_residual", c_dbl)]


# name -> (restype, argtypes); every symbol of include/sk_cuda.h
SIGNATURES = {
    "sk_last_error": (C.c_char_p, []),
    "sk_status_name": (C.c_char_p, [c_int]),
    "sk_version": (c_int, []),
    "sk_device_init": (c_int, [c_int]),
    "sk_device_alloc": (c_int, [C.c_size_t, C.POINTER(vp)]),
    "sk_device_free": (c_int, [vp]),
    "sk_memcpy_h2d": (c_int, [vp, vp, C.c_size_t, vp]),
    "sk_memcpy_d2h": (c_int, [vp, vp, C.c_size_t, vp]),
    "sk_stream_sync": (c_int, [vp]),
    "sk_ipc_get_handle": (c_int, [vp, vp]),
    "sk_ipc_open_handle": (c_int, [vp, C.POINTER(vp)]),
    "sk_ipc_close_handle": (c_int, [vp]),
    "sk_stream_create": (c_int, [C.POINTER(vp)]),
    "sk_stream_destroy": (c_int, [vp]),
    "sk_fill_uniform_host": (c_int, [C.c_uint64, c_i64, c_dbl, c_dbl, vp]),
    "sk_launch_count": (c_i64, []),
    "sk_host_register": (c_int, [vp, C.c_size_t]),
    "sk_host_unregister": (c_int, [vp]),
    "sk_event_create": (c_int, [C.POINTER(vp)]),
    "sk_event_destroy": (c_int, [vp]),
    "sk_event_record": (c_int, [vp, vp]),
    "sk_event_elapsed_ms": (c_int, [vp, vp, C.POINTER(C.c_float)]),
    "sk_l2_flush": (c_int, [vp]),
    "sk_set_option": (c_int, [c_int, c_int]),
    "sk_get_option": (c_int, [c_int, C.POINTER(c_int)]),
    "sk_stencil_create": (c_int, [c_int, c_int, vp, vp, c_int, C.POINTER(vp)]),
    "sk_stencil_destroy": (c_int, [vp]),
    "sk_stencil_kernel_class": (c_int, [vp]),
    "sk_composed_apply": (c_int, [vp, C.POINTER(GridDesc), vp, vp, vp]),
    "sk_composed_apply_repeat": (c_int, [vp, C.POINTER(GridDesc), vp, vp, vp, c_int, vp]),
    "sk_composed_apply_host": (c_int, [vp, C.POINTER(GridDesc), vp, vp]),
    "sk_ch_explicit": (c_int, [vp, vp, C.POINTER(GridDesc), C.POINTER(ChParams), c_dbl, c_i64, vp, vp,
                               C.POINTER(c_int), vp]),
    "sk_ch_explicit_slab": (c_int, [vp, vp, C.POINTER(GridDesc), C.POINTER(ChParams), c_dbl, vp, vp, vp]),
    "sk_ch_explicit_slab_peer": (c_int, [vp, vp, C.POINTER(GridDesc), C.POINTER(ChParams), c_dbl, vp, vp, vp, vp,
                                         vp]),
    "sk_ch_explicit_host": (c_int, [vp, vp, C.POINTER(GridDesc), C.POINTER(ChParams), c_dbl, c_i64, vp]),
    "sk_free_energy": (c_int, [C.POINTER(GridDesc), C.POINTER(ChParams), vp, pd, vp]),
    "sk_ch_imex_create": (c_int, [C.POINTER(GridDesc), C.POINTER(ChParams), C.POINTER(SolveOptionsC),
                                  C.POINTER(vp)]),
    "sk_ch_imex_destroy": (c_int, [vp]),
    "sk_ch_imex_reset_history": (c_int, [vp]),
    "sk_ch_imex_step": (c_int, [vp, vp, c_dbl, c_int, c_i64, C.POINTER(SolveReportC), C.POINTER(c_i64), vp]),
    "sk_ch_imex_matrix": (c_int, [vp, c_int, C.POINTER(vp)]),
    "sk_ch_init_host": (c_int, [C.POINTER(GridDesc), c_dbl, c_dbl, vp]),
    "sk_csr_matmul": (c_int, [vp, vp, C.POINTER(vp), vp]),
    "sk_power_iteration": (c_int, [vp, c_dbl, C.c_uint64, c_i64, pd, C.POINTER(c_i64), vp]),
    "sk_periodic_spectrum": (c_int, [vp, C.POINTER(GridDesc), c_dbl, c_dbl, vp, pd, pd, pd]),
    "sk_csr_assemble": (c_int, [vp, C.POINTER(GridDesc), c_int, C.POINTER(vp), vp]),
    "sk_csr_assemble_into": (c_int, [vp, C.POINTER(GridDesc), vp, vp]),
    "sk_csr_upload": (c_int, [c_i64, c_i64, c_i64, vp, vp, vp, c_int, C.POINTER(vp)]),
    "sk_csr_info": (c_int, [vp, C.POINTER(c_i64), C.POINTER(c_i64), C.POINTER(c_i64), C.POINTER(c_int)]),
    "sk_csr_download": (c_int, [vp, vp, vp, vp]),
    "sk_csr_destroy": (c_int, [vp]),
    "sk_csr_matvec": (c_int, [vp, vp, vp, vp]),
    "sk_csr_matvec_host": (c_int, [vp, vp, vp]),
    "sk_dot": (c_int, [c_i64, vp, vp, pd, vp]),
    "sk_nrm2": (c_int, [c_i64, vp, pd, vp]),
    "sk_sum": (c_int, [c_i64, vp, pd, vp]),
    "sk_minmax": (c_int, [c_i64, vp, pd, pd, vp]),
    "sk_axpy": (c_int, [c_i64, c_dbl, vp, vp, vp]),
    "sk_xpby": (c_int, [c_i64, vp, c_dbl, vp, vp]),
    "sk_cg_solve": (c_int, [vp, vp, vp, C.POINTER(SolveOptionsC), C.POINTER(SolveReportC), vp]),
    "sk_cg_solve_host": (c_int, [vp, vp, vp, C.POINTER(SolveOptionsC), C.POINTER(SolveReportC)]),
    "sk_cg_solve_stencil": (c_int, [vp, C.POINTER(GridDesc), vp, vp, C.POINTER(SolveOptionsC), C.POINTER(SolveReportC),
                                    vp]),
    "sk_stencil_create_exact": (c_int, [c_int, c_int, vp, vp, vp, c_int, C.POINTER(vp)]),
    "sk_residual_refined": (c_int, [vp, C.POINTER(GridDesc), vp, vp, vp, vp]),
    "sk_cg_solve_stencil_refined": (c_int, [vp, C.POINTER(GridDesc), vp, vp, C.POINTER(SolveOptionsC), c_dbl, c_int,
                                            C.POINTER(RefineReportC), vp]),
}

_lib: Optional[C.CDLL] = None


def load(path: Optional[Path] = None) -> C.CDLL:
    """Load libsk_cuda.so and declare every signature. Raises if it is absent.

    `path` (tools only): an explicitly named alternative build of the same ABI."""
    global _lib
    if _lib is not None:
        return _lib
    explicit = path is not None
    path = Path(path) if explicit else LIB_PATH
    if not path.exists():
        raise RuntimeError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(the CUDA path has no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        if explicit and not hasattr(lib, name):  # an older A/B build may lack newer entry points
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# sk_set_option ids (include/sk_cuda.h enum sk_option)
OPTIONS = {"pdl": 0, "ch_padded": 1, "cg_device_loop": 2, "cg_fused": 3, "cg_coop": 4, "cg_pq": 5,
           "imex_matrix_free": 6, "apply73_factored": 7, "cg_padded": 8,
           "ch_host_pipeline": 9}


def set_option(name: str, value: int) -> int:
    """Set one execution option (explicit; the library never reads the environment); returns the old value."""
    lib = load()
    old = c_int()
    check(lib.sk_get_option(OPTIONS[name], C.byref(old)))
    check(lib.sk_set_option(OPTIONS[name], int(value)))
    return old.value


class options:
    """Context manager: `with options(ch_padded=0): ...` restores the previous values on exit."""

    def __init__(self, **kw: int):
        self.kw = kw
        self.saved: dict = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.saved[k] = set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_option(k, v)


def check(status: int) -> None:
    """Raise StencilkitError for a non-zero status (the reference's throw)."""
    if status == 0:
        return
    msg = load().sk_last_error().decode(errors="replace")
    raise StencilkitError(Errc(status - 1), msg)


_initialised = False


def ensure_device(device: int = 0) -> C.CDLL:
    global _initialised
    lib = load()
    if not _initialised:
        check(lib.sk_device_init(device))
        _initialised = True
    return lib
