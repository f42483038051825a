"""CPU: the C-ABI library loads, exports every symbol include/sk_cuda.h declares,
and its host-only entry points behave (no GPU needed)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2205_03354_b200 import _lib
from paper_2205_03354_b200.errors import ERRC_NAMES, Errc

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sk_cuda.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["sk_composed_apply", "sk_ch_explicit", "sk_csr_assemble", "sk_csr_matvec", "sk_cg_solve",
                 "sk_dot", "sk_axpy", "sk_xpby", "sk_free_energy", "sk_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_status_names_follow_errc():
    lib = _lib.load()
    for code, name in ERRC_NAMES.items():
        assert lib.sk_status_name(int(code) + 1).decode() == name
    assert lib.sk_status_name(0).decode() == "Ok"
    assert lib.sk_version() >= 1


def test_host_generator_matches_reference_fixture():
    """sk_fill_uniform_host == std::mt19937_64 + uniform_real_distribution as drawn by the reference."""
    lib = _lib.load()
    z = np.load(ROOT / "tests" / "golden" / "uniform.npz")
    for s in (0, 1, 2, 3, 99):
        out = np.empty(2000)
        assert lib.sk_fill_uniform_host(s, out.size, -1.0, 1.0, out.ctypes.data) == 0
        assert np.array_equal(out, z[f"seed{s}"])


def test_device_entry_points_fail_loudly_without_gpu():
    """No CPU fallback: on this GPU-less host a device call reports an error code."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = _lib.load()
    st = lib.sk_device_init(0)
    assert st in (Errc.no_device + 1, Errc.cuda_error + 1)
    assert lib.sk_last_error().decode()


def test_missing_library_raises(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "libsk_cuda.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_struct_layouts_match_header():
    # sk_grid_desc {int; int64[3]; double; int[3]} with natural alignment
    assert C.sizeof(_lib.GridDesc) == 4 + 4 + 24 + 8 + 12 + 4
    assert C.sizeof(_lib.ChParams) == 5 * 8 + 8
    assert C.sizeof(_lib.SolveOptionsC) == 8 + 8 + 4 + 4 + 4 + 4
    assert C.sizeof(_lib.SolveReportC) == 32


def test_options_are_explicit_and_validated():
    # execution options are set through sk_set_option only (host-side, no GPU needed)
    lib = _lib.load()
    v = C.c_int()
    for name, opt in _lib.OPTIONS.items():
        assert lib.sk_get_option(opt, C.byref(v)) == 0
    assert lib.sk_set_option(99, 1) == Errc.invalid_argument + 1
    assert lib.sk_set_option(_lib.OPTIONS["ch_padded"], 7) == Errc.invalid_argument + 1
    with _lib.options(ch_padded=0, cg_coop=1):
        lib.sk_get_option(_lib.OPTIONS["ch_padded"], C.byref(v))
        assert v.value == 0
    lib.sk_get_option(_lib.OPTIONS["ch_padded"], C.byref(v))
    assert v.value == 1


def test_product_never_reads_the_environment():
    # a stray environment variable must not change which kernel runs
    csrc = ROOT / "paper_2205_03354_b200" / "csrc"
    for f in list(csrc.glob("*.cu")) + list(csrc.glob("*.cuh")) + list(csrc.glob("*.hpp")):
        assert "getenv" not in f.read_text(), f.name
    for f in (ROOT / "paper_2205_03354_b200").glob("*.py"):
        if f.name == "build_ext.py":  # the build tool may locate nvcc through $NVCC
            continue
        text = f.read_text()
        assert "os.environ" not in text and "getenv" not in text, f.name
