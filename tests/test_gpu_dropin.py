"""GPU: the reference's own C++ API vs the stencilkit::cuda drop-in header.

Runs oracle/_ref/dropin_parity (tests/cpp/dropin_parity.cpp), built here by
`make -C oracle` against the unmodified reference headers and library plus
libsk_cuda.so; the prebuilt binary travels with the repo snapshot.
"""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "dropin_parity"


def test_dropin_header_matches_reference_library():
    if not BIN.exists():
        pytest.skip("dropin_parity not built (needs /root/reference at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "PASSED" in res.stdout
