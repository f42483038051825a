import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    from oracle.ffi import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.ffi import Reference

    if not Reference.available():
        pytest.skip("compiled reference (oracle/_ref/libstencilkit_ref.so) not built here")
    return Reference()


@pytest.fixture(scope="session")
def lib():
    from paper_2205_03354_b200 import _lib

    return _lib.ensure_device(0)
