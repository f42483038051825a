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


@pytest.fixture
def sk_option():
    """Set library execution options (sk_set_option) for one test; every changed
    option is restored afterwards."""
    from paper_2205_03354_b200 import _lib

    saved = {}

    def setter(name, value):
        old = _lib.set_option(name, value)
        saved.setdefault(name, old)

    yield setter
    for name, value in saved.items():
        _lib.set_option(name, value)
