import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


@pytest.fixture(scope="session")
def gpu():
    """The product library with at least one visible CUDA device. On a GPU box
    a missing/unloadable library is an error, never a skip."""
    import ctypes

    from paper_2310_12403_b200 import _lib
    L = _lib.load()
    n = ctypes.c_int(0)
    if L.cb_device_count(ctypes.byref(n)) != 0 or n.value == 0:
        pytest.skip("no CUDA device visible")
    return L
