import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running oracle pin (still part of the CPU suite)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import refpy

    refpy.lib()
    return refpy


@pytest.fixture(scope="session")
def gpu():
    """The CUDA extension; a GPU test must run the native path or fail loudly (never skip)."""
    import paper_1707_00164_b200 as G
    from paper_1707_00164_b200 import _lib

    _lib.lib()
    return G
