import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


import pytest


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Make sure the in-tree libtm_w4a16.so is current (nvcc cross-compiles; no GPU needed)."""
    from paper_2508_15601_b200 import build
    build.build()
    yield
