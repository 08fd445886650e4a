import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")


import pytest  # noqa: E402


@pytest.fixture(autouse=True)
def _close_gpu_contexts():
    """After each test, destroy the libaqua contexts its Rigs created, even if
    the test kept references alive (a leak check then sees every library
    allocation freed by aqua_destroy)."""
    yield
    mod = sys.modules.get("gpu_util")
    if mod is not None:
        mod.close_all()
