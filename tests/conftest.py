import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built extension")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session", autouse=True)
def _poisoned_device_memory():
    """RCP_POISON=1: start the session with the caching allocator's blocks full of 0xFF
    (NaN as fp64), so reads of never-written device memory fail every time."""
    if os.environ.get("RCP_POISON", "") == "1" and cuda_ok():
        import torch
        from paper_2210_05105_b200.device import poison_allocator
        poison_allocator(torch.device("cuda", 0))
    yield
