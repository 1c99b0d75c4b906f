import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI CUDA library)")
    config.addinivalue_line("markers", "slow: long CPU test (still part of the default suite unless deselected)")


@pytest.fixture(scope="session")
def repo_root():
    return ROOT


@pytest.fixture(scope="module")
def smc():
    """The C-ABI library with torch's allocator and stream (GPU tests only)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a GPU")
    import paper_0912_2551_b200 as smc
    smc.use_torch()
    return smc
