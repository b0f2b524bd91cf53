import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA product library; fails loudly (never skips to a fallback)."""
    import torch
    assert torch.cuda.is_available(), "gpu test collected without a CUDA device"
    from paper_math_0508111_b200 import binding
    return binding
