import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: longer CPU stress")


@pytest.fixture(scope="session")
def cuda():
    """GPU tests never skip: a missing GPU or library is a failure."""
    import torch
    assert torch.cuda.is_available(), "gpu test without a GPU"
    from paper_2504_18211_b200 import lib
    lib()
    torch.cuda.init()
    return torch
