import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")
    config.addinivalue_line("markers", "slow: reproduces a paper table on the CPU oracle (tens of seconds)")


@pytest.fixture(scope="session")
def cuda_lib():
    """The product library; GPU tests fail loudly when it is missing."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_11235_b200 import qtip
    qtip.load()
    return qtip
