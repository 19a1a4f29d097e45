import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhefv.so")
    config.addinivalue_line("markers", "slow: long-running (retina-scale) checks")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def gpu_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
