import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libphif_b200.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
