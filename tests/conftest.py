import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libnekb200.so")


@pytest.fixture(scope="session")
def golden_basis():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "basis_ref.npz"))


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
