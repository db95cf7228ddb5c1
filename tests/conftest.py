import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))
    return load


@pytest.fixture(scope="session")
def reference():
    """The real reference package (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference package not available here")
    sys.path.insert(0, REFERENCE_SRC)
    import mlrpca
    return mlrpca


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
