import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")
    config.addinivalue_line("markers", "multigpu: needs N > 1 GPUs in one node (skips otherwise)")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def acg():
    """The product package; on a GPU box it must load its CUDA build (no fallback)."""
    import paper_1302_7193_b200 as p
    return p


def max_rel(a, b):
    """max|a-b| / max|b|  (test_operator.cpp:30-37, verify.cpp:31-39)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max() if b.size else 0.0
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0)) if a.size else 0.0
