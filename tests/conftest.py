import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def normwise(a, b):
    """max|a - b| / max|b| -- the SURVEY §8c parity measure."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if b.size == 0:
        return 0.0
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / den) if den > 0 else float(np.abs(a - b).max())


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(params=["v1", "v2"])
def k1_generation(request, monkeypatch):
    """Run a tensor-core test on both K1 generations: v1 (two 256-thread CTAs
    per SM, one 32-row chunk at a time) and v2 (warp-specialized tcgen05
    pipeline, gmf_tc2.cuh).  gmf_create reads GMF_TC_VERSION."""
    monkeypatch.setenv("GMF_TC_VERSION", "1" if request.param == "v1" else "2")
    return request.param
