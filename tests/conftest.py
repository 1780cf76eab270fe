import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libhrt.so")
    config.addinivalue_line("markers", "reference: needs the reference package at /root/reference")


def reference_available():
    return os.path.isdir(os.path.join(REFERENCE_SRC, "hybridrt"))


@pytest.fixture(scope="session")
def hybridrt():
    """The real reference package (build container only)."""
    if not reference_available():
        pytest.skip("reference package not present (GPU box / CI)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import hybridrt as h
    return h


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)
