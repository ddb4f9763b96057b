"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu and call the CUDA path
through the C-ABI library; everything else runs on CPU (oracle vs golden
fixtures, host logic, library exports, gloo world_size-2 transport tests)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def golden():
    return load_golden
