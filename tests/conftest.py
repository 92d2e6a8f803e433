import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU-only case")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def grid_from(arr):
    """(dims, spacing, origin) from the 9-vector written by make_golden.garr."""
    from oracle import ngf_oracle as O
    a = np.asarray(arr, dtype=np.float64)
    return O.grid(tuple(int(v) for v in a[:3]), tuple(a[3:6]), tuple(a[6:9]))


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
