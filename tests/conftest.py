import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libopcfe.so")


@pytest.fixture
def rng():
    # same seed as the reference suite's shared fixture (tests/conftest.py:5-7)
    return np.random.default_rng(12345)


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        out = {}
        for key in z.files:
            case, field = key.split("/", 1)
            out.setdefault(case, {})[field] = z[key]
        return out


def grid_opc(M, N, z=0.0):
    u, v = np.meshgrid(np.arange(M, dtype=float), np.arange(N, dtype=float), indexing="ij")
    return np.stack([v, -u, np.full_like(u, z)], axis=2)
