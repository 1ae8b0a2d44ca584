import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(HERE, "golden")
GOLDEN_FILES = {"c0": "c0_0_128.npz", "c1": "c1_0_24.npz", "c2": "c2_0_7.npz", "c4": "c4_0_256.npz"}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running checks")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, GOLDEN_FILES[name])))


@pytest.fixture(scope="session")
def golden():
    return load_golden


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)
