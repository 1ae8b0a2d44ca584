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


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running checks")


def _golden_files(name):
    import glob
    fs = [f for f in glob.glob(os.path.join(GOLDEN, f"{name}_*_*.npz"))
          if "_devmodel" not in f and "_sel" not in f]
    return sorted(fs, key=lambda f: int(os.path.basename(f).split("_")[1]))


def _concat(parts):
    out = {}
    for k in parts[0]:
        arrs = [np.asarray(p[k]) for p in parts]
        if arrs[0].ndim == 0:
            out[k] = arrs[0]
            continue
        if arrs[0].ndim == 2 and k in ("e_values", "surplus", "rounds", "sweeps"):
            w = max(a.shape[1] for a in arrs)
            arrs = [np.pad(a, ((0, 0), (0, w - a.shape[1])), constant_values=np.nan) for a in arrs]
        out[k] = np.concatenate(arrs)
    return out


def load_golden(name):
    """Reference outputs (tests/golden/make_golden.py) of every draw file of a config."""
    return _concat([dict(np.load(f)) for f in _golden_files(name)])


def load_selected(name):
    """Reference outputs of hand-picked draws (make_golden.py --list): the draws
    whose device outcome is infeasible, products-active or otherwise rare."""
    import glob
    fs = sorted(glob.glob(os.path.join(GOLDEN, f"{name}_*_sel.npz")))
    return _concat([dict(np.load(f)) for f in fs]) if fs else None


def load_devmodel(name):
    """Oracle restatement of the B200 default SIC model for the same draws
    (tests/golden/make_device_model.py); None when not generated."""
    fs = [f.replace(".npz", "_devmodel.npz") for f in _golden_files(name)]
    if not all(os.path.exists(f) for f in fs):
        return None
    return _concat([dict(np.load(f)) for f in fs])


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def selected():
    return load_selected


@pytest.fixture(scope="session")
def devmodel():
    return load_devmodel


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)
