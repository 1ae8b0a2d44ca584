"""Sweep batcher (sweep.py, a23): the reference's run_sweep rows
(scenarios.py:266-296, golden tests/golden/sweep_rows.json from
make_sweep_golden.py) reproduced with one batched solve per sweep value.
CPU: the host build of the device solver (tests/emu) stands in for the
library; GPU: the sm_100a library."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1803_07772_b200.sweep import Scenario, run_sweep, config_for

ROWS = json.load(open(os.path.join(GOLDEN, "sweep_rows.json")))


def _emu_solve_batch(cfg, gamma):
    from emu import runner
    return runner.run(cfg, gamma, np.full(gamma.shape[1:], cfg.noise_density * cfg.subcarrier_bandwidth))


def _compare(rows, ref):
    assert len(rows) == len(ref)
    for r, g in zip(rows, ref):
        assert r.value == g["value"] and r.n_draws == g["n_draws"] and r.n_feasible == g["n_feasible"]
        for k in ("mean_ee", "mean_rate", "mean_power"):
            assert abs(getattr(r, k) - g[k]) <= 1e-4 * abs(g[k]), (k, getattr(r, k), g[k])
        assert r.mean_iterations == g["mean_iterations"]


@pytest.mark.parametrize("name", sorted(ROWS))
def test_sweep_rows_host_build(name):
    sc = ROWS[name]["scenario"]
    sc = Scenario(**{k: tuple(v) if isinstance(v, list) else v for k, v in sc.items()})
    _compare(run_sweep(sc, solve_batch=_emu_solve_batch), ROWS[name]["rows"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(ROWS))
def test_sweep_rows_gpu(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sc = ROWS[name]["scenario"]
    sc = Scenario(**{k: tuple(v) if isinstance(v, list) else v for k, v in sc.items()})
    _compare(run_sweep(sc), ROWS[name]["rows"])


def test_config_for_matches_sweep_variable():
    sc = Scenario(sweep="lpn", values=(1, 3), k_total=6, k_streaming=2, n_subcarriers=8)
    cfg = config_for(sc, 3, np.random.default_rng([1, 0]))
    assert cfg.n_rrh == 4 and cfg.n_users == 6
    sc = Scenario(sweep="streaming", values=(0,), k_total=6, k_streaming=2, n_subcarriers=8)
    cfg = config_for(sc, 0, np.random.default_rng([1, 0]))
    assert cfg.streaming_users() == []
