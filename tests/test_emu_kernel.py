"""CPU check of the DEVICE solver's logic: hcran_solver.cuh compiled for the
host (tests/emu, one CTA of one thread) against the reference's golden
outputs.  Same source as the sm_100a kernel; the GPU parity tests
(test_gpu_parity.py) repeat these checks on the B200."""

import numpy as np
import pytest

from conftest import rel
from emu import runner
from paper_1803_07772_b200.scenarios import workload_batch


def _check_dinkelbach(g, out, idx):
    bad = []
    for j, i in enumerate(idx):
        if g["near_tie"][i]:
            continue
        ok = (out["status"][j] == g["status"][i]
              and rel(out["ee"][j], g["ee"][i]) <= 1e-4
              and rel(out["total_power"][j], g["total_power"][i]) <= 1e-4
              and np.array_equal(out["rho"][j], g["rho"][i])
              and np.array_equal(out["a"][j], g["a"][i]))
        if not ok:
            bad.append(int(i))
    return bad


@pytest.mark.parametrize("engine", [True, False], ids=["smem-engine", "global-engine"])
@pytest.mark.parametrize("name", ["c0", "c1"])
def test_emu_dinkelbach_golden(golden, name, engine):
    g = golden(name)
    idx = np.arange(len(g["draw"]))
    b = workload_batch(name, g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=0, engine=engine)
    assert _check_dinkelbach(g, out, idx) == []
    assert np.all(out["feasible"][g["feasible"][idx]] == 1)
    # iteration counts follow the reference's trajectory
    n_ref = np.sum(~np.isnan(g["e_values"][idx]), axis=1)
    assert np.mean(out["outer_iters"] == n_ref) >= 0.95


@pytest.mark.parametrize("engine", [True, False], ids=["smem-engine", "global-engine"])
def test_emu_fixed_e_golden(golden, engine):
    g = golden("c4")
    idx = np.arange(len(g["draw"]))
    b = workload_batch("c4", g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=1, elastic=b.elastic, min_rates=b.min_rates,
                     e_fixed=b.e_fixed, engine=engine)
    for j in idx:
        assert out["status"][j] == g["status"][j]
        assert rel(out["objective"][j], g["objective"][j]) <= 1e-4, j
        assert np.array_equal(out["rho"][j], g["rho"][j]) and np.array_equal(out["a"][j], g["a"][j])


def test_emu_seated_pairs_flag_floor_ties(golden):
    """Without the dense re-solve the seated-pair SIC model is exact except on
    floor-tie instances, and every such divergence is flagged."""
    g = golden("c0")
    idx = np.arange(len(g["draw"]))
    b = workload_batch("c0", g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=0, dense_off=True)
    bad = _check_dinkelbach(g, out, idx)
    flagged = set(np.nonzero(out["flags"] & 1)[0].tolist())
    assert set(bad) <= flagged
    assert len(flagged) <= 0.1 * len(idx)


def test_emu_warm_start_never_worse(golden):
    """scale.py:536-540: with a warm start the result is never worse than it."""
    g = golden("c0")
    b = workload_batch("c0", range(8))
    first = runner.run(b.cfg, b.gamma, b.sigma, mode=1, e_fixed=np.zeros(8))
    e = first["sum_rate"] / first["total_power"]
    second = runner.run(b.cfg, b.gamma, b.sigma, mode=1, e_fixed=e, warm_p=first["p"])
    warm_obj = first["sum_rate"] - e * first["total_power"]
    assert np.all(second["objective"] >= warm_obj - 1e-9)
