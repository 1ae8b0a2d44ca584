"""CPU check of the DEVICE solver's logic: hcran_solver.cuh compiled for the
host (tests/emu, one CTA of one thread) against the reference's golden
outputs.  Same source as the sm_100a kernel; the GPU parity tests
(test_gpu_parity.py) repeat these checks on the B200."""

import numpy as np
import pytest

from conftest import rel
from emu import runner
from paper_1803_07772_b200.scenarios import workload_batch


def _ok(o, ref, j, i, key="ee"):
    good = o["status"][j] == ref["status"][i] and rel(o[key][j], ref[key][i]) <= 1e-4
    if key == "ee":
        good = good and rel(o["total_power"][j], ref["total_power"][i]) <= 1e-4
    return good and np.array_equal(o["rho"][j], ref["rho"][i]) and np.array_equal(o["a"][j], ref["a"][i])


def _check_dinkelbach(g, out, idx, skip=None):
    return [int(i) for j, i in enumerate(idx)
            if not g["near_tie"][i] and not (skip is not None and skip[i]) and not _ok(out, g, j, i)]


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_emu_default_mode(golden, devmodel, name):
    g, dm = golden(name), devmodel(name)
    idx = np.arange(len(g["draw"]))
    b = workload_batch(name, g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=0)
    fs = dm["floor_sensitive"] if dm is not None else None
    assert _check_dinkelbach(g, out, idx, fs) == []
    if dm is not None:
        assert _check_dinkelbach(dm | {"near_tie": g["near_tie"]}, out, idx) == []
    assert np.all(out["feasible"][g["feasible"][idx]] == 1)
    n_ref = np.sum(~np.isnan(g["e_values"][idx]), axis=1)
    assert np.mean(out["outer_iters"] == n_ref) >= 0.9


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_emu_exact_mode(golden, name):
    g = golden(name)
    idx = np.arange(len(g["draw"]))
    b = workload_batch(name, g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=0, exact=True)
    assert _check_dinkelbach(g, out, idx) == []


def test_emu_fixed_e_golden(golden, devmodel):
    g, dm = golden("c4"), devmodel("c4")
    ref = g if dm is None else dm
    idx = np.arange(len(g["draw"]))
    b = workload_batch("c4", g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=1, elastic=b.elastic, min_rates=b.min_rates,
                     e_fixed=b.e_fixed)
    for j in idx:
        assert _ok(out, ref, j, j, key="objective"), j


def test_emu_seated_pairs_flag_floor_ties(golden):
    """Without the dense re-solve the seated-pair SIC model is exact except on
    floor-tie instances, and every such divergence is flagged."""
    g = golden("c0")
    idx = np.arange(len(g["draw"]))
    b = workload_batch("c0", g["draw"][idx])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=0, dense_off=True)
    bad = _check_dinkelbach(g, out, idx)
    flagged = set(np.nonzero(out["flags"] & 1)[0].tolist())
    # c0's floor-sensitive draws are all floor ties, so every divergence is flagged
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

