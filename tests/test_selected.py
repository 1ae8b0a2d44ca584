"""Rare outcomes pinned against the reference (make_golden.py --list): the
draws of the config[1] / config[2] bench batches on which the device reports
an infeasible first inner solve (the reference raises InfeasibleProblemError,
dinkelbach.py:81-86) or a non-exclusive greedy seating (the products-active
theta' family, scale.py:561-566, 861-895).

Documented exception: on products-active draws the repair's top-l_max cut
(scale.py:941-945) meets exactly equal seat powers (the greedy start's
budget-scaled mask on every seat of the overfull column), and numpy's
unstable argsort (x86-simd-sort on AVX-512 hosts) decides which seat goes;
the reference's own tie order is host-dependent there, so those draws are
checked for status, feasibility and EE within 1e-3."""

import numpy as np
import pytest

from conftest import rel

TIE_CUT = {("c1", 690)}


def _compare(name, g, out):
    bad = []
    for j, d in enumerate(g["draw"]):
        d = int(d)
        if int(out["status"][j]) != int(g["status"][j]):
            bad.append((d, "status", int(out["status"][j]), int(g["status"][j])))
            continue
        if int(g["status"][j]) == 3:
            continue
        tol = 1e-3 if (name, d) in TIE_CUT else 1e-4
        if rel(out["ee"][j], g["ee"][j]) > tol or rel(out["total_power"][j], g["total_power"][j]) > tol:
            bad.append((d, "ee", float(out["ee"][j]), float(g["ee"][j])))
        if (name, d) not in TIE_CUT and not (np.array_equal(out["rho"][j], g["rho"][j])
                                              and np.array_equal(out["a"][j], g["a"][j])):
            bad.append((d, "rho/a"))
        if not out["feasible"][j]:
            bad.append((d, "infeasible output"))
    return bad


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_selected_host_build(selected, name):
    from emu import runner
    from paper_1803_07772_b200.scenarios import workload_batch
    g = selected(name)
    if g is None:
        pytest.skip("no selected fixtures")
    b = workload_batch(name, g["draw"])
    out = runner.run(b.cfg, b.gamma, b.sigma, mode=0)
    assert _compare(name, g, out) == []
    assert not np.any(out["status"] == 4)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_selected_b200(selected, name):
    from paper_1803_07772_b200 import solve_batch
    from paper_1803_07772_b200.scenarios import workload_batch
    g = selected(name)
    if g is None:
        pytest.skip("no selected fixtures")
    b = workload_batch(name, g["draw"])
    o = solve_batch(b.cfg, b.gamma, b.sigma)
    out = {k: v.cpu().numpy() for k, v in o.items() if hasattr(v, "cpu")}
    assert _compare(name, g, out) == []
    assert not np.any(out["status"] == 4)
