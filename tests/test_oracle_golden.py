"""The CPU oracle (oracle/hcran_oracle.py) is pinned against golden outputs of
the unmodified reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import rel
from oracle import hcran_oracle as O
from paper_1803_07772_b200.scenarios import workload_instance


@pytest.mark.parametrize("i", range(0, 128, 8))
def test_c0_dinkelbach(golden, i):
    g = golden("c0")
    cfg, ch, _ = workload_instance("c0", int(g["draw"][i]))
    P = O.Prob.from_config(cfg, ch)
    tr = O.dinkelbach(P)
    r, pw, ee = O.report(P, tr.p)
    assert rel(ee, g["ee"][i]) <= 1e-12 and rel(pw, g["total_power"][i]) <= 1e-12
    assert np.array_equal(tr.rho, g["rho"][i]) and np.array_equal(tr.a, g["a"][i])
    assert len(tr.e_values) == np.sum(~np.isnan(g["e_values"][i]))


@pytest.mark.parametrize("i", range(0, 256, 16))
def test_c4_fixed_e(golden, i):
    g = golden("c4")
    cfg, ch, e = workload_instance("c4", int(g["draw"][i]))
    P = O.Prob.from_config(cfg, ch)
    res = O.solve_fixed_e(P, e)
    assert res.status == "ok"
    r, pw, _ = O.report(P, res.p)
    assert rel(r - e * pw, g["objective"][i]) <= 1e-12
    assert res.stats.rounds == g["rounds"][i][0] and res.stats.total_sweeps == g["sweeps"][i][0]


def test_c1_one(golden):
    g = golden("c1")
    cfg, ch, _ = workload_instance("c1", int(g["draw"][5]))
    P = O.Prob.from_config(cfg, ch)
    tr = O.dinkelbach(P)
    _, pw, ee = O.report(P, tr.p)
    assert rel(ee, g["ee"][5]) <= 1e-10 and rel(pw, g["total_power"][5]) <= 1e-10
