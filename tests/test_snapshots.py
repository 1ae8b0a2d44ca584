"""Localising parity harness: the device solver source (host
build) against reference mid-solve snapshots (tests/golden/snapshots.npz,
make_snapshots.py), so a divergence is pinned to one sweep or to the budget
multiplier instead of an end-to-end EE.

* budget multiplier: every non-trivial `scale._budget_dual` call of the
  captured solves (scale.py:444-475), replayed through the device's
  Newton-estimate / replay / verify algorithm with the reference's load
  function -- bit-identical multipliers;
* one sweep from the start of SCA rounds 0-2 of the first inner solve
  (scale.py:575-594): p_next, xi, zeta and the seated pairs' zeta_t within
  1e-12 relative."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from emu import runner
from paper_1803_07772_b200.scenarios import workload_instance

Z = np.load(os.path.join(GOLDEN, "snapshots.npz"))
KEYS = sorted({tuple(k.split("/")[:3]) for k in Z.files})


def _get(name, d, tag):
    pre = f"{name}/{d}/{tag}/"
    return {k[len(pre):]: Z[k] for k in Z.files if k.startswith(pre)}


def test_budget_multiplier_bit_exact():
    n = 0
    for name, d, tag in KEYS:
        if not tag.startswith("bud"):
            continue
        b = _get(name, d, tag)
        xi, ev = runner.budget(b["num"], b["den"], b["mask"], b["budget"], b["warm"])
        assert np.array_equal(xi, b["xi"]), (name, d, tag, xi, b["xi"])
        n += 1
    assert n >= 200


def _rel(a, b):
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) if a.size else 0.0


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_one_sweep_from_snapshot(name):
    n = 0
    for nm, d, tag in KEYS:
        if nm != name or not tag.startswith("snap"):
            continue
        s = _get(nm, d, tag)
        if "p_next" not in s:
            continue
        cfg, ch, _ = workload_instance(name, int(d))
        p, xi, zeta, zt, fg = runner.sweep_snapshot(cfg, ch.gamma, ch.sigma, s["p"], s["xi"],
                                                    s["zeta"], s["zeta_t"])
        assert not fg, (name, d, tag)
        seats = s["p"] > 1e-30 * cfg.max_mask
        assert _rel(p[seats], s["p_next"][seats]) <= 1e-12, (name, d, tag)
        assert np.array_equal(p[~seats], s["p_next"][~seats])
        assert _rel(xi, s["xi_next"]) <= 1e-12
        assert _rel(zeta, s["zeta_next"]) <= 1e-12
        # seated pairs: both members seated on (m, n)
        st, wk = s["strong"], s["weak"]
        mm = np.arange(cfg.n_rrh)[:, None, None]
        nn = np.arange(cfg.n_subcarriers)[None, None, :]
        both = seats[mm, st, nn] & seats[mm, wk, nn]
        assert _rel(zt[both], s["zeta_t_next"][both]) <= 1e-12, (name, d, tag)
        n += 1
    assert n >= 4
