"""The reference's own Dinkelbach / SCALE edge cases (test_dinkelbach.py:62-132,
test_scale.py:343-383) through this package's reference-shaped API on the
B200: `solve(ch, cfg, inner)` (device loop with the B200 ScaleSolver; the
reference's host loop for any other InnerSolver, surplus/EE on the device),
`ScaleSolver().solve_fixed_e` with the reference's SolveStats fields."""

from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1803_07772_b200 import (InfeasibleProblemError, InnerResult, PowerAllocation,  # noqa: E402
                                   ScaleSolver, SolveStats, Tolerances, energy_report, solve)
from refcases import make_channel, make_config  # noqa: E402


@pytest.fixture
def small():
    cfg = make_config()
    return cfg, make_channel(cfg)


class FixedInner:
    """Always returns the same allocation (test_dinkelbach.py:12-21)."""

    def __init__(self, alloc):
        self.alloc = alloc

    def solve_fixed_e(self, ch, cfg, e, warm_start=None):
        return InnerResult(self.alloc, "ok", SolveStats())


class Wrapped:
    """The B200 inner solver behind the reference's host-driven loop."""

    def __init__(self):
        self.s = ScaleSolver()

    def solve_fixed_e(self, ch, cfg, e, warm_start=None):
        return self.s.solve_fixed_e(ch, cfg, e, warm_start)


def test_degenerate_two_iterations(small):
    cfg, ch = small
    fixed = PowerAllocation(p=np.random.default_rng(4).uniform(0.0, 0.3, ch.gamma.shape))
    tr = solve(ch, cfg, FixedInner(fixed))
    ee = float(energy_report(ch, cfg, fixed.p)["ee"][0])
    assert tr.status == "converged" and len(tr.iterations) <= 2
    assert abs(tr.final_e - ee) <= 1e-9 * ee
    assert tr.iterations[-1].surplus <= cfg.tolerances.xi


def test_monotone_e_and_termination():
    cfg = make_config(m=2, k=4, n=3, streaming=(0,))
    ch = make_channel(cfg, seed=5)
    tr = solve(ch, cfg, ScaleSolver())
    es = tr.e_values
    assert all(b > a for a, b in zip(es, es[1:]))
    assert -cfg.tolerances.xi <= tr.iterations[-1].surplus <= cfg.tolerances.xi
    assert tr.final_allocation is not None


def test_device_loop_equals_reference_host_loop():
    """The device Dinkelbach loop and the reference's host loop over the B200
    inner solver produce the same trace."""
    cfg = make_config(m=2, k=4, n=3, streaming=(0,))
    ch = make_channel(cfg, seed=5)
    a = solve(ch, cfg, ScaleSolver())
    b = solve(ch, cfg, Wrapped())
    assert a.status == b.status and len(a.iterations) == len(b.iterations)
    assert np.allclose(a.e_values, b.e_values, rtol=1e-12, atol=0)
    assert abs(a.final_e - b.final_e) <= 1e-12 * a.final_e
    assert np.array_equal(a.final_allocation.p, b.final_allocation.p)


def test_infeasible_streaming_raises():
    cfg = make_config(m=1, k=2, n=1, streaming=(0,), bandwidth=1e-3)
    ch = make_channel(cfg, seed=6)
    with pytest.raises(InfeasibleProblemError):
        solve(ch, cfg, ScaleSolver())
    with pytest.raises(InfeasibleProblemError):
        solve(ch, cfg, Wrapped())


def test_cap_hit_flag(small):
    cfg, ch = small

    class ImprovingInner:
        def __init__(self):
            self.scale = 2.0

        def solve_fixed_e(self, ch, cfg, e, warm_start=None):
            self.scale *= 0.5
            return InnerResult(PowerAllocation(p=cfg.p_mask * self.scale), "ok", SolveStats())

    cfg = replace(cfg, tolerances=Tolerances(xi=1e-12, outer_max=3))
    tr = solve(ch, cfg, ImprovingInner())
    assert tr.cap_hit and tr.status == "cap"


def test_matches_grid_oracle_on_tiny_instance():
    cfg = make_config(m=1, k=2, n=2, p_max=[1.0])
    ch = make_channel(cfg, seed=9, gamma_scale=1e-8)
    tr = solve(ch, cfg, ScaleSolver())
    levels = 20
    axes = [np.linspace(0, cfg.p_mask.reshape(-1)[i], levels) for i in range(4)]
    mesh = np.meshgrid(*axes, indexing="ij")
    p = np.stack([m.reshape(-1) for m in mesh], axis=1).reshape(-1, 1, 2, 2)
    ok = p.sum(axis=(1, 2, 3)) <= cfg.p_max[0] * (1 + 1e-12)
    rep = energy_report(ch, cfg, p[ok])
    assert tr.final_e >= 0.98 * rep["ee"].max()


def test_round_objectives_nondecreasing():
    for seed in range(6):
        cfg = make_config(m=2, k=4, n=3, streaming=(0,))
        ch = make_channel(cfg, seed=30 + seed)
        res = ScaleSolver().solve_fixed_e(ch, cfg, e=float(seed) * 0.5)
        objs = res.stats.round_objectives
        assert len(objs) == res.stats.rounds >= 1
        assert all(b >= a - 1e-9 for a, b in zip(objs, objs[1:])), objs


def test_output_feasible():
    for seed in range(5):
        cfg = make_config(m=2, k=4, n=3, streaming=(0, 1))
        ch = make_channel(cfg, seed=40 + seed)
        res = ScaleSolver().solve_fixed_e(ch, cfg, e=0.3)
        assert res.status == "ok"
        assert energy_report(ch, cfg, res.allocation.p)["feasible"][0]


def test_fixed_point_residual_and_stats():
    cfg = make_config(m=1, k=2, n=2)
    ch = make_channel(cfg, seed=50)
    res = ScaleSolver().solve_fixed_e(ch, cfg, e=0.5)
    assert res.stats.fixed_point_residual < cfg.tolerances.varpi1_rel * 10
    assert res.stats.max_dual > 0 and res.stats.denominator_floor_hits >= 0
    assert res.stats.wall_time > 0


def test_infeasible_detection():
    cfg = make_config(m=1, k=2, n=1, streaming=(0,), bandwidth=1e-3)
    ch = make_channel(cfg, seed=51)
    res = ScaleSolver().solve_fixed_e(ch, cfg, e=0.0)
    assert res.status == "infeasible" and res.stats.infeasible_reason


def test_never_worse_than_warm_start():
    cfg = make_config(m=2, k=4, n=3, streaming=(0,))
    ch = make_channel(cfg, seed=52)
    s = ScaleSolver()
    first = s.solve_fixed_e(ch, cfg, e=0.0)
    res = s.solve_fixed_e(ch, cfg, 1.0, warm_start=first.allocation)
    a = energy_report(ch, cfg, res.allocation.p, 1.0)["objective"][0]
    b = energy_report(ch, cfg, first.allocation.p, 1.0)["objective"][0]
    assert a >= b - 1e-9


def test_knobs():
    ScaleSolver(workers=8, collect_trace=True)  # accepted: no effect on the device path
    with pytest.raises(NotImplementedError):
        ScaleSolver(damping=0.5)
