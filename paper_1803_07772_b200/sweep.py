"""Sweep batcher: the reference's `run_sweep` / `run_draw` campaign runner on
the B200 path.

Mirrors /root/reference/pkg/src/hcran_noma/scenarios.py:160-296:
`Scenario`, `DrawResult`, `SweepRow`, `_config_for` (users / streaming /
arrival / lpn / none sweeps), `run_draw` semantics (InfeasibleProblemError ->
feasible=False; otherwise feasibility of the final allocation, EE, sum rate,
power and outer-iteration count) and the aggregation into per-value means
over feasible draws in deterministic (value, draw) order.  Instead of a
process pool over draws, every sweep value is one batched device solve.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .model import ConfigError
from .scenarios import ARCHITECTURES, build_config, draw_rng, gen_channel


@dataclass(frozen=True)
class Scenario:
    architecture: str = "hcran"
    sweep: str = "users"      # "users" | "streaming" | "arrival" | "lpn" | "none"
    values: tuple = (8, 12, 16)
    k_total: int = 12
    k_streaming: int = 6
    arrival_rate: float = 125.0
    l_max: int = 3
    n_subcarriers: int = 32
    bandwidth_hz: float = 1.0e6
    draws: int = 50
    seed: int = 1
    solver: str = "scale"
    workers: int = 1
    include_timing: bool = False

    def __post_init__(self) -> None:
        if self.architecture not in ARCHITECTURES:
            raise ConfigError(f"unknown architecture {self.architecture!r}")
        if self.sweep not in ("users", "streaming", "arrival", "lpn", "none"):
            raise ConfigError(f"unknown sweep variable {self.sweep!r}")
        if self.solver not in ("scale", "polyblock"):
            raise ConfigError(f"unknown solver {self.solver!r}")


@dataclass
class DrawResult:
    value: float
    draw: int
    feasible: bool
    ee: float = float("nan")
    sum_rate: float = float("nan")
    power: float = float("nan")
    iterations: int = 0
    wall_s: float = 0.0


@dataclass
class SweepRow:
    value: float
    mean_ee: float
    mean_rate: float
    mean_power: float
    mean_iterations: float
    n_feasible: int
    n_draws: int
    mean_wall_s: float


def config_for(scenario: Scenario, value, rng: np.random.Generator):
    """scenarios.py:220-234."""
    kw = dict(architecture=scenario.architecture, k_total=scenario.k_total,
              k_streaming=scenario.k_streaming, rng=rng, arrival_rate=scenario.arrival_rate,
              l_max=scenario.l_max, n_subcarriers=scenario.n_subcarriers,
              bandwidth_hz=scenario.bandwidth_hz)
    if scenario.sweep == "users":
        kw["k_total"] = int(value)
    elif scenario.sweep == "streaming":
        kw["k_streaming"] = int(value)
    elif scenario.sweep == "arrival":
        kw["arrival_rate"] = float(value)
    elif scenario.sweep == "lpn":
        kw["m_f"] = int(value)
    return build_config(**kw)


def _same_template(a, b) -> bool:
    return (a.n_rrh == b.n_rrh and a.n_users == b.n_users and a.n_subcarriers == b.n_subcarriers
            and a.l_max == b.l_max and np.array_equal(a.p_mask, b.p_mask)
            and np.array_equal(a.p_max, b.p_max) and np.array_equal(a.eta, b.eta)
            and np.array_equal(a.weights, b.weights) and a.static_power() == b.static_power()
            and np.array_equal(a.elastic_mask(), b.elastic_mask())
            and np.array_equal(a.min_rates(), b.min_rates()))


def run_value(scenario: Scenario, value, solve_batch=None) -> list[DrawResult]:
    """All draws of one sweep value as one batched device solve."""
    if scenario.solver != "scale":
        raise NotImplementedError("the polyblock oracle is out of the B200 path's scope")
    if solve_batch is None:
        from .solver import solve_batch
    cfgs, gam = [], []
    for d in range(scenario.draws):
        rng = draw_rng(scenario.seed, d)
        cfg = config_for(scenario, value, rng)
        cfgs.append(cfg)
        gam.append(gen_channel(cfg, rng).gamma)
    tmpl = cfgs[0]
    for c in cfgs[1:]:
        if not _same_template(tmpl, c):
            raise ConfigError("draws of one sweep value must share their network template")
    t0 = time.perf_counter()
    out = solve_batch(tmpl, np.stack(gam))
    wall = (time.perf_counter() - t0) / max(scenario.draws, 1)
    o = {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v))
         for k, v in out.items() if not k.startswith("_") and k != "launches"}
    res = []
    for d in range(scenario.draws):
        st = int(o["status"][d])
        if st == 4:  # a capacity limit of the device state (hcran_b200.h), not an outcome
            raise NotImplementedError(f"draw {d}: seating exceeds the device's per-column "
                                      "seat / tuple capacity (HCRAN_ST_UNSUPPORTED)")
        if st == 3:  # InfeasibleProblemError (scenarios.py:248-252)
            res.append(DrawResult(value=value, draw=d, feasible=False, wall_s=wall))
            continue
        res.append(DrawResult(value=value, draw=d, feasible=bool(o["feasible"][d]),
                              ee=float(o["ee"][d]), sum_rate=float(o["sum_rate"][d]),
                              power=float(o["total_power"][d]),
                              iterations=int(o["outer_iters"][d]), wall_s=wall))
    return res


def aggregate(scenario: Scenario, results: list[DrawResult]) -> list[SweepRow]:
    """Per-value means over feasible draws (scenarios.py:278-296)."""
    rows = []
    for value in scenario.values:
        group = [r for r in results if r.value == value]
        good = [r for r in group if r.feasible]
        if good:
            rows.append(SweepRow(value=float(value), mean_ee=float(np.mean([r.ee for r in good])),
                                 mean_rate=float(np.mean([r.sum_rate for r in good])),
                                 mean_power=float(np.mean([r.power for r in good])),
                                 mean_iterations=float(np.mean([r.iterations for r in good])),
                                 n_feasible=len(good), n_draws=len(group),
                                 mean_wall_s=float(np.mean([r.wall_s for r in good]))))
        else:
            rows.append(SweepRow(value=float(value), mean_ee=float("nan"),
                                 mean_rate=float("nan"), mean_power=float("nan"),
                                 mean_iterations=0.0, n_feasible=0, n_draws=len(group),
                                 mean_wall_s=0.0))
    return rows


def run_sweep(scenario: Scenario, solve_batch=None) -> list[SweepRow]:
    results = []
    for value in scenario.values:
        results.extend(run_value(scenario, value, solve_batch))
    return aggregate(scenario, results)
