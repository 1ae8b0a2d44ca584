"""Reference mid-solve snapshots for the localising parity harness
(scale.py:553-615): the state at the start of SCA round s of
the first inner solve (e = 0, greedy start) of a draw -- p, the carried
multipliers xi / zeta / zeta_t -- and the state after that round's first
sweep (p_next, xi, zeta, zeta_t), plus every `_budget_dual` call of the
solve (inputs and result) for a bit-exact test of the device's budget
multiplier.  Runs the UNMODIFIED reference:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_snapshots.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

DRAWS = {"c1": (0, 1, 2, 3), "c0": (0, 1, 2, 3, 4, 5)}
ROUNDS = (0, 1, 2)


def capture(name, draw):
    from hcran_noma import scale
    from make_golden import _instance
    cfg, ch, _ = _instance(name, draw)
    snaps, bud = [], []
    orig_bd = scale._budget_dual

    def bd(num, den, mask, budget, warm=None, iters=42):
        xi = orig_bd(num, den, mask, budget, warm, iters)
        # the non-trivial calls (some head over budget at 0), a bounded number per draw
        if np.any(xi > 0) and len(bud) < (60 if name == "c0" else 12):
            bud.append(dict(num=num.copy(), den=den.copy(), mask=mask.copy(), budget=budget.copy(),
                            warm=np.zeros_like(budget) if warm is None else warm.copy(), xi=xi.copy()))
        return xi
    scale._budget_dual = bd
    orig_an = scale._SolveContext.analyze
    state = {"round": -1, "v": 0}
    orig_coeffs = scale.coeffs_at

    def coeffs_at(p, ch_, stronger=None):  # called once per round start
        state["round"] += 1
        state["v"] = 0
        return orig_coeffs(p, ch_, stronger)

    def analyze(self, p, duals, coeffs, lin, products_active=True):
        state["v"] += 1
        if state["v"] == 1 and state["round"] in ROUNDS and self.e == 0.0:
            snaps.append(dict(round=state["round"], p=p.copy(), xi=duals.xi.copy(),
                              zeta=duals.zeta.copy(), zeta_t=duals.zeta_t.copy(),
                              strong=self.strong_idx.copy(), weak=self.weak_idx.copy()))
            state["want"] = True
        return orig_an(self, p, duals, coeffs, lin, products_active)
    orig_du = scale.dual_update

    def dual_update(duals, slacks, step, v=1):
        out = orig_du(duals, slacks, step, v)
        if state.get("want"):  # runs after _sweep (scale.py:581-583)
            snaps[-1]["zeta_next"] = out.zeta.copy()
            snaps[-1]["zeta_t_next"] = out.zeta_t.copy()
            state["want"] = False
        return out
    orig_sweep = scale.ScaleSolver._sweep

    def sweep(self, ctx, snap, xi, mask):
        out = orig_sweep(self, ctx, snap, xi, mask)
        if state.get("want"):
            snaps[-1]["p_next"] = out.copy()
            snaps[-1]["xi_next"] = xi.copy()
        return out
    scale._SolveContext.analyze = analyze
    scale.dual_update = dual_update
    scale.coeffs_at = coeffs_at
    scale.ScaleSolver._sweep = sweep
    try:
        scale.ScaleSolver().solve_fixed_e(ch, cfg, 0.0)
    finally:
        scale._budget_dual = orig_bd
        scale._SolveContext.analyze = orig_an
        scale.dual_update = orig_du
        scale.coeffs_at = orig_coeffs
        scale.ScaleSolver._sweep = orig_sweep
    return snaps, bud


def main():
    flat = {}
    for name, draws in DRAWS.items():
        for d in draws:
            snaps, bud = capture(name, d)
            for i, sn in enumerate(snaps):
                for k, v in sn.items():
                    flat[f"{name}/{d}/snap{i}/{k}"] = np.asarray(v)
            for i, b in enumerate(bud):
                for k, v in b.items():
                    flat[f"{name}/{d}/bud{i}/{k}"] = np.asarray(v)
            print(name, d, len(snaps), "snapshots", len(bud), "budget calls", flush=True)
    np.savez_compressed(os.path.join(HERE, "snapshots.npz"), **flat)


if __name__ == "__main__":
    main()
