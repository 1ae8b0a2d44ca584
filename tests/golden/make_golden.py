"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference package (read-only at /root/reference/pkg/src) in this container.

This script is the provenance of every fixture; it is never run on the GPU box
(the reference does not exist there).  Usage:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py c0 --draws 0:128
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py c1 --draws 0:24
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py c4 --draws 0:256
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py c1 --list 598,644,690

Instances are built exactly as `scenarios.run_draw` builds them
(/root/reference/pkg/src/hcran_noma/scenarios.py:237-242): rng =
default_rng([seed=1, draw]); build_config(..., rng=rng); gen_channel(cfg, rng).
c4 follows `tiny_instance` (scenarios.py:310-327) at a fixed 2x4x4 shape and is a
fixed-e inner solve (`ScaleSolver.solve_fixed_e`, scale.py:506-551).

Per instance the fixture stores the reference outputs (p, rho, a, EE, R, P,
final e, Dinkelbach e/surplus trace, rounds/sweeps per outer iteration, status)
and a near-tie flag: the reference re-run 3x with its budget multiplier
perturbed by xi*(1+1e-12*U(-1,1)) at `scale._budget_dual`.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

CONFIGS = {
    # name: (m_f, k_total, k_streaming, n_subcarriers, bandwidth_hz)
    "c0": (2, 6, 2, 8, 1.0e6),
    "c1": (3, 20, 6, 64, 2.0e6),
    "c2": (7, 48, 16, 128, 4.0e6),
    "c3": (15, 128, 42, 256, 8.0e6),
}
NEAR_TIE_REPEATS = 3
NEAR_TIE_DELTA = 1e-12
PARITY_REL = 1e-4


def gamma_digest(gamma: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(gamma, dtype=np.float64).tobytes()).hexdigest()[:16]


def _instance(name: str, draw: int):
    from hcran_noma.scenarios import build_config, gen_channel, tiny_instance
    rng = np.random.default_rng([1, draw])
    if name == "c4":
        inst = tiny_instance(rng, sizes=((2,), (4,), (4,)))
        return inst.cfg, inst.ch, inst.e
    m_f, k, ks, n, bw = CONFIGS[name]
    cfg = build_config(architecture="hcran", m_f=m_f, k_total=k, k_streaming=ks,
                       n_subcarriers=n, bandwidth_hz=bw, rng=rng)
    ch = gen_channel(cfg, rng)
    return cfg, ch, None


def _solve(name: str, draw: int, perturb_seed: int | None):
    from hcran_noma import dinkelbach, model, scale
    orig = scale._budget_dual
    if perturb_seed is not None:
        prng = np.random.default_rng(perturb_seed)

        def perturbed(*args, **kw):
            xi = orig(*args, **kw)
            return xi * (1.0 + NEAR_TIE_DELTA * prng.uniform(-1.0, 1.0, size=xi.shape))
        scale._budget_dual = perturbed
    try:
        cfg, ch, e_fixed = _instance(name, draw)
        out = {}
        if name == "c4":
            res = scale.ScaleSolver().solve_fixed_e(ch, cfg, e_fixed)
            alloc = res.allocation
            out["status"] = res.status
            out["e_fixed"] = e_fixed
            out["rounds"] = np.array([res.stats.rounds])
            out["sweeps"] = np.array([res.stats.total_sweeps])
            out["objective"] = (model.weighted_sum_rate(alloc, ch, cfg)
                                - e_fixed * model.total_power(alloc, cfg))
            rep = model.energy_efficiency(alloc, ch, cfg)
            out["feasible"] = bool(model.check_feasibility(alloc, ch, cfg).ok) if res.status == "ok" else False
        else:
            try:
                trace = dinkelbach.solve(ch, cfg, scale.ScaleSolver())
            except dinkelbach.InfeasibleProblemError:
                out["status"] = "infeasible"
                return out
            alloc = trace.final_allocation
            rep = model.energy_efficiency(alloc, ch, cfg)
            out["status"] = trace.status
            out["final_e"] = trace.final_e
            out["e_values"] = np.array([it.e for it in trace.iterations])
            out["surplus"] = np.array([it.surplus for it in trace.iterations])
            out["rounds"] = np.array([it.inner_stats.rounds for it in trace.iterations])
            out["sweeps"] = np.array([it.inner_stats.total_sweeps for it in trace.iterations])
            out["feasible"] = bool(model.check_feasibility(alloc, ch, cfg).ok)
        out["p"] = alloc.p
        out["rho"] = alloc.rho if alloc.rho is not None else np.zeros(alloc.p.shape, np.uint8)
        out["a"] = alloc.a if alloc.a is not None else np.zeros(alloc.p.shape[:2], np.uint8)
        out["ee"] = rep.ee
        out["sum_rate"] = rep.sum_rate
        out["total_power"] = rep.total_power
        return out
    finally:
        scale._budget_dual = orig


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def run_one(args):
    name, draw = args
    t0 = time.perf_counter()
    base = _solve(name, draw, None)
    wall = time.perf_counter() - t0
    cfg, ch, _ = _instance(name, draw)
    near_tie = False
    if base["status"] not in ("infeasible",):
        for rep in range(NEAR_TIE_REPEATS):
            alt = _solve(name, draw, 1000003 * draw + rep + 1)
            if alt["status"] != base["status"] or alt["status"] == "infeasible":
                near_tie = True
                continue
            if (_rel(alt["ee"], base["ee"]) > PARITY_REL
                    or _rel(alt["total_power"], base["total_power"]) > PARITY_REL
                    or not np.array_equal(alt["rho"], base["rho"])
                    or not np.array_equal(alt["a"], base["a"])):
                near_tie = True
    base["near_tie"] = near_tie
    base["wall_s"] = wall
    base["gamma_digest"] = gamma_digest(ch.gamma)
    base["draw"] = draw
    return base


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--draws", default="0:16")
    ap.add_argument("--list", default=None,
                    help="comma-separated draws (e.g. the draws whose device status is "
                         "infeasible / products-active); written to <config>_<min>_<max+1>_sel.npz")
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--no-near-tie", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    if args.no_near_tie:
        global NEAR_TIE_REPEATS
        NEAR_TIE_REPEATS = 0
    if args.list:
        draws = sorted(int(x) for x in args.list.split(","))
        lo, hi = draws[0], draws[-1] + 1
    else:
        lo, hi = (int(x) for x in args.draws.split(":"))
        draws = list(range(lo, hi))
    tasks = [(args.config, d) for d in draws]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=args.workers) as pool:
        results = list(pool.map(run_one, tasks, chunksize=1))
    print(f"{args.config}: {len(results)} instances in {time.perf_counter() - t0:.1f}s",
          file=sys.stderr)

    # pack: scalars as arrays, tensors stacked (ragged traces padded with nan)
    n = len(results)
    status_codes = {"converged": 0, "cap": 1, "stalled": 2, "infeasible": 3, "ok": 0}
    pack = {
        "config": np.array(args.config),
        "draw": np.array([r["draw"] for r in results], np.int64),
        "status": np.array([status_codes[r["status"]] for r in results], np.int8),
        "near_tie": np.array([r["near_tie"] for r in results], bool),
        "gamma_digest": np.array([r["gamma_digest"] for r in results]),
        "wall_s": np.array([r["wall_s"] for r in results]),
    }
    for key in ("ee", "sum_rate", "total_power", "final_e", "e_fixed", "objective"):
        if any(key in r for r in results):
            pack[key] = np.array([r.get(key, np.nan) for r in results], np.float64)
    pack["feasible"] = np.array([r.get("feasible", False) for r in results], bool)
    ref = next(r for r in results if "p" in r)
    shape = ref["p"].shape
    pack["p"] = np.stack([r.get("p", np.zeros(shape)) for r in results])
    pack["rho"] = np.stack([r.get("rho", np.zeros(shape, np.uint8)) for r in results]).astype(np.uint8)
    pack["a"] = np.stack([r.get("a", np.zeros(shape[:2], np.uint8)) for r in results]).astype(np.uint8)
    t_max = max(len(r.get("rounds", [])) for r in results)
    for key in ("e_values", "surplus", "rounds", "sweeps"):
        arr = np.full((n, max(t_max, 1)), np.nan)
        for i, r in enumerate(results):
            v = r.get(key)
            if v is not None:
                arr[i, :len(v)] = v
        pack[key] = arr
    tag = "_sel" if args.list else ""
    out = args.out or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                   f"{args.config}_{lo}_{hi}{tag}.npz")
    np.savez_compressed(out, **pack)
    print(f"wrote {out}", file=sys.stderr)


if __name__ == "__main__":
    main()
