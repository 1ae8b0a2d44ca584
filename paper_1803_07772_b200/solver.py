"""B200 solve entry points with the reference's names and result layout.

Drop-in surface:

* `ScaleSolver().solve_fixed_e(ch, cfg, e, warm_start)` -> `InnerResult`
  (scale.py:489-551; the `InnerSolver` protocol of dinkelbach.py:28-33)
* `solve(ch, cfg, inner=None)` -> `DinkelbachTrace` (dinkelbach.py:65-112),
  with the whole outer loop on the device
* `solve_batch(cfg, gamma, ...)` -> dict of per-instance tensors: the batched
  form the C ABI exposes (one launch pair for the whole batch)

Host code only packs arguments and moves buffers (torch is the device-memory
and stream plumbing); all arithmetic runs in libhcran_b200.so.  There is no
CPU fallback: without the library or a CUDA device every call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi, pack
from .model import PowerAllocation

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HCRAN_LIB", os.path.join(_HERE, "libhcran_b200.so"))


class InfeasibleProblemError(RuntimeError):
    """The streaming constraints cannot be met (dinkelbach.py:24-25)."""


class B200Unavailable(RuntimeError):
    """libhcran_b200.so or a CUDA device is missing: there is no fallback."""


_lib = None


def library() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise B200Unavailable(f"{LIB_PATH} not built (run __graft_entry__.build())")
        _lib = _abi.bind_device_lib(C.CDLL(LIB_PATH))
    return _lib


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise B200Unavailable("no CUDA device: the B200 solver has no CPU path")
    return torch


_TORCH_DT = {"f8": "float64", "u1": "uint8", "i4": "int32", "i1": "int8"}


class DeviceProblem:
    """Batch-constant config arrays resident on the device + the C struct
    (hcran_problem_t).  Build once per (config, noise, SIC mode) and pass as
    `solve_batch(..., problem=)` to keep per-batch host work to the launch."""

    def __init__(self, cfg, sigma=None, device=None, exact=False):
        torch = _torch()
        library()
        if sigma is None:
            sigma = _flat_sigma(cfg)
        arrs = pack.problem_arrays(cfg, sigma)
        self.device = torch.device(device or "cuda")
        self.t = {k: torch.from_numpy(np.array(v)).to(self.device) for k, v in arrs.items()}
        self.struct = pack.problem_struct(cfg, {k: v.data_ptr() for k, v in self.t.items()},
                                          exact=exact)
        self.shape = (cfg.n_rrh, cfg.n_users, cfg.n_subcarriers)
        self.exact = exact


_DeviceProblem = DeviceProblem


def _flat_sigma(cfg):
    M, K, N = cfg.n_rrh, cfg.n_users, cfg.n_subcarriers
    return np.full((M, K, N), cfg.noise_density * cfg.subcarrier_bandwidth)


def _on_device(x, dtype, dev):
    """numpy / torch (pinned host or device) -> contiguous device tensor, stream-ordered."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(dev, dtype, non_blocking=True).contiguous()
    np_dt = np.uint8 if dtype == torch.uint8 else np.float64
    return torch.as_tensor(np.ascontiguousarray(x, np_dt)).to(dev)


def solve_batch(cfg, gamma, sigma=None, elastic=None, min_rates=None, *, mode="dinkelbach",
                e_fixed=None, warm_p=None, stream=None, outputs=None, device=None,
                workspace=None, sync=True, exact=False, problem=None):
    """Solve every instance of a batch on the device.

    cfg        template NetworkConfig (p_max, p_mask, eta, weights, l_max, tolerances)
    gamma      (B, M, K, N) float64 channel gains: numpy (copied in) or a CUDA tensor
    sigma      (M, K, N) noise powers (default: the config's flat noise floor)
    elastic    (B, K) bool / min_rates (B, K): per-instance user classes (default: cfg's)
    mode       "dinkelbach" (full solve), "fixed_e" (one inner solve per instance) or
               "report" (energy report of the allocations in warm_p at e_fixed)
    exact      False (default): seated SIC family, inner solves that meet a floor tie
               are redone with the dense family (HCRAN_SIC_SEATED); True: dense family
               everywhere (HCRAN_SIC_DENSE); "fast": seated family only, floor ties not
               redone (HCRAN_SIC_SEATED_FAST, ~3% of config[1] draws then differ)
    outputs    subset of _abi.OUT_FIELDS names to produce (default: all)
    problem    a DeviceProblem for (cfg, sigma, exact) built earlier (sigma/exact ignored)
    Array inputs may be numpy or torch tensors (host tensors should be pinned:
    they are copied with non_blocking=True on the current stream).
    Returns a dict of CUDA tensors keyed like hcran_batch_out_t (plus "launches").
    """
    torch = _torch()
    lib = library()
    dev = problem.device if problem is not None else torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    # every allocation, copy and the launch are ordered on `s`, with `dev` current
    # (the library launches on the calling thread's current device)
    with torch.cuda.device(dev), torch.cuda.stream(s):
        outs = _solve_batch_on(torch, lib, dev, s, cfg, gamma, sigma, elastic, min_rates, mode,
                               e_fixed, warm_p, outputs, workspace, exact, problem)
    if sync:
        s.synchronize()
    return outs


def _solve_batch_on(torch, lib, dev, s, cfg, gamma, sigma, elastic, min_rates, mode, e_fixed,
                    warm_p, outputs, workspace, exact, problem):
    prob = problem if problem is not None else DeviceProblem(cfg, sigma, dev, exact=exact)
    M, K, N = cfg.n_rrh, cfg.n_users, cfg.n_subcarriers
    g = _on_device(gamma, torch.float64, dev)
    B = int(g.shape[0])
    if elastic is None:
        elastic = np.broadcast_to(cfg.elastic_mask(), (B, K))
    if min_rates is None:
        min_rates = np.broadcast_to(cfg.min_rates(), (B, K))
    el = _on_device(elastic, torch.uint8, dev)
    mr = _on_device(min_rates, torch.float64, dev)
    ef = None
    if mode in ("fixed_e", "report"):
        if not isinstance(e_fixed, torch.Tensor):
            e_fixed = np.broadcast_to(e_fixed, (B,))
        ef = _on_device(e_fixed, torch.float64, dev)
    wp = None
    if warm_p is not None:
        wp = _on_device(warm_p, torch.float64, dev)
    T = cfg.tolerances.outer_max
    outs = {}
    for name, dt, kind in _abi.OUT_FIELDS:
        if outputs is not None and name not in outputs:
            continue
        outs[name] = torch.empty(_abi.out_shape(kind, B, M, K, N, T, cfg.tolerances.s_max),
                                 dtype=getattr(torch, _TORCH_DT[dt]), device=dev)
    bi = _abi.BatchIn(B=B, gamma=g.data_ptr(), elastic=el.data_ptr(), min_rates=mr.data_ptr(),
                      e_fixed=ef.data_ptr() if ef is not None else None,
                      warm_p=wp.data_ptr() if wp is not None else None)
    bo = _abi.BatchOut(**{k: v.data_ptr() for k, v in outs.items()})
    grid, wsb = C.c_int32(), C.c_size_t()
    rc = lib.hcran_b200_plan(C.byref(prob.struct), B, dev.index, C.byref(grid), C.byref(wsb))
    if rc:
        raise ValueError(f"hcran_b200_plan: {_abi.ERRORS.get(rc, rc)}")
    if workspace is None or workspace.numel() < wsb.value:
        workspace = torch.empty(wsb.value, dtype=torch.uint8, device=dev)
    fn = {"dinkelbach": lib.hcran_b200_solve_batch, "fixed_e": lib.hcran_b200_solve_fixed_e_batch,
          "report": lib.hcran_b200_report_batch}[mode]
    rc = fn(C.byref(prob.struct), C.byref(bi), C.byref(bo), workspace.data_ptr(), wsb.value,
            s.cuda_stream)
    if rc:
        raise RuntimeError(f"hcran_b200 solve failed: {_abi.ERRORS.get(rc, rc)}")
    outs["launches"] = int(lib.hcran_b200_last_launches())
    outs["_keepalive"] = (prob, g, el, mr, ef, wp, workspace)
    return outs


# --------------------------------------------------------------------------
# reference-shaped results
# --------------------------------------------------------------------------

@dataclass
class SolveStats:
    """scale.SolveStats (scale.py:405-418).  Every field is reported by the
    device for the inner solve; `trace` (per-sweep records of
    collect_trace=True) stays empty: the sweeps never leave the device.
    `denominator_floor_hits` counts seated cells (unseated cells are pinned at
    p_floor and their denominators are floor-level noise)."""
    status: str = "ok"
    rounds: int = 0
    total_sweeps: int = 0
    round_objectives: list = field(default_factory=list)
    true_objective: float = float("nan")
    used_warm_start: bool = False
    denominator_floor_hits: int = 0
    max_dual: float = 0.0
    fixed_point_residual: float = float("nan")
    infeasible_reason: str | None = None
    wall_time: float = 0.0
    trace: list = field(default_factory=list)
    budget_evals: int = 0   # device counters (no reference counterpart)
    flags: int = 0


@dataclass
class InnerResult:
    allocation: PowerAllocation
    status: str
    stats: SolveStats


@dataclass(frozen=True)
class DinkelbachIteration:
    e: float
    surplus: float
    inner_stats: object


@dataclass
class DinkelbachTrace:
    iterations: list = field(default_factory=list)
    final_e: float = 0.0
    final_allocation: PowerAllocation | None = None
    cap_hit: bool = False
    status: str = "converged"
    xi: np.ndarray | None = None
    zeta: np.ndarray | None = None

    @property
    def e_values(self) -> list[float]:
        return [it.e for it in self.iterations]


def _host(outs: dict) -> dict:
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v)
            for k, v in outs.items() if not k.startswith("_")}


class ScaleSolver:
    """B200 inner solver with the reference's InnerSolver interface
    (scale.py:489-551, dinkelbach.py:28-33).

    `solve_fixed_e` runs one fixed-e solve on the device and returns an
    `InnerResult` with the reference's `SolveStats`; `solve(ch, cfg,
    ScaleSolver())` runs the whole Dinkelbach loop on the device.  The
    reference's constructor knobs are accepted: `workers` (the reference's
    serial == parallel contract holds trivially) and `collect_trace` (no
    per-sweep records) change nothing; the step gains, damping, min_sweeps and
    multistart_cells are compiled into the device solver at the reference's
    defaults, so other values raise NotImplementedError."""

    def __init__(self, workers: int = 1, collect_trace: bool = False,
                 gains=(0.6, 0.8, 0.6, 0.6, 0.6), damping: float = 1.0, min_sweeps: int = 8,
                 multistart_cells: int = 16, device=None):
        if (tuple(gains) != (0.6, 0.8, 0.6, 0.6, 0.6) or damping != 1.0 or min_sweeps != 8
                or multistart_cells != 16):
            raise NotImplementedError("the B200 solver implements the reference defaults only")
        self.workers = workers
        self.collect_trace = collect_trace
        self.device = device

    def solve_fixed_e(self, ch, cfg, e: float, warm_start: PowerAllocation | None = None):
        if e < 0:
            raise ValueError("the efficiency parameter must be non-negative")
        t0 = time.perf_counter()
        warm = None if warm_start is None else np.asarray(warm_start.p, np.float64)[None]
        o = _host(solve_batch(cfg, np.asarray(ch.gamma)[None], np.asarray(ch.sigma),
                              mode="fixed_e", e_fixed=float(e), warm_p=warm,
                              device=self.device))
        st = int(o["status"][0])
        if st == 4:
            raise NotImplementedError("seating beyond the device's per-column capacity "
                                      "(HCRAN_ST_UNSUPPORTED)")
        status = _abi.HCRAN_ST_FIXED.get(st, "infeasible")
        ro = o["round_obj"][0]
        stats = SolveStats(status=status, rounds=int(o["rounds"][0]),
                           total_sweeps=int(o["sweeps"][0]),
                           round_objectives=[float(x) for x in ro[~np.isnan(ro)]],
                           used_warm_start=warm_start is not None,
                           denominator_floor_hits=int(o["floor_hits"][0]),
                           max_dual=float(o["max_dual"][0]),
                           fixed_point_residual=float(o["fp_residual"][0]),
                           budget_evals=int(o["bisect_evals"][0]), flags=int(o["flags"][0]))
        alloc = PowerAllocation(p=o["p"][0].copy())
        if status == "ok":
            alloc.rho, alloc.a = o["rho"][0].copy(), o["a"][0].copy()
            stats.true_objective = float(o["objective"][0])
        else:
            stats.infeasible_reason = "repair could not meet the streaming rates"
        stats.wall_time = time.perf_counter() - t0
        return InnerResult(alloc, status, stats)


def energy_report(ch, cfg, allocations, e: float = 0.0, device=None) -> dict:
    """(sum_rate, total_power, ee, objective at e, feasible, rho, a) of given
    allocations, computed on the device (hcran_b200_report_batch): the
    reference's model.energy_efficiency / check_feasibility / derive_binaries."""
    p = np.asarray(allocations, np.float64)
    if p.ndim == 3:
        p = p[None]
    g = np.broadcast_to(np.asarray(ch.gamma), p.shape)
    return _host(solve_batch(cfg, np.ascontiguousarray(g), np.asarray(ch.sigma), mode="report",
                             e_fixed=float(e), warm_p=p, device=device,
                             outputs=["sum_rate", "total_power", "ee", "objective", "feasible",
                                      "rho", "a", "status"]))


def solve(ch, cfg, inner=None, e0: float = 0.0) -> DinkelbachTrace:
    """dinkelbach.solve (dinkelbach.py:65-112).

    With the B200 ScaleSolver (or no inner solver) and e0 = 0 the whole outer
    loop runs on the device in one launch.  Any other InnerSolver (the
    reference's protocol: `solve_fixed_e(ch, cfg, e, warm_start)` returning
    `.allocation`, `.status`, `.stats`) is driven by the reference's host loop,
    with the surplus and EE of each allocation evaluated on the device."""
    if e0 < 0:
        raise ValueError("the efficiency parameter must be non-negative")
    if (inner is None or isinstance(inner, ScaleSolver)) and e0 == 0.0:
        dev = inner.device if inner is not None else None
        o = _host(solve_batch(cfg, np.asarray(ch.gamma)[None], np.asarray(ch.sigma), device=dev))
        return trace_from_batch(o, 0)
    if inner is None:
        inner = ScaleSolver()
    dev = getattr(inner, "device", None)
    tol = cfg.tolerances
    tr = DinkelbachTrace()
    e, warm = e0, None
    for _ in range(tol.outer_max):
        result = inner.solve_fixed_e(ch, cfg, e, warm_start=warm)
        if result.status != "ok":
            if warm is None:
                raise InfeasibleProblemError(
                    "inner solver found no feasible allocation at e="
                    f"{e:g}: {getattr(result.stats, 'infeasible_reason', None)}")
            tr.status = "stalled"
            break
        warm = result.allocation
        rep = energy_report(ch, cfg, warm.p, e, device=dev)
        s = float(rep["objective"][0])  # R - e P (dinkelbach.surplus)
        tr.iterations.append(DinkelbachIteration(e=e, surplus=s, inner_stats=result.stats))
        ee = float(rep["ee"][0])
        if s <= tol.xi:
            tr.final_e, tr.final_allocation, tr.status = ee, warm, "converged"
            return tr
        if ee <= e:
            tr.status = "stalled"
            break
        e = ee
    else:
        tr.cap_hit = True
        tr.status = "cap"
    if warm is None:
        raise InfeasibleProblemError("inner solver produced no allocation")
    tr.final_e = float(energy_report(ch, cfg, warm.p, device=dev)["ee"][0])
    tr.final_allocation = warm
    return tr


def trace_from_batch(o: dict, b: int) -> DinkelbachTrace:
    st = int(o["status"][b])
    if st == 3:
        raise InfeasibleProblemError("inner solver found no feasible allocation at e=0")
    if st == 4:
        raise NotImplementedError("seating beyond the device's per-column capacity "
                                  "(HCRAN_ST_UNSUPPORTED)")
    tr = DinkelbachTrace()
    n_it = int(o["outer_iters"][b])
    for i in range(n_it):
        stats = SolveStats(rounds=int(o["rounds_trace"][b, i]),
                           total_sweeps=int(o["sweeps_trace"][b, i]))
        tr.iterations.append(DinkelbachIteration(e=float(o["e_trace"][b, i]),
                                                 surplus=float(o["surplus_trace"][b, i]),
                                                 inner_stats=stats))
    tr.status = _abi.HCRAN_ST[st]
    tr.cap_hit = st == 1
    tr.final_e = float(o["final_e"][b])
    tr.final_allocation = PowerAllocation(p=o["p"][b].copy(), rho=o["rho"][b].copy(),
                                          a=o["a"][b].copy())
    tr.xi = o["xi"][b].copy()
    tr.zeta = o["zeta"][b].copy()
    return tr
