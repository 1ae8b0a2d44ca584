"""Host-side packing of reference-shaped inputs into the C ABI's flat arrays.

Takes any reference-compatible NetworkConfig (hcran_noma.model.NetworkConfig
or paper_1803_07772_b200.model.NetworkConfig, duck-typed) and builds the
per-batch constant arrays plus the per-instance arrays, as numpy.  Moving them
to the device (torch) and binding pointers happens in `solver.py`.
"""

from __future__ import annotations

import numpy as np

from . import _abi

F8 = np.float64


def tolerances(cfg) -> _abi.Tolerances:
    t = cfg.tolerances
    return _abi.Tolerances(xi=t.xi, varpi1_rel=t.varpi1_rel, varpi2_rel=t.varpi2_rel,
                           s_max=t.s_max, v_max=t.v_max, outer_max=t.outer_max,
                           rho1=float(cfg.rho1), rho2=float(cfg.rho2), dual_cap=t.dual_cap,
                           c13_rate_tol=t.c13_rate_tol, c14_rel_tol=t.c14_rel_tol,
                           box_rel_tol=t.box_rel_tol)


def problem_arrays(cfg, sigma: np.ndarray) -> dict:
    """Batch-constant arrays (NetworkConfig fields, model.py:83-185)."""
    M, K, N = cfg.n_rrh, cfg.n_users, cfg.n_subcarriers
    sig = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma, F8), (M, K, N)))
    return {"p_max": np.ascontiguousarray(cfg.p_max, F8),
            "p_mask": np.ascontiguousarray(cfg.p_mask, F8),
            "eta": np.ascontiguousarray(cfg.eta, F8),
            "weights": np.ascontiguousarray(cfg.weights, F8),
            "sigma": sig}


def problem_struct(cfg, ptrs: dict, exact=False) -> _abi.Problem:
    """exact: False -> HCRAN_SIC_SEATED (default), True -> HCRAN_SIC_DENSE,
    "fast" -> HCRAN_SIC_SEATED_FAST."""
    return _abi.Problem(M=cfg.n_rrh, K=cfg.n_users, N=cfg.n_subcarriers, l_max=cfg.l_max,
                        p_max=ptrs["p_max"], p_mask=ptrs["p_mask"], eta=ptrs["eta"],
                        weights=ptrs["weights"], sigma=ptrs["sigma"],
                        static_power=float(cfg.static_power()), tol=tolerances(cfg),
                        sic_mode=2 if exact == "fast" else (1 if exact else 0))


def instance_arrays(cfgs_or_cfg, gamma: np.ndarray, elastic=None, min_rates=None,
                    e_fixed=None, warm_p=None) -> dict:
    """Per-instance arrays.  `elastic` / `min_rates` default to the template
    config's (model.py:151-152, 178-185)."""
    gamma = np.ascontiguousarray(gamma, F8)
    B = gamma.shape[0]
    cfg = cfgs_or_cfg
    if elastic is None:
        elastic = np.broadcast_to(cfg.elastic_mask(), (B, cfg.n_users))
    if min_rates is None:
        min_rates = np.broadcast_to(cfg.min_rates(), (B, cfg.n_users))
    out = {"gamma": gamma,
           "elastic": np.ascontiguousarray(elastic, np.uint8),
           "min_rates": np.ascontiguousarray(min_rates, F8)}
    if e_fixed is not None:
        out["e_fixed"] = np.ascontiguousarray(np.broadcast_to(e_fixed, (B,)), F8)
    if warm_p is not None:
        out["warm_p"] = np.ascontiguousarray(warm_p, F8)
    return out


def out_arrays(B: int, M: int, K: int, N: int, T: int, want=None, S: int = 20) -> dict:
    arrs = {}
    for name, dt, kind in _abi.OUT_FIELDS:
        if want is not None and name not in want:
            continue
        arrs[name] = np.zeros(_abi.out_shape(kind, B, M, K, N, T, S), dtype=dt)
    return arrs
