"""ctypes mirror of include/hcran_b200.h (the C ABI of libhcran_b200.so).

The structures are plain C: device pointers are passed as integers (torch
tensors' data_ptr()), so the library never sees a torch type.
"""

from __future__ import annotations

import ctypes as C

HCRAN_ST = {0: "converged", 1: "cap", 2: "stalled", 3: "infeasible", 4: "unsupported"}
HCRAN_ST_FIXED = {0: "ok", 3: "infeasible", 4: "unsupported"}
ERRORS = {-1: "bad argument", -2: "unsupported size", -3: "workspace too small",
          -4: "CUDA launch failure"}


class Tolerances(C.Structure):
    _fields_ = [("xi", C.c_double), ("varpi1_rel", C.c_double), ("varpi2_rel", C.c_double),
                ("s_max", C.c_int32), ("v_max", C.c_int32), ("outer_max", C.c_int32),
                ("rho1", C.c_double), ("rho2", C.c_double), ("dual_cap", C.c_double),
                ("c13_rate_tol", C.c_double), ("c14_rel_tol", C.c_double),
                ("box_rel_tol", C.c_double)]


class Problem(C.Structure):
    _fields_ = [("M", C.c_int32), ("K", C.c_int32), ("N", C.c_int32), ("l_max", C.c_int32),
                ("p_max", C.c_void_p), ("p_mask", C.c_void_p), ("eta", C.c_void_p),
                ("weights", C.c_void_p), ("sigma", C.c_void_p),
                ("static_power", C.c_double), ("tol", Tolerances), ("sic_mode", C.c_int32)]


class Synth(C.Structure):
    _fields_ = [("M", C.c_int32), ("K", C.c_int32), ("N", C.c_int32),
                ("rrh_xy", C.c_void_p), ("disc_radius", C.c_double),
                ("pathloss_exp", C.c_double), ("seed", C.c_uint64)]


class BatchIn(C.Structure):
    _fields_ = [("B", C.c_int64), ("gamma", C.c_void_p), ("elastic", C.c_void_p),
                ("min_rates", C.c_void_p), ("e_fixed", C.c_void_p), ("warm_p", C.c_void_p)]


OUT_FIELDS = [
    # name, dtype, shape-kind
    ("p", "f8", "MKN"), ("rho", "u1", "MKN"), ("a", "u1", "MK"),
    ("ee", "f8", ""), ("sum_rate", "f8", ""), ("total_power", "f8", ""),
    ("final_e", "f8", ""), ("objective", "f8", ""),
    ("outer_iters", "i4", ""), ("rounds", "i4", ""), ("sweeps", "i4", ""),
    ("bisect_evals", "i4", ""), ("status", "i1", ""), ("feasible", "u1", ""),
    ("xi", "f8", "M"), ("zeta", "f8", "K"),
    ("e_trace", "f8", "T"), ("surplus_trace", "f8", "T"),
    ("rounds_trace", "i4", "T"), ("sweeps_trace", "i4", "T"),
    ("flags", "u1", ""), ("work", "f8", ""),
    ("round_obj", "f8", "S"), ("fp_residual", "f8", ""), ("max_dual", "f8", ""),
    ("floor_hits", "i4", ""),
]


class BatchOut(C.Structure):
    _fields_ = [(name, C.c_void_p) for name, _, _ in OUT_FIELDS]


def out_shape(kind: str, B: int, M: int, K: int, N: int, T: int, S: int = 20) -> tuple:
    return {"MKN": (B, M, K, N), "MK": (B, M, K), "": (B,), "M": (B, M), "K": (B, K),
            "T": (B, T), "S": (B, S)}[kind]


def bind_device_lib(lib: C.CDLL) -> C.CDLL:
    lib.hcran_b200_plan.argtypes = [C.POINTER(Problem), C.c_int64, C.c_int,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_size_t)]
    lib.hcran_b200_plan.restype = C.c_int
    for fn in (lib.hcran_b200_solve_batch, lib.hcran_b200_solve_fixed_e_batch,
               lib.hcran_b200_report_batch):
        fn.argtypes = [C.POINTER(Problem), C.POINTER(BatchIn), C.POINTER(BatchOut),
                       C.c_void_p, C.c_size_t, C.c_void_p]
        fn.restype = C.c_int
    lib.hcran_b200_engine.argtypes = [C.POINTER(Problem), C.c_int64, C.c_int,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_size_t)]
    lib.hcran_b200_engine.restype = C.c_int
    lib.hcran_b200_last_launches.argtypes = []
    lib.hcran_b200_last_launches.restype = C.c_int32
    lib.hcran_b200_synth_gamma.argtypes = [C.POINTER(Synth), C.c_int64, C.c_int64, C.c_void_p,
                                           C.c_void_p]
    lib.hcran_b200_synth_gamma.restype = C.c_int
    lib.hcran_b200_version.argtypes = []
    lib.hcran_b200_version.restype = C.c_char_p
    return lib


EXPORTED = ("hcran_b200_plan", "hcran_b200_solve_batch", "hcran_b200_solve_fixed_e_batch",
            "hcran_b200_engine", "hcran_b200_last_launches", "hcran_b200_synth_gamma",
            "hcran_b200_report_batch",
            "hcran_b200_version")
