"""TEST-ONLY: build and drive the host emulation of the device solver
(tests/emu/hcran_emu.cpp) on numpy buffers.  Used by the CPU test-suite to
check the kernel logic against the oracle without a GPU."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1803_07772_b200 import _abi, pack

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SRC = os.path.join(HERE, "hcran_emu.cpp")
LIB = os.path.join(HERE, "libhcran_emu.so")
DEPS = [SRC] + [os.path.join(ROOT, "paper_1803_07772_b200", "csrc", f)
                for f in ("hcran_solver.cuh", "hcran_exec.cuh", "hcran_work.cuh")] + \
       [os.path.join(ROOT, "include", "hcran_b200.h")]

_lib = None


def build(force: bool = False) -> str:
    stale = not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB)
                                           for d in DEPS)
    if force or stale:
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC",
                        "-I" + os.path.join(ROOT, "include"), "-o", LIB, SRC], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.hcran_emu_solve.argtypes = [C.POINTER(_abi.Problem), C.POINTER(_abi.BatchIn),
                                         C.POINTER(_abi.BatchOut), C.c_int, C.c_int64,
                                         C.c_int64, C.c_int]
        _lib.hcran_emu_solve.restype = C.c_int
    return _lib


def run(cfg, gamma, sigma, mode=0, elastic=None, min_rates=None, e_fixed=None, warm_p=None,
        dense_off=False, exact=False):
    pa = pack.problem_arrays(cfg, sigma)
    ia = pack.instance_arrays(cfg, gamma, elastic, min_rates, e_fixed, warm_p)
    B, M, K, N = ia["gamma"].shape
    T = cfg.tolerances.outer_max
    oa = pack.out_arrays(B, M, K, N, T, S=cfg.tolerances.s_max)
    prob = pack.problem_struct(cfg, {k: v.ctypes.data for k, v in pa.items()}, exact=exact)
    bi = _abi.BatchIn(B=B, gamma=ia["gamma"].ctypes.data, elastic=ia["elastic"].ctypes.data,
                      min_rates=ia["min_rates"].ctypes.data,
                      e_fixed=ia["e_fixed"].ctypes.data if "e_fixed" in ia else None,
                      warm_p=ia["warm_p"].ctypes.data if "warm_p" in ia else None)
    bo = _abi.BatchOut(**{k: v.ctypes.data for k, v in oa.items()})
    rc = lib().hcran_emu_solve(C.byref(prob), C.byref(bi), C.byref(bo), mode, 0, B,
                               1 if dense_off else 0)
    assert rc == 0
    return oa
