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
        P = C.POINTER(C.c_double)
        _lib.hcran_emu_budget.argtypes = [P, P, P, C.c_int, C.c_int, P, P, P,
                                          C.POINTER(C.c_int)]
        _lib.hcran_emu_budget.restype = None
        _lib.hcran_emu_sweep_snapshot.argtypes = [C.POINTER(_abi.Problem), C.POINTER(_abi.BatchIn),
                                                  P, P, P, P, P, P, P]
        _lib.hcran_emu_sweep_snapshot.restype = C.c_int
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def budget(num, den, mask, budget_, warm):
    """The device budget multiplier on the reference's (M, K, N) inputs."""
    num, den, mask = (np.ascontiguousarray(x, np.float64) for x in (num, den, mask))
    M = num.shape[0]
    KN = num.size // M
    b = np.ascontiguousarray(budget_, np.float64)
    w = np.ascontiguousarray(warm, np.float64)
    xi = np.zeros(M)
    ev = (C.c_int * M)()
    lib().hcran_emu_budget(_dp(num), _dp(den), _dp(mask), M, KN, _dp(b), _dp(w), _dp(xi), ev)
    return xi, np.array(ev[:])


def sweep_snapshot(cfg, gamma, sigma, p0, xi0, zeta0, zeta_t0):
    """One device sweep from a reference round-start snapshot."""
    pa = pack.problem_arrays(cfg, sigma)
    ia = pack.instance_arrays(cfg, gamma[None])
    prob = pack.problem_struct(cfg, {k: v.ctypes.data for k, v in pa.items()})
    bi = _abi.BatchIn(B=1, gamma=ia["gamma"].ctypes.data, elastic=ia["elastic"].ctypes.data,
                      min_rates=ia["min_rates"].ctypes.data, e_fixed=None, warm_p=None)
    p0, xi0, zeta0 = (np.ascontiguousarray(x, np.float64) for x in (p0, xi0, zeta0))
    zt = np.ascontiguousarray(zeta_t0, np.float64).copy()
    p_out, xi_out, z_out = np.zeros_like(p0), np.zeros_like(xi0), np.zeros_like(zeta0)
    fg = lib().hcran_emu_sweep_snapshot(C.byref(prob), C.byref(bi), _dp(p0), _dp(xi0), _dp(zeta0),
                                        _dp(zt), _dp(p_out), _dp(xi_out), _dp(z_out))
    return p_out, xi_out, z_out, zt, bool(fg)


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
