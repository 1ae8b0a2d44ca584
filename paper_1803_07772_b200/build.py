"""Build the in-tree sm_100a library libhcran_b200.so (nvcc, no JIT cache).

The library is the product's only compute path; it is built next to this file
so it travels with the repository snapshot to the GPU box.  The translation
units (the C ABI, one per kernel launch shape) compile in parallel.
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhcran_b200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("hcran_kernel.cu", "hcran_k256.cu", "hcran_k512.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("hcran_solver.cuh", "hcran_exec.cuh", "hcran_work.cuh",
                                           "hcran_kernel.cuh")] + \
    [os.path.join(ROOT, "include", "hcran_b200.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++17",
                 "--fmad=false",  # the reference rounds every product (numpy): keep cancellations identical
                 "-Xptxas", "-v", "-Xcompiler", "-fPIC"]
# kept for tools that compile the sources in one nvcc call (profiling variants)
NVCC_FLAGS = CFLAGS + ["-shared", "-lcudart"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build_lib(out: str, extra=(), verbose: bool = False) -> str:
    """Compile every translation unit in parallel and link `out`."""
    inc = "-I" + os.path.join(ROOT, "include")
    with tempfile.TemporaryDirectory() as tmp:
        def one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            r = subprocess.run([nvcc()] + CFLAGS + list(extra) + [inc, "-c", "-o", obj, src],
                               capture_output=True, text=True)
            return src, obj, r
        with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
            res = list(pool.map(one, SOURCES))
        log = ""
        for src, obj, r in res:
            log += r.stdout + r.stderr
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
        r = subprocess.run([nvcc()] + ARCH + ["-shared", "-o", out] + [o for _, o, _ in res] +
                           ["-lcudart"], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    if verbose:
        sys.stderr.write(log)
    return log


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    log = build_lib(LIB, verbose=verbose)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
