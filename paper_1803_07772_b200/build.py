"""Build the in-tree sm_100a library libhcran_b200.so (nvcc, no JIT cache).

The library is the product's only compute path; it is built next to this file
so it travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhcran_b200.so")
SOURCES = [os.path.join(CSRC, "hcran_kernel.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("hcran_solver.cuh", "hcran_exec.cuh", "hcran_work.cuh")] + \
    [os.path.join(ROOT, "include", "hcran_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "--fmad=false",  # the reference rounds every product (numpy): keep cancellations identical
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC", "-lcudart"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + ["-I" + os.path.join(ROOT, "include"), "-o", LIB] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libhcran_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
