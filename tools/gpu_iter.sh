#!/bin/bash
# One optimisation iteration on a B200: branch-free reciprocal check, GPU parity
# suite, phase profiles + bench lines of the default vs HCRAN_FAST=0.
TAG=${1:-it}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I. -Iinclude -o /tmp/rcptest tools/rcptest.cu > gpurun_out/rcptest_$TAG.txt 2>&1 && /tmp/rcptest >> gpurun_out/rcptest_$TAG.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
VARIANTS="${VARIANTS:-2 0}" bash tools/gpu_phase_ab.sh $TAG
