#!/bin/bash
# One optimisation iteration on a B200: branch-free reciprocal / division check,
# GPU parity suite, phase profiles and short bench lines at c1 / c2, and the
# c2 launch-shape alternatives (HCRAN_SHAPE).
TAG=${1:-it}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I. -Iinclude -o /tmp/rcptest tools/rcptest.cu > gpurun_out/rcptest_$TAG.txt 2>&1 && /tmp/rcptest >> gpurun_out/rcptest_$TAG.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
python tools/phase_profile.py c1 1024 > gpurun_out/phase_${TAG}_c1.txt 2>&1
python tools/phase_profile.py c2 296 > gpurun_out/phase_${TAG}_c2.txt 2>&1
python bench.py --config c1 --batch 1024 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c1.json 2>&1
python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2.json 2>&1
for sh in ${SHAPES:-}; do
  HCRAN_SHAPE=$sh python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2_shape${sh/:/_}.json 2>&1
done
