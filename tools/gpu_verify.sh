#!/bin/bash
# Verification of the final build on one B200: GPU suite, smoke, short c1 / c2 lines.
TAG=${1:-r02v}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2_b2960.json 2>&1
python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c1.json 2>&1
