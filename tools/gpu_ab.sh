#!/bin/bash
# A/B of a kernel change on one B200: GPU parity suite, then c1 / c2 bench lines
# with the change (default) and without it (the env switch given as $1, e.g. HCRAN_FAST=0).
mkdir -p gpurun_out
OFF=${1:-HCRAN_FAST=0}
TAG=${2:-ab}
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for cfg in "c1 1024" "c2 2960"; do
  set -- $cfg
  python bench.py --config $1 --batch $2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_on_$1.json 2> gpurun_out/${TAG}_on_$1.err
  env $OFF python bench.py --config $1 --batch $2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_off_$1.json 2> gpurun_out/${TAG}_off_$1.err
done
echo done
