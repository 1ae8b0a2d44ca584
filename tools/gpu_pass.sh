#!/bin/bash
# One B200 measurement pass (run under gpurun): GPU parity suite, bench lines for
# the named configs, optional ncu captures.  Usage: tools/gpu_pass.sh TAG [configs...]
TAG=${1:-run}; shift
CONFIGS=${@:-c2 c1}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for c in $CONFIGS; do
  case $c in
    c2s) args="--config c2 --batch 2960 --steps 2 --warmup 1 --cpu-sample 4";;
    c2) args="--config c2 --steps 3 --warmup 3 --cpu-sample 8";;
    *) args="--config $c";;
  esac
  timeout 1500 python bench.py $args > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
tail -3 gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/bench_${TAG}_*.json | cut -c1-400
