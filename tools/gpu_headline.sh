#!/bin/bash
# Headline pass on one B200: GPU suite, phase profiles, a short c2 line, then the
# driver's default bench command (c2 / 16,384, --steps 20 --warmup 5) with its wall time.
TAG=${1:-r02h}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
python tools/phase_profile.py c2 296 > gpurun_out/phase_${TAG}_c2.txt 2>&1
python tools/phase_profile.py c1 1024 > gpurun_out/phase_${TAG}_c1.txt 2>&1
python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2_b2960.json 2>&1
python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c1.json 2>&1
t0=$(date +%s)
timeout 1750 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
echo "c2 default (--steps 20 --warmup 5) wall $(( $(date +%s) - t0 )) s" > gpurun_out/bench_${TAG}_walls.txt
