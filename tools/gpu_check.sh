#!/bin/bash
# One GPU-box pass: parity suite, bench line, phase profile, work scan, launch list.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python tools/phase_profile.py c1 1024 > gpurun_out/phase_c1.txt 2>&1
python tools/work_scan.py c1 0 1024 > gpurun_out/work_c1.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
