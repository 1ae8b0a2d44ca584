#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01_last.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r01_last.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_last.log
python bench.py > gpurun_out/bench_last_c1.json 2> gpurun_out/bench_last_c1.err
python bench.py --config c0 --no-cpu-baseline > gpurun_out/bench_last_c0.json 2> gpurun_out/bench_last_c0.err
python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_last_c4.json 2> gpurun_out/bench_last_c4.err
