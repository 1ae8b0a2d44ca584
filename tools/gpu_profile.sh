#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, one GPU):
#  1. launch list of a short bench run (gpu__time_duration per launch)
#  2. one --set full capture of the solve kernel on a c2 batch of $2 instances
#     (default 2960), reduced on the box to the raw-metric CSV and the top
#     source lines (the .ncu-rep and the source CSV exceed gpurun's 64 MiB)
TAG=${1:-r02}; NB=${2:-2960}; CFG=${3:-c2}
mkdir -p gpurun_out
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:hcran_solve_kernel -c 1 -o /tmp/full_${TAG} \
    python tools/ncu_one.py $CFG $NB > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu -i /tmp/full_${TAG}.ncu-rep --page raw --csv > gpurun_out/ncu_full_${TAG}_${CFG}_b${NB}_raw.csv 2>/dev/null
ncu -i /tmp/full_${TAG}.ncu-rep --page details --csv > gpurun_out/ncu_full_${TAG}_${CFG}_b${NB}_details.csv 2>/dev/null
ncu -i /tmp/full_${TAG}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_${TAG}.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_${TAG}.csv 60 > gpurun_out/ncu_lines_${TAG}_${CFG}_b${NB}.txt 2>&1
echo done
