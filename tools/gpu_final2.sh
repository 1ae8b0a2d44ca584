#!/bin/bash
# Round-end measurement pass (one B200): parity, smoke, bench lines for every config, reference arm,
# launch list and full ncu captures of config[1] and config[2].
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
for i in 1 2; do
  HCRAN_LIB=tools/variants/lib_ch8.so python tools/variant_time.py c1 1024 >> gpurun_out/ab.txt 2>&1
  python tools/variant_time.py c1 1024 >> gpurun_out/ab.txt 2>&1
done
python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config c0 > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
python bench.py --config c4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c2 --batch 2960 --steps 3 --cpu-sample 4 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c1.json 2> gpurun_out/bench_ref_c1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:hcran_solve_kernel -c 1 -o gpurun_out/c1_bench_full \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
python tools/phase_profile.py c1 1024 > gpurun_out/phase_c1.txt 2>&1
python tools/phase_profile.py c2 148 > gpurun_out/phase_c2.txt 2>&1
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
echo done
