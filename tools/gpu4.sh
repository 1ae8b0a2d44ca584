python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
rm -f gpurun_out/variants.txt
python tools/variant_time.py c1 4096 >> gpurun_out/variants.txt 2>&1
python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
