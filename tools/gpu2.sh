python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python tools/work_scan.py c1 0 1024 > gpurun_out/work_c1.txt 2>&1
for v in t256_b1 t256_b2 t128_b4; do HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1; done
for v in t256_b1 t256_b2; do HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1; done
