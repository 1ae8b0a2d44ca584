python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python tools/phase_profile.py c1 1024 > gpurun_out/phase_c1.txt 2>&1
python tools/phase_profile.py c2 148 > gpurun_out/phase_c2.txt 2>&1
rm -f gpurun_out/variants.txt
python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_ch8.so python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_ch8.so python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
