rm -f gpurun_out/variants.txt
HCRAN_LIB=tools/variants/lib_grp.so python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_grp.so python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
done
python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_grp.so python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
python tools/variant_time.py c0 128 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_grp.so python tools/variant_time.py c0 128 >> gpurun_out/variants.txt 2>&1
