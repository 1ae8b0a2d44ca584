rm -f gpurun_out/variants.txt
for i in 1 2; do
python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_load4.so python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
done
python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_load4.so python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
