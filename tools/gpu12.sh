rm -f gpurun_out/variants.txt
for v in base l1 ca; do
HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c2 592 >> gpurun_out/variants.txt 2>&1
done
