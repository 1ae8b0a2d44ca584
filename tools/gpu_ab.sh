#!/bin/bash
# A/B device time of library variants (tools/variants/lib_*.so) against the default build, then the
# GPU parity suite on the default build.  Usage: bash tools/gpu_ab.sh "base new" [configs...]
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
for i in 1 2; do
  for v in $1; do
    HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c1 1024 >> gpurun_out/ab.txt 2>&1
  done
  python tools/variant_time.py c1 1024 >> gpurun_out/ab.txt 2>&1
done
for v in $1; do
  HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c2 592 >> gpurun_out/ab.txt 2>&1
  HCRAN_LIB=tools/variants/lib_$v.so python tools/variant_time.py c0 128 >> gpurun_out/ab.txt 2>&1
done
python tools/variant_time.py c2 592 >> gpurun_out/ab.txt 2>&1
python tools/variant_time.py c0 128 >> gpurun_out/ab.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_ab.log
