#!/bin/bash
# Shared-memory residency sweep: device time vs HCRAN_HOT_KB (Work::HOT_* arrays in dynamic smem),
# then the GPU parity suite with the arrays in shared memory.
mkdir -p gpurun_out
rm -f gpurun_out/hot.txt
for i in 1 2; do
  for kb in 0 12 92 132 172 212; do
    echo -n "hot_kb=$kb " >> gpurun_out/hot.txt
    HCRAN_HOT_KB=$kb python tools/variant_time.py c1 1024 >> gpurun_out/hot.txt 2>&1
  done
done
for kb in 0 100; do echo -n "hot_kb=$kb " >> gpurun_out/hot.txt; HCRAN_HOT_KB=$kb python tools/variant_time.py c2 592 >> gpurun_out/hot.txt 2>&1; done
for kb in 0 12 92 212; do echo -n "hot_kb=$kb " >> gpurun_out/hot.txt; HCRAN_HOT_KB=$kb python tools/variant_time.py c0 128 >> gpurun_out/hot.txt 2>&1; done
for kb in 0 212; do echo -n "hot_kb=$kb " >> gpurun_out/hot.txt; HCRAN_HOT_KB=$kb python tools/variant_time.py c4 4096 >> gpurun_out/hot.txt 2>&1; done
HCRAN_HOT_KB=212 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_hot.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_hot.log
