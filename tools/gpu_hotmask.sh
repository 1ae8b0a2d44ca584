#!/bin/bash
# Which Work::HOT_* arrays to keep in shared memory at config[1]: device time per bit mask
# (bits: Work::HOT_* order: 0 ord, 1 slot, 2 p, 3 gains, 4 alpha, 5 u, 6 t).
mkdir -p gpurun_out
rm -f gpurun_out/hotmask.txt
for i in 1 2; do
  for m in 0x00 0x1F 0x2F 0x37 0x3B 0x3C 0x17 0x0F 0x4F; do
    echo -n "mask=$m " >> gpurun_out/hotmask.txt
    HCRAN_HOT_KB=200 HCRAN_HOT_MASK=$m python tools/variant_time.py c1 1024 >> gpurun_out/hotmask.txt 2>&1
  done
done
