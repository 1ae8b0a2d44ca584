#!/bin/bash
# Shared-memory residency / launch-shape sweep at c1 and c2.
# HOT order: 0 CSR 1 CSQ 2 TOT 3 FULL 4 UTOT 5 RNK 6 GAM 7 ALPHA 8 U 9 SLOT 10 P
for cfg in "c1 1024"; do
  set -- $cfg
  for sh in 256:256 512:512; do
  for mk in 0x0 0x7 0x1f 0x20 0x60 0xe0 0x1e0 0x1ff; do
    r=$(HCRAN_SHAPE=$sh HCRAN_HOT_KB=200 HCRAN_HOT_MASK=$mk timeout 300 python bench.py --config $1 --batch $2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
    echo "$1 shape=$sh mask=$mk $r"
  done
  done
done
for mk in 0x0 0x7 0x1f 0x20; do
  r=$(HCRAN_HOT_KB=200 HCRAN_HOT_MASK=$mk timeout 300 python bench.py --config c2 --batch 592 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
  echo "c2 mask=$mk $r"
done
