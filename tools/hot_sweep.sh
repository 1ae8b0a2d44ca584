#!/bin/bash
# Shared-memory residency sweep (Work::HOT_* bit masks / budgets) at c1 and c2.
# HOT order: 0 CSR 1 CSQ 2 TOT 3 FULL 4 UTOT 5 RNK 6 GAM 7 ALPHA 8 U 9 SLOT 10 P
for cfg in "c1 1024" "c2 296"; do
  set -- $cfg
  for mk in 0x0 0x1f 0x3f 0x1 0x3 0x23 0x60 0x7f 0xff 0x7ff; do
    r=$(HCRAN_HOT_MASK=$mk timeout 300 python bench.py --config $1 --batch $2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
    echo "$1 mask=$mk $r"
  done
done
