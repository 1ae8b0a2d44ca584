#!/bin/bash
# Shared-memory residency budget (HCRAN_HOT_KB) at c2 / c1 on the current build.
mkdir -p gpurun_out
for kb in ${KBS:-16 56 100}; do
  HCRAN_HOT_KB=$kb python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/hot${kb}_c2.json 2>&1
  HCRAN_HOT_KB=$kb python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/hot${kb}_c1.json 2>&1
done
