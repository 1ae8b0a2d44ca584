#!/bin/bash
# Phase profiles and short bench lines of the analysis variants (HCRAN_FAST=0/1/2) at c1 and c2.
mkdir -p gpurun_out
TAG=${1:-ab}
for m in ${VARIANTS:-2 0}; do
  HCRAN_FAST=$m python tools/phase_profile.py c1 1024 > gpurun_out/phase_${TAG}_fast${m}_c1.txt 2>&1
  HCRAN_FAST=$m python tools/phase_profile.py c2 296 > gpurun_out/phase_${TAG}_fast${m}_c2.txt 2>&1
  HCRAN_FAST=$m python bench.py --config c1 --batch 1024 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_fast${m}_c1.json 2>&1
  HCRAN_FAST=$m python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_fast${m}_c2.json 2>&1
done
