for sh in 256:256 512:512 512:256 512:128; do
  echo "== c1 $sh"; HCRAN_SHAPE=$sh timeout 300 python bench.py --config c1 --no-cpu-baseline --no-e2e --steps 3 2>&1 | cut -c1-200
done
for sh in 512:512 512:256 512:128; do
  echo "== c2 $sh"; HCRAN_SHAPE=$sh timeout 600 python bench.py --config c2 --batch 2960 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | cut -c1-200
done
