#!/bin/bash
# Round measurement pass on one B200 (run under gpurun): the driver's default
# bench command with its wall time, the reference arm, and the other configs.
TAG=${1:-r02}
mkdir -p gpurun_out
t0=$(date +%s)
timeout 1750 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
echo "c2 default wall $(( $(date +%s) - t0 )) s" > gpurun_out/bench_${TAG}_walls.txt
t0=$(date +%s)
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_reference_c2.json 2> gpurun_out/bench_${TAG}_reference_c2.err
echo "reference c2 wall $(( $(date +%s) - t0 )) s" >> gpurun_out/bench_${TAG}_walls.txt
for c in c1 c0 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err
timeout 600 python bench.py --impl reference --config c1 --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference_c1.json 2> gpurun_out/bench_${TAG}_reference_c1.err
cat gpurun_out/bench_${TAG}_walls.txt
for f in gpurun_out/bench_${TAG}_*.json; do echo $f; cut -c1-300 $f; done
