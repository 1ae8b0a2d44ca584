#!/bin/bash
# Round measurement pass on one B200 (run under gpurun): GPU parity suite and
# smoke, the driver's default bench command (c2 / 16,384, --steps 20 --warmup 5)
# with its wall time, the reference arm, ncu evidence (launch list + one
# --set full capture), phase profiles, and the other configs.
TAG=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
t0=$(date +%s)
timeout 1750 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
echo "c2 default (--steps 20 --warmup 5) wall $(( $(date +%s) - t0 )) s" > gpurun_out/bench_${TAG}_walls.txt
t0=$(date +%s)
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_reference_c2.json 2> gpurun_out/bench_${TAG}_reference_c2.err
echo "reference c2 wall $(( $(date +%s) - t0 )) s" >> gpurun_out/bench_${TAG}_walls.txt
bash tools/gpu_profile.sh ${TAG} 148 c2
python tools/phase_profile.py c2 296 > gpurun_out/phase_${TAG}_c2.txt 2>&1
python tools/phase_profile.py c1 1024 > gpurun_out/phase_${TAG}_c1.txt 2>&1
for c in c1 c0 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err
timeout 600 python bench.py --impl reference --config c1 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference_c1.json 2> gpurun_out/bench_${TAG}_reference_c1.err
cat gpurun_out/bench_${TAG}_walls.txt
for f in gpurun_out/bench_${TAG}_*.json; do echo $f; cut -c1-300 $f; done
