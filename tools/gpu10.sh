python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
rm -f gpurun_out/variants.txt
python tools/variant_time.py c1 1024 4096 >> gpurun_out/variants.txt 2>&1
python tools/variant_time.py c2 592 2960 >> gpurun_out/variants.txt 2>&1
timeout 600 python tools/c3_probe.py 148 fast > gpurun_out/c3.txt 2>&1
