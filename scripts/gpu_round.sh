set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python scripts/bench_kernels.py > gpurun_out/kernels.json 2> gpurun_out/kernels.log; echo rc=$?
grep -v "^\[" gpurun_out/kernels.log | cut -c1-400
