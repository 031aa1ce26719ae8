set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30
timeout 600 python bench.py --n 200000 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/b_small.json 2> gpurun_out/b_small.log; echo rc=$?
tail -5 gpurun_out/b_small.log; cat gpurun_out/b_small.json
timeout 900 python bench.py --steps 1000 --warmup 20 > gpurun_out/b_full.json 2> gpurun_out/b_full.log; echo rc=$?
tail -5 gpurun_out/b_full.log; cat gpurun_out/b_full.json
