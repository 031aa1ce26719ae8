set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.log; echo rc=$?; tail -2 gpurun_out/b_c3.log; cat gpurun_out/b_c3.json | cut -c1-1500
timeout 1500 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.log; echo rc=$?; tail -2 gpurun_out/b_c4.log; cat gpurun_out/b_c4.json | cut -c1-1500
