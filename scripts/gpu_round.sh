mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_highdim.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --config c5 --n 200000 --steps 20 --warmup 3 > gpurun_out/c5s.json 2> gpurun_out/c5s.log; echo "exit $?"; tail -3 gpurun_out/c5s.log; cat gpurun_out/c5s.json
timeout 1500 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.log; echo "exit $?"; tail -3 gpurun_out/c5.log; cat gpurun_out/c5.json
