mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_highdim.py tests/test_gpu_build.py -x -q -m gpu > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
timeout 600 python scripts/c5_kernel.py > gpurun_out/c5k.txt 2>&1; echo "exit $?"; tail -3 gpurun_out/c5k.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gauss -s 3 -c 1 -o gpurun_out/c5_gauss_packed -f python scripts/c5_kernel.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu exit $?"
