mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
timeout 900 python scripts/bench_kernels.py --only c2,c3 > gpurun_out/bk.json 2> gpurun_out/bk.log; echo "exit $?"; grep -E "^c[23]|^perm" gpurun_out/bk.log | cut -c1-100
