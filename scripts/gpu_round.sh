set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
KNNX_NONSTAT_VARIANT=3 timeout 900 python -m pytest tests -x -q -m gpu -k "gauss or meanshift or variable" 2>&1 | tail -2
for V in 0 3 1; do KNNX_NONSTAT_VARIANT=$V timeout 900 python scripts/bench_kernels.py --only c2,c3 > gpurun_out/kernels_v$V.json 2> gpurun_out/kernels_v$V.log; echo V=$V rc=$?; grep -E "gauss_spmv|meanshift" gpurun_out/kernels_v$V.log | cut -c1-110; done
