mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "tsne" > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
timeout 600 python scripts/c4_kernel.py > gpurun_out/c4k.txt 2>&1; echo "exit $?"; tail -4 gpurun_out/c4k.txt
