#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONPATH=.
mkdir -p gpurun_out
make -s -C tests/cpp > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_shim.py -x -q > gpurun_out/shim.log 2>&1; echo "rc=$?" >> gpurun_out/shim.log
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "rc=$?" >> gpurun_out/c5.err
timeout 1800 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "rc=$?" >> gpurun_out/c4.err
