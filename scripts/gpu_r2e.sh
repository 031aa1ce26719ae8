#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "rc=$?" >> gpurun_out/c5.err
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err; echo "rc=$?" >> gpurun_out/c3.err
