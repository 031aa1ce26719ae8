#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 1200 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4w.json 2> gpurun_out/bench_c4w.err; echo "rc=$?" >> gpurun_out/bench_c4w.err
