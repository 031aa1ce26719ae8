#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python scripts/probe_shard_scaling.py > gpurun_out/shards.log 2>&1
KNNX_BENCH_FUNCTIONAL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --e2e-steps 5 > gpurun_out/c2_n2f.json 2> gpurun_out/c2_n2f.err
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4.json 2> gpurun_out/c4.err
