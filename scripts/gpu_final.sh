#!/bin/bash
# Round-2 record run: headline + reference arm + C3-C5 lines, the N = 2 code
# paths run functionally on one GPU, the shard-scaling forecast and one ncu
# capture of the headline kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
timeout 600 python scripts/probe_shard_scaling.py > gpurun_out/f_shards.log 2>&1
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err
timeout 1500 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err
KNNX_BENCH_FUNCTIONAL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --e2e-steps 5 > gpurun_out/f_c2_n2f.json 2> gpurun_out/f_c2_n2f.err
KNNX_BENCH_FUNCTIONAL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config c3 --steps 10 --warmup 3 > gpurun_out/f_c3_n2f.json 2> gpurun_out/f_c3_n2f.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/f_small.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tiles_g -s 3 -c 1 -o gpurun_out/r2_c2_spmv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/f_ncu.log 2>&1
