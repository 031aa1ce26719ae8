#!/bin/bash
# Round-2 validation: full-size parity tests, the C3-C5 lines with their
# teacher-forced checks, and the N=2 code path run functionally on one GPU.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/scale_test.log 2>&1; echo "rc=$?" >> gpurun_out/scale_test.log
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "rc=$?" >> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
KNNX_BENCH_FUNCTIONAL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --e2e-steps 5 > gpurun_out/bench_c2_n2f.json 2> gpurun_out/bench_c2_n2f.err; echo "rc=$?" >> gpurun_out/bench_c2_n2f.err
timeout 1200 python bench.py --config c4 --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "rc=$?" >> gpurun_out/bench_c4.err
