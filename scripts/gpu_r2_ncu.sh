#!/bin/bash
# Round-2 full ncu captures of the default non-stationary kernels at the
# BASELINE sizes (C3 mean shift, C5 wide Gaussian recompute, C4 t-SNE); each
# profiled command is first run plain (the box refuses ncu otherwise).
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 280 python scripts/c3_kernel.py > gpurun_out/c3_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:meanshift_lane --launch-skip 49 --launch-count 1 -o gpurun_out/r2_c3_meanshift -f python scripts/c3_kernel.py > gpurun_out/ncu_c3.log 2>&1; echo "ncu3 rc=$?"
timeout 280 python scripts/c5_kernel.py > gpurun_out/c5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gauss_warp --launch-skip 16 --launch-count 1 -o gpurun_out/r2_c5_gauss_warp -f python scripts/c5_kernel.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu5 rc=$?"
timeout 280 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tsne_group --launch-skip 4 --launch-count 1 -o gpurun_out/r2_c4_tsne_group -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu4 rc=$?"
