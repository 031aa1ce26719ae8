#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONPATH=.
mkdir -p gpurun_out

timeout 900 python scripts/probe_c5_reuse.py > gpurun_out/c5_reuse.log 2>&1; echo "rc=$?" >> gpurun_out/c5_reuse.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:screen_kernel -c 1 -o gpurun_out/r2_knn_wide_screen python scripts/probe_knn_wide.py 200000 > gpurun_out/ncu_knn.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_knn.log
