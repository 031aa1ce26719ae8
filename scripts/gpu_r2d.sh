#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 300 python scripts/probe_knn_wide.py 1000000 --no-tool > gpurun_out/knnw_plain.log 2>&1 || exit 1
# launch list of the whole call, then one full capture of the last (main) screen launch
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_knn_wide_launches.csv python scripts/probe_knn_wide.py 1000000 --no-tool > gpurun_out/ncu_knnw_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen_kernel -s 5 -c 1 -o gpurun_out/r2_knn_wide_screen_part python scripts/probe_knn_wide.py 1000000 --no-tool > gpurun_out/ncu_knnw_s.log 2>&1
timeout 300 python scripts/probe_knn_c4.py 1000000 > gpurun_out/knn_c4_1m.log 2>&1
