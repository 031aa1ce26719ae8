#!/bin/bash
# Round-2 closing validation on a B200 box: sanitize script, smoke, the bench
# lines of every config, the reference arm, a launch list of the C2 bench and
# one full capture of the main kNN screen launch.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python tests/sanitize_small.py > gpurun_out/sanitize_small.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_small.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "rc=$?" >> gpurun_out/bench_c2.err
timeout 1500 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "rc=$?" >> gpurun_out/c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen_kernel -s 2 -c 1 -o gpurun_out/r2_knn_wide_screen_main python scripts/probe_knn_wide.py 1000000 --no-tool > gpurun_out/ncu_knnw_main.log 2>&1
