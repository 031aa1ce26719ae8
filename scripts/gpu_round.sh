set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 1000 --warmup 20 > gpurun_out/b_full.json 2> gpurun_out/b_full.log; echo rc=$?
tail -3 gpurun_out/b_full.log; python -c "import json;d=json.load(open('gpurun_out/b_full.json'));print(json.dumps({k:d[k] for k in ['value','ms_per_step','e2e','roofline','cpu_baseline','extra','checks','setup_s']},indent=1))"
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tiles_g -s 3 -c 1 -o gpurun_out/prof_spmv_g $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_orig -s 3 -c 1 -o gpurun_out/prof_spmv_orig $CMD > gpurun_out/ncu_full2.log 2>&1; echo ncu3=$?
