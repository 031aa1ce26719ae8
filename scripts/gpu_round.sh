timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --steps 1000 --warmup 20 > gpurun_out/b_full.json 2> gpurun_out/b_full.log; echo rc=$?
python -c "
import json;d=json.load(open('gpurun_out/b_full.json'))
print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['frac_format'], d['e2e']['value'], d['cpu_baseline']['value'])
for k,v in d['extra'].items(): print(k, v.get('launch_us'))
print(d['checks'])"
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tiles_g -s 3 -c 1 -o gpurun_out/prof_spmv_g $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
