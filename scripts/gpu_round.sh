# Full round validation on one B200: GPU tests, smoke, bench lines for C2-C5,
# C2 launch list under ncu.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t.txt 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/t.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.log; echo "c2 exit $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.log; echo "ref exit $?"
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.log; echo "c3 exit $?"
timeout 1500 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.log; echo "c4 exit $?"
timeout 1500 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.log; echo "c5 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
for c in c2 c3 c4 c5; do python -c "
import json
d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value') if isinstance(d.get('e2e'),dict) else None, d.get('clocks'))
"; done
