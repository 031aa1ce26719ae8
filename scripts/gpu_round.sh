mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.log; echo "c2 exit $?"
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.log; echo "c3 exit $?"
timeout 1500 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.log; echo "c4 exit $?"
timeout 1500 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.log; echo "c5 exit $?"
for c in c2 c3 c4 c5; do python -c "
import json,sys
d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value') if isinstance(d.get('e2e'),dict) else None)
"; done
