set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for L in flat tiles; do KNNX_LAYOUT=$L timeout 900 python bench.py --config c4 --n 1000000 --steps 20 --warmup 3 > gpurun_out/b_c4_$L.json 2> gpurun_out/b_c4_$L.log; echo L=$L rc=$?; python -c "import json;d=json.load(open('gpurun_out/b_c4_$L.json'));print(d['ms_per_step'], d['value'], d['config']['nnz'])"; done
