mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "tsne or shim or golden" > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
run() { timeout 900 env "$@" python bench.py --config c4 --n 1000000 --steps 20 --warmup 3 2> /dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],3), 'ms')"; }
run KNNX_TSNE_VARIANT=0
run KNNX_TSNE_VARIANT=0 KNNX_LAYOUT=flat
run KNNX_TSNE_VARIANT=1
run KNNX_TSNE_VARIANT=1 KNNX_LAYOUT=flat
