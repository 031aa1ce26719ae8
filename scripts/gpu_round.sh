timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python scripts/bench_kernels.py --only c2,c3 2>&1 | grep -E "gauss|meanshift|update|tsne" | cut -c1-110
