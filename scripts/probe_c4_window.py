"""C4 y-window hit rate (diagnostic for KNNX_OPT_Y_WINDOW): for scheduled,
relabelled row tiles, the fraction of entries whose relabelled column falls in
the tile's window (median-centred, host rule of runtime.cu)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c4", n) if n != 4_000_000 else workloads.CONFIGS["c4"]
wl = workloads.build(cfg, ctx, 0, log=print)
rp, cols, _ = wl.csr_c.export()
sched = wl.csr_c.locality_schedule()
rel = np.empty(n, np.int64)
rel[sched] = np.arange(n)
for R in (64, 128):
    for W in (8192, 16384, 65536):
        hit = tot = 0
        for t0 in range(0, n - R, R * 50):
            rows = sched[t0:t0 + R]
            c = np.concatenate([rel[cols[rp[r]:rp[r + 1]]] for r in rows])
            lo = max(0, min(int(np.median(c)) - W // 2, n - W)) & ~3
            hit += np.sum((c >= lo) & (c < lo + W))
            tot += c.size
        print("tile", R, "window", W, "hit", hit / tot, flush=True)
