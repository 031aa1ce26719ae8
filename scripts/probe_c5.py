"""C5 tile statistics: halo size per tile for several tile heights."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c5", n) if n != 1_000_000 else workloads.CONFIGS["c5"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
ids = wl.knn_ids_c
m_, n_, _, _ = wl.csr_c.shape
rp, cols, _ = wl.csr_c.export()
sched = wl.csr_c.locality_schedule()
pos = np.empty(n, np.int64)
pos[sched] = np.arange(n)
for tr in (64, 128, 256, 512, 1024):
    op = api.Operator.from_csr_scheduled(ctx, m_, n_, rp, cols, None, api.CLUSTER, tr)
    inf = op.info
    intile = np.mean((pos[ids] // tr) == (pos[:, None] // tr))
    print("sched", tr, {k: inf[k] for k in ("n_tiles", "halo_total", "max_halo")},
          "avg_halo", inf["halo_total"] / inf["n_tiles"], "in_tile_frac", round(float(intile), 3))
    op.close()
for tr in (64, 128, 256, 512, 1024):
    op = api.Operator.from_host_csr(ctx, wl.csr_c, api.CLUSTER, tr)
    inf = op.info
    rows = np.arange(n)
    intile = np.mean((ids // tr) == (rows[:, None] // tr))
    print(tr, {k: inf[k] for k in ("n_tiles", "halo_total", "max_halo")},
          "avg_halo", inf["halo_total"] / inf["n_tiles"], "in_tile_frac", round(float(intile), 3))
    op.close()
