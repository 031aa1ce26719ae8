"""C3 tile halo statistics (distinct sources per row tile) for the staged kernel design."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
cfg = workloads.CONFIGS["c3"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
ids = wl.knn_ids_c
n, k = ids.shape
for tr in (32, 64, 128, 256):
    t = ids.reshape(-1, tr * k) if n % tr == 0 else ids[: n // tr * tr].reshape(-1, tr * k)
    s = np.sort(t, axis=1)
    h = 1 + (np.diff(s, axis=1) != 0).sum(1)
    print(tr, "tiles", h.size, "mean", h.mean().round(1), "p50", np.percentile(h, 50),
          "p90", np.percentile(h, 90), "p99", np.percentile(h, 99), "max", h.max(),
          "KB@208B p99", round(np.percentile(h, 99) * 208 / 1024, 1))
