"""C5 graph: fraction of kNN entries whose pair is mutual (i in nn(j) and
j in nn(i)), i.e. how many Gaussian distances a pair-once operator would
skip when targets = sources."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c5", n) if n != 1_000_000 else workloads.CONFIGS["c5"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
ids = wl.knn_ids_c.astype(np.int64)
m, k = ids.shape
rows = np.repeat(np.arange(m), k)
cols = ids.ravel()
offdiag = cols != rows
mutual = np.zeros(cols.size, bool)
for c0 in range(0, cols.size, 1 << 22):
    sl = slice(c0, c0 + (1 << 22))
    mutual[sl] = (ids[cols[sl]] == rows[sl, None]).any(1)
mutual &= offdiag
res = {"n": m, "k": k, "entries": int(cols.size), "diagonal": int((~offdiag).sum()),
       "mutual_entries": int(mutual.sum()), "mutual_frac": float(mutual.mean()),
       "distances_saved_frac": float(mutual.mean() / 2),
       "mutual_within_256_rows_frac": float((mutual & (np.abs(cols - rows) < 256)).mean())}
print(json.dumps(res))
