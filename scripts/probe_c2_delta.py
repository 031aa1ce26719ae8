"""C2 index-compression feasibility: encode every row's
halo-local column indices (256-row tiles, cluster order) as 8-bit deltas
from the previous entry of the row (first entry from 0), a delta >= 256
costing one zero-valued stepping entry per 255.  Reports the stored bytes
per launch against today's 16-bit indices."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c2", n) if n != 1_000_000 else workloads.CONFIGS["c2"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
rp, cols, _ = wl.csr_c.export()
rp = rp.astype(np.int64)
m = rp.size - 1
R = 256
rows = np.repeat(np.arange(m), np.diff(rp))
tile = rows // R
lidx = np.empty(cols.size, np.int64)
halo_total = 0
for t0 in range(0, m, R):
    a, b = rp[t0], rp[min(t0 + R, m)]
    h = np.unique(cols[a:b])
    halo_total += h.size
    lidx[a:b] = np.searchsorted(h, cols[a:b])
steps = 0
hist = np.zeros(4, np.int64)
first = np.zeros(cols.size, bool)
first[rp[:-1][np.diff(rp) > 0]] = True
srt = lidx.copy()
for i in range(m):  # rows sorted by local index (sum order changes only by +0 terms)
    srt[rp[i]:rp[i + 1]] = np.sort(lidx[rp[i]:rp[i + 1]])
prev = np.where(first, 0, np.concatenate(([0], srt[:-1])))
delta = srt - prev
extra = np.maximum(0, (delta - 1) // 255)
nnz = cols.size
stored = nnz + int(extra.sum())
res = {"n": m, "nnz": int(nnz), "halo_total": int(halo_total),
       "delta_p50": float(np.median(delta)), "delta_p99": float(np.percentile(delta, 99)),
       "frac_delta_ge_256": float((delta >= 256).mean()), "stepping_entries": int(extra.sum()),
       "bytes_u16": int(6 * nnz), "bytes_u8_delta": int(5 * stored),
       "saving_frac_of_entries": 1 - 5 * stored / (6 * nnz)}
print(json.dumps(res))
