"""C5 (N=1M, D=960, k=16): how many distinct source rows do R consecutive
scheduled rows reference?  (Source-row reuse available to a kernel that
processes R rows per warp.)  Also times the workload build with the tcgen05
kNN.  Usage: probe_c5_reuse.py [n]"""
import sys
import time

import numpy as np
import torch

from paper_1709_03671_b200 import api, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = api.Context(0)
cfg = workloads.scaled("c5", n) if n != 1_000_000 else workloads.CONFIGS["c5"]
t0 = time.perf_counter()
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
print("build", time.perf_counter() - t0, wl.timings, flush=True)
rp, cols, _ = wl.csr_c.export()
k = cfg.k
ids = cols.reshape(n, k).astype(np.int64)
sched = wl.csr_c.locality_schedule()
for name, order in (("tree order", np.arange(n)), ("graph schedule", sched.astype(np.int64))):
    rows = ids[order]
    for R in (2, 4, 8, 16, 32, 64):
        g = n // R
        blk = rows[: g * R].reshape(g, R * k)
        blk = np.sort(blk, axis=1)
        distinct = 1 + (np.diff(blk, axis=1) != 0).sum(1)
        # sources that are also target rows of the same group (self rows are loaded anyway)
        print(f"{name}: R={R}: distinct sources per group {distinct.mean():.1f} of {R * k} "
              f"(reuse {R * k / distinct.mean():.2f}x)", flush=True)
# mutual-pair greedy matching: pair each row with its nearest not-yet-paired neighbour
paired = np.full(n, -1, np.int64)
for i in range(n):
    if paired[i] >= 0:
        continue
    for j in ids[i]:
        if paired[j] < 0 and j != i:
            paired[i] = j
            paired[j] = i
            break
pairs = np.flatnonzero((paired >= 0) & (paired > np.arange(n)))
a, b = pairs, paired[pairs]
blk = np.sort(np.concatenate([ids[a], ids[b]], axis=1), axis=1)
distinct = 1 + (np.diff(blk, axis=1) != 0).sum(1)
print(f"greedy neighbour pairs: {2 * len(pairs) / n:.3f} of rows paired, distinct {distinct.mean():.1f} of {2 * k} "
      f"(reuse {2 * k / distinct.mean():.2f}x)")
# Dense-block form of the operator: which (128-row target tile, 256-row source
# tile) pairs contain at least one graph entry?  Each such pair costs one
# 128 x 256 x 960 tile product (9.5 us at the measured 979 TFLOP/s TF32 rate,
# three of them in 3xTF32).
for name, order in (("tree order", np.arange(n)), ("graph schedule", sched.astype(np.int64))):
    pos = np.empty(n, np.int64)
    pos[order] = np.arange(n)
    tq = np.repeat(pos // 128, k)
    ts = pos[ids.reshape(-1)] // 256
    pairs = np.unique(tq * ((n + 255) // 256) + ts).size
    t_tf32 = pairs * 9.5e-6 / 148
    print(f"{name}: {pairs} tile pairs hold the {n * k} entries ({n * k / pairs:.1f} entries per 128 x 256 block, "
          f"density {n * k / pairs / (128 * 256):.2e}); at 9.5 us per tile product on 148 SMs: "
          f"{t_tf32 * 1e3:.1f} ms in TF32, {3 * t_tf32 * 1e3:.1f} ms in 3xTF32")
