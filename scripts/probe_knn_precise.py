"""The 3xTF32 second pass at scale: C2's 3-level mixture (leaf clusters tight
against their distance from the mean) generated in 96 dimensions, N = 1M,
k = 16 -- no SIMT fallback applies, so every row the TF32 screen cannot certify
is screened again with 3xTF32 operands.  Sampled rows against an fp64 brute force."""
import time

import numpy as np
import torch

from paper_1709_03671_b200 import api

n, dim, k = 1_000_000, 96, 16
ctx = api.Context(0)
pts = api.gen_points(api.GEN_3LEVEL, n, dim, 0, 0.125, 7)
dp = api.to_device_points(pts)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ids, d2, st = ctx.knn_wide(dp, dp, n, n, dim, k, True, want_stats=True)
    ctx.sync(); dt = time.perf_counter() - t0
print(f"n={n} dim={dim} k={k} (unordered input): {dt:.3f} s {st}")
rows = torch.from_numpy(np.random.default_rng(1).choice(n, 256, replace=False)).cuda()
p = dp[:, :dim].double()
same, worst = 0.0, 0.0
for r0 in range(0, 256, 32):
    rr = rows[r0:r0 + 32]
    q = p[rr]
    dd = (q * q).sum(1)[:, None] + (p * p).sum(1)[None, :] - 2.0 * q @ p.t()
    dd[torch.arange(len(rr)), rr] = float("inf")
    cand = torch.topk(dd, k + 16, dim=1, largest=False).indices
    ex = ((p[cand] - q[:, None, :]) ** 2).sum(-1)
    o = torch.argsort(ex, dim=1, stable=True)[:, :k]
    bi, bd = torch.gather(cand, 1, o), torch.gather(ex, 1, o)
    same += (ids[rr].long() == bi).float().mean().item() / 8
    worst = max(worst, ((d2[rr].double() - bd).abs() / bd).max().item())
print(f"sampled rows: ids == fp64 brute force {same:.5f}, d2 rel {worst:.2e}")
