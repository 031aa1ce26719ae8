"""Full-size agreement of the two kNN builders on C2's points (1M x 49, k = 30):
the provably exact SIMT search (knnx_knn_dev) and the tensor-core screen +
exact re-rank (knnx_knn_wide_dev).  Rows that differ are classified: a
near-tie (same distance multiset to fp32 rounding) or a real miss."""
import time

import numpy as np
import torch

from paper_1709_03671_b200 import api, workloads

cfg = workloads.CONFIGS["c2"]
ctx = api.Context(0)
pts = api.gen_points(cfg.kind, cfg.n, cfg.dim, cfg.n_clusters, cfg.p0, workloads.SEED_POINTS)
tree = api.order_tree(pts.astype(np.float64), 3, pca_device=0)
pc = np.empty_like(pts)
pc[tree.forward] = pts
dp = api.to_device_points(pc)
n, dim, k = cfg.n, cfg.dim, cfg.k
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ids_s, d2_s = ctx.knn(dp, dp, n, n, dim, k, True)
    ctx.sync(); t_s = time.perf_counter() - t0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ids_w, d2_w, st = ctx.knn_wide(dp, dp, n, n, dim, k, True, want_stats=True)
    ctx.sync(); t_w = time.perf_counter() - t0
same_rows = (ids_s == ids_w).all(1)
print(f"n={n} dim={dim} k={k}: SIMT exact {t_s:.3f} s, tensor-core {t_w:.3f} s, {st}")
print(f"rows with identical id lists: {same_rows.float().mean().item():.6f} ({int((~same_rows).sum())} differ)")
bad = torch.nonzero(~same_rows).flatten()
if bad.numel():
    a, b = torch.sort(d2_s[bad], 1).values, torch.sort(d2_w[bad], 1).values
    rel = ((a - b).abs() / a.clamp_min(1e-30)).max(1).values
    sets_equal = (torch.sort(ids_s[bad], 1).values == torch.sort(ids_w[bad], 1).values).all(1)
    print(f"  of those: same id set in another order {int(sets_equal.sum())}, "
          f"distance lists equal to 1e-6 rel {int((rel <= 1e-6).sum())}, worst rel {rel.max().item():.2e}")
print(f"distances bitwise equal on identical rows: {(d2_s[same_rows] == d2_w[same_rows]).float().mean().item():.6f}, "
      f"max rel diff {((d2_s - d2_w).abs() / d2_s.clamp_min(1e-30))[same_rows].max().item():.2e}")
# the exact search itself against an fp64 brute force on sampled rows
rows = torch.from_numpy(np.random.default_rng(1).choice(n, 256, replace=False)).cuda()
p = dp[:, :dim].double()
agree = 0.0
worst = 0.0
for r0 in range(0, 256, 64):
    rr = rows[r0:r0 + 64]
    q = p[rr]
    dd = (q * q).sum(1)[:, None] + (p * p).sum(1)[None, :] - 2.0 * q @ p.t()
    dd[torch.arange(len(rr)), rr] = float("inf")
    cand = torch.topk(dd, k + 16, dim=1, largest=False).indices
    ex = ((p[cand] - q[:, None, :]) ** 2).sum(-1)
    o = torch.argsort(ex, dim=1, stable=True)[:, :k]
    bi, bd = torch.gather(cand, 1, o), torch.gather(ex, 1, o)
    agree += (ids_s[rr].long() == bi).float().mean().item() / 4
    worst = max(worst, ((d2_s[rr].double() - bd).abs() / bd).max().item())
print(f"knnx_knn_dev vs fp64 brute force on 256 sampled rows: ids equal {agree:.5f}, d2 rel {worst:.2e}")
