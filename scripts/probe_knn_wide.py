"""knnx_knn_wide_dev (tcgen05 screen + exact re-rank) against a torch fp32/fp64
brute force on sampled rows, and its run time against the cuBLAS + topk tool
(workloads.knn_wide) at growing sizes.  Usage: probe_knn_wide.py [n ...]"""
import sys
import time

import numpy as np
import torch

from paper_1709_03671_b200 import api, workloads


def torch_tool(pts, dim, k, self_set=True, n_cand=64, chunk=4096):
    """The library path this kernel replaced (round 1): cuBLAS TF32 Gram +
    torch.topk screen, fp32 re-rank."""
    n = pts.shape[0]
    p = pts[:, :dim].float()
    pc = p - p.mean(0, keepdim=True)
    norms = (pc * pc).sum(1)
    ids = torch.empty(n, k, dtype=torch.int32, device=p.device)
    d2o = torch.empty(n, k, dtype=torch.float32, device=p.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        for q0 in range(0, n, chunk):
            q1 = min(n, q0 + chunk)
            g = torch.mm(pc[q0:q1], pc.t())
            g.mul_(-2.0).add_(norms[None, :]).add_(norms[q0:q1, None])
            if self_set:
                r = torch.arange(q0, q1, device=p.device)
                g[r - q0, r] = float("inf")
            cand = torch.topk(g, min(n_cand, n), dim=1, largest=False, sorted=False).indices
            del g
            cand, _ = torch.sort(cand, dim=1)
            diff = p[cand] - p[q0:q1, None, :]
            d2 = (diff * diff).sum(-1)
            if self_set:
                d2 = torch.where(cand == torch.arange(q0, q1, device=p.device)[:, None],
                                 torch.full_like(d2, float("inf")), d2)
            d2s, order = torch.sort(d2, dim=1, stable=True)
            ids[q0:q1] = torch.gather(cand, 1, order[:, :k]).int()
            d2o[q0:q1] = d2s[:, :k]
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return ids, d2o


def brute_rows(pts, rows, k, self_set):
    p = pts.double()
    q = p[rows]
    d2 = (q * q).sum(1)[:, None] + (p * p).sum(1)[None, :] - 2.0 * q @ p.t()
    if self_set:
        d2[torch.arange(len(rows)), rows] = float("inf")
    cand = torch.topk(d2, k + 8, dim=1, largest=False).indices
    diff = p[cand] - q[:, None, :]
    ex = (diff * diff).sum(-1)
    o = torch.argsort(ex, dim=1, stable=True)[:, :k]
    return torch.gather(cand, 1, o), torch.gather(ex, 1, o)


def main():
    no_tool = "--no-tool" in sys.argv
    sizes = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [1500, 20000, 200000]
    ctx = api.Context(0)
    for n in sizes:
        for dim, k in ((960, 16), (200, 10)):
            if dim != 960 and n > 20000:
                continue
            pts = api.gen_points(api.GEN_ANISO, n, dim, (32 << 16) | 32, 1.0, 17)
            tree = api.order_tree(pts.astype(np.float64), 3, pca_device=0)
            pc = np.empty_like(pts)
            pc[tree.forward] = pts
            dp = api.to_device_points(pc)
            torch.cuda.synchronize()
            for rep in range(2):
                t0 = time.perf_counter()
                ids, d2, st = ctx.knn_wide(dp, dp, n, n, dim, k, True, want_stats=True)
                ctx.sync()
                torch.cuda.synchronize()
                t_new = time.perf_counter() - t0
            t0 = time.perf_counter()
            ids_o, d2_o = (ids, d2) if no_tool else torch_tool(dp, dim, k, True)
            torch.cuda.synchronize()
            t_old = time.perf_counter() - t0
            rows = torch.from_numpy(np.random.default_rng(1).choice(n, min(n, 512), replace=False)).cuda()
            bi, bd = brute_rows(dp[:, :dim], rows, k, True)
            same = (ids[rows].long() == bi).float().mean().item()
            same_o = (ids_o[rows].long() == bi).float().mean().item()
            rel = ((d2[rows].double() - bd).abs() / bd).max().item()
            full = (ids == ids_o).float().mean().item()
            print(f"n={n} dim={dim} k={k}: wide {t_new*1e3:.1f} ms, torch tool {t_old*1e3:.1f} ms, "
                  f"ids==brute {same:.5f} (tool {same_o:.5f}), d2 rel {rel:.2e}, ids==tool {full:.5f}, {st}",
                  flush=True)


if __name__ == "__main__":
    main()
