"""Runs the C5 Gaussian-recompute SpMV once scheduled and once in plain tree
order (for ncu captures of the wide kernels)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tile_rows = int(os.environ.get("C5_TILE_ROWS", "256"))
cfg = workloads.scaled("c5", n) if n != 1_000_000 else workloads.CONFIGS["c5"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
m, nn, _, _ = wl.csr_c.shape
rp, cols, _ = wl.csr_c.export()
s = api.to_device_points(wl.points_c)
x = torch.from_numpy(wl.x_c).cuda()
ys = []
for sched, tile_rows in ((True, 32), (True, 256), (False, 32)):
    op = (api.Operator.from_csr_scheduled(ctx, m, nn, rp, cols, None, api.CLUSTER, tile_rows) if sched
          else api.Operator.from_csr(ctx, m, nn, rp, cols, None, api.CLUSTER, tile_rows))
    y = torch.empty(n, device="cuda")
    for _ in range(3):
        op.gauss_spmv(s, s, cfg.dim, wl.h_ref, x, y)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.gauss_spmv(s, s, cfg.dim, wl.h_ref, x, y)
    e1.record()
    torch.cuda.synchronize()
    print("sched" if sched else "plain", tile_rows, f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us",
          "max_halo", op.info["max_halo"], "halo_total", op.info["halo_total"], flush=True)
    ys.append(y)
    op.close()
for y in ys[1:]:
    print("rel vs first", float((y - ys[0]).abs().max() / ys[0].abs().max()))
