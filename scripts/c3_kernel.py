"""C3 mean-shift step once (for ncu captures): N=1M, D=49, k=30 incl. self."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c3", n) if n != 1_000_000 else workloads.CONFIGS["c3"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
m, nn, _, _ = wl.csr_c.shape
rp, cols, _ = wl.csr_c.export()
s = api.to_device_points(wl.points_c)
out = torch.empty_like(s)
for sched, lay in ((False, api.CLUSTER), (True, api.CLUSTER), (True, api.ORIGINAL)):
  tr = int(os.environ.get("C3_TILE_ROWS", "256"))
  op = (api.Operator.from_csr_scheduled(ctx, m, nn, rp, cols, None, lay, tr) if sched
        else api.Operator.from_csr(ctx, m, nn, rp, cols, None, lay, tr))
  for _ in range(3):
    op.meanshift(s, s, cfg.dim, wl.h_ref, out)
  torch.cuda.synchronize()
  e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
  e0.record()
  for _ in range(20):
    op.meanshift(s, s, cfg.dim, wl.h_ref, out)
  e1.record()
  torch.cuda.synchronize()
  print("sched" if sched else "plain", "flat" if lay == api.ORIGINAL else "tiles", f"meanshift {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", op.info["halo_total"])
