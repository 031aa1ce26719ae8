"""C5 (N=1M, D=960, k=16) Gaussian-recompute SpMV: chunk-major kernel
(gauss_chunk_kernel, CH float4 per chunk) vs the warp-per-row kernel
(KNNX_CHUNK_CH=0), graph schedule, 256-row tiles; every variant checked
against the first (same y up to fp32 summation order) and 2048 rows against
the double oracle."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c5", n) if n != 1_000_000 else workloads.CONFIGS["c5"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
m, nn, _, _ = wl.csr_c.shape
rp, cols, _ = wl.csr_c.export()
s = api.to_device_points(wl.points_c)
x = torch.from_numpy(wl.x_c).cuda()
ys = {}
for lay in ("tiles", "flat"):
    order = api.CLUSTER if lay == "tiles" else api.ORIGINAL
    op = api.Operator.from_csr_scheduled(ctx, m, nn, rp, cols, None, order, 256)
    for ch in ("0", "2", "4", "8"):
        os.environ["KNNX_CHUNK_CH"] = ch
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
        ys[(lay, ch)] = y
        y0 = ys[("tiles", "0")]
        print(lay, "CH", ch, f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us",
              "rel vs warp", float((y - y0).abs().max() / y0.abs().max()), flush=True)
    op.close()
if n <= 1_000_000:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    rows = bench.sample_rows(n)
    for key, y in ys.items():
        print(key, "oracle rows rel", bench.gauss_rows_check(wl, cfg, y.cpu().numpy(), rows))
