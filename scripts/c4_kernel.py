"""C4-shaped t-SNE attraction once per layout (for ncu): N (default 1M), D=50, k=90 symmetrised."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c4", n) if n != 4_000_000 else workloads.CONFIGS["c4"]
wl = workloads.build(cfg, ctx, 0, log=print)
y0 = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)
y = torch.from_numpy(y0[wl.inverse]).cuda()
f = torch.empty(n, 2, device="cuda")
yo = torch.empty(n, 2, device="cuda")
m_, n_, _, _ = wl.csr_c.shape
rp, cols, vals = wl.csr_c.export()
ref = None
for layout, tr, sched, opts in ((api.ORIGINAL, 256, True, 0), (api.ORIGINAL, 256, True, 1),
                                (api.ORIGINAL, 256, True, 2), (api.ORIGINAL, 256, True, 3),
                                (api.CLUSTER, 256, True, 1), (api.CLUSTER, 32, True, 0)):
    op = (api.Operator.from_csr_scheduled(ctx, m_, n_, rp, cols, vals, layout, tr, None, 0, opts)
          if sched else api.Operator.from_host_csr(ctx, wl.csr_c, layout, tr))
    for _ in range(3):
        op.tsne(y, 2, f, False, 1.0, yo)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.tsne(y, 2, f, False, 1.0, yo)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = f.clone()
    rel = float((f - ref).abs().max() / ref.abs().max())
    print("layout", layout, tr, "sched" if sched else "", "opts", opts, "rel_vs_first", rel,
          f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us", op.info["nnz"],
          "max_halo", op.info["max_halo"], "halo_total", op.info["halo_total"])
    op.close()
