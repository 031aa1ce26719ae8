"""C4 t-SNE step: persistent window kernel (options 3 = relabel + interleave,
tsne_window_kernel) vs the interleaved group kernel (options 2), and the
window hit rate of the breadth-first relabelling (fraction of entries whose
relabelled column lies in the chunk window [c0 - 8192, c0 + 16384))."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c4", n) if n != 4_000_000 else workloads.CONFIGS["c4"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
m, nn, nnz, _ = wl.csr_c.shape
rp, cols, p = wl.csr_c.export()
t0 = time.time()
sched = wl.csr_c.locality_schedule(0)
rel = np.empty(n, np.int64)
rel[sched] = np.arange(n)
lab = rel[cols]
row_lab = np.repeat(rel, np.diff(rp))
c0 = (row_lab // 8192) * 8192
hit = (lab >= c0 - 8192) & (lab < c0 + 16384)
print(f"window hit rate {hit.mean():.4f}  (|label - own| median {np.median(np.abs(lab - row_lab)):.0f}, "
      f"p90 {np.percentile(np.abs(lab - row_lab), 90):.0f}, p99 {np.percentile(np.abs(lab - row_lab), 99):.0f}) "
      f"[{time.time() - t0:.1f} s]", flush=True)
y0 = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)
yd = torch.from_numpy(y0[wl.inverse]).cuda()
res = {}
for opts in (2, 3):
    op = api.Operator.from_csr_scheduled(ctx, m, nn, rp, cols, p, api.ORIGINAL, 256, None, 0, opts)
    f = torch.empty(n, 2, device="cuda")
    yo = torch.empty(n, 2, device="cuda")
    for _ in range(3):
        op.tsne(yd, 2, f, False, 1.0, yo)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.tsne(yd, 2, f, False, 1.0, yo)
    e1.record()
    torch.cuda.synchronize()
    res[opts] = f.clone()
    print("options", opts, f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
    op.close()
print("rel diff", float((res[2] - res[3]).abs().max() / res[2].abs().max()))
