"""C4 t-SNE kernel at the full BASELINE size for an ncu capture.

The C4 workload build (PCA, k = 90 kNN, symmetrisation: ~250 s) does not fit
the GPU box's 300-s plain run that gates ncu, so: `save` builds it once and
writes the cluster-ordered P and the starting embedding to /tmp/c4cache;
`run` (the profiled command, on the same box within its 5-min reuse window)
loads them and runs the bench's C4 operator (int32-column rows, graph
schedule, group interleave, fused y update) for 3 warm-up + 2 steps.
Profiling evidence only: no test or bench number reads the cache."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api, workloads

CACHE = "/tmp/c4cache"
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
if sys.argv[1] == "save":
    cfg = workloads.CONFIGS["c4"]
    wl = workloads.build(cfg, ctx, 0, log=print)
    rp, cols, vals = wl.csr_c.export()
    y0 = api.gen_points(api.GEN_NORMAL, cfg.n, 2, 0, 1e-2, 2)[wl.inverse]
    os.makedirs(CACHE, exist_ok=True)
    for name, a in (("rp", rp), ("cols", cols), ("vals", vals), ("y0", y0)):
        np.save(os.path.join(CACHE, name + ".npy"), np.ascontiguousarray(a))
    print("saved", rp.size - 1, cols.size)
else:
    rp, cols, vals, y0 = (np.load(os.path.join(CACHE, k + ".npy")) for k in ("rp", "cols", "vals", "y0"))
    n = rp.size - 1
    op = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, api.ORIGINAL, 256, None, 0, 2)
    ybuf = [torch.from_numpy(y0).cuda(), torch.zeros(n, 2, device="cuda")]
    f = torch.empty(n, 2, device="cuda")
    eta = 4.0 * n / 12.0
    for i in range(5):
        op.tsne(ybuf[i & 1], 2, f, False, eta, ybuf[(i + 1) & 1])
    torch.cuda.synchronize()
    print("ran", n, cols.size, float(f.abs().max()))
