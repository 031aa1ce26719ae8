"""A/B of the C3 mean-shift kernels in one process (KNNX_NONSTAT_VARIANT is read
per launch): lean lane groups (0) vs neighbour-parallel warp per row (10).
N=1M, D=49, k=30, scheduled flat rows as bench.py --config c3 runs them."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api, workloads
from oracle.oracle import scale_rel
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c3", n) if n != 1_000_000 else workloads.CONFIGS["c3"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
m, nn, _, _ = wl.csr_c.shape
rp, cols, _ = wl.csr_c.export()
s = api.to_device_points(wl.points_c)
res = {}
outs = {}
for lay, name in ((api.ORIGINAL, "flat"), (api.CLUSTER, "tiles")):
    op = api.Operator.from_csr_scheduled(ctx, m, nn, rp, cols, None, lay, 256)
    for var in ("0", "10"):
        os.environ["KNNX_NONSTAT_VARIANT"] = var
        out = torch.empty_like(s)
        for _ in range(3):
            op.meanshift(s, s, cfg.dim, wl.h_ref, out)
        torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                op.meanshift(s, s, cfg.dim, wl.h_ref, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20 * 1e3)
        outs[(name, var)] = out.cpu().numpy()[:, :cfg.dim]
        res[f"{name}_var{var}_us"] = ts
        print(name, var, [f"{t:.1f}" for t in ts], flush=True)
    res[f"{name}_rel_np_vs_lane"] = scale_rel(outs[(name, "10")], outs[(name, "0")].astype(np.float64))
os.environ.pop("KNNX_NONSTAT_VARIANT")
print(json.dumps(res))
