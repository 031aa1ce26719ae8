"""A/B of the C4 t-SNE kernel's y_j gather cache policy (KNNX_TSNE_YLOAD, read
per launch: 0 ld.global.nc, 1 ld.global.cg, 2 nc + L1::evict_last) on the cached
full-size C4 operator (scripts/c4_capture.py save first)."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api
CACHE = "/tmp/c4cache"
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
rp, cols, vals, y0 = (np.load(os.path.join(CACHE, k + ".npy")) for k in ("rp", "cols", "vals", "y0"))
n = rp.size - 1
op = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, api.ORIGINAL, 256, None, 0, 2)
y = torch.from_numpy(y0).cuda()
yo = torch.empty(n, 2, device="cuda")
f = torch.empty(n, 2, device="cuda")
res, ref = {}, None
for mb in sys.argv[1].split(",") if len(sys.argv) > 1 else ("0", "1", "2", "0", "1", "2"):
    os.environ["KNNX_TSNE_YLOAD"] = mb
    for _ in range(3):
        op.tsne(y, 2, f, False, 1.0, yo)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        op.tsne(y, 2, f, False, 1.0, yo)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = f.clone()
    res.setdefault(f"yload{mb}_us", []).append(e0.elapsed_time(e1) / 20 * 1e3)
    res[f"yload{mb}_equal"] = bool(torch.equal(f, ref))
print(json.dumps(res))
