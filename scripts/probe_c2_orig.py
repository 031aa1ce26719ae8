"""C2 original-order y = A x (spmv_flat path): spmv_orig_kernel vs explicit
U-entry batches (KNNX_ORIG_U = 8 / 15 / 30), bitwise equal results."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_03671_b200 import api, workloads
ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
wl = workloads.build(workloads.CONFIGS["c2"], ctx, 0, log=print)
op = api.Operator.from_host_csr(ctx, wl.csr_o, api.ORIGINAL)
x = torch.from_numpy(wl.x).cuda()
ref = None
for u in ("0", "8", "15", "16", "30", "31", "0"):
    os.environ["KNNX_ORIG_U"] = u
    y = torch.empty(wl.cfg.n, device="cuda")
    for _ in range(5):
        op.spmv(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        op.spmv(x, y)
    e1.record()
    torch.cuda.synchronize()
    ref = y if ref is None else ref
    print("U", u, f"{e0.elapsed_time(e1) / 200 * 1e3:.1f} us", "bitwise", bool(torch.equal(y, ref)),
          flush=True)
