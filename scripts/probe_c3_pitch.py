"""C3 mean-shift step and the D=49 Gaussian-recompute SpMV with the source rows
at a 208-B pitch (ld = 52) against a 256-B pitch (ld = 64: every 128-B lane-group
request is one cache line).  Usage: probe_c3_pitch.py [n]"""
import sys

import torch

from paper_1709_03671_b200 import api, workloads

ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = workloads.scaled("c3", n) if n != 1_000_000 else workloads.CONFIGS["c3"]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
m, nn, _, _ = wl.csr_c.shape
rp, cols, _ = wl.csr_c.export()
op = api.Operator.from_csr_scheduled(ctx, m, nn, rp, cols, None, api.ORIGINAL, 256)
x = torch.from_numpy(wl.x_c).cuda()
y = torch.empty(n, device="cuda")
ref = None
for align in (4, 32, 4, 32):
    s = api.to_device_points(wl.points_c, align=align)
    out = torch.empty_like(s)
    for name, fn in (("meanshift", lambda: op.meanshift(s, s, cfg.dim, wl.h_ref, out)),
                     ("gauss_spmv", lambda: op.gauss_spmv(s, s, cfg.dim, wl.h_ref, x, y))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"ld={s.shape[1]} {name} {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
    res = out[:, :cfg.dim].clone()
    if ref is None:
        ref = res
    else:
        print("  max |diff| vs first", float((res - ref).abs().max()))
