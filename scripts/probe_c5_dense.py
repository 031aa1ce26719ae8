"""Dense-block distance probe (evidence for DESIGN.md §3.2-3.3, not product code).

Usage: probe_c5_dense.py [N] [c5|c3] -- C5 by default; c3 runs the same
measurements on the mean-shift point set (D = 49, k = 30 with self).

Asks whether the north star's tensor-core formulation d2 = |t|^2 + |s|^2 - 2 t.s
over dense (tile x halo) blocks can beat the CUDA-core gauss_warp_kernel at C5
(N=1M, D=960, k=16).  For each scheduled tile of R rows the dense block is
R x H (H = the tile's distinct sources), of which only R*k pairs are needed.

Measures, on the real C5 workload:
  * halo statistics per tile height (the overcompute factor H/k),
  * cuBLAS batched GEMM time for the dense blocks at the mean halo size, in
    TF32 and BF16 (library GEMMs stand in for an ideal tcgen05 kernel: they
    are an upper bound on what the tensor pipe can deliver for these shapes),
  * the gather of S[halo] into GEMM operands (the traffic a fused kernel would
    move L2 -> SMEM),
  * the accuracy of 1xTF32 / BF16 / 3xTF32 distances on the needed pairs,
    propagated to y = A x against the fp64 result (the 1e-5 gate).
"""
import os
import sys
import json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1709_03671_b200 import api, workloads

ctx = api.Context(0)
ctx.use_stream(torch.cuda.current_stream())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cname = sys.argv[2] if len(sys.argv) > 2 else "c5"  # c3: the mean-shift point set (D = 49, k = 30)
cfg = workloads.scaled(cname, n) if n != 1_000_000 else workloads.CONFIGS[cname]
wl = workloads.build(cfg, ctx, 0, with_values=False, log=print)
D, k = cfg.dim, cfg.k
ids = wl.knn_ids_c.astype(np.int64)
sched = wl.csr_c.locality_schedule()
pts = torch.from_numpy(wl.points_c).cuda()
h2 = wl.h_baseline ** 2
out = {"n": n, "dim": D, "k": k}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for R in ((32, 64, 128, 256) if cname == "c3" else (64, 128, 256)):
    rows = sched[: (n // R) * R].reshape(-1, R)
    nb = ids[rows]                                           # tiles x R x k
    halos = [np.unique(t) for t in nb[:200]]
    H = int(np.mean([len(h) for h in halos]))
    Hp = (H + 15) // 16 * 16
    T = rows.shape[0]
    rec = {"tiles": T, "mean_halo_first200": H, "overcompute": round(Hp / k, 1)}
    flops = 2.0 * T * R * Hp * D
    for dt, name in ((torch.float32, "tf32"), (torch.bfloat16, "bf16")):
        torch.backends.cuda.matmul.allow_tf32 = True
        chunk = max(1, min(T, int(6e9 // ((R + Hp) * D * 4 + R * Hp * 4))))
        a = torch.randn(chunk, R, D, device="cuda", dtype=dt)
        b = torch.randn(chunk, D, Hp, device="cuda", dtype=dt)
        ms = timed(lambda: torch.bmm(a, b)) * T / chunk
        rec[f"bmm_{name}_ms"] = round(ms, 3)
        rec[f"bmm_{name}_tflops"] = round(flops / ms / 1e9, 1)
        del a, b
    # gather of the halo rows into contiguous operands (fused-kernel L2->SMEM bytes)
    rec["gather_bytes_GB"] = round(T * Hp * D * 4 / 1e9, 2)
    idx = torch.from_numpy(np.concatenate([np.resize(h, Hp) for h in halos])).cuda()
    ms_g = timed(lambda: pts.index_select(0, idx)) * T / len(halos)
    rec["gather_ms"] = round(ms_g, 3)
    out[f"R{R}"] = rec
    print(R, rec, flush=True)

# accuracy of tensor-core distances on the needed pairs (first 2,048 rows)
m = 2048
t = torch.from_numpy(wl.points_c[:m]).double().cuda()
nbr = torch.from_numpy(ids[:m]).cuda()
s = pts.double()[nbr]                                        # m x k x D
x = torch.from_numpy(wl.x_c.astype(np.float64)).cuda()
d2_ref = ((s - t[:, None, :]) ** 2).sum(-1)
y_ref = (torch.exp(-d2_ref / h2) * x[nbr]).sum(-1)
c = pts.double().mean(0)                                     # centring (global mean)
tc, sc = (t - c).float(), (s - c).float()


def split_tf32(v):
    hi = v.view(torch.int32) & ~0x1FFF
    hi = hi.view(torch.float32)
    return hi, v - hi


def dot(a, b, mode):
    if mode == "bf16":
        return (a.bfloat16().double() * b.bfloat16().double()).sum(-1)
    ah, al = split_tf32(a)
    bh, bl = split_tf32(b)
    r = (ah.double() * bh.double()).sum(-1)
    if mode == "3xtf32":
        r = r + (ah.double() * bl.double()).sum(-1) + (al.double() * bh.double()).sum(-1)
    return r


# tile-local centring: each 64-row tile (cluster order) centred on its own mean
ct = t.reshape(-1, 64, D).mean(1).repeat_interleave(64, 0)   # m x D
tcl, scl = (t - ct).float(), (s - ct[:, None, :]).float()
for centring, (tt, ss) in (("global", (tc, sc)), ("tile64", (tcl, scl))):
    for mode in ("tf32", "3xtf32", "bf16"):
        tn = dot(tt, tt, mode)[:, None]
        sn = dot(ss, ss, mode)
        ts = dot(tt[:, None, :].expand_as(ss), ss, mode)
        d2 = (tn + sn - 2 * ts).clamp_min(0)
        y = (torch.exp(-d2 / h2) * x[nbr]).sum(-1)
        rel = float((y - y_ref).abs().max() / y_ref.abs().max())
        key = f"y_rel_{mode}" if centring == "global" else f"y_rel_{mode}_{centring}"
        out[key] = rel
        print(centring, mode, "y rel err", rel, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/probe_{cname}_dense.json", "w") as f:
    json.dump(out, f, indent=1)
