"""C5 dense-block distance probe (evidence for DESIGN.md §3.3, not product code).

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
cfg = workloads.scaled("c5", n) if n != 1_000_000 else workloads.CONFIGS["c5"]
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


for R in (64, 128, 256):
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

# accuracy of tensor-core distances on the needed pairs (first 2,000 rows)
m = 2000
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


for mode in ("tf32", "3xtf32", "bf16"):
    tn = dot(tc, tc, mode)[:, None]
    sn = dot(sc, sc, mode)
    ts = dot(tc[:, None, :].expand_as(sc), sc, mode)
    d2 = (tn + sn - 2 * ts).clamp_min(0)
    y = (torch.exp(-d2 / h2) * x[nbr]).sum(-1)
    rel = float((y - y_ref).abs().max() / y_ref.abs().max())
    out[f"y_rel_{mode}"] = rel
    print(mode, "y rel err", rel, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/probe_c5_dense.json", "w") as f:
    json.dump(out, f, indent=1)
