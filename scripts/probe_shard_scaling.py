"""Strong-scaling forecast for `bench.py --gpus N` at C2 on one GPU: the
per-rank step of every N-way row-block shard (nnz-balanced, tile-aligned;
the slowest one counts) timed with the L2 flushed before each step (what
bench.py does when a shard fits the L2), as one CUDA-graph replay of K
steps, and as K stream launches, for N = 1, 2, 4, 8.  The forecast
efficiency is t(1) / (N t(N))."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_03671_b200 import api, workloads
from paper_1709_03671_b200.distributed import partition_rows
ctx = api.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.use_stream(stream)
wl = workloads.build(workloads.CONFIGS["c2"], ctx, 0, log=print)
rp, _, _ = wl.csr_c.export()
x = torch.from_numpy(wl.x_c).cuda()
K = 1000
out = {}
for n in (1, 2, 4, 8):
    worst = {}
    for r in range(n):
        r0, r1 = partition_rows(rp, n, 256)[r]
        op = api.Operator.from_host_csr(ctx, wl.csr_c.row_block(r0, r1), api.CLUSTER)
        op.set_row_base(r0)
        y = torch.empty(r1 - r0, device="cuda")
        res = {}
        scrub = torch.empty(64 * 2 ** 20, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(200)]
        for e0, e1 in evs:  # bench.py's method when a shard fits in L2
            scrub.zero_()
            e0.record(stream)
            op.spmv(x, y)
            e1.record(stream)
        torch.cuda.synchronize()
        res["flushed"] = sum(e0.elapsed_time(e1) for e0, e1 in evs) * 1e3 / len(evs)
        for mode in ("graph", "stream"):
            for _ in range(3):
                op.spmv(x, y)
            op.spmv_repeat(K, x, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if mode == "graph":
                op.spmv_repeat(K, x, y)
            else:
                for _ in range(K):
                    op.spmv(x, y)
            e1.record(stream)
            torch.cuda.synchronize()
            res[mode] = e0.elapsed_time(e1) * 1e3 / K
        op.close()
        for m, t in res.items():
            worst[m] = max(worst.get(m, 0.0), t)
    out[n] = worst
    print(n, {m: f"{t:.2f} us" for m, t in worst.items()},
          {m: f"eff {out[1][m] / (n * t):.2f}" for m, t in worst.items()}, flush=True)
print(json.dumps(out))
