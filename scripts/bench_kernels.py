#!/usr/bin/env python3
"""Per-kernel timings at BASELINE scale (C2/C3 shapes: N=1M, D=49, k=30).

Times every hot-path kernel with CUDA events on the library's stream (median
of `--reps` launches after warm-up) and reports algorithmic bytes / FLOPs per
launch (SURVEY.md §8d formulas) against MEASURED_PEAKS.json.  Output: one JSON
object on stdout.  Not the driver's bench line (that is bench.py).
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--only", default="")
    ap.add_argument("--align", type=int, default=4, help="point row pitch alignment (floats)")
    args = ap.parse_args()
    import torch

    from paper_1709_03671_b200 import api, workloads

    peaks = json.load(open(os.path.join(os.path.dirname(HERE), "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    dev = 0
    ctx = api.Context(dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.use_stream(stream)
    res = {"n": args.n, "peak_hbm_gbs": hbm}

    def timeit(fn, reps=args.reps, warm=5):
        for _ in range(warm):
            fn()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        torch.cuda.synchronize()
        ev[0].record(stream)
        for r in range(reps):
            fn()
            ev[r + 1].record(stream)
        torch.cuda.synchronize()
        ts = [ev[r].elapsed_time(ev[r + 1]) for r in range(reps)]
        ctx.sync()
        return float(np.median(ts)) * 1e-3  # s

    def report(name, t, alg_bytes=None, flops=None, nnz=None, **kw):
        d = {"us": t * 1e6}
        if nnz:
            d["interactions_per_s"] = nnz / t
        if alg_bytes:
            d["alg_bytes"] = alg_bytes
            d["gbs"] = alg_bytes / t / 1e9
            d["frac_hbm"] = d["gbs"] / hbm
        if flops:
            d["gflops"] = flops / t / 1e9
        d.update(kw)
        res[name] = d
        print(name, json.dumps(d), file=sys.stderr, flush=True)

    for cname in ("c2", "c3"):
        if args.only and cname not in args.only:
            continue
        cfg = workloads.scaled(cname, args.n) if args.n != 1_000_000 else workloads.CONFIGS[cname]
        wl = workloads.build(cfg, ctx, dev, with_values=(cname == "c2"),
                             log=lambda m: print(m, file=sys.stderr))
        n, D, k = cfg.n, cfg.dim, cfg.k
        nnz = wl.nnz
        pc = api.to_device_points(wl.points_c, align=args.align)
        ld = pc.shape[1]
        rp, cols, vals = wl.csr_c.export()
        x = torch.from_numpy(wl.x_c).cuda()
        y = torch.empty(n, device="cuda")
        if cname == "c2":
            op = api.Operator.from_csr(ctx, n, n, rp, cols, vals, api.CLUSTER)
            report("c2_spmv_cluster", timeit(lambda: op.spmv(x, y)),
                   8 * nnz + 4 * (n + 1) + 8 * n, nnz=nnz)
            for tr in (64, 128, 256):
                opn = api.Operator.from_csr(ctx, n, n, rp, cols, None, api.CLUSTER, tr)
                t = timeit(lambda: opn.gauss_spmv(pc, pc, D, wl.h_ref, x, y))
                report(f"c2_gauss_spmv_cluster_t{tr}", t, 4 * D * n + 4 * nnz + 4 * (n + 1) + 8 * n,
                       flops=(3 * D + 4) * nnz, nnz=nnz)
            ops = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, None, api.ORIGINAL, 256)
            t = timeit(lambda: ops.gauss_spmv(pc, pc, D, wl.h_ref, x, y))
            report("c2_gauss_spmv_sched_flat", t, 4 * D * n + 4 * nnz + 4 * (n + 1) + 8 * n,
                   flops=(3 * D + 4) * nnz, nnz=nnz)
            t = timeit(lambda: opn.update_gaussian(pc, pc, D, wl.h_ref), reps=5)
            report("c2_update_gaussian_cluster", t, 4 * D * n + 8 * nnz, nnz=nnz)
            rpo, colso, valso = wl.csr_o.export()
            opo = api.Operator.from_csr(ctx, n, n, rpo, colso, None, api.ORIGINAL)
            po = api.to_device_points(wl.points, align=args.align)
            t = timeit(lambda: opo.gauss_spmv(po, po, D, wl.h_ref, x, y), reps=10)
            report("c2_gauss_spmv_original", t, 4 * D * n + 4 * nnz + 4 * (n + 1) + 8 * n, nnz=nnz)
            # t-SNE attractive force on the symmetrised C2 graph, random p
            sym = wl.csr_c.symmetrize()
            srp, scol, _ = sym.export()
            rng = np.random.default_rng(0)
            p = rng.random(scol.size).astype(np.float32)
            p /= p.sum()
            opt = api.Operator.from_csr(ctx, n, n, srp, scol, p, api.CLUSTER)
            yy = (1e-2 * torch.randn(n, 2, device="cuda")).contiguous()
            f = torch.empty_like(yy)
            y2 = torch.empty_like(yy)
            snnz = scol.size
            report("c2sym_tsne_cluster", timeit(lambda: opt.tsne(yy, 2, f, False, 1.0, y2)),
                   8 * snnz + 4 * (n + 1) + 8 * n + 8 * n + 8 * n, nnz=snnz)
            # permutation of the 1M x 52 point set (gather)
            inv = torch.from_numpy(wl.inverse).cuda()
            out = torch.empty_like(pc)
            report("permute_points_gather", timeit(lambda: ctx.gather_rows(pc, inv, out)),
                   2 * pc.numel() * 4 + 4 * n)
        else:
            tout = torch.empty_like(pc)
            for tr in (64, 128, 256):
                op = api.Operator.from_csr(ctx, n, n, rp, cols, None, api.CLUSTER, tr)
                t = timeit(lambda: op.meanshift(pc, pc, D, wl.h_ref, tout))
                report(f"c3_meanshift_cluster_t{tr}", t, 4 * D * n * 3 + 4 * nnz + 4 * (n + 1),
                       flops=(4 * D + 10) * nnz, nnz=nnz, max_halo=op.info["max_halo"],
                       halo_total=op.info["halo_total"])
            ops = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, None, api.ORIGINAL, 256)
            t = timeit(lambda: ops.meanshift(pc, pc, D, wl.h_ref, tout))
            report("c3_meanshift_sched_flat", t, 4 * D * n * 3 + 4 * nnz + 4 * (n + 1),
                   flops=(4 * D + 10) * nnz, nnz=nnz)
            rpo, colso, _ = wl.csr_o.export()
            opo = api.Operator.from_csr(ctx, n, n, rpo, colso, None, api.ORIGINAL)
            po = api.to_device_points(wl.points, align=args.align)
            touto = torch.empty_like(po)
            t = timeit(lambda: opo.meanshift(po, po, D, wl.h_ref, touto), reps=10)
            report("c3_meanshift_original", t, 4 * D * n * 3 + 4 * nnz + 4 * (n + 1), nnz=nnz)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
