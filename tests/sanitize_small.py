"""Every default kernel of libknnx.so once on small inputs, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool racecheck python tests/sanitize_small.py

Covers the shared-memory / PDL kernels (spmv_tiles_g_kernel with
griddepcontrol, tsne_tiles_group_kernel) and the rest of
the hot path, then checks the results against the double oracle so a run
that passes the tool also computed the right numbers."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle.oracle import Oracle, scale_rel
from paper_1709_03671_b200 import api, workloads

ctx = api.Context(0)
orc = Oracle()
wl = workloads.build(workloads.scaled("c1", 1500), ctx, 0, pca_device=-1)
n, dim, k = wl.cfg.n, wl.cfg.dim, wl.cfg.k
rp, cols, vals = wl.csr_c.export()
errs = {}
x = torch.from_numpy(wl.x_c).cuda()
y = torch.empty(n, device="cuda")
want_y = orc.spmv(rp, cols, vals.astype(np.float64), wl.x_c.astype(np.float64))
for order, tile in ((api.CLUSTER, 256), (api.CLUSTER, 64), (api.ORIGINAL, 256)):
    op = api.Operator.from_csr(ctx, n, n, rp, cols, vals, order, tile)
    op.spmv(x, y)
    op.spmv(y.clone(), y)  # back-to-back PDL launches reading the previous output
    op.spmv(x, y)
    ctx.sync()
    errs[f"spmv_{order}_{tile}"] = scale_rel(y.cpu().numpy(), want_y)
    ys = torch.empty(4, n, device="cuda")
    op.spmv_repeat(4, x, ys, 0, n)  # CUDA-graph replay
    ctx.sync()
    errs[f"spmv_graph_{order}"] = scale_rel(ys[3].cpu().numpy(), want_y)
s = wl.points_c
s64 = s.astype(np.float64)
sd = api.to_device_points(s)
op = api.Operator.from_csr(ctx, n, n, rp, cols, None, api.CLUSTER)
op.gauss_spmv(sd, sd, dim, wl.h_ref, x, y)
out = torch.empty_like(sd)
op.meanshift(sd, sd, dim, wl.h_ref, out)
op.update_gaussian(sd, sd, dim, wl.h_ref)
ctx.sync()
errs["gauss"] = scale_rel(y.cpu().numpy(), orc.gauss_spmv(rp, cols, s64, s64, wl.h_ref,
                                                           wl.x_c.astype(np.float64)))
errs["meanshift"] = scale_rel(out.cpu().numpy()[:, :dim],
                              orc.meanshift_step(cols.reshape(n, k), s64, s64, wl.h_ref))
# wide rows (warp per row)
for wd, kk in ((128, 16), (131, 12)):
    pts = api.gen_points(api.GEN_ANISO, 1200, wd, (4 << 16) | 4, 1.0, 3)
    p64 = pts.astype(np.float64)
    ids, _ = orc.build_knn(p64, None, kk, True)
    c = api.HostCsr.from_knn(ids.reshape(1200, kk), 1200)
    wrp, wcols, _ = c.export()
    opw = api.Operator.from_csr(ctx, 1200, 1200, wrp, wcols, None, api.CLUSTER)
    pd = api.to_device_points(pts)
    xw = torch.rand(1200, device="cuda")
    yw = torch.empty(1200, device="cuda")
    opw.gauss_spmv(pd, pd, wd, 2.0, xw, yw)
    ow = torch.empty_like(pd)
    opw.meanshift(pd, pd, wd, 2.0, ow)
    ctx.sync()
    errs[f"gauss_wide_{wd}"] = scale_rel(yw.cpu().numpy(), orc.gauss_spmv(
        wrp, wcols, p64, p64, 2.0, xw.cpu().numpy().astype(np.float64)))
# t-SNE: rows / tiles-group / group / interleaved / window kernels
sym = wl.csr_c.symmetrize_values(1.0 / (2.0 * n))
prp, pcols, pv = sym.export()
yv = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)
want_f = orc.tsne(prp, pcols, pv.astype(np.float64), yv.astype(np.float64), direct=True)
yd = torch.from_numpy(yv).cuda()
f = torch.empty(n, 2, device="cuda")
for name, mk in (("tiles64", lambda: api.Operator.from_csr(ctx, n, n, prp, pcols, pv, api.CLUSTER, 64)),
                 ("group", lambda: api.Operator.from_csr(ctx, n, n, prp, pcols, pv, api.CLUSTER, 256)),
                 ("inter", lambda: api.Operator.from_csr_scheduled(ctx, n, n, prp, pcols, pv,
                                                                   api.ORIGINAL, 0, None, 0, 2)),
                 ("relabel", lambda: api.Operator.from_csr_scheduled(ctx, n, n, prp, pcols, pv,
                                                                     api.ORIGINAL, 0, None, 0, 3))):
    opt = mk()
    yo = torch.empty_like(yd)
    opt.tsne(yd, 2, f, False, 0.5, yo)
    ctx.sync()
    errs[f"tsne_{name}"] = scale_rel(f.cpu().numpy(), want_f)
# permutation + kNN tool
fwd = torch.from_numpy(wl.forward).cuda()
src = torch.from_numpy(wl.points).cuda()
dst = torch.empty_like(src)
ctx.permute_rows(src, fwd, dst)
ids_d, _ = ctx.knn(sd, sd, n, n, dim, k, self_set=True)
ctx.sync()
assert np.array_equal(dst.cpu().numpy(), orc.permute_rows(wl.points, wl.forward))
# tensor-core kNN (TMA ring, tcgen05.mma, TMEM loads, mbarrier pipeline, warp
# radix select), unpartitioned and with the pivot-cell partition
for wn, wd, wk in ((900, 96, 8), (20000, 64, 12)):
    wp = api.gen_points(api.GEN_ANISO, wn, wd, (4 << 16) | 4, 1.0, 9)
    wdev = api.to_device_points(wp)
    wids, wd2, wst = ctx.knn_wide(wdev, wdev, wn, wn, wd, wk, True, want_stats=True)
    ctx.sync()
    rows = np.random.default_rng(0).choice(wn, 300, replace=False)
    w64 = wp.astype(np.float64)
    got = wids.cpu().numpy()[rows].astype(np.int64)
    full = ((w64[rows, None, :] - w64[None, :, :]) ** 2).sum(-1) if wn <= 2000 else (
        (w64[rows] ** 2).sum(1)[:, None] + (w64 ** 2).sum(1)[None, :] - 2.0 * w64[rows] @ w64.T)
    full[np.arange(300), rows] = np.inf
    want = np.argsort(full, axis=1, kind="stable")[:, :wk]
    assert np.mean(got == want) > 0.995, f"knn_wide ids {np.mean(got == want)}"
    dd = ((w64[rows, None, :] - w64[got]) ** 2).sum(-1)
    errs[f"knn_wide_{wn}"] = float(np.max(np.abs(wd2.cpu().numpy()[rows] - dd) / dd))
    assert wst["rows_nonpositive_margin"] == 0
# device operator build (validate / BFS schedule / tile sort / placement kernels)
d_rp, d_cols, d_vals = (torch.from_numpy(a).cuda() for a in (prp, pcols, pv))
opd = api.Operator.from_csr_device(ctx, n, n, d_rp, d_cols, d_vals, schedule="graph", options=2)
opd.tsne(yd, 2, f)
ctx.sync()
errs["tsne_device_built"] = scale_rel(f.cpu().numpy(), want_f)
bad = {a: b for a, b in errs.items() if not b <= 1e-5}
print({a: f"{b:.1e}" for a, b in errs.items()})
assert not bad, bad
print("sanitize_small ok")
