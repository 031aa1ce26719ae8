"""Workload builders at small scale (GPU): the C4 t-SNE affinities and the
sharded operator paths used by bench.py, checked against the CPU oracle."""
import numpy as np
import pytest

from oracle.oracle import scale_rel

pytestmark = pytest.mark.gpu
TOL = 1e-5


def test_c4_affinities_and_tsne_iterations(ctx, oracle):
    import torch

    from paper_1709_03671_b200 import api, workloads
    cfg = workloads.scaled("c4", 3000)
    wl = workloads.build(cfg, ctx, 0)
    rp, cols, p = wl.csr_c.export()
    assert abs(float(p.astype(np.float64).sum()) - 1.0) < 1e-4
    # symmetric: p_ij == p_ji
    n = cfg.n
    dense = {}
    for i in range(0, n, 37):
        for e in range(rp[i], rp[i + 1]):
            j = cols[e]
            lo, hi = rp[j], rp[j + 1]
            k = lo + np.searchsorted(cols[lo:hi], i)
            assert cols[k] == i and p[k] == p[e]
    # three teacher-forced iterations of F + y update through the sharded path
    from paper_1709_03671_b200.distributed import ShardedOperator
    sop = ShardedOperator(ctx, wl.csr_c, 1, 0)
    y = torch.from_numpy(api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)).cuda()
    f = torch.empty_like(y)
    y2 = torch.empty_like(y)
    eta = 4.0 * n / 12.0
    for _ in range(3):
        sop.op.tsne(y, 2, f, False, eta, y2)
        ctx.sync()
        want = oracle.tsne(rp, cols, p.astype(np.float64), y.cpu().numpy().astype(np.float64),
                           direct=True)
        assert scale_rel(f.cpu().numpy(), want) <= TOL
        yn = y.cpu().numpy() - eta * f.cpu().numpy()
        assert np.allclose(y2.cpu().numpy(), yn, rtol=1e-6, atol=1e-9)
        y, y2 = y2, y


def test_row_block_shards_match_whole_operator(ctx):
    """Two row blocks of one operator reproduce the whole operator bit-for-bit
    (each row's sum stays in one block): spmv, Gaussian SpMV, mean shift, t-SNE."""
    import torch

    from paper_1709_03671_b200 import api, workloads
    from paper_1709_03671_b200.distributed import ShardedOperator
    cfg = workloads.scaled("c1", 3000)
    wl = workloads.build(cfg, ctx, 0)
    n = cfg.n
    whole = ShardedOperator(ctx, wl.csr_c, 1, 0)
    parts = [ShardedOperator(ctx, wl.csr_c, 2, r) for r in range(2)]
    x = torch.from_numpy(wl.x_c).cuda()
    y = torch.empty(n, device="cuda")
    whole.spmv(x, y)
    pts = api.to_device_points(wl.points_c)
    ms = torch.empty_like(pts)
    whole.op.meanshift(pts, pts, cfg.dim, wl.h_ref, ms)
    g = torch.empty(n, device="cuda")
    whole.op.gauss_spmv(pts, pts, cfg.dim, wl.h_ref, x, g)
    emb = torch.from_numpy(api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)).cuda()
    fw = torch.empty_like(emb)
    whole.op.tsne(emb, 2, fw, False, 0.0, None)
    for sop in parts:
        r0, r1 = sop.rows
        yl = torch.empty(r1 - r0, device="cuda")
        sop.spmv(x, yl)
        msl = torch.empty(r1 - r0, pts.shape[1], device="cuda")
        sop.op.meanshift(pts[r0:r1], pts, cfg.dim, wl.h_ref, msl)
        gl = torch.empty(r1 - r0, device="cuda")
        sop.op.gauss_spmv(pts[r0:r1], pts, cfg.dim, wl.h_ref, x, gl)
        fl = torch.empty(r1 - r0, 2, device="cuda")
        sop.op.tsne(emb, 2, fl, False, 0.0, None)
        ctx.sync()
        assert torch.equal(yl, y[r0:r1])
        assert torch.equal(msl, ms[r0:r1])
        assert torch.equal(gl, g[r0:r1])
        assert torch.equal(fl, fw[r0:r1])


def test_device_built_shards_match_whole_operator(ctx):
    """The C4 pipeline on the device end to end at test scale: tensor-core kNN,
    device-built symmetrised P, and two row-block shards built on the device
    from the full device CSR (scheduled, group-interleaved) -- five t-SNE steps
    with the fused embedding update equal the single-rank run bit for bit."""
    import torch

    from paper_1709_03671_b200 import api, workloads
    from paper_1709_03671_b200.distributed import ShardedOperator
    cfg = workloads.scaled("c4", 6000)
    wl = workloads.build(cfg, ctx, 0, keep_device_csr=True)
    assert wl.dev_csr is not None and wl.timings["knn_wide"]["rows_nonpositive_margin"] == 0
    n = cfg.n
    opts = api.OPT_GROUP_INTERLEAVE
    whole = ShardedOperator(ctx, wl.csr_c, 1, 0, layout=api.ORIGINAL, schedule=True, options=opts,
                            dev_csr=wl.dev_csr)
    parts = [ShardedOperator(ctx, wl.csr_c, 2, r, layout=api.ORIGINAL, schedule=True, options=opts,
                             dev_csr=wl.dev_csr) for r in range(2)]
    host = ShardedOperator(ctx, wl.csr_c, 1, 0, layout=api.ORIGINAL, schedule=True, options=opts)
    y0 = torch.from_numpy(api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)).cuda()
    eta = 4.0 * n / 12.0

    def run(ops):
        y, out = y0.clone(), torch.empty_like(y0)
        fs = []
        for _ in range(5):
            f = torch.empty(n, 2, device="cuda")
            for sop in ops:
                r0, r1 = sop.rows
                sop.op.tsne(y, 2, f[r0:r1], False, eta, out[r0:r1])
            ctx.sync()
            fs.append(f)
            y, out = out, y
        return fs, y

    fw, yw = run([whole])
    fp, yp = run(parts)
    fh, yh = run([host])
    for a, b, c in zip(fw, fp, fh):
        assert torch.equal(a, b) and torch.equal(a, c)
    assert torch.equal(yw, yp) and torch.equal(yw, yh)
