"""Device construction of the cluster-tile format
against the host builder: same halos, same 16-bit indices -> bitwise equal
results for every kernel."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k", [(3000, 30), (2049, 16), (700, 7)])
def test_device_tile_build_matches_host(ctx, n, k):
    import torch

    from paper_1709_03671_b200 import api
    pts = api.gen_points(api.GEN_3LEVEL, n, 49, 0, 0.125, 5)
    tree = api.order_tree(pts.astype(np.float64), 3, pca_device=0)
    pc = np.empty_like(pts)
    pc[tree.forward] = pts
    dp = api.to_device_points(pc)
    ids, _ = ctx.knn(dp, dp, n, n, 49, k, True)
    ctx.sync()
    op_dev = api.Operator.from_knn_device(ctx, ids, n)
    csr = api.HostCsr.from_knn(ids.cpu().numpy(), n)
    rp, cols, _ = csr.export()
    op_host = api.Operator.from_csr(ctx, n, n, rp, cols, None, api.CLUSTER, 256)
    for key in ("nnz", "stored", "n_tiles", "max_halo", "halo_total", "tile_rows"):
        assert op_dev.info[key] == op_host.info[key], key
    vals = np.random.default_rng(1).random(cols.size).astype(np.float32)
    op_dev.set_values(vals)
    op_host.set_values(vals)
    assert np.array_equal(op_dev.get_values(), vals)
    x = np.random.default_rng(2).random(n).astype(np.float32)
    assert np.array_equal(op_dev.spmv_host(x), op_host.spmv_host(x))
    h = 1.3
    xd = torch.from_numpy(x).cuda()
    y1, y2 = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    op_dev.gauss_spmv(dp, dp, 49, h, xd, y1)
    op_host.gauss_spmv(dp, dp, 49, h, xd, y2)
    o1, o2 = torch.empty_like(dp), torch.empty_like(dp)
    op_dev.meanshift(dp, dp, 49, h, o1)
    op_host.meanshift(dp, dp, 49, h, o2)
    ctx.sync()
    assert torch.equal(y1, y2) and torch.equal(o1, o2)


@pytest.mark.parametrize("tile_rows,order", [(256, 1), (128, 1), (256, 0)])
def test_scheduled_operator_is_bitwise_the_plain_one(ctx, tile_rows, order):
    """A row schedule (KNNX_SCHEDULE_GRAPH / GIVEN) changes only when rows run:
    every result equals the unscheduled operator's bit for bit."""
    import torch

    from paper_1709_03671_b200 import api
    n, k, dim = 3000, 12, 49
    pts = api.gen_points(api.GEN_3LEVEL, n, dim, 0, 0.125, 21)
    dp = api.to_device_points(pts)
    ids, _ = ctx.knn(dp, dp, n, n, dim, k, True)
    ctx.sync()
    ids = ids.cpu().numpy()
    # ragged rows too: drop a few entries from every 7th row
    rp = np.arange(0, n * k + 1, k, dtype=np.int64)
    cols = np.sort(ids, 1)
    keep = np.ones((n, k), bool)
    keep[::7, : 3] = False
    cols = cols[keep]
    rp = np.concatenate([[0], np.cumsum(keep.sum(1))]).astype(np.int64)
    vals = np.random.default_rng(4).random(cols.size).astype(np.float32) + 0.1
    plain = api.Operator.from_csr(ctx, n, n, rp, cols, vals, order, tile_rows)
    sched = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, order, tile_rows)
    perm = np.random.default_rng(5).permutation(n).astype(np.int32)
    given = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, order, tile_rows, perm)
    x = np.random.default_rng(6).random(n).astype(np.float32)
    want = plain.spmv_host(x)
    xd = torch.from_numpy(x).cuda()
    h = 0.9
    outs = {}
    for name, op in (("plain", plain), ("sched", sched), ("given", given)):
        assert np.array_equal(op.get_values(), vals)
        y0 = op.spmv_host(x)
        y = torch.empty(n, device="cuda")
        op.gauss_spmv(dp, dp, dim, h, xd, y)
        m = torch.empty_like(dp)
        op.meanshift(dp, dp, dim, h, m)
        emb = dp[:, :2].contiguous()
        f = torch.empty(n, 2, device="cuda")
        op.tsne(emb, 2, f, True, 0.0, None)
        ctx.sync()
        op.update_gaussian(dp, dp, dim, h)
        ctx.sync()
        outs[name] = (y0, y.cpu(), m.cpu(), f.cpu(), op.get_values(), op.spmv_host(x))
    assert np.array_equal(outs["plain"][0], want)
    for name in ("sched", "given"):
        for a, b in zip(outs["plain"], outs[name]):
            assert np.array_equal(np.asarray(a), np.asarray(b)), name


def test_tsne_affinities_on_device(ctx, ref):
    """knnx_tsne_affinities_dev (C4's P built on the device: conditional
    Gaussian rows, both orientations, radix sort + reduce by key) against a
    double-precision numpy construction on the same kNN rows, and its pattern
    against the reference library's own symmetrize (proj/src/knn.cpp:72-84)."""
    import math

    from paper_1709_03671_b200 import api
    n, dim, k = 3001, 50, 30
    pts = api.gen_points(api.GEN_C1_MIXTURE, n, dim, 16, 1.0, 4)
    dp = api.to_device_points(pts)
    ids, d2 = ctx.knn(dp, dp, n, n, dim, k, self_set=True)
    ctx.sync()
    idn, d2n = ids.cpu().numpy(), d2.cpu().numpy().astype(np.float64)
    h = float(np.median(np.sqrt(d2n)))
    rp, cols, vals = ctx.tsne_affinities(ids, d2, h / math.sqrt(2.0), 1.0 / (2.0 * n))
    w = np.exp(-d2n / (h * h))
    w /= w.sum(1, keepdims=True)
    rows = np.repeat(np.arange(n), k)
    key = np.concatenate([rows * n + idn.ravel(), idn.ravel().astype(np.int64) * n + rows])
    val = np.concatenate([w.ravel(), w.ravel()]) / (2.0 * n)
    uk, inv = np.unique(key, return_inverse=True)
    want = np.bincount(inv, weights=val)
    assert rp[-1] == uk.size and np.array_equal(cols, (uk % n).astype(np.int32))
    assert np.array_equal(rp, np.concatenate([[0], np.cumsum(np.bincount(uk // n, minlength=n))]))
    assert np.max(np.abs(vals - want) / want) < 1e-5
    assert abs(float(vals.astype(np.float64).sum()) - 1.0) < 1e-5
    # the pattern is the reference's structural union of the kNN pattern
    krp = np.arange(n + 1, dtype=np.int64) * k
    kcols = np.sort(idn, axis=1).ravel().astype(np.int32)
    sr, sc = ref.symmetrize(krp, kcols)
    order = np.lexsort((sc, sr))
    assert np.array_equal(np.asarray(sc)[order], cols)
