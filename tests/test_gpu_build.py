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


def _ragged_symmetric_csr(ctx, n, k, dim, seed):
    """A symmetrised kNN pattern with values (variable row lengths, several
    components are possible): the shape of C4's P."""
    from paper_1709_03671_b200 import api
    pts = api.gen_points(api.GEN_C1_MIXTURE, n, dim, 7, 1.0, seed)
    dp = api.to_device_points(pts)
    ids, d2 = ctx.knn(dp, dp, n, n, dim, k, True)
    ctx.sync()
    csr = api.HostCsr.from_knn(ids.cpu().numpy(), n)
    csr.set_values(np.exp(-d2.cpu().numpy().astype(np.float64).ravel() / 20.0).astype(np.float32))
    return csr.symmetrize_values(1.0 / (2.0 * n)).export()


@pytest.mark.parametrize("n,k,options", [(3000, 12, 0), (3000, 12, 2), (5000, 30, 2), (257, 5, 0)])
@pytest.mark.parametrize("schedule", ["graph", None])
def test_device_csr_build_equals_host_build(ctx, n, k, options, schedule):
    """knnx_op_create_csr_dev (schedule, tile sort, slice offsets and entry
    placement on the device) builds the operator knnx_op_create_csr_ex builds
    on the host: same slot -> row map (so the same breadth-first schedule),
    same sizes, same stored values, bitwise equal results."""
    import torch

    from paper_1709_03671_b200 import api
    assert api.OPT_GROUP_INTERLEAVE == 2
    rp, cols, vals = _ragged_symmetric_csr(ctx, n, k, 10, 3)
    d_rp, d_cols, d_vals = (torch.from_numpy(a).cuda() for a in (rp, cols, vals))
    op_dev = api.Operator.from_csr_device(ctx, n, n, d_rp, d_cols, d_vals, schedule=schedule,
                                          options=options)
    if schedule == "graph":
        op_host = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, api.ORIGINAL, 256,
                                                  options=options)
    else:
        op_host = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, api.ORIGINAL, 256,
                                                  schedule=np.arange(n, dtype=np.int32), options=options)
    assert np.array_equal(op_dev.slot_rows(), op_host.slot_rows())
    for key in ("nnz", "stored", "n_tiles", "tile_rows", "uniform_row_len", "has_values"):
        assert op_dev.info[key] == op_host.info[key], key
    assert np.array_equal(op_dev.get_values(), vals)
    y = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)
    yd = torch.from_numpy(y).cuda()
    f1, f2 = torch.empty(n, 2, device="cuda"), torch.empty(n, 2, device="cuda")
    op_dev.tsne(yd, 2, f1)
    op_host.tsne(yd, 2, f2)
    ctx.sync()
    assert torch.equal(f1, f2)
    if options == 0:
        x = np.random.default_rng(2).random(n).astype(np.float32)
        assert np.array_equal(op_dev.spmv_host(x), op_host.spmv_host(x))
    new_vals = np.random.default_rng(4).random(cols.size).astype(np.float32)
    op_dev.set_values(new_vals)
    assert np.array_equal(op_dev.get_values(), new_vals)


def test_device_csr_build_rejects_bad_input(ctx):
    import torch

    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import KnnxError
    rp = torch.tensor([0, 2, 4], dtype=torch.int64).cuda()
    for bad_cols in ([0, 1, 1, 0], [0, 5, 0, 1]):      # unsorted row, column out of range
        cols = torch.tensor(bad_cols, dtype=torch.int32).cuda()
        with pytest.raises(KnnxError):
            api.Operator.from_csr_device(ctx, 2, 2, rp, cols, None)
    cols = torch.tensor([0, 1, 0, 1], dtype=torch.int32).cuda()
    vals = torch.tensor([1.0, float("nan"), 1.0, 1.0]).cuda()
    with pytest.raises(KnnxError):
        api.Operator.from_csr_device(ctx, 2, 2, rp, cols, vals)
    with pytest.raises(KnnxError):
        api.Operator.from_csr_device(ctx, 2, 2, rp, cols, None, schedule=np.array([0, 0], np.int32))


@pytest.mark.parametrize("options", [0, 2])
def test_device_csr_build_of_a_row_block(ctx, options):
    """A rank of a multi-GPU run builds its row block from the full device
    CSR (shifted row_ptr, unshifted cols / vals, col_base = r0): the same
    operator as the host build of HostCsr.row_block."""
    import torch

    from paper_1709_03671_b200 import api
    n, k = 4000, 14
    rp, cols, vals = _ragged_symmetric_csr(ctx, n, k, 10, 8)
    r0, r1 = 768, 2816
    full = api.HostCsr.from_arrays(n, n, rp, cols, vals)
    brp, bcols, bvals = full.row_block(r0, r1).export()
    op_host = api.Operator.from_csr_scheduled(ctx, r1 - r0, n, brp, bcols, bvals, api.ORIGINAL, 256,
                                              None, r0, options)
    op_host.set_row_base(r0)
    d_rp, d_cols, d_vals = (torch.from_numpy(a).cuda() for a in (rp, cols, vals))
    dev = api.DeviceCsr.from_tensors(ctx, n, n, d_rp, d_cols, d_vals)
    op_dev = api.Operator.from_csr_device(ctx, 0, 0, dev, schedule="graph", options=options, col_base=r0,
                                          rows=(r0, r1), block_nnz=int(rp[r1] - rp[r0]))
    op_dev.set_row_base(r0)
    assert np.array_equal(op_dev.slot_rows(), op_host.slot_rows())
    assert op_dev.info["stored"] == op_host.info["stored"] and op_dev.info["nnz"] == op_host.info["nnz"]
    assert np.array_equal(op_dev.get_values(), bvals)
    y = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)
    yd = torch.from_numpy(y).cuda()
    f1, f2 = torch.empty(r1 - r0, 2, device="cuda"), torch.empty(r1 - r0, 2, device="cuda")
    op_dev.tsne(yd, 2, f1)
    op_host.tsne(yd, 2, f2)
    ctx.sync()
    assert torch.equal(f1, f2)


def test_device_csr_build_many_components(ctx):
    """A pattern of 30,000 two-row components exhausts the level-synchronous
    walk's step budget; the schedule is then finished by the host function and
    the operator still equals the host build."""
    import torch

    from paper_1709_03671_b200 import api
    n = 60000
    rp = np.arange(n + 1, dtype=np.int64)
    cols = (np.arange(n, dtype=np.int32) ^ 1)           # row 2i <-> row 2i + 1
    vals = np.random.default_rng(0).random(n).astype(np.float32)
    op_host = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, api.ORIGINAL, 256)
    d = [torch.from_numpy(a).cuda() for a in (rp, cols, vals)]
    op_dev = api.Operator.from_csr_device(ctx, n, n, d[0], d[1], d[2], schedule="graph")
    assert np.array_equal(op_dev.slot_rows(), op_host.slot_rows())
    x = np.random.default_rng(2).random(n).astype(np.float32)
    assert np.array_equal(op_dev.spmv_host(x), op_host.spmv_host(x))


def test_device_csr_build_with_empty_rows_and_ragged_tail(ctx):
    """Empty rows, a row count that is not a multiple of 32, and one long row."""
    import torch

    from paper_1709_03671_b200 import api
    n = 1001
    rng = np.random.default_rng(9)
    lens = rng.integers(0, 9, n)
    lens[::5] = 0
    lens[17] = 300
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    vals = rng.random(cols.size).astype(np.float32)
    for options in (0, 2):
        op_host = api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, vals, api.ORIGINAL, 256, options=options)
        d = [torch.from_numpy(a).cuda() for a in (rp, cols, vals)]
        op_dev = api.Operator.from_csr_device(ctx, n, n, d[0], d[1], d[2], schedule="graph", options=options)
        assert np.array_equal(op_dev.slot_rows(), op_host.slot_rows())
        assert op_dev.info["stored"] == op_host.info["stored"]
        assert np.array_equal(op_dev.get_values(), vals)
        y = api.gen_points(api.GEN_NORMAL, n, 2, 0, 1e-2, 2)
        yd = torch.from_numpy(y).cuda()
        f1, f2 = torch.empty(n, 2, device="cuda"), torch.empty(n, 2, device="cuda")
        op_dev.tsne(yd, 2, f1)
        op_host.tsne(yd, 2, f2)
        ctx.sync()
        assert torch.equal(f1, f2)
