"""GPU parity: every hot-path kernel through the C ABI vs the CPU oracles.

Tolerances (BASELINE north_star): permutations and permuted
data bit-exact; y, mean-shift positions and forces within 1e-5 relative in
the scale-aware metric max|g - r| / max|r| against the double-precision
oracle, on identical fp32 inputs widened to double.
"""
import math

import numpy as np
import pytest

from oracle.oracle import RefHier, scale_rel

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


@pytest.fixture(scope="module")
def mini(ctx):
    """C1-shaped workload at N=4000 (D=49, k=30, 64-component mixture)."""
    from paper_1709_03671_b200 import workloads
    cfg = workloads.scaled("c1", 4000)
    return workloads.build(cfg, ctx, 0)


def _coo_rows(row_ptr):
    return np.repeat(np.arange(row_ptr.size - 1), np.diff(row_ptr))


def test_knn_matches_oracle(mini, oracle):
    """Device exact kNN vs the brute-force oracle (proj/src/knn.cpp:9-62)."""
    pts = mini.points.astype(np.float64)
    ids_o, d2_o = oracle.build_knn(pts, None, mini.cfg.k, True)
    # device ids are cluster positions of cluster-ordered rows -> original ids
    ids_dev = mini.inverse[mini.knn_ids_c[mini.forward]]
    same_rows = np.all(ids_dev == ids_o, axis=1)
    assert same_rows.mean() > 0.995
    # rows that differ only swap near-tied neighbors (fp32 vs fp64 distances)
    for i in np.nonzero(~same_rows)[0]:
        kth = d2_o[i, -1]
        d_dev = ((pts[ids_dev[i]] - pts[i]) ** 2).sum(1)
        assert np.all(d_dev <= kth * (1 + 1e-5))


@pytest.mark.parametrize("k", [90, 200])
def test_knn_large_k(ctx, oracle, torch, k):
    """Large k (C4's k = 90; up to 256): candidates are buffered in registers
    and merged into the sorted list 8 at a time.  Rows against the
    brute-force oracle (near-ties only may differ), and the result does not
    depend on the point order (the selection is exact in the (fp32 distance,
    index) order): a shuffled copy of the points gives the same distances and
    neighbour sets (up to exact fp32 ties at the k-th place)."""
    from paper_1709_03671_b200 import api
    n, dim = 3000, 50
    pts = api.gen_points(api.GEN_C1_MIXTURE, n, dim, 8, 1.0, 6)
    dp = api.to_device_points(pts)
    ids, d2 = ctx.knn(dp, dp, n, n, dim, k, self_set=True)
    ctx.sync()
    ids, d2 = ids.cpu().numpy(), d2.cpu().numpy()
    assert np.all(np.diff(d2, axis=1) >= 0)
    p64 = pts.astype(np.float64)
    ids_o, d2_o = oracle.build_knn(p64, None, k, True)
    ids_o = ids_o.reshape(n, k)
    same = np.all(ids == ids_o, axis=1)
    assert same.mean() > 0.99
    for i in np.nonzero(~same)[0]:
        d_dev = ((p64[ids[i]] - p64[i]) ** 2).sum(1)
        assert np.all(d_dev <= d2_o.reshape(n, k)[i, -1] * (1 + 1e-5))
    perm = np.random.default_rng(1).permutation(n)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(n)
    dq = api.to_device_points(np.ascontiguousarray(pts[perm]))
    ids_q, d2_q = ctx.knn(dq, dq, n, n, dim, k, self_set=True)
    ctx.sync()
    ids_q = perm[ids_q.cpu().numpy()][inv]
    d2_q = d2_q.cpu().numpy()[inv]
    # same sorted distances; the same neighbours except where an fp32 distance
    # tie at the k-th place is broken by the (permuted) index
    assert np.array_equal(d2_q, d2)
    for i in range(n):
        a, b = set(ids[i]), set(ids_q[i])
        if a != b:
            for j in a ^ b:
                dj = np.float32(((pts[j].astype(np.float32) - pts[i]) ** 2).sum())
                assert abs(float(d2[i, -1]) - float(dj)) <= 1e-5 * float(d2[i, -1])


def test_ordering_bit_exact_vs_reference(mini, ref):
    """Tree ordering (device PCA + host tree) == reference make_ordering('tree3')."""
    fwd_ref, _ = ref.make_ordering("tree3", mini.points.astype(np.float64))
    assert np.array_equal(fwd_ref, mini.forward)


def test_device_pca_is_bitwise_host_pca(mini):
    from paper_1709_03671_b200 import api
    pts = mini.points.astype(np.float64)
    a = api.fit_pca(pts, 3, pca_device=-1)
    b = api.fit_pca(pts, 3, pca_device=0)
    assert a["iterations"] == b["iterations"]
    assert np.array_equal(a["axes"], b["axes"])
    assert np.array_equal(a["projected"], b["projected"])


def test_gaussian_values(mini, oracle):
    rp, cols, vals = mini.csr_c.export()
    pc = mini.points_c.astype(np.float64)
    want = oracle.gaussian_values(rp, cols, pc, pc, mini.h_ref)
    assert scale_rel(vals, want) <= TOL


@pytest.mark.parametrize("order", ["cluster", "original"])
def test_spmv(mini, oracle, ctx, torch, order):
    """spmv_hier (cluster tiles) / spmv_flat (original CSR) vs the oracle."""
    from paper_1709_03671_b200 import api
    csr = mini.csr_c if order == "cluster" else mini.csr_o
    x = mini.x_c if order == "cluster" else mini.x
    rp, cols, vals = csr.export()
    op = api.Operator.from_csr(ctx, mini.cfg.n, mini.cfg.n, rp, cols, vals,
                               api.CLUSTER if order == "cluster" else api.ORIGINAL)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(mini.cfg.n, device="cuda")
    op.spmv(xd, yd)
    ctx.sync()
    want = oracle.spmv(rp, cols, vals.astype(np.float64), x.astype(np.float64))
    assert scale_rel(yd.cpu().numpy(), want) <= TOL
    assert scale_rel(op.spmv_host(x), want) <= TOL


def test_spmv_matches_reference_hier(mini, ref, ctx):
    """Against the reference library's own spmv_hier on its HierBlockMatrix."""
    from paper_1709_03671_b200 import api
    rp_o, cols_o, vals_o = mini.csr_o.export()
    h, fwd = RefHier.from_original(ref, rp_o, cols_o, vals_o.astype(np.float64), mini.embedding)
    assert np.array_equal(fwd, mini.forward)
    want = h.spmv(mini.x_c.astype(np.float64))
    want_par = h.spmv(mini.x_c.astype(np.float64), workers=4)
    assert np.array_equal(want, want_par)
    rp, cols, vals = mini.csr_c.export()
    op = api.Operator.from_csr(ctx, mini.cfg.n, mini.cfg.n, rp, cols, vals, api.CLUSTER)
    assert scale_rel(op.spmv_host(mini.x_c), want) <= TOL


def test_gauss_spmv(mini, oracle, ctx, torch):
    """iterate_interactions step with the Gaussian value model, weights recomputed."""
    from paper_1709_03671_b200 import api
    rp, cols, _ = mini.csr_c.export()
    op = api.Operator.from_csr(ctx, mini.cfg.n, mini.cfg.n, rp, cols, None, api.CLUSTER)
    pc = mini.points_c
    dp = api.to_device_points(pc)
    xd = torch.from_numpy(mini.x_c).cuda()
    yd = torch.empty(mini.cfg.n, device="cuda")
    op.gauss_spmv(dp, dp, mini.cfg.dim, mini.h_ref, xd, yd)
    ctx.sync()
    want = oracle.gauss_spmv(rp, cols, pc.astype(np.float64), pc.astype(np.float64), mini.h_ref,
                             mini.x_c.astype(np.float64))
    assert scale_rel(yd.cpu().numpy(), want) <= TOL


def test_meanshift_step(ctx, oracle, torch):
    """meanshift_step over fixed neighbor rows (self included), teacher-forced 5 steps."""
    from paper_1709_03671_b200 import api, workloads
    cfg = workloads.scaled("c3", 3000)
    wl = workloads.build(cfg, ctx, 0, with_values=False)
    rp, cols, _ = wl.csr_c.export()
    op = api.Operator.from_csr(ctx, cfg.n, cfg.n, rp, cols, None, api.CLUSTER)
    s = wl.points_c
    sd = api.to_device_points(s)
    t = s.copy()
    ids = cols.reshape(cfg.n, cfg.k)
    for _ in range(5):
        td = api.to_device_points(t)
        out = torch.empty_like(td)
        op.meanshift(td, sd, cfg.dim, wl.h_ref, out)
        ctx.sync()
        got = out.cpu().numpy()[:, :cfg.dim]
        want = oracle.meanshift_step(ids, t.astype(np.float64), s.astype(np.float64), wl.h_ref)
        assert scale_rel(got, want) <= TOL
        t = got


@pytest.mark.parametrize("tile_rows,dim", [(256, 2), (32, 2), (64, 2), (32, 3), (64, 1)])
def test_tsne_attractive(ctx, oracle, torch, tile_rows, dim):
    """tsne_attractive_step on a symmetrised kNN affinity matrix, both formulas
    (tiles <= 64 rows run the shared-memory-staged lane-group kernel)."""
    from paper_1709_03671_b200 import api, workloads
    cfg = workloads.scaled("c1", 3000)
    wl = workloads.build(cfg, ctx, 0)
    sym = wl.csr_c.symmetrize()
    rp, cols, _ = sym.export()
    rng = np.random.default_rng(0)
    p = rng.random(cols.size).astype(np.float32)
    p /= p.sum()
    y = (1e-2 * rng.standard_normal((cfg.n, dim))).astype(np.float32)
    op = api.Operator.from_csr(ctx, cfg.n, cfg.n, rp, cols, p, api.CLUSTER, tile_rows)
    f = op.tsne_host(y)
    want_direct = oracle.tsne(rp, cols, p.astype(np.float64), y.astype(np.float64), direct=True)
    want_ref, a = oracle.tsne(rp, cols, p.astype(np.float64), y.astype(np.float64))
    assert scale_rel(f, want_direct) <= TOL
    assert scale_rel(f, want_ref) <= TOL  # reference form = direct form to ~1e-15 in fp64
    f2 = op.tsne_host(y, store=True)
    assert np.array_equal(f, f2)
    assert scale_rel(op.get_values(), a) <= TOL


@pytest.mark.parametrize("order,options", [
    (0, 1), (0, 2), (0, 3), (1, 1)])  # (ORIGINAL|CLUSTER, RELABEL|INTERLEAVE|both)
def test_tsne_relabel_interleave_layouts(ctx, oracle, torch, order, options):
    """The C4 t-SNE layouts (KNNX_OPT_RELABEL_COLS / KNNX_OPT_GROUP_INTERLEAVE)
    give the oracle's forces; values, get/set and the in-place a_ij mutation
    stay in canonical order; the fused y update matches; a row-block shard
    (col_base = its first row) relabels only its own columns; every other
    entry point rejects these layouts."""
    from paper_1709_03671_b200 import api, workloads
    from paper_1709_03671_b200._lib import KnnxError
    cfg = workloads.scaled("c1", 3000)
    wl = workloads.build(cfg, ctx, 0)
    sym = wl.csr_c.symmetrize()
    rp, cols, _ = sym.export()
    rng = np.random.default_rng(5)
    p = rng.random(cols.size).astype(np.float32)
    p /= p.sum()
    y = (1e-2 * rng.standard_normal((cfg.n, 2))).astype(np.float32)
    op = api.Operator.from_csr_scheduled(ctx, cfg.n, cfg.n, rp, cols, p, order, 0, None, 0, options)
    want_direct = oracle.tsne(rp, cols, p.astype(np.float64), y.astype(np.float64), direct=True)
    _, a = oracle.tsne(rp, cols, p.astype(np.float64), y.astype(np.float64))
    assert np.array_equal(op.get_values(), p)
    f = op.tsne_host(y)
    assert scale_rel(f, want_direct) <= TOL
    yd = torch.from_numpy(y).cuda()
    fd = torch.empty_like(yd)
    yo = torch.empty_like(yd)
    op.tsne(yd, 2, fd, False, 0.5, yo)
    ctx.sync()
    assert np.array_equal(fd.cpu().numpy(), f)
    assert np.array_equal(yo.cpu().numpy(), y - np.float32(0.5) * f)
    f2 = op.tsne_host(y, store=True)
    assert np.array_equal(f, f2)
    assert scale_rel(op.get_values(), a) <= TOL
    op.set_values(p)
    assert np.array_equal(op.get_values(), p)
    x = torch.ones(cfg.n, device="cuda")
    with pytest.raises(KnnxError):
        op.spmv(x, torch.empty_like(x))
    # row-block shard [r0, r1): relabels columns r0..r1-1 only
    r0, r1 = 1024, 2048
    blk = sym.row_block(r0, r1)
    brp, bcols, _ = blk.export()
    bp = p[rp[r0]:rp[r1]]
    sop = api.Operator.from_csr_scheduled(ctx, r1 - r0, cfg.n, brp, bcols, bp, order, 0, None,
                                          r0, options)
    sop.set_row_base(r0)
    fs = torch.empty(r1 - r0, 2, device="cuda")
    sop.tsne(yd, 2, fs, False, 0.0, None)
    ctx.sync()
    assert scale_rel(fs.cpu().numpy(), want_direct[r0:r1]) <= TOL


def test_permute_rows_bit_exact(ctx, oracle, torch):
    from paper_1709_03671_b200 import api
    rng = np.random.default_rng(3)
    for width in (1, 3, 52):
        a = rng.standard_normal((1000, width)).astype(np.float32)
        fwd = api.order_scattered(1000, 7)
        want = oracle.permute_rows(a, fwd)
        ad = torch.from_numpy(a).cuda()
        out = torch.empty_like(ad)
        ctx = api.Context(0)
        ctx.permute_rows(ad, torch.from_numpy(fwd).cuda(), out)
        ctx.sync()
        assert np.array_equal(out.cpu().numpy(), want)
        back = torch.empty_like(ad)
        ctx.gather_rows(out, torch.from_numpy(fwd).cuda(), back)
        ctx.sync()
        assert np.array_equal(back.cpu().numpy(), a)


def test_zero_weight_error(ctx):
    """proj/tests/test_kernels.cpp:356-368: far target -> ZeroWeight with its index."""
    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import KnnxError
    op = api.Operator.from_csr(ctx, 1, 1, np.array([0, 1]), np.array([0]), None, api.CLUSTER)
    with pytest.raises(KnnxError) as e:
        op.meanshift_host(np.array([[0.0]], np.float32), np.array([[1e6]], np.float32), 1.0)
    assert e.value.name == "ZeroWeight"
    assert "target 0" in str(e.value)
    with pytest.raises(KnnxError) as e:
        op.meanshift_host(np.array([[0.0]], np.float32), np.array([[1.0]], np.float32), 0.0)
    assert e.value.name == "NonPositiveBandwidth"


@pytest.mark.parametrize("order", ["cluster", "original"])
def test_variable_length_rows_all_ops(ctx, oracle, torch, order):
    """Symmetrised pattern (row lengths vary): SELL-sigma slot order must be
    invisible -- spmv, Gaussian recompute, update_values and mean shift."""
    from paper_1709_03671_b200 import api, workloads
    cfg = workloads.scaled("c1", 2500)
    wl = workloads.build(cfg, ctx, 0, with_values=False)
    sym = wl.csr_c.symmetrize()
    rp, cols, _ = sym.export()
    n = cfg.n
    assert len(set(np.diff(rp).tolist())) > 1
    rng = np.random.default_rng(5)
    vals = rng.random(cols.size).astype(np.float32)
    o = api.CLUSTER if order == "cluster" else api.ORIGINAL
    op = api.Operator.from_csr(ctx, n, n, rp, cols, vals, o)
    assert op.info["stored"] < 1.5 * cols.size  # slots sorted by length pad little
    x = wl.x_c
    want = oracle.spmv(rp, cols, vals.astype(np.float64), x.astype(np.float64))
    assert scale_rel(op.spmv_host(x), want) <= TOL
    assert np.array_equal(op.get_values(), vals)
    pc = wl.points_c
    dp = api.to_device_points(pc)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(n, device="cuda")
    op.gauss_spmv(dp, dp, cfg.dim, wl.h_ref, xd, yd)
    ctx.sync()
    p64 = pc.astype(np.float64)
    want_g = oracle.gauss_spmv(rp, cols, p64, p64, wl.h_ref, x.astype(np.float64))
    assert scale_rel(yd.cpu().numpy(), want_g) <= TOL
    op.update_gaussian(dp, dp, cfg.dim, wl.h_ref)
    ctx.sync()
    assert scale_rel(op.get_values(), oracle.gaussian_values(rp, cols, p64, p64, wl.h_ref)) <= TOL
    # mean shift over variable-length neighbor rows (dense reference loop)
    out = torch.empty_like(dp)
    op.meanshift(dp, dp, cfg.dim, wl.h_ref, out)
    ctx.sync()
    got = out.cpu().numpy()[:, :cfg.dim]
    inv = 1.0 / (2.0 * wl.h_ref ** 2)
    for i in range(0, n, 97):
        js = cols[rp[i]:rp[i + 1]]
        w = np.exp(-((p64[js] - p64[i]) ** 2).sum(1) * inv)
        ref_i = (w[:, None] * p64[js]).sum(0) / w.sum()
        assert np.max(np.abs(got[i] - ref_i)) <= TOL * np.max(np.abs(p64))


@pytest.mark.parametrize("dim", [1, 3, 4, 5, 8, 16, 17, 20, 21, 33, 48, 49, 52, 64])
@pytest.mark.parametrize("order", [0, 1])
def test_meanshift_dims(ctx, oracle, torch, dim, order):
    """meanshift_step across dims (whole 16-float rounds, scalar and float4
    tails) and row lengths 3..40 (groups of a row with no neighbour), both
    layouts; fixed k = 24 rows against the oracle, ragged rows against the
    dense loop of proj/src/kernels.cpp:188-208."""
    from paper_1709_03671_b200 import api
    rng = np.random.default_rng(dim)
    n, k = 1500, 24
    pts = (rng.random((n, dim)) * 4.0).astype(np.float32)
    ids = np.empty((n, k), np.int32)
    for i in range(n):
        ids[i] = np.sort(np.concatenate(([i], rng.choice(np.delete(np.arange(n), i), k - 1, False))))
    h = float(np.sqrt(dim))
    op = api.Operator.from_csr(ctx, n, n, np.arange(n + 1) * k, ids.ravel(), None, order)
    dp = api.to_device_points(pts)
    out = torch.empty_like(dp)
    op.meanshift(dp, dp, dim, h, out)
    ctx.sync()
    p64 = pts.astype(np.float64)
    want = oracle.meanshift_step(ids, p64, p64, h)
    assert scale_rel(out.cpu().numpy()[:, :dim], want) <= TOL
    lens = rng.integers(3, 41, n)
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(n, l, False)) for l in lens]).astype(np.int32)
    op = api.Operator.from_csr(ctx, n, n, rp, cols, None, order)
    op.meanshift(dp, dp, dim, h, out)
    ctx.sync()
    got = out.cpu().numpy()[:, :dim]
    inv = 1.0 / (2.0 * h * h)
    for i in range(0, n, 7):
        js = cols[rp[i]:rp[i + 1]]
        w = np.exp(-((p64[js] - p64[i]) ** 2).sum(1) * inv)
        ref_i = (w[:, None] * p64[js]).sum(0) / w.sum()
        assert np.max(np.abs(got[i] - ref_i)) <= TOL * np.max(np.abs(p64)), i


def _same_tree(a, b):
    for f in ("forward", "begin", "end", "depth", "parent", "is_leaf"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("n,dim,cap,max_depth", [(5000, 3, 128, 12), (5000, 2, 16, 12), (3000, 1, 8, 20),
                                                 (100, 3, 128, 12), (1, 3, 128, 12), (40000, 3, 64, 4),
                                                 (200000, 3, 128, 12)])
def test_device_tree_equals_host_tree(n, dim, cap, max_depth):
    """knnx_tree_build_dev (orthant paths + two stable radix sorts) builds the
    tree of the host recursion (proj/src/tree.cpp:15-112) field for field:
    leaf order, node ids in creation order, ranges, depths, parents."""
    from paper_1709_03671_b200 import api
    rng = np.random.default_rng(n + dim + cap)
    centers = rng.standard_normal((7, dim)) * 5.0
    emb = centers[rng.integers(0, 7, n)] + rng.standard_normal((n, dim)) * rng.random((n, 1))
    _same_tree(api.build_tree(emb, cap, max_depth), api.build_tree(emb, cap, max_depth, device=0))


def test_device_tree_with_coincident_points():
    """Many identical points cannot be separated: the chain of single-child
    nodes runs to max_depth on both builds; ties keep ascending original index."""
    from paper_1709_03671_b200 import api
    rng = np.random.default_rng(3)
    emb = rng.standard_normal((4000, 3))
    emb[500:1500] = emb[500]          # 1000 copies of one point
    emb[3000:3100, 1] = emb[3000, 1]  # a degenerate line
    for cap, md in ((32, 12), (128, 6)):
        _same_tree(api.build_tree(emb, cap, md), api.build_tree(emb, cap, md, device=0))
