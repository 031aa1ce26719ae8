"""Wide points (D > 64: warp-per-row kernels, C5's D = 960 path) against the
double oracle: Gaussian-recompute SpMV, update_values, mean shift."""
import numpy as np
import pytest

from oracle.oracle import scale_rel

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("dim", [67, 960])
@pytest.mark.parametrize("order", ["cluster", "original"])
def test_wide_points_all_nonstationary_ops(ctx, oracle, dim, order):
    import torch

    from paper_1709_03671_b200 import api
    n, k = 700, 16
    pts = api.gen_points(api.GEN_ANISO, n, dim, (4 << 16) | 4, 1.0, 11)
    p64 = pts.astype(np.float64)
    ids, d2 = oracle.build_knn(p64, None, k, True)
    csr = api.HostCsr.from_knn(ids, n)
    rp, cols, _ = csr.export()
    h_ref = float(np.median(np.sqrt(d2))) / np.sqrt(2.0)
    o = api.CLUSTER if order == "cluster" else api.ORIGINAL
    op = api.Operator.from_csr(ctx, n, n, rp, cols, None, o)
    dp = api.to_device_points(pts)
    x = np.random.default_rng(3).random(n).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(n, device="cuda")
    op.gauss_spmv(dp, dp, dim, h_ref, xd, yd)
    ctx.sync()
    want = oracle.gauss_spmv(rp, cols, p64, p64, h_ref, x.astype(np.float64))
    assert scale_rel(yd.cpu().numpy(), want) <= TOL
    op.update_gaussian(dp, dp, dim, h_ref)
    ctx.sync()
    assert scale_rel(op.get_values(), oracle.gaussian_values(rp, cols, p64, p64, h_ref)) <= TOL
    out = torch.empty_like(dp)
    op.meanshift(dp, dp, dim, h_ref, out)
    ctx.sync()
    want_ms = oracle.meanshift_step(cols.reshape(n, k), p64, p64, h_ref)
    assert scale_rel(out.cpu().numpy()[:, :dim], want_ms) <= TOL


@pytest.mark.parametrize("dim,k,sched", [(960, 16, True), (960, 16, False), (131, 32, True),
                                         (960, 5, True)])
def test_wide_gauss_32row_tiles(ctx, oracle, dim, k, sched):
    """Gaussian SpMV on 32-row cluster tiles vs the double oracle, with a
    ragged last tile (n % 32 != 0), a symmetrised graph with variable row
    lengths and scheduled / tree-order rows."""
    import torch

    from paper_1709_03671_b200 import api
    n = 1000 + 13
    pts = api.gen_points(api.GEN_ANISO, n, dim, (4 << 16) | 4, 1.0, 12)
    p64 = pts.astype(np.float64)
    ids, d2 = oracle.build_knn(p64, None, k, True)
    csr = api.HostCsr.from_knn(ids, n)
    if k == 5:
        csr = csr.symmetrize()  # variable row lengths
    rp, cols, _ = csr.export()
    h_ref = float(np.median(np.sqrt(d2))) / np.sqrt(2.0)
    op = (api.Operator.from_csr_scheduled(ctx, n, n, rp, cols, None, api.CLUSTER, 32) if sched
          else api.Operator.from_csr(ctx, n, n, rp, cols, None, api.CLUSTER, 32))
    dp = api.to_device_points(pts)
    x = np.random.default_rng(4).random(n).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    yd = torch.full((n,), float("nan"), device="cuda")
    for _ in range(2):  # the ring's phases continue across launches
        op.gauss_spmv(dp, dp, dim, h_ref, xd, yd)
    ctx.sync()
    want = oracle.gauss_spmv(rp, cols, p64, p64, h_ref, x.astype(np.float64))
    assert scale_rel(yd.cpu().numpy(), want) <= TOL


@pytest.mark.parametrize("dim", [200, 960])
def test_wide_device_pca_bitwise_and_reference_ordering(ref, dim):
    """Column-blocked device covariance (D * p > 512 chains): bitwise the host
    PCA, and the resulting tree order == reference make_ordering('tree3')."""
    from paper_1709_03671_b200 import api
    pts = api.gen_points(api.GEN_ANISO, 2500, dim, (4 << 16) | 4, 1.0, 13).astype(np.float64)
    a = api.fit_pca(pts, 3, pca_device=-1)
    b = api.fit_pca(pts, 3, pca_device=0)
    assert a["iterations"] == b["iterations"]
    assert np.array_equal(a["axes"], b["axes"])
    assert np.array_equal(a["projected"], b["projected"])
    tree = api.order_tree(pts, 3, pca_device=0)
    fwd_ref, _ = ref.make_ordering("tree3", pts)
    assert np.array_equal(fwd_ref, tree.forward)


@pytest.mark.parametrize("n,dim,k,self_set", [(1500, 960, 16, True), (700, 67, 5, False),
                                              (3000, 200, 30, True), (130, 96, 8, True),
                                              (5000, 50, 90, True), (2000, 33, 200, False),
                                              (600, 8, 4, True), (20, 70, 3, True), (9, 130, 8, True)])
def test_wide_knn_matches_oracle(ctx, oracle, n, dim, k, self_set):
    """knnx_knn_wide_dev (tcgen05 TF32 screen, exact fp32 re-rank) against the
    brute-force oracle (proj/src/knn.cpp:9-62): identical rows up to fp32
    near-ties, distances to fp32 rounding, a positive margin on every row."""
    from paper_1709_03671_b200 import api
    pts = api.gen_points(api.GEN_ANISO, n, dim, (4 << 16) | 4, 1.0, 17)
    dp = api.to_device_points(pts)
    ids, d2, st = ctx.knn_wide(dp, dp, n, n, dim, k, self_set, want_stats=True)
    ctx.sync()
    p64 = pts.astype(np.float64)
    want_ids, want_d2 = oracle.build_knn(p64, p64, k, self_set)
    got = ids.cpu().numpy()
    assert got.min() >= 0 and got.max() < n
    assert np.mean(got == want_ids.reshape(n, k)) > 0.999
    assert np.allclose(d2.cpu().numpy(), want_d2.reshape(n, k), rtol=1e-4, atol=1e-6)
    assert st["rows_nonpositive_margin"] == 0 and st["tiles_multiplied"] <= st["tiles_dense"]


def test_wide_knn_distinct_queries_and_order_independence(ctx, oracle):
    """Queries that are not the sources (the mean-shift refresh case), and the
    same neighbours whatever order the sources come in (pruning only changes
    which tiles are visited)."""
    import torch

    from paper_1709_03671_b200 import api
    n, m, dim, k = 5000, 777, 128, 12
    src = api.gen_points(api.GEN_ANISO, n, dim, (8 << 16) | 8, 1.0, 5)
    qry = api.gen_points(api.GEN_ANISO, m, dim, (8 << 16) | 8, 1.0, 6)
    ds, dq = api.to_device_points(src), api.to_device_points(qry)
    ids, d2 = ctx.knn_wide(dq, ds, m, n, dim, k, False)
    ctx.sync()
    want_ids, want_d2 = oracle.build_knn(qry.astype(np.float64), src.astype(np.float64), k, False)
    assert np.mean(ids.cpu().numpy() == want_ids.reshape(m, k)) > 0.999
    assert np.allclose(d2.cpu().numpy(), want_d2.reshape(m, k), rtol=1e-4)
    perm = np.random.default_rng(0).permutation(n)
    ds2 = api.to_device_points(src[perm])
    ids2, d22 = ctx.knn_wide(dq, ds2, m, n, dim, k, False)
    ctx.sync()
    back = torch.from_numpy(perm.astype(np.int64)).cuda()[ids2.long()]
    assert (back == ids.long()).float().mean().item() > 0.999
    assert torch.allclose(d22, d2, rtol=1e-5)


@pytest.mark.parametrize("n,dim,k,shuffle", [(40000, 96, 16, False), (40000, 96, 16, True),
                                             (70000, 50, 90, True)])
def test_wide_knn_partitioned_matches_brute_force(ctx, n, dim, k, shuffle):
    """n >= 16384: the points are re-partitioned into pivot cells before the
    screen (tile pruning no longer depends on the caller's order).  Sampled
    rows against an fp64 brute force; a shuffled input gives the same graph."""
    import torch

    from paper_1709_03671_b200 import api
    pts = api.gen_points(api.GEN_ANISO, n, dim, (8 << 16) | 8, 1.0, 23)
    if shuffle:
        pts = pts[np.random.default_rng(5).permutation(n)]
    dp = api.to_device_points(pts)
    ids, d2, st = ctx.knn_wide(dp, dp, n, n, dim, k, True, want_stats=True)
    ctx.sync()
    assert st["rows_nonpositive_margin"] == 0
    assert st["tiles_multiplied"] < 0.7 * st["tiles_dense"]      # the pruning works in any order
    rows = torch.from_numpy(np.random.default_rng(1).choice(n, 256, replace=False)).cuda()
    p = dp[:, :dim].double()
    q = p[rows]
    dd = (q * q).sum(1)[:, None] + (p * p).sum(1)[None, :] - 2.0 * q @ p.t()
    dd[torch.arange(256), rows] = float("inf")
    cand = torch.topk(dd, k + 8, dim=1, largest=False).indices
    ex = ((p[cand] - q[:, None, :]) ** 2).sum(-1)
    o = torch.argsort(ex, dim=1, stable=True)[:, :k]
    want_ids, want_d2 = torch.gather(cand, 1, o), torch.gather(ex, 1, o)
    assert (ids[rows].long() == want_ids).float().mean().item() > 0.999
    assert torch.allclose(d2[rows].double(), want_d2, rtol=1e-4)
    got = ids.cpu().numpy()
    assert got.min() >= 0 and got.max() < n and not (got == np.arange(n)[:, None]).any()


def test_wide_knn_certificate_and_exact_fallback(ctx):
    """Leaf clusters that are tight against their distance from the global
    mean (C2's 3-level mixture) defeat a TF32 screen: the per-row certificate
    must notice, and for dim <= 64 those rows are searched again by the exact
    SIMT kernel, so the result is the exact one."""
    import torch

    from paper_1709_03671_b200 import api
    n, dim, k = 30000, 49, 30
    pts = api.gen_points(api.GEN_3LEVEL, n, dim, 0, 0.125, 7)
    tree = api.order_tree(pts.astype(np.float64), 3, pca_device=-1)
    pc = np.empty_like(pts)
    pc[tree.forward] = pts
    dp = api.to_device_points(pc)
    ids_e, d2_e = ctx.knn(dp, dp, n, n, dim, k, True)
    ids_w, d2_w, st = ctx.knn_wide(dp, dp, n, n, dim, k, True, want_stats=True)
    ctx.sync()
    assert st["rows_recomputed_exactly"] > 0 and st["rows_nonpositive_margin"] == 0
    # certified rows keep the screen's result: equal to the exact search up to
    # fp32 near-ties (same distance lists), never a missed neighbour
    same = (ids_e == ids_w).all(1)
    assert same.float().mean().item() > 0.99
    rel = ((d2_e - d2_w).abs() / d2_e.clamp_min(1e-30)).max().item()
    assert rel < 1e-5, rel
    # the same geometry in 96 dimensions has no SIMT fallback: the failed rows
    # are screened again with 3xTF32 operands and come out right
    nw, dw_, kw = 20000, 96, 16
    wide = api.gen_points(api.GEN_3LEVEL, nw, dw_, 0, 0.125, 7)
    dw = api.to_device_points(wide)
    ids2, d22, st2 = ctx.knn_wide(dw, dw, nw, nw, dw_, kw, True, want_stats=True)
    ctx.sync()
    assert st2["rows_recomputed_exactly"] == 0 and st2["rows_screened_3xtf32"] > 0
    assert st2["rows_nonpositive_margin"] == 0
    rows = torch.from_numpy(np.random.default_rng(1).choice(nw, 256, replace=False)).cuda()
    p = dw[:, :dw_].double()
    q = p[rows]
    dd = ((q[:, None, :] - p[None, :, :]) ** 2).sum(-1)
    dd[torch.arange(256), rows] = float("inf")
    want_d2, want_ids = torch.sort(dd, dim=1, stable=True)
    assert (ids2[rows].long() == want_ids[:, :kw]).float().mean().item() > 0.995
    assert torch.allclose(d22[rows].double(), want_d2[:, :kw], rtol=1e-4)
    ids3, _ = ctx.knn_wide(dw, dw, nw, nw, dw_, kw, True)     # no stats array: must succeed too
    ctx.sync()
    assert torch.equal(ids3, ids2)


def test_knn_entry_point_forwards_wide_points(ctx, oracle):
    """knnx_knn_dev with dim > 64 is served by the tensor-core builder."""
    from paper_1709_03671_b200 import api
    n, dim, k = 900, 96, 8
    pts = api.gen_points(api.GEN_ANISO, n, dim, (4 << 16) | 4, 1.0, 31)
    dp = api.to_device_points(pts)
    ids, d2 = ctx.knn(dp, dp, n, n, dim, k, True)
    ctx.sync()
    p64 = pts.astype(np.float64)
    want_ids, want_d2 = oracle.build_knn(p64, p64, k, True)
    assert np.mean(ids.cpu().numpy() == want_ids.reshape(n, k)) > 0.999
    assert np.allclose(d2.cpu().numpy(), want_d2.reshape(n, k), rtol=1e-4)


def test_wide_knn_argument_errors(ctx):
    from paper_1709_03671_b200 import api
    from paper_1709_03671_b200._lib import KnnxError
    pts = api.gen_points(api.GEN_ANISO, 64, 96, (2 << 16) | 2, 1.0, 1)
    dp = api.to_device_points(pts)
    with pytest.raises(KnnxError):
        ctx.knn_wide(dp, dp, 64, 64, 96, 64, True)      # k > n - 1
    big = api.to_device_points(api.gen_points(api.GEN_ANISO, 400, 96, (2 << 16) | 2, 1.0, 1))
    with pytest.raises(KnnxError):
        ctx.knn_wide(big, big, 400, 400, 96, 300, False)  # k > 256
