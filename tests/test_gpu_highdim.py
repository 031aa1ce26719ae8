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
