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
