"""GPU kernels through the C ABI against the reference-generated golden vectors
(tests/golden/golden_small.npz), fp32 tolerance 1e-5 scale-aware."""
import os

import numpy as np
import pytest

from oracle.oracle import scale_rel

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_small.npz"))
TOL = 1e-5


def _op(ctx, rp, cols, vals, order):
    from paper_1709_03671_b200 import api
    n = rp.size - 1
    return api.Operator.from_csr(ctx, n, n, rp, cols, vals, order)


def test_spmv_flat_and_hier(ctx):
    from paper_1709_03671_b200 import api
    op = _op(ctx, G["row_ptr"], G["cols"], G["vals"].astype(np.float32), api.ORIGINAL)
    assert scale_rel(op.spmv_host(G["x"].astype(np.float32)), G["y_flat"]) <= TOL
    n = G["x"].size
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, G["hier_rows"] + 1, 1)
    rp = np.cumsum(rp)
    for tile_rows in (32, 128, 256):
        op = api.Operator.from_csr(ctx, n, n, rp, G["hier_cols"], G["hier_vals"].astype(np.float32),
                                   api.CLUSTER, tile_rows)
        assert scale_rel(op.spmv_host(G["x_cluster"].astype(np.float32)), G["y_hier"]) <= TOL


def test_hbm1_loader(ctx):
    """A HierBlockMatrix dumped by the reference (dump_hbm1) loads straight
    into a device operator: same y as the reference's spmv_hier."""
    from paper_1709_03671_b200 import api
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_small.hbm1")
    op, rf, cf = api.Operator.from_hbm1(ctx, path)
    assert np.array_equal(rf, G["hier_forward"]) and np.array_equal(cf, G["hier_forward"])
    assert op.info["nnz"] == G["cols"].size
    assert scale_rel(op.spmv_host(G["x_cluster"].astype(np.float32)), G["y_hier"]) <= TOL


def test_gaussian_update_and_recompute(ctx):
    import torch

    from paper_1709_03671_b200 import api
    n = G["x"].size
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, G["hier_rows"] + 1, 1)
    rp = np.cumsum(rp)
    op = api.Operator.from_csr(ctx, n, n, rp, G["hier_cols"], None, api.CLUSTER)
    pc = api.to_device_points(G["points_cluster"].astype(np.float32))
    h = float(G["h"])
    for kappa in range(2):
        x = torch.from_numpy(G["iterate_xs"][kappa].astype(np.float32)).cuda()
        y = torch.empty(n, device="cuda")
        op.gauss_spmv(pc, pc, G["points"].shape[1], h, x, y)
        ctx.sync()
        assert scale_rel(y.cpu().numpy(), G["iterate_ys"][kappa]) <= TOL
    op.update_gaussian(pc, pc, G["points"].shape[1], h)
    ctx.sync()
    assert scale_rel(op.get_values(), G["hier_vals"]) <= TOL


def test_meanshift(ctx):
    from paper_1709_03671_b200 import api
    n, k = G["knn_ids"].shape
    cols = np.sort(G["knn_ids"], axis=1).ravel()
    op = api.Operator.from_csr(ctx, n, n, np.arange(n + 1) * k, cols, None, api.ORIGINAL)
    got = op.meanshift_host(G["ms_targets"].astype(np.float32), G["points"].astype(np.float32),
                            float(G["h"]))
    assert scale_rel(got, G["ms_out"]) <= TOL


def test_tsne(ctx):
    from paper_1709_03671_b200 import api
    op = _op(ctx, G["tsne_row_ptr"], G["tsne_cols"], G["tsne_p"].astype(np.float32), api.CLUSTER)
    f = op.tsne_host(G["tsne_y"].astype(np.float32), store=True)
    # golden inputs are fp32-representable (make_golden.py): same gate as every other output
    assert scale_rel(f, G["tsne_f"]) <= TOL
    assert scale_rel(op.get_values(), G["tsne_a"]) <= TOL
