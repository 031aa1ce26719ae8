"""Golden vectors produced by the reference library itself
(tests/golden/make_golden.py) pin the C oracle and the product's host code
without needing /root/reference at test time."""
import os

import numpy as np
import pytest

from oracle.oracle import scale_rel
from paper_1709_03671_b200 import api

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_small.npz"))


@pytest.mark.parametrize("seed", [0, 1, 42])
def test_rng_streams(oracle, seed):
    assert np.array_equal(oracle.rng_u64(seed, 64), G[f"rng_u64_{seed}"])
    assert np.array_equal(oracle.rng_uniform01(seed, 64), G[f"rng_uniform01_{seed}"])
    assert np.array_equal(oracle.rng_normal(seed, 65), G[f"rng_normal_{seed}"])
    assert np.array_equal(oracle.order_scattered(300, seed), G[f"order_scattered_{seed}"])
    assert np.array_equal(api.rng_u64(seed, 64), G[f"rng_u64_{seed}"])
    assert np.array_equal(api.rng_normal(seed, 65), G[f"rng_normal_{seed}"])
    assert np.array_equal(api.order_scattered(300, seed), G[f"order_scattered_{seed}"])


def test_knn(oracle):
    ids, d2 = oracle.build_knn(G["points"], None, G["knn_ids"].shape[1], True)
    assert np.array_equal(ids, G["knn_ids"]) and np.array_equal(d2, G["knn_d2"])


@pytest.mark.parametrize("scheme", ["tree2", "tree3"])
def test_ordering(scheme):
    t = api.order_tree(G["points"], int(scheme[-1]))
    assert np.array_equal(t.forward, G[f"forward_{scheme}"])
    assert t.captured_ratio == float(G[f"ratio_{scheme}"])


def test_pca():
    p = api.fit_pca(G["points"], 3)
    assert p["iterations"] == int(G["pca_iterations"])
    assert np.array_equal(p["axes"], G["pca_axes"])
    assert np.array_equal(p["projected"], G["pca_projected"])


def test_gaussian_spmv_meanshift(oracle):
    rp, cols, h = G["row_ptr"], G["cols"], float(G["h"])
    vals = oracle.gaussian_values(rp, cols, G["points"], G["points"], h)
    assert np.array_equal(vals, G["vals"])
    assert np.array_equal(oracle.spmv(rp, cols, vals, G["x"]), G["y_flat"])
    ms = oracle.meanshift_step(G["knn_ids"], G["ms_targets"], G["points"], h)
    assert np.array_equal(ms, G["ms_out"])


def test_cluster_order(oracle):
    """Blocked operator in tree order == canonical-order oracle, bitwise."""
    n = G["x"].size
    fwd = G["hier_forward"]
    assert np.array_equal(api.build_tree(G["pca_projected"], 32, 12).forward, fwd)
    r, c, v = G["hier_rows"], G["hier_cols"], G["hier_vals"]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    assert np.array_equal(oracle.spmv(rp, c, v, G["x_cluster"]), G["y_hier"])
    # the product's host permute reproduces the reference's permuted matrix
    a = api.HostCsr.from_arrays(n, n, G["row_ptr"], G["cols"], G["vals"].astype(np.float32))
    rp2, c2, v2 = a.permute(fwd).export()
    assert np.array_equal(rp2, rp) and np.array_equal(c2, c)
    assert np.array_equal(v2, v.astype(np.float32))
    pc = oracle.permute_rows(G["points"], fwd)
    assert np.array_equal(pc, G["points_cluster"])
    for kappa in range(2):
        y = oracle.gauss_spmv(rp, c, pc, pc, float(G["h"]), G["iterate_xs"][kappa])
        assert np.max(np.abs(y - G["iterate_ys"][kappa])) <= 1e-12 * np.max(np.abs(y))


def test_hbm1_header_and_leaf_orders():
    """The reference's own HBM1 dump (tests/golden/golden_small.hbm1) parses
    to the same shape, cut level and leaf order as the reference matrix."""
    import ctypes as C

    from paper_1709_03671_b200._lib import check, lib
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_small.hbm1").encode()
    m, n, nnz, cut = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
    check(lib.knnx_hbm1_info(path, C.byref(m), C.byref(n), C.byref(nnz), C.byref(cut)))
    assert (m.value, n.value, nnz.value) == (G["x"].size, G["x"].size, G["cols"].size)
    assert cut.value == int(G["hier_cut_level"])
    from paper_1709_03671_b200._lib import KnnxError
    with pytest.raises(KnnxError) as e:
        check(lib.knnx_hbm1_info(__file__.encode(), C.byref(m), C.byref(n), C.byref(nnz),
                                 C.byref(cut)))
    assert e.value.name == "MalformedRecord"


def test_tsne(oracle):
    f, a = oracle.tsne(G["tsne_row_ptr"], G["tsne_cols"], G["tsne_p"], G["tsne_y"])
    assert np.array_equal(f, G["tsne_f"])
    assert np.array_equal(a, G["tsne_a"])
    fd = oracle.tsne(G["tsne_row_ptr"], G["tsne_cols"], G["tsne_p"], G["tsne_y"], direct=True)
    assert scale_rel(fd, G["tsne_f"]) < 1e-9
