"""Pinning the CPU oracle (oracle/knn_oracle.c) -- no GPU.

1. Known-answer tests restated from the reference's own unit tests
   (proj/tests/test_kernels.cpp, test_knn.cpp, test_orderings.cpp, test_core.cpp).
2. Bitwise agreement with the reference library itself (oracle/_ref, built
   from /root/reference by oracle/Makefile) on seeded random inputs.
"""
import numpy as np
import pytest

from oracle.oracle import OracleError, Ref, RefHier

# ---------------------------------------------------------------------------
# 1. hand-value KATs


def csr(n_rows, entries):
    """canonical CSR from (i, j, v) triples"""
    entries = sorted(entries)
    row_ptr = np.zeros(n_rows + 1, np.int64)
    for i, _, _ in entries:
        row_ptr[i + 1] += 1
    row_ptr = np.cumsum(row_ptr)
    cols = np.array([j for _, j, _ in entries], np.int32)
    vals = np.array([v for _, _, v in entries], np.float64)
    return row_ptr, cols, vals


def test_spmv_identity(oracle):  # test_kernels.cpp:65-71
    rp, c, v = csr(3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    x = np.array([0.5, -2.0, 7.25])
    assert np.array_equal(oracle.spmv(rp, c, v, x), x)


def test_spmv_2x2(oracle):  # test_kernels.cpp:73-77
    rp, c, v = csr(2, [(0, 0, 1.0), (0, 1, 2.0), (1, 1, 3.0)])
    assert np.array_equal(oracle.spmv(rp, c, v, np.ones(2)), [3.0, 3.0])


def test_spmv_dense_oracle(oracle):  # test_kernels.cpp:79-91
    rng = np.random.default_rng(3)
    dense = np.where(rng.random((64, 64)) < 0.2, rng.random((64, 64)) + 0.1, 0.0)
    ent = [(i, j, dense[i, j]) for i in range(64) for j in range(64) if dense[i, j] != 0]
    rp, c, v = csr(64, ent)
    x = rng.standard_normal(64)
    assert np.max(np.abs(oracle.spmv(rp, c, v, x) - dense @ x)) < 1e-13


def test_tsne_two_points(oracle):  # test_kernels.cpp:179-190
    rp, c, p = csr(2, [(0, 1, 0.5), (1, 0, 0.5)])
    y = np.array([[0.0, 0.0], [1.0, 0.0]])
    f, a = oracle.tsne(rp, c, p, y)
    assert np.array_equal(f, [[-0.25, 0.0], [0.25, 0.0]])
    assert np.array_equal(a, [0.25, 0.25])


def test_tsne_coincident_points(oracle):  # test_kernels.cpp:192-204
    rp, c, p = csr(3, [(0, 1, 0.3), (1, 0, 0.3), (1, 2, 0.2), (2, 1, 0.2)])
    f, a = oracle.tsne(rp, c, p, np.zeros((3, 3)))
    assert np.array_equal(a, p)
    assert np.all(f == 0.0)


def test_meanshift_single_source(oracle):  # test_kernels.cpp:277-285
    out = oracle.meanshift_step(np.array([[0]]), np.array([[10.0, 10.0]]),
                                np.array([[3.0, -1.0]]), 5.0)
    assert np.array_equal(out, [[3.0, -1.0]])


def test_meanshift_symmetric_sources(oracle):  # test_kernels.cpp:287-293
    out = oracle.meanshift_step(np.array([[0, 1]]), np.array([[0.0]]), np.array([[-1.0], [1.0]]), 1.0)
    assert out[0, 0] == 0.0


def test_meanshift_coincident_sources(oracle):  # test_kernels.cpp:295-301
    t = np.array([[0.0, 0.0], [1.0, 5.0], [-2.0, 3.0]])
    out = oracle.meanshift_step(np.tile(np.arange(4), (3, 1)), t, np.full((4, 2), 6.0), 100.0)
    assert np.allclose(out, 6.0, rtol=1e-14)


def test_meanshift_zero_weight(oracle):  # test_kernels.cpp:356-368
    with pytest.raises(OracleError) as e:
        oracle.meanshift_step(np.array([[0]]), np.array([[0.0]]), np.array([[1e6]]), 1.0)
    assert e.value.code == 20 and "target 0" in str(e.value)


def test_iterate_2x2(oracle):  # test_kernels.cpp:433-447 (value_fn (kappa+1)(1+2i+j))
    rp, c, _ = csr(2, [(0, 0, 0.0), (0, 1, 0.0), (1, 0, 0.0), (1, 1, 0.0)])
    rows = np.repeat(np.arange(2), np.diff(rp))
    out = []
    for kappa, x in enumerate([np.array([1.0, 1.0]), np.array([1.0, -1.0])]):
        v = (kappa + 1) * (1 + 2 * rows + c).astype(np.float64)
        out.append(oracle.spmv(rp, c, v, x))
    assert np.array_equal(out[0], [3.0, 7.0])
    assert np.array_equal(out[1], [-2.0, -2.0])


def test_knn_three_points(oracle):  # test_knn.cpp:31-39
    ids, d2 = oracle.build_knn(np.array([[0.0], [1.0], [3.0]]), None, 1, True)
    assert ids[:, 0].tolist() == [1, 0, 1]
    assert d2[0, 0] == 1.0 and d2[2, 0] == 4.0


def test_knn_self_kept_for_distinct_sets(oracle):  # test_knn.cpp:68-74
    p = np.array([[0.0], [5.0]])
    ids, d2 = oracle.build_knn(p, p.copy(), 1, False)
    assert ids[0, 0] == 0 and d2[0, 0] == 0.0


def test_knn_tie_break(oracle):  # test_knn.cpp:76-84
    s = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [0.0, -1.0]])
    ids, _ = oracle.build_knn(np.array([[0.0, 0.0]]), s, 3, False)
    assert ids[0].tolist() == [0, 1, 2]


def test_knn_k_validation(oracle):  # test_knn.cpp:86-94
    p = np.random.default_rng(1).standard_normal((4, 2))
    with pytest.raises(OracleError):
        oracle.build_knn(p, None, 4, True)
    with pytest.raises(OracleError):
        oracle.build_knn(p, None, 0, True)
    assert oracle.build_knn(p, p.copy(), 4, False)[0].shape == (4, 4)


def test_tree_1d_split(oracle):  # test_orderings.cpp:199-210
    fwd, _ = oracle.build_tree(np.array([[0.1], [0.9], [0.15], [0.85]]), 1, 12)
    assert fwd.tolist() == [0, 3, 1, 2]


def test_tree_identical_points_chain(oracle):  # test_orderings.cpp:212-227
    fwd, (begin, end, depth, parent, is_leaf) = oracle.build_tree(np.full((5, 2), 3.0), 1, 4)
    assert depth.max() == 4 and begin.size == 5 and is_leaf.sum() == 1


def test_permute_moves_whole_points(oracle):  # test_core.cpp:148-154
    ps = np.array([[0.0, 1.0], [10.0, 11.0], [20.0, 21.0]])
    moved = oracle.permute_rows(ps, np.array([2, 0, 1]))
    assert moved[2, 1] == 1.0 and moved[0, 0] == 10.0 and moved[1, 0] == 20.0


# ---------------------------------------------------------------------------
# 2. bitwise vs the reference library itself


@pytest.mark.parametrize("seed", [0, 1, 7, 42, 2**63 + 5])
def test_rng_streams_bitwise(oracle, ref, seed):
    assert np.array_equal(oracle.rng_u64(seed, 2000), ref.rng_u64(seed, 2000))
    assert np.array_equal(oracle.rng_uniform01(seed, 2000), ref.rng_uniform01(seed, 2000))
    assert np.array_equal(oracle.rng_normal(seed, 2001), ref.rng_normal(seed, 2001))
    assert np.array_equal(oracle.order_scattered(999, seed), ref.order_scattered(999, seed))


def _random_problem(seed, n=300, dim=5, k=7):
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, dim)) * 3
    return pts, k


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_knn_and_operators_bitwise(oracle, ref, seed):
    pts, k = _random_problem(seed)
    ids_r, d2_r = ref.build_knn(pts, None, k, True)
    ids_o, d2_o = oracle.build_knn(pts, None, k, True)
    assert np.array_equal(ids_r, ids_o) and np.array_equal(d2_r, d2_o)
    n = pts.shape[0]
    order = np.argsort(ids_r, axis=1, kind="stable")
    cols = np.take_along_axis(ids_r, order, 1).ravel().astype(np.int32)
    rp = np.arange(n + 1, dtype=np.int64) * k
    h = 1.7
    vals = oracle.gaussian_values(rp, cols, pts, pts, h)
    rows = np.repeat(np.arange(n, dtype=np.int32), k)
    import ctypes as C
    want = np.empty(cols.size)
    from oracle.oracle import _p
    ref._ok(ref.lib.ref_gaussian_values(n, n, cols.size, _p(rows), _p(cols), _p(pts), _p(pts), 5, h,
                                        _p(want)))
    assert np.array_equal(vals, want)
    x = np.random.default_rng(seed + 9).random(n)
    assert np.array_equal(oracle.spmv(rp, cols, vals, x), ref.spmv_flat(n, rp, cols, vals, x))
    # meanshift over the reference's neighbor rows (kNN order, self excluded here)
    t = pts + 0.1
    got = oracle.meanshift_step(ids_r, t, pts, h)
    assert np.array_equal(got, ref.meanshift_step(pts, t, ids_r, h))


def test_hier_equals_flat_oracle(oracle, ref):
    """spmv_hier on the reference's blocked storage == canonical-order oracle."""
    pts, k = _random_problem(5, n=500, dim=3, k=6)
    ids, _ = ref.build_knn(pts, None, k, True)
    n = pts.shape[0]
    cols = np.sort(ids, axis=1).ravel().astype(np.int32)
    rp = np.arange(n + 1, dtype=np.int64) * k
    vals = np.random.default_rng(2).random(cols.size)
    for cut in (0, 1, 2, -1):
        h, fwd = RefHier.from_original(ref, rp, cols, vals, pts, 16, 12, cut)
        r, c, v = h.flatten()
        rpp = np.zeros(n + 1, np.int64)
        np.add.at(rpp, r + 1, 1)
        rpp = np.cumsum(rpp)
        x = np.random.default_rng(cut + 10).random(n)
        # same per-row accumulation order: bitwise
        assert np.array_equal(h.spmv(x), oracle.spmv(rpp, c, v, x))


def test_tsne_matches_reference(oracle, ref):
    rng = np.random.default_rng(4)
    n = 64
    ent = {}
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < 0.2:
                p = 0.1 + 0.9 * rng.random()
                ent[(i, j)] = p
                ent[(j, i)] = p
    rp, c, p = csr(n, [(i, j, v) for (i, j), v in ent.items()])
    y = rng.random((n, 2))
    h = RefHier.flat(ref, n, n, rp, c, p)
    f_ref = h.tsne(y)
    f_orc, _ = oracle.tsne(rp, c, p, y)
    assert np.array_equal(f_ref, f_orc)
    f_dir = oracle.tsne(rp, c, p, y, direct=True)
    assert np.max(np.abs(f_dir - f_ref)) < 1e-12  # acceptance.cpp:573-590 oracle


def test_tree_matches_reference(oracle, ref):
    rng = np.random.default_rng(11)
    for dim in (1, 2, 3):
        pts = rng.standard_normal((2000, dim))
        fwd_r, arrs, _ = ref.build_tree(pts, 16, 12)
        fwd_o, oarrs = oracle.build_tree(pts, 16, 12)
        assert np.array_equal(fwd_r, fwd_o)
        for a, b in zip(arrs[:5], oarrs):
            assert np.array_equal(a, b)


def test_oracle_generators_match_product(oracle):
    """The oracle's restatement of the BASELINE workload generators (used by
    the reference arm of bench.py, which never loads libknnx.so) is bitwise
    the product's knnx_gen_points / knnx_gen_uniform01."""
    from paper_1709_03671_b200 import api
    assert np.array_equal(oracle.gen_mixture_3level(3000, 49, 0.125, 0),
                          api.gen_points(api.GEN_3LEVEL, 3000, 49, 0, 0.125, 0))
    assert np.array_equal(oracle.gen_mixture_c1(3000, 50, 256, 1.0, 5),
                          api.gen_points(api.GEN_C1_MIXTURE, 3000, 50, 256, 1.0, 5))
    # two 8192-point blocks of the anisotropic mixture (per-block substreams)
    assert np.array_equal(oracle.gen_mixture_aniso(8192 + 100, 64, 4, 4, 3),
                          api.gen_points(api.GEN_ANISO, 8192 + 100, 64, (4 << 16) | 4, 1.0, 3))
    assert np.array_equal(oracle.gen_uniform01(5000, 1), api.gen_uniform01(5000, 1))


def test_refbench_knn_matches_reference_build_knn(ref):
    """The reference arm's exact kNN tool (cKDTree, all host threads) gives
    the reference build_knn's rows exactly (ascending distance, self excluded)."""
    from oracle import refbench
    from oracle.oracle import Oracle
    pts = Oracle().gen_mixture_3level(2500, 49, 0.125, 7).astype(np.float64)
    ids, d2 = refbench.knn_cpu(pts, 30, True)
    want_ids, want_d2 = ref.build_knn(pts, pts, 30, True)
    assert np.array_equal(ids, want_ids.reshape(ids.shape))
    assert np.allclose(d2, want_d2.reshape(d2.shape), rtol=1e-12, atol=1e-12)
    # mean-shift semantics (self included) on a query subset
    q = np.arange(0, 2500, 7)
    ids_q, _ = refbench.knn_cpu(pts, 30, False, queries=q)
    want_q, _ = ref.build_knn(pts[q], pts, 30, False)
    assert np.array_equal(ids_q, want_q.reshape(ids_q.shape))
