"""Host-side product code (libknnx.so host half) vs the reference -- no GPU.

Ordering must be bit-exact (BASELINE north_star): Rng streams, PCA axes and
projections, partition tree, level blocking, make_ordering('tree2/3'); the
format conversions (permute, symmetrize, kNN rows) must reproduce the
reference's canonical matrices exactly.  Also checks the library exports
every symbol the C headers declare.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1709_03671_b200 import api
from paper_1709_03671_b200._lib import KnnxError, LIB_PATH

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB_PATH)
    names = []
    for hdr in ("knnx.h", "knnx_host.h"):
        text = open(os.path.join(REPO, "include", hdr)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"^\s*(?:[\w\*]+\s+)+\**(knnx_\w+)\s*\(", text, flags=re.M)
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.parametrize("seed", [0, 1, 42, 2**64 - 1])
def test_rng_bitwise(ref, seed):
    assert np.array_equal(api.rng_u64(seed, 3000), ref.rng_u64(seed, 3000))
    assert np.array_equal(api.rng_uniform01(seed, 3000), ref.rng_uniform01(seed, 3000))
    assert np.array_equal(api.rng_normal(seed, 3001), ref.rng_normal(seed, 3001))
    assert np.array_equal(api.order_scattered(1234, seed), ref.order_scattered(1234, seed))


def test_gen_mixture_uses_the_reference_stream(ref):
    """C1 generator = reference Rng draws (centers U[0,1]*20-10, then normals)."""
    pts = api.gen_points(api.GEN_C1_MIXTURE, 200, 5, 8, 1.0, 3)
    u = ref.rng_uniform01(3, 40)
    centers = -10.0 + 20.0 * u.reshape(8, 5)
    assert np.allclose(pts[:8], centers, atol=6)  # one sigma-1 draw away
    assert np.array_equal(pts, api.gen_points(api.GEN_C1_MIXTURE, 200, 5, 8, 1.0, 3))


@pytest.mark.parametrize("n,dim,d", [(1500, 49, 3), (800, 12, 2), (600, 7, 3)])
def test_pca_bitwise(ref, n, dim, d):
    pts = api.gen_points(api.GEN_C1_MIXTURE, n, dim, 16, 1.0, n).astype(np.float64)
    a = ref.fit_pca(pts, d)
    b = api.fit_pca(pts, d)
    assert a["iterations"] == b["iterations"]
    assert np.array_equal(a["mean"], b["mean"])
    assert np.array_equal(a["axes"], b["axes"])
    assert np.array_equal(a["singular_values"], b["singular_values"])
    assert np.array_equal(a["projected"], b["projected"])


def test_pca_exact_case(ref):  # d == dim: axis-aligned (pca.cpp:160-180)
    pts = np.random.default_rng(1).standard_normal((100, 3)) * [1.0, 3.0, 2.0]
    a = ref.fit_pca(pts, 3)
    b = api.fit_pca(pts, 3)
    assert np.array_equal(a["axes"], b["axes"])


@pytest.mark.parametrize("scheme,gen", [("tree3", 1), ("tree2", 1), ("tree3", 2)])
def test_make_ordering_bitwise(ref, scheme, gen):
    n = 3000
    pts = api.gen_points(gen, n, 49, 64, 1.0 if gen == 1 else 0.125, 0).astype(np.float64)
    fwd_ref, ratio_ref = ref.make_ordering(scheme, pts)
    tree = api.order_tree(pts, int(scheme[-1]))
    assert np.array_equal(fwd_ref, tree.forward)
    assert tree.captured_ratio == ratio_ref


@pytest.mark.parametrize("dim,cap,depth", [(1, 1, 12), (2, 8, 6), (3, 16, 12), (3, 128, 12)])
def test_tree_and_level_blocking(ref, dim, cap, depth):
    emb = np.random.default_rng(dim * 7 + cap).standard_normal((2500, dim))
    fwd_r, arrs, blocks = ref.build_tree(emb, cap, depth)
    t = api.build_tree(emb, cap, depth)
    assert np.array_equal(fwd_r, t.forward)
    for a, b in zip(arrs[:5], [t.begin, t.end, t.depth, t.parent, t.is_leaf]):
        assert np.array_equal(a, b)
    for lvl, off in blocks.items():
        assert np.array_equal(off, t.level_blocking(lvl))
    with pytest.raises(KnnxError):
        t.level_blocking(t.max_depth + 1)


def test_tree_rejects_bad_dim():
    with pytest.raises(KnnxError) as e:
        api.build_tree(np.zeros((4, 4)))
    assert e.value.name == "DimTooHigh"


def _knn_csr(ref, n=400, dim=6, k=8, seed=0):
    pts = np.random.default_rng(seed).standard_normal((n, dim))
    ids, _ = ref.build_knn(pts, None, k, True)
    return pts, ids


def test_csr_from_knn_and_permute_match_reference(ref):
    pts, ids = _knn_csr(ref)
    n, k = ids.shape
    a = api.HostCsr.from_knn(ids, n)
    rp, cols, _ = a.export()
    assert np.array_equal(rp, np.arange(n + 1) * k)
    assert np.array_equal(cols.reshape(n, k), np.sort(ids, axis=1))
    vals = np.random.default_rng(1).random(cols.size).astype(np.float32)
    a.set_values(vals)
    fwd = api.order_scattered(n, 5)
    orow, ocol, oval = ref.permute_matrix(rp, cols, vals.astype(np.float64), fwd)
    rp2, c2, v2 = a.permute(fwd).export()
    rows2 = np.repeat(np.arange(n), np.diff(rp2))
    assert np.array_equal(rows2, orow) and np.array_equal(c2, ocol)
    assert np.array_equal(v2.astype(np.float64), oval)


def test_symmetrize_matches_reference(ref):
    _, ids = _knn_csr(ref, seed=3)
    n = ids.shape[0]
    a = api.HostCsr.from_knn(ids, n)
    rp, cols, _ = a.export()
    orow, ocol = ref.symmetrize(rp, cols)
    rp2, c2, _ = a.symmetrize().export()
    assert np.array_equal(np.repeat(np.arange(n), np.diff(rp2)), orow)
    assert np.array_equal(c2, ocol)


def test_row_block_shards_reassemble(ref):
    _, ids = _knn_csr(ref, seed=4)
    n = ids.shape[0]
    a = api.HostCsr.from_knn(ids, n)
    rp, cols, _ = a.export()
    parts = [a.row_block(0, 130), a.row_block(130, 131), a.row_block(131, n)]
    got = np.concatenate([p.export()[1] for p in parts])
    assert np.array_equal(got, cols)
    assert parts[1].shape[:3] == (1, n, rp[131] - rp[130])


def test_csr_validation():
    with pytest.raises(KnnxError) as e:
        api.HostCsr.from_arrays(2, 2, [0, 2, 2], [1, 0])
    assert e.value.name == "DuplicateEntry"
    with pytest.raises(KnnxError) as e:
        api.HostCsr.from_arrays(2, 2, [0, 1, 1], [5])
    assert e.value.name == "OutOfBounds"
    with pytest.raises(KnnxError) as e:
        api.HostCsr.from_knn(np.array([[0, 0]], np.int32), 3)
    assert e.value.name == "OutOfBounds"


def test_median_distance():
    d2 = np.array([1.0, 4.0, 9.0, 16.0], np.float32)
    assert api.median_distance(d2) == 2.5
    assert api.median_distance(np.array([4.0, 1.0, 9.0], np.float32)) == 2.0


def test_symmetrize_values_and_row_normalize(ref):
    """t-SNE joint affinities: P = (P_cond + P_cond^T) / 2N, sums to 1."""
    _, ids = _knn_csr(ref, n=300, seed=9)
    n = ids.shape[0]
    a = api.HostCsr.from_knn(ids, n)
    rp, cols, _ = a.export()
    vals = np.random.default_rng(2).random(cols.size).astype(np.float32) + 0.1
    a.set_values(vals)
    a.row_normalize()
    _, _, pc = a.export()
    dense = np.zeros((n, n))
    for i in range(n):
        dense[i, cols[rp[i]:rp[i + 1]]] = vals[rp[i]:rp[i + 1]].astype(np.float64)
    dense /= dense.sum(1, keepdims=True)
    assert np.allclose(pc, dense[np.repeat(np.arange(n), np.diff(rp)), cols], rtol=1e-6)
    p = a.symmetrize_values(1.0 / (2 * n))
    srp, scol, sv = p.export()
    want = (dense + dense.T) / (2 * n)
    assert np.allclose(sv, want[np.repeat(np.arange(n), np.diff(srp)), scol], rtol=1e-6)
    assert abs(float(sv.astype(np.float64).sum()) - 1.0) < 1e-5
    orow, ocol = ref.symmetrize(rp, cols)
    assert np.array_equal(scol, ocol)


def test_locality_schedule_groups_components():
    """Two interleaved disjoint neighbourhoods (even / odd rows) are laid out
    one after the other; the schedule is a permutation; col_base shifts ids."""
    from paper_1709_03671_b200 import api
    n, k = 64, 4
    ids = np.array([[(i + 2 * (q + 1)) % n for q in range(k)] for i in range(n)], np.int32)
    csr = api.HostCsr.from_knn(ids, n)
    s = csr.locality_schedule()
    assert np.array_equal(np.sort(s), np.arange(n))
    assert np.all(s[: n // 2] % 2 == 0) and np.all(s[n // 2:] % 2 == 1)
    # row block shard: columns outside [col_base, col_base + m) are not followed
    blk = csr.row_block(16, 48)
    s2 = blk.locality_schedule(16)
    assert np.array_equal(np.sort(s2), np.arange(32))
