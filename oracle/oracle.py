"""TEST INFRASTRUCTURE ONLY -- numpy wrappers of the CPU oracles.

* ``Oracle``: the plain-C restatement oracle/knn_oracle.c (always built).
* ``Ref``: the reference library itself, compiled from /root/reference by
  oracle/Makefile into oracle/_ref/libpatchord_ref.so (present when it was
  built here; the file travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  The product (paper_1709_03671_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_oracle", "libknn_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpatchord_ref.so")

vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code} {msg}")
        self.code = code


def _csr_arrays(row_ptr, cols):
    return np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(cols, np.int32)


class Oracle:
    """Double-precision restatement (oracle/knn_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        self.lib = C.CDLL(ORACLE_SO)
        L = self.lib
        for name, args in {
            "orc_rng_u64": [u64, i64, vp], "orc_rng_uniform01_stream": [u64, i64, vp],
            "orc_rng_normal_stream": [u64, i64, vp], "orc_order_scattered": [i32, u64, vp],
            "orc_spmv_csr": [i32, vp, vp, vp, vp, vp],
            "orc_gaussian_values": [i32, vp, vp, vp, vp, i32, f64, vp],
            "orc_gauss_spmv": [i32, vp, vp, vp, vp, i32, f64, vp, vp],
            "orc_meanshift_step": [i32, i32, vp, vp, vp, i32, f64, vp, vp],
            "orc_tsne_attractive": [i32, vp, vp, vp, vp, i32, vp, vp],
            "orc_tsne_direct": [i32, vp, vp, vp, vp, i32, vp],
            "orc_permute_rows": [i32, i64, vp, vp, vp],
            "orc_build_knn": [vp, i32, vp, i32, i32, i32, C.c_int, vp, vp],
            "orc_build_tree": [vp, i32, i32, i32, i32, vp, i32, vp, vp, vp, vp, vp, vp],
            "orc_gen_mixture_c1": [i32, i32, i32, f64, u64, vp],
            "orc_gen_mixture_3level": [i32, i32, f64, u64, vp],
            "orc_gen_uniform01_f32": [i64, u64, vp],
            "orc_gen_mixture_aniso": [i32, i32, i32, i32, u64, vp],
        }.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = None if name in ("orc_rng_u64", "orc_rng_uniform01_stream",
                                          "orc_rng_normal_stream", "orc_order_scattered",
                                          "orc_permute_rows", "orc_gen_uniform01_f32") else C.c_int

    @staticmethod
    def _ok(rc):
        if rc != 0:
            raise OracleError(rc)

    def rng_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.orc_rng_u64(seed, n, _p(out))
        return out

    def rng_uniform01(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.orc_rng_uniform01_stream(seed, n, _p(out))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.orc_rng_normal_stream(seed, n, _p(out))
        return out

    def order_scattered(self, n, seed):
        out = np.empty(n, np.int32)
        self.lib.orc_order_scattered(n, seed, _p(out))
        return out

    # BASELINE workload generators (the reference arm's inputs)
    def gen_mixture_c1(self, n, dim, n_clusters, sigma, seed):
        out = np.empty((n, dim), np.float32)
        self._ok(self.lib.orc_gen_mixture_c1(n, dim, n_clusters, sigma, seed, _p(out)))
        return out

    def gen_mixture_3level(self, n, dim, noise, seed):
        out = np.empty((n, dim), np.float32)
        self._ok(self.lib.orc_gen_mixture_3level(n, dim, noise, seed, _p(out)))
        return out

    def gen_mixture_aniso(self, n, dim, n_top, n_sub, seed):
        out = np.empty((n, dim), np.float32)
        self._ok(self.lib.orc_gen_mixture_aniso(n, dim, n_top, n_sub, seed, _p(out)))
        return out

    def gen_uniform01(self, n, seed):
        out = np.empty(n, np.float32)
        self.lib.orc_gen_uniform01_f32(n, seed, _p(out))
        return out

    def spmv(self, row_ptr, cols, vals, x):
        row_ptr, cols = _csr_arrays(row_ptr, cols)
        vals = np.ascontiguousarray(vals, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(row_ptr.size - 1)
        self._ok(self.lib.orc_spmv_csr(row_ptr.size - 1, _p(row_ptr), _p(cols), _p(vals), _p(x), _p(y)))
        return y

    def gaussian_values(self, row_ptr, cols, t, s, h):
        row_ptr, cols = _csr_arrays(row_ptr, cols)
        t = np.ascontiguousarray(t, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        out = np.empty(cols.size)
        self._ok(self.lib.orc_gaussian_values(row_ptr.size - 1, _p(row_ptr), _p(cols), _p(t), _p(s),
                                              t.shape[1], h, _p(out)))
        return out

    def gauss_spmv(self, row_ptr, cols, t, s, h, x):
        row_ptr, cols = _csr_arrays(row_ptr, cols)
        t = np.ascontiguousarray(t, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(row_ptr.size - 1)
        self._ok(self.lib.orc_gauss_spmv(row_ptr.size - 1, _p(row_ptr), _p(cols), _p(t), _p(s),
                                         t.shape[1], h, _p(x), _p(y)))
        return y

    def meanshift_step(self, ids, t, s, h):
        ids = np.ascontiguousarray(ids, np.int32)
        t = np.ascontiguousarray(t, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        out = np.empty_like(t)
        bad = C.c_int32(-1)
        rc = self.lib.orc_meanshift_step(t.shape[0], ids.shape[1], _p(ids), _p(t), _p(s), t.shape[1],
                                         h, _p(out), C.byref(bad))
        if rc != 0:
            raise OracleError(rc, f"target {bad.value}")
        return out

    def tsne(self, row_ptr, cols, p, y, direct=False):
        row_ptr, cols = _csr_arrays(row_ptr, cols)
        p = np.ascontiguousarray(p, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        f = np.empty_like(y)
        if direct:
            self._ok(self.lib.orc_tsne_direct(y.shape[0], _p(row_ptr), _p(cols), _p(p), _p(y),
                                              y.shape[1], _p(f)))
            return f
        a = np.empty_like(p)
        self._ok(self.lib.orc_tsne_attractive(y.shape[0], _p(row_ptr), _p(cols), _p(p), _p(y),
                                              y.shape[1], _p(a), _p(f)))
        return f, a

    def tsne_rows(self, row_ptr, cols, p, y, m):
        """Direct attractive force for the first m rows of a square P
        (orc_tsne_direct restricted to rows < m; y holds every point)."""
        row_ptr, cols = _csr_arrays(row_ptr, cols)
        p = np.ascontiguousarray(p, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        f = np.empty((m, y.shape[1]))
        self._ok(self.lib.orc_tsne_direct(m, _p(row_ptr), _p(cols), _p(p), _p(y), y.shape[1],
                                          _p(f)))
        return f

    def permute_rows(self, arr, forward):
        arr = np.ascontiguousarray(arr)
        forward = np.ascontiguousarray(forward, np.int32)
        out = np.empty_like(arr)
        n = arr.shape[0]
        self.lib.orc_permute_rows(n, arr.nbytes // max(n, 1), _p(arr), _p(forward), _p(out))
        return out

    def build_knn(self, t, s, k, self_set):
        t = np.ascontiguousarray(t, np.float64)
        s = t if self_set else np.ascontiguousarray(s, np.float64)
        m = t.shape[0]
        ids = np.empty((m, k), np.int32)
        d2 = np.empty((m, k), np.float64)
        self._ok(self.lib.orc_build_knn(_p(t), m, _p(s), s.shape[0], t.shape[1], k,
                                        1 if self_set else 0, _p(ids), _p(d2)))
        return ids, d2

    def build_tree(self, pts, leaf_capacity=128, max_depth=12):
        pts = np.ascontiguousarray(pts, np.float64)
        n, dim = pts.shape
        cap = 2 * n + 16 * max_depth + 16
        fwd = np.empty(n, np.int32)
        arrs = [np.empty(cap, np.int32) for _ in range(5)]
        nn = C.c_int32()
        self._ok(self.lib.orc_build_tree(_p(pts), n, dim, leaf_capacity, max_depth, _p(fwd), cap,
                                         C.byref(nn), *[_p(a) for a in arrs]))
        return fwd, [a[:nn.value] for a in arrs]


class Ref:
    """The reference library itself (oracle/_ref/libpatchord_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        sig = {
            "ref_rng_u64": [u64, i64, vp], "ref_rng_uniform01": [u64, i64, vp],
            "ref_rng_normal": [u64, i64, vp], "ref_rng_bounded": [u64, u64, i64, vp],
            "ref_order_scattered": [i32, u64, vp],
            "ref_gen_gaussian_mixture": [i32, i32, i32, f64, f64, u64, vp],
            "ref_build_knn": [vp, i32, vp, i32, i32, i32, C.c_int, vp, vp],
            "ref_gaussian_values": [i32, i32, i64, vp, vp, vp, vp, i32, f64, vp],
            "ref_spmv_flat": [i32, i32, i64, vp, vp, vp, vp, vp],
            "ref_bench_spmv_flat": [i32, i32, i64, vp, vp, vp, vp, i32, vp, vp],
            "ref_make_ordering": [C.c_char_p, i32, i32, vp, i32, i32, u64, vp, vp],
            "ref_fit_pca": [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp],
            "ref_tree_create": [vp, i32, i32, i32, i32, C.POINTER(vp)],
            "ref_tree_nodes": [vp, vp, vp, vp, vp, vp, vp, vp],
            "ref_tree_forward": [vp, vp],
            "ref_tree_level_blocking": [vp, i32, vp, vp],
            "ref_permute_points": [vp, i32, i32, vp, vp],
            "ref_permute_matrix": [i32, i64, vp, vp, vp, vp, vp, vp, vp],
            "ref_symmetrize": [i32, i64, vp, vp, vp, vp, vp],
            "ref_hier_create": [i32, i64, vp, vp, vp, vp, i32, i32, i32, i32, vp, C.POINTER(vp)],
            "ref_hier_create_flat": [i32, i32, i64, vp, vp, vp, C.POINTER(vp)],
            "ref_hier_info": [vp, vp, vp, vp, vp, vp],
            "ref_hier_flatten": [vp, vp, vp, vp],
            "ref_hier_spmv": [vp, vp, vp, i32],
            "ref_hier_bench": [vp, vp, i32, i32, vp, vp],
            "ref_hier_update_gaussian": [vp, vp, vp, i32, f64, vp],
            "ref_hier_iterate_gaussian": [vp, vp, vp, i32, f64, i32, vp, vp, vp],
            "ref_hier_tsne": [vp, vp, i32, vp],
            "ref_meanshift_step": [vp, i32, vp, i32, i32, vp, i32, f64, vp],
            "ref_meanshift_run": [vp, i32, vp, i32, i32, i32, f64, i32, i32, vp, vp],
            "ref_meanshift_bench": [vp, i32, vp, i32, i32, vp, i32, f64, i32, vp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.ref_tree_destroy.argtypes = [vp]
        L.ref_tree_destroy.restype = None
        L.ref_hier_destroy.argtypes = [vp]
        L.ref_hier_destroy.restype = None
        L.ref_tree_n_nodes.argtypes = [vp]
        L.ref_tree_n_nodes.restype = i32
        L.ref_tree_depth.argtypes = [vp]
        L.ref_tree_depth.restype = i32
        L.ref_hardware_threads.restype = i32

    def _ok(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode(errors="replace"))

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def machine_descriptor(self) -> str:
        """The reference's machine_descriptor() (proj/src/pipeline.cpp:75-89)."""
        buf = C.create_string_buffer(512)
        self._ok(self.lib.ref_machine_descriptor(buf, 512))
        return buf.value.decode()

    def rng_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self._ok(self.lib.ref_rng_u64(seed, n, _p(out)))
        return out

    def rng_uniform01(self, seed, n):
        out = np.empty(n)
        self._ok(self.lib.ref_rng_uniform01(seed, n, _p(out)))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n)
        self._ok(self.lib.ref_rng_normal(seed, n, _p(out)))
        return out

    def order_scattered(self, n, seed):
        out = np.empty(n, np.int32)
        self._ok(self.lib.ref_order_scattered(n, seed, _p(out)))
        return out

    def build_knn(self, t, s, k, self_set):
        t = np.ascontiguousarray(t, np.float64)
        s = t if self_set else np.ascontiguousarray(s, np.float64)
        ids = np.empty((t.shape[0], k), np.int32)
        d2 = np.empty((t.shape[0], k))
        self._ok(self.lib.ref_build_knn(_p(t), t.shape[0], _p(s), s.shape[0], t.shape[1], k,
                                        1 if self_set else 0, _p(ids), _p(d2)))
        return ids, d2

    @staticmethod
    def _coo(row_ptr, cols):
        row_ptr = np.asarray(row_ptr, np.int64)
        rows = np.repeat(np.arange(row_ptr.size - 1, dtype=np.int32), np.diff(row_ptr))
        return np.ascontiguousarray(rows), np.ascontiguousarray(cols, np.int32)

    def spmv_flat(self, n_cols, row_ptr, cols, vals, x):
        rows, cols = self._coo(row_ptr, cols)
        vals = np.ascontiguousarray(vals, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(len(row_ptr) - 1)
        self._ok(self.lib.ref_spmv_flat(len(row_ptr) - 1, n_cols, cols.size, _p(rows), _p(cols),
                                        _p(vals), _p(x), _p(y)))
        return y

    def bench_spmv_flat(self, n_cols, row_ptr, cols, vals, x, reps):
        rows, cols = self._coo(row_ptr, cols)
        vals = np.ascontiguousarray(vals, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(len(row_ptr) - 1)
        times = np.empty(reps, np.int64)
        self._ok(self.lib.ref_bench_spmv_flat(len(row_ptr) - 1, n_cols, cols.size, _p(rows),
                                              _p(cols), _p(vals), _p(x), reps, _p(times), _p(y)))
        return y, times

    def make_ordering(self, scheme, pts, leaf_capacity=128, max_depth=12, seed=1):
        pts = np.ascontiguousarray(pts, np.float64)
        fwd = np.empty(pts.shape[0], np.int32)
        ratio = C.c_double()
        self._ok(self.lib.ref_make_ordering(scheme.encode(), pts.shape[0], pts.shape[1], _p(pts),
                                            leaf_capacity, max_depth, seed, _p(fwd), C.byref(ratio)))
        return fwd, ratio.value

    def fit_pca(self, pts, d):
        pts = np.ascontiguousarray(pts, np.float64)
        n, dim = pts.shape
        mean, axes, sv, proj = np.empty(dim), np.empty((d, dim)), np.empty(d), np.empty((n, d))
        it, conv = C.c_int32(), C.c_int()
        self._ok(self.lib.ref_fit_pca(_p(pts), n, dim, d, _p(mean), _p(axes), _p(sv), C.byref(it),
                                      C.byref(conv), _p(proj)))
        return dict(mean=mean, axes=axes, singular_values=sv, iterations=it.value,
                    converged=bool(conv.value), projected=proj)

    def build_tree(self, emb, leaf_capacity=128, max_depth=12):
        emb = np.ascontiguousarray(emb, np.float64)
        h = vp()
        self._ok(self.lib.ref_tree_create(_p(emb), emb.shape[0], emb.shape[1], leaf_capacity,
                                          max_depth, C.byref(h)))
        try:
            nn = self.lib.ref_tree_n_nodes(h)
            fwd = np.empty(emb.shape[0], np.int32)
            self._ok(self.lib.ref_tree_forward(h, _p(fwd)))
            arrs = [np.empty(nn, np.int32) for _ in range(5)] + [np.empty(3 * nn), np.empty(3 * nn)]
            self._ok(self.lib.ref_tree_nodes(h, *[_p(a) for a in arrs]))
            depth = self.lib.ref_tree_depth(h)
            blocks = {}
            for lvl in range(depth + 1):
                off = np.empty(nn + 1, np.int32)
                cnt = C.c_int32()
                self._ok(self.lib.ref_tree_level_blocking(h, lvl, _p(off), C.byref(cnt)))
                blocks[lvl] = off[:cnt.value].copy()
            return fwd, arrs, blocks
        finally:
            self.lib.ref_tree_destroy(h)

    def permute_points(self, pts, forward):
        pts = np.ascontiguousarray(pts, np.float64)
        out = np.empty_like(pts)
        self._ok(self.lib.ref_permute_points(_p(pts), pts.shape[0], pts.shape[1],
                                             _p(np.ascontiguousarray(forward, np.int32)), _p(out)))
        return out

    def permute_matrix(self, row_ptr, cols, vals, forward):
        rows, cols = self._coo(row_ptr, cols)
        n = len(row_ptr) - 1
        vals = np.ascontiguousarray(vals, np.float64)
        orow, ocol, oval = np.empty_like(rows), np.empty_like(cols), np.empty_like(vals)
        self._ok(self.lib.ref_permute_matrix(n, cols.size, _p(rows), _p(cols), _p(vals),
                                             _p(np.ascontiguousarray(forward, np.int32)),
                                             _p(orow), _p(ocol), _p(oval)))
        return orow, ocol, oval

    def symmetrize(self, row_ptr, cols):
        rows, cols = self._coo(row_ptr, cols)
        n = len(row_ptr) - 1
        nnz = C.c_int64()
        cap = 2 * cols.size
        orow, ocol = np.empty(cap, np.int32), np.empty(cap, np.int32)
        self._ok(self.lib.ref_symmetrize(n, cols.size, _p(rows), _p(cols), C.byref(nnz), _p(orow),
                                         _p(ocol)))
        return orow[:nnz.value], ocol[:nnz.value]

    def gaussian_values(self, n_cols, row_ptr, cols, t, s, h):
        """gaussian_values (proj/src/knn.cpp:86-108) on a flat pattern."""
        rows, cols = self._coo(row_ptr, cols)
        t = np.ascontiguousarray(t, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        out = np.empty(cols.size)
        self._ok(self.lib.ref_gaussian_values(len(row_ptr) - 1, n_cols, cols.size, _p(rows),
                                              _p(cols), _p(t), _p(s), t.shape[1], h, _p(out)))
        return out

    def meanshift_step(self, sources, targets, ids, h):
        s = np.ascontiguousarray(sources, np.float64)
        t = np.ascontiguousarray(targets, np.float64)
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.empty_like(t)
        self._ok(self.lib.ref_meanshift_step(_p(s), s.shape[0], _p(t), t.shape[0], t.shape[1],
                                             _p(ids), ids.shape[1], h, _p(out)))
        return out


def _ref_bench_meanshift(self, sources, targets, ids, h, reps):
    """Per-call times (ns) of the reference's meanshift_step (copies outside)."""
    s = np.ascontiguousarray(sources, np.float64)
    t = np.ascontiguousarray(targets, np.float64)
    ids = np.ascontiguousarray(ids, np.int32)
    times = np.empty(reps, np.int64)
    self._ok(self.lib.ref_meanshift_bench(_p(s), s.shape[0], _p(t), t.shape[0], t.shape[1],
                                          _p(ids), ids.shape[1], h, reps, _p(times)))
    return times


Ref.bench_meanshift = _ref_bench_meanshift


class RefHier:
    """A reference HierBlockMatrix built by the reference pipeline steps."""

    def __init__(self, ref: Ref, handle, n_rows, n_cols):
        self.ref, self.h, self.n_rows, self.n_cols = ref, handle, n_rows, n_cols

    @classmethod
    def from_original(cls, ref: Ref, row_ptr, cols, vals, emb, leaf_capacity=128, max_depth=12,
                      cut_level=-1):
        rows, cols = Ref._coo(row_ptr, cols)
        n = len(row_ptr) - 1
        vals = np.ascontiguousarray(vals, np.float64)
        emb = np.ascontiguousarray(emb, np.float64)
        fwd = np.empty(n, np.int32)
        h = vp()
        ref._ok(ref.lib.ref_hier_create(n, cols.size, _p(rows), _p(cols), _p(vals), _p(emb),
                                        emb.shape[1], leaf_capacity, max_depth, cut_level, _p(fwd),
                                        C.byref(h)))
        return cls(ref, h, n, n), fwd

    @classmethod
    def flat(cls, ref: Ref, n_rows, n_cols, row_ptr, cols, vals):
        rows, cols = Ref._coo(row_ptr, cols)
        vals = np.ascontiguousarray(vals, np.float64)
        h = vp()
        ref._ok(ref.lib.ref_hier_create_flat(n_rows, n_cols, cols.size, _p(rows), _p(cols), _p(vals),
                                             C.byref(h)))
        return cls(ref, h, n_rows, n_cols)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_hier_destroy(self.h)
            self.h = None

    def info(self):
        cut, nb, nl, nt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        nnz = C.c_int64()
        self.ref._ok(self.ref.lib.ref_hier_info(self.h, C.byref(cut), C.byref(nb), C.byref(nl),
                                                C.byref(nt), C.byref(nnz)))
        return dict(cut_level=cut.value, n_blocks=nb.value, n_leaf_blocks=nl.value,
                    n_top_blocks=nt.value, nnz=nnz.value)

    def dump(self, path):
        self.ref.lib.ref_hier_dump.argtypes = [vp, C.c_char_p]
        self.ref.lib.ref_hier_dump.restype = C.c_int
        self.ref._ok(self.ref.lib.ref_hier_dump(self.h, path.encode()))

    def flatten(self):
        nnz = self.info()["nnz"]
        rows, cols, vals = np.empty(nnz, np.int32), np.empty(nnz, np.int32), np.empty(nnz)
        self.ref._ok(self.ref.lib.ref_hier_flatten(self.h, _p(rows), _p(cols), _p(vals)))
        return rows, cols, vals

    def spmv(self, x, workers=0):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n_rows)
        self.ref._ok(self.ref.lib.ref_hier_spmv(self.h, _p(x), _p(y), workers))
        return y

    def bench(self, x, workers, reps):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n_rows)
        times = np.empty(reps, np.int64)
        self.ref._ok(self.ref.lib.ref_hier_bench(self.h, _p(x), workers, reps, _p(times), _p(y)))
        return y, times

    def update_gaussian(self, t, s, h):
        t = np.ascontiguousarray(t, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        cnt = C.c_int32()
        self.ref._ok(self.ref.lib.ref_hier_update_gaussian(self.h, _p(t), _p(s), t.shape[1], h,
                                                           C.byref(cnt)))
        return cnt.value

    def iterate_gaussian(self, t, s, h, xs):
        t = np.ascontiguousarray(t, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        xs = np.ascontiguousarray(xs, np.float64)
        ys = np.empty((xs.shape[0], self.n_rows))
        times = np.empty(xs.shape[0], np.int64)
        self.ref._ok(self.ref.lib.ref_hier_iterate_gaussian(self.h, _p(t), _p(s), t.shape[1], h,
                                                            xs.shape[0], _p(xs), _p(ys), _p(times)))
        return ys, times

    def tsne(self, y):
        y = np.ascontiguousarray(y, np.float64)
        f = np.empty_like(y)
        self.ref._ok(self.ref.lib.ref_hier_tsne(self.h, _p(y), y.shape[1], _p(f)))
        return f


def scale_rel(g, r) -> float:
    """SURVEY.md §8d parity metric: max|g - r| / max|r| (scale-aware L-inf)."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    den = np.max(np.abs(r)) if r.size else 0.0
    return float(np.max(np.abs(g - r)) / den) if den > 0 else float(np.max(np.abs(g - r), initial=0.0))


def ref_rel(g, r) -> float:
    """The reference's metric |a-b| / max(1,|a|,|b|) (proj/tests/acceptance.cpp:63-71)."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    if g.size == 0:
        return 0.0
    return float(np.max(np.abs(g - r) / np.maximum(1.0, np.maximum(np.abs(g), np.abs(r)))))
