"""Python view of libknnx (the B200 kNN-interaction operator).

Thin wrappers over the C ABI in include/knnx.h / include/knnx_host.h.  Host
arrays are numpy; device arrays are torch CUDA tensors (torch is used only for
device memory and streams).  Every compute call lands in the sm_100a kernels
of libknnx.so -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import KnnxError, OpInfo, check, lib

ORIGINAL = 0
CLUSTER = 1
SCHEDULE_NONE, SCHEDULE_GRAPH, SCHEDULE_GIVEN = 0, 1, 2
OPT_RELABEL_COLS, OPT_GROUP_INTERLEAVE = 1, 2

# generator kinds (knnx_gen_points)
GEN_C1_MIXTURE = 1
GEN_3LEVEL = 2
GEN_ANISO = 3
GEN_NORMAL = 4


def _np_ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return C.c_void_p(a.ctypes.data)


def _dev_ptr(t):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device arrays must be contiguous CUDA tensors"
    return C.c_void_p(t.data_ptr())


def padded_ld(dim: int) -> int:
    return (dim + 3) // 4 * 4


# ---------------------------------------------------------------------------
# host-side helpers (knnx_host.h)

def rng_u64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    check(lib.knnx_rng_u64(seed, n, _np_ptr(out)), host=True)
    return out


def rng_uniform01(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    check(lib.knnx_rng_uniform01(seed, n, _np_ptr(out)), host=True)
    return out


def rng_normal(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    check(lib.knnx_rng_normal(seed, n, _np_ptr(out)), host=True)
    return out


def order_scattered(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.int32)
    check(lib.knnx_order_scattered(n, seed, _np_ptr(out)), host=True)
    return out


def gen_points(kind: int, n: int, dim: int, n_clusters: int, p0: float, seed: int) -> np.ndarray:
    out = np.empty((n, dim), np.float32)
    check(lib.knnx_gen_points(kind, n, dim, n_clusters, p0, seed, _np_ptr(out)), host=True)
    return out


def gen_uniform01(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    check(lib.knnx_gen_uniform01(n, seed, _np_ptr(out)), host=True)
    return out


def median_distance(d2: np.ndarray) -> float:
    d2 = np.ascontiguousarray(d2, np.float32).ravel()
    out = C.c_double()
    check(lib.knnx_median_distance(_np_ptr(d2), d2.size, C.byref(out)), host=True)
    return out.value


class HostCsr:
    """Canonical CSR owned by the host library (knnx_csr_t)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter exit
            lib.knnx_csr_destroy(self.h)
            self.h = None

    @classmethod
    def from_knn(cls, ids: np.ndarray, n_cols: int) -> "HostCsr":
        ids = np.ascontiguousarray(ids, np.int32)
        m, k = ids.shape
        h = C.c_void_p()
        check(lib.knnx_csr_from_knn(_np_ptr(ids), m, n_cols, k, C.byref(h)), host=True)
        return cls(h)

    @classmethod
    def from_arrays(cls, n_rows, n_cols, row_ptr, cols, vals=None) -> "HostCsr":
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = None if vals is None else np.ascontiguousarray(vals, np.float32)
        h = C.c_void_p()
        check(lib.knnx_csr_from_arrays(n_rows, n_cols, cols.size, _np_ptr(row_ptr), _np_ptr(cols),
                                       _np_ptr(vals), C.byref(h)), host=True)
        return cls(h)

    def symmetrize(self) -> "HostCsr":
        h = C.c_void_p()
        check(lib.knnx_csr_symmetrize(self.h, C.byref(h)), host=True)
        return HostCsr(h)

    def symmetrize_values(self, scale: float) -> "HostCsr":
        h = C.c_void_p()
        check(lib.knnx_csr_symmetrize_values(self.h, scale, C.byref(h)), host=True)
        return HostCsr(h)

    def row_normalize(self) -> None:
        check(lib.knnx_csr_row_normalize(self.h), host=True)

    def permute(self, forward: np.ndarray) -> "HostCsr":
        forward = np.ascontiguousarray(forward, np.int32)
        h = C.c_void_p()
        check(lib.knnx_csr_permute(self.h, _np_ptr(forward), C.byref(h)), host=True)
        return HostCsr(h)

    def row_block(self, r0: int, r1: int) -> "HostCsr":
        h = C.c_void_p()
        check(lib.knnx_csr_row_block(self.h, r0, r1, C.byref(h)), host=True)
        return HostCsr(h)

    def locality_schedule(self, col_base: int = 0) -> np.ndarray:
        """Row schedule of KNNX_SCHEDULE_GRAPH (breadth-first over the graph)."""
        out = np.empty(self.shape[0], np.int32)
        check(lib.knnx_csr_locality_schedule(self.h, col_base, _np_ptr(out)), host=True)
        return out

    def set_values(self, vals) -> None:
        vals = None if vals is None else np.ascontiguousarray(vals, np.float32)
        check(lib.knnx_csr_set_values(self.h, _np_ptr(vals)), host=True)

    @property
    def shape(self):
        m, n, hv = C.c_int32(), C.c_int32(), C.c_int32()
        nnz = C.c_int64()
        check(lib.knnx_csr_shape(self.h, C.byref(m), C.byref(n), C.byref(nnz), C.byref(hv)), host=True)
        return m.value, n.value, nnz.value, bool(hv.value)

    def export(self):
        m, _n, nnz, hv = self.shape
        row_ptr = np.empty(m + 1, np.int64)
        cols = np.empty(nnz, np.int32)
        vals = np.empty(nnz, np.float32) if hv else None
        check(lib.knnx_csr_export(self.h, _np_ptr(row_ptr), _np_ptr(cols), _np_ptr(vals)), host=True)
        return row_ptr, cols, vals


@dataclass
class Tree:
    forward: np.ndarray
    begin: np.ndarray
    end: np.ndarray
    depth: np.ndarray
    parent: np.ndarray
    is_leaf: np.ndarray
    captured_ratio: float = 1.0
    pca_iterations: int = 0

    @property
    def max_depth(self) -> int:
        return int(self.depth.max()) if self.depth.size else 0

    def level_blocking(self, level: int) -> np.ndarray:
        """Cluster offsets at `level` (proj/src/tree.cpp:114-124)."""
        if level < 0 or level > self.max_depth:
            raise KnnxError(10, f"LevelOutOfRange: level {level} exceeds tree depth {self.max_depth}")
        sel = (self.depth == level) | (self.is_leaf.astype(bool) & (self.depth < level))
        return np.sort(np.concatenate([self.begin[sel], [self.forward.size]])).astype(np.int32)


def _tree_from_handle(h, ratio=1.0, iters=0) -> Tree:
    try:
        nn, dp, npts = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib.knnx_tree_info(h, C.byref(nn), C.byref(dp), C.byref(npts)), host=True)
        fwd = np.empty(npts.value, np.int32)
        check(lib.knnx_tree_forward(h, _np_ptr(fwd)), host=True)
        arrs = [np.empty(nn.value, np.int32) for _ in range(5)]
        check(lib.knnx_tree_nodes(h, *[_np_ptr(a) for a in arrs]), host=True)
        return Tree(fwd, *arrs, captured_ratio=ratio, pca_iterations=iters)
    finally:
        lib.knnx_tree_destroy(h)


def order_tree(points: np.ndarray, d: int = 3, leaf_capacity: int = 128, max_depth: int = 12,
               pca_device: int = -1) -> Tree:
    """make_ordering("tree<d>") (proj/src/pipeline.cpp:91-129): PCA to d then tree."""
    pts = np.ascontiguousarray(points, np.float64)
    n, dim = pts.shape
    h = C.c_void_p()
    ratio, iters = C.c_double(), C.c_int32()
    check(lib.knnx_order_tree(_np_ptr(pts), n, dim, d, leaf_capacity, max_depth, pca_device,
                              C.byref(h), C.byref(ratio), C.byref(iters)), host=True)
    return _tree_from_handle(h, ratio.value, iters.value)


def build_tree(emb: np.ndarray, leaf_capacity: int = 128, max_depth: int = 12, device: int = -1) -> Tree:
    """Partition tree over a 1..3-D embedding; device >= 0 builds it on that
    CUDA device (knnx_tree_build_dev, the same tree)."""
    emb = np.ascontiguousarray(emb, np.float64)
    n, dim = emb.shape
    h = C.c_void_p()
    if device >= 0:
        check(lib.knnx_tree_build_dev(_np_ptr(emb), n, dim, leaf_capacity, max_depth, device, C.byref(h)),
              host=True)
    else:
        check(lib.knnx_tree_build(_np_ptr(emb), n, dim, leaf_capacity, max_depth, C.byref(h)), host=True)
    return _tree_from_handle(h)


def fit_pca(points: np.ndarray, d: int, pca_device: int = -1):
    pts = np.ascontiguousarray(points, np.float64)
    n, dim = pts.shape
    mean = np.empty(dim)
    axes = np.empty((d, dim))
    sv = np.empty(d)
    proj = np.empty((n, d))
    it, conv = C.c_int32(), C.c_int32()
    check(lib.knnx_fit_pca(_np_ptr(pts), n, dim, d, pca_device, _np_ptr(mean), _np_ptr(axes),
                           _np_ptr(sv), C.byref(it), C.byref(conv), _np_ptr(proj)), host=True)
    return dict(mean=mean, axes=axes, singular_values=sv, iterations=it.value,
                converged=bool(conv.value), projected=proj)


# ---------------------------------------------------------------------------
# device side (knnx.h)

class Context:
    """One device + one stream (the library's launch queue)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(lib.knnx_ctx_create(device, C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            lib.knnx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def use_stream(self, stream) -> None:
        """Launch on a torch.cuda.Stream (or raw cudaStream_t int); None = own stream."""
        if stream is None:
            check(lib.knnx_ctx_use_own_stream(self.h))
            return
        handle = int(getattr(stream, "cuda_stream", stream))
        check(lib.knnx_ctx_set_stream(self.h, C.c_void_p(handle)))

    def sync(self) -> None:
        """Synchronise and raise any deferred kernel error (ZeroWeight, ...)."""
        check(lib.knnx_ctx_sync(self.h))

    @property
    def launches(self) -> int:
        return int(lib.knnx_ctx_launches(self.h))

    def knn(self, t, s, m: int, n: int, dim: int, k: int, self_set: bool):
        """Exact fp32 kNN (device tool); t, s: padded CUDA tensors (rows x ld)."""
        import torch
        ld = t.shape[1]
        ids = torch.empty((m, k), dtype=torch.int32, device=t.device)
        d2 = torch.empty((m, k), dtype=torch.float32, device=t.device)
        check(lib.knnx_knn_dev(self.h, _dev_ptr(t), m, _dev_ptr(s), n, ld, dim, k,
                               1 if self_set else 0, _dev_ptr(ids), _dev_ptr(d2)))
        return ids, d2

    def knn_wide(self, t, s, m: int, n: int, dim: int, k: int, self_set: bool, n_cand: int = 0,
                 want_stats: bool = False):
        """kNN for wide points (dim > 64): tcgen05 TF32 distance screen + exact
        fp32 re-rank (knnx_knn_wide_dev).  Returns (ids, d2[, stats dict])."""
        import torch
        ld = t.shape[1]
        ids = torch.empty((m, k), dtype=torch.int32, device=t.device)
        d2 = torch.empty((m, k), dtype=torch.float32, device=t.device)
        stats = (C.c_double * 6)()
        check(lib.knnx_knn_wide_dev(self.h, _dev_ptr(t), m, _dev_ptr(s), n, ld, dim, k, n_cand,
                                    1 if self_set else 0, _dev_ptr(ids), _dev_ptr(d2),
                                    stats if want_stats else None))
        if want_stats:
            return ids, d2, {"min_margin": stats[0], "rows_nonpositive_margin": int(stats[1]),
                             "tiles_multiplied": int(stats[2]), "tiles_dense": int(stats[3]),
                             "rows_recomputed_exactly": int(stats[4]),
                             "rows_screened_3xtf32": int(stats[5])}
        return ids, d2

    def tsne_affinities(self, ids, d2, h: float, scale: float, keep_device: bool = False):
        """t-SNE joint P from device kNN rows, built on the device
        (knnx_tsne_affinities_dev): returns (row_ptr, cols, vals) numpy arrays;
        keep_device=True appends the DeviceCsr the arrays were read from (for
        Operator.from_csr_device) instead of freeing it."""
        n, k = ids.shape
        rp, cols, vals = C.c_void_p(), C.c_void_p(), C.c_void_p()
        nnz = C.c_int64()
        check(lib.knnx_tsne_affinities_dev(self.h, _dev_ptr(ids), _dev_ptr(d2), n, k, h, scale,
                                           C.byref(rp), C.byref(cols), C.byref(vals),
                                           C.byref(nnz)))
        dev = DeviceCsr(self, n, n, nnz.value, rp, cols, vals)
        try:
            out_rp = np.empty(n + 1, np.int64)
            out_c = np.empty(nnz.value, np.int32)
            out_v = np.empty(nnz.value, np.float32)
            check(lib.knnx_download_points(self.h, rp, 2 * (n + 1), 1, 1, _np_ptr(out_rp)))
            check(lib.knnx_download_points(self.h, cols, nnz.value, 1, 1, _np_ptr(out_c)))
            check(lib.knnx_download_points(self.h, vals, nnz.value, 1, 1, _np_ptr(out_v)))
        except Exception:
            dev.free()
            raise
        if keep_device:
            return out_rp, out_c, out_v, dev
        dev.free()
        return out_rp, out_c, out_v

    def permute_rows(self, src, forward, out) -> None:
        """out[forward[i]] = src[i] (whole rows, bit-exact)."""
        n = src.shape[0]
        row_bytes = src.element_size() * (src.numel() // max(n, 1))
        check(lib.knnx_permute_rows_dev(self.h, n, row_bytes, _dev_ptr(src), _dev_ptr(forward),
                                        _dev_ptr(out)))

    def gather_rows(self, src, index, out) -> None:
        """out[i] = src[index[i]]."""
        n = out.shape[0]
        row_bytes = out.element_size() * (out.numel() // max(n, 1))
        check(lib.knnx_gather_rows_dev(self.h, n, row_bytes, _dev_ptr(src), _dev_ptr(index),
                                       _dev_ptr(out)))


class DeviceCsr:
    """A canonical CSR in device buffers owned by the library (row_ptr int64,
    cols int32, vals fp32; e.g. the output of knnx_tsne_affinities_dev)."""

    def __init__(self, ctx: Context, n_rows: int, n_cols: int, nnz: int, row_ptr, cols, vals,
                 owned: bool = True, keep=None):
        self.ctx, self.n_rows, self.n_cols, self.nnz = ctx, n_rows, n_cols, nnz
        self.row_ptr, self.cols, self.vals = row_ptr, cols, vals
        self.owned, self._keep = owned, keep

    @classmethod
    def from_tensors(cls, ctx: Context, n_rows: int, n_cols: int, row_ptr, cols, vals=None) -> "DeviceCsr":
        """View of CUDA tensors (int64 row_ptr, int32 cols, fp32 vals) that stay owned by torch."""
        return cls(ctx, n_rows, n_cols, cols.numel(), _dev_ptr(row_ptr), _dev_ptr(cols),
                   None if vals is None else _dev_ptr(vals), owned=False, keep=(row_ptr, cols, vals))

    def free(self) -> None:
        for name in ("row_ptr", "cols", "vals"):
            p = getattr(self, name)
            if self.owned and p is not None and self.ctx.h:
                lib.knnx_free(self.ctx.h, p)
            setattr(self, name, None)
        self._keep = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Comm:
    """One rank of a multi-device communicator (include/knnx.h "multi-device"):
    NCCL inside, opened at run time.  Comm.unique_id() on one rank, shared
    by the host (e.g. torch.distributed.broadcast_object_list), then
    Comm(ctx, nranks, rank, uid) on every rank."""

    NCCL, LOCAL = 1, 2

    def __init__(self, ctx: Context, nranks: int, rank: int, uid: bytes):
        self.h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        check(lib.knnx_comm_init_rank(ctx.h, nranks, rank, buf, C.byref(self.h)))
        self.ctx, self.nranks, self.rank = ctx, nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.knnx_comm_unique_id(buf))
        return buf.raw

    def allgather_rows(self, buf, rows_per_rank: int) -> None:
        """In place: rank r's rows [r*rows, (r+1)*rows) of buf to every rank."""
        n = buf.shape[0]
        row_bytes = buf.element_size() * (buf.numel() // max(n, 1))
        check(lib.knnx_allgather_rows_dev(self.h, _dev_ptr(buf), rows_per_rank, row_bytes))

    def barrier(self) -> None:
        check(lib.knnx_comm_barrier(self.h))

    def close(self):
        if self.h:
            lib.knnx_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    """A kNN interaction operator resident on one device."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle
        inf = OpInfo()
        check(lib.knnx_op_info(self.h, C.byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in OpInfo._fields_}

    @classmethod
    def from_csr(cls, ctx: Context, n_rows: int, n_cols: int, row_ptr, cols, vals=None,
                 order: int = ORIGINAL, tile_rows: int = 0) -> "Operator":
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = None if vals is None else np.ascontiguousarray(vals, np.float32)
        h = C.c_void_p()
        check(lib.knnx_op_create_csr(ctx.h, n_rows, n_cols, cols.size, _np_ptr(row_ptr),
                                     _np_ptr(cols), _np_ptr(vals), order, tile_rows, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_csr_scheduled(cls, ctx: Context, n_rows: int, n_cols: int, row_ptr, cols, vals=None,
                           order: int = CLUSTER, tile_rows: int = 0, schedule=None,
                           col_base: int = 0, options: int = 0) -> "Operator":
        """Operator whose rows run in a locality schedule (knnx_op_create_csr_ex):
        schedule=None -> breadth-first over the graph, else the given row order.
        options: OPT_RELABEL_COLS / OPT_GROUP_INTERLEAVE (t-SNE layouts)."""
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = None if vals is None else np.ascontiguousarray(vals, np.float32)
        sched = None if schedule is None else np.ascontiguousarray(schedule, np.int32)
        kind = SCHEDULE_GRAPH if sched is None else SCHEDULE_GIVEN
        h = C.c_void_p()
        check(lib.knnx_op_create_csr_ex(ctx.h, n_rows, n_cols, cols.size, _np_ptr(row_ptr),
                                        _np_ptr(cols), _np_ptr(vals), order, tile_rows, kind,
                                        col_base, _np_ptr(sched), options, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_csr_device(cls, ctx: Context, n_rows: int, n_cols: int, row_ptr, cols=None, vals=None,
                        schedule="graph", col_base: int = 0, options: int = 0, rows=None,
                        block_nnz: int = 0) -> "Operator":
        """Original-order operator built on the device from a device CSR
        (knnx_op_create_csr_dev): row_ptr int64 / cols int32 / vals fp32 CUDA
        tensors, or a DeviceCsr as row_ptr.  schedule: "graph" (breadth-first, on the device), None, or
        a host row order."""
        if isinstance(row_ptr, DeviceCsr):
            d = row_ptr
            n_rows, n_cols, nnz, p_rp, p_cols, p_vals = d.n_rows, d.n_cols, d.nnz, d.row_ptr, d.cols, d.vals
            if rows is not None:   # row block [r0, r1): shifted row_ptr, unshifted cols / vals
                r0, r1 = rows
                n_rows, nnz = r1 - r0, block_nnz
                p_rp = C.c_void_p(p_rp.value + 8 * r0)
        else:
            nnz, p_rp, p_cols = cols.numel(), _dev_ptr(row_ptr), _dev_ptr(cols)
            p_vals = None if vals is None else _dev_ptr(vals)
        if schedule is None:
            kind, sched = SCHEDULE_NONE, None
        elif isinstance(schedule, str):
            kind, sched = SCHEDULE_GRAPH, None
        else:
            kind, sched = SCHEDULE_GIVEN, np.ascontiguousarray(schedule, np.int32)
        h = C.c_void_p()
        check(lib.knnx_op_create_csr_dev(ctx.h, n_rows, n_cols, nnz, p_rp, p_cols, p_vals,
                                         kind, col_base, _np_ptr(sched), options, C.byref(h)))
        return cls(ctx, h)

    def slot_rows(self) -> np.ndarray:
        """slot -> row map the kernels run in (knnx_op_slot_rows)."""
        out = np.empty(self.info["n_rows"], np.int32)
        check(lib.knnx_op_slot_rows(self.h, _np_ptr(out)))
        return out

    @classmethod
    def from_knn_device(cls, ctx: Context, ids, n_cols: int) -> "Operator":
        """Cluster operator built on the device from device kNN rows (m x k)."""
        m, k = ids.shape
        h = C.c_void_p()
        check(lib.knnx_op_create_knn_dev(ctx.h, _dev_ptr(ids), m, n_cols, k, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_hbm1(cls, ctx: Context, path: str, tile_rows: int = 0):
        """Load a reference HBM1 dump; returns (operator, row_forward, col_forward)."""
        m, n, nnz, cut = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
        check(lib.knnx_hbm1_info(path.encode(), C.byref(m), C.byref(n), C.byref(nnz), C.byref(cut)))
        rf = np.empty(m.value, np.int32)
        cf = np.empty(n.value, np.int32)
        h = C.c_void_p()
        check(lib.knnx_op_load_hbm1(ctx.h, path.encode(), tile_rows, _np_ptr(rf), _np_ptr(cf),
                                    C.byref(h)))
        return cls(ctx, h), rf, cf

    @classmethod
    def from_host_csr(cls, ctx: Context, csr: HostCsr, order: int = ORIGINAL,
                      tile_rows: int = 0) -> "Operator":
        m, n, _nnz, _hv = csr.shape
        row_ptr, cols, vals = csr.export()
        return cls.from_csr(ctx, m, n, row_ptr, cols, vals, order, tile_rows)

    def close(self):
        if self.h:
            lib.knnx_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_rows(self) -> int:
        return self.info["n_rows"]

    @property
    def n_cols(self) -> int:
        return self.info["n_cols"]

    def set_row_base(self, row_base: int) -> None:
        check(lib.knnx_op_set_row_base(self.h, row_base))
        self.info["row_base"] = row_base

    def set_values(self, vals: np.ndarray) -> None:
        vals = np.ascontiguousarray(vals, np.float32)
        check(lib.knnx_op_set_values(self.h, _np_ptr(vals)))
        self.info["has_values"] = 1

    def get_values(self) -> np.ndarray:
        out = np.empty(self.info["nnz"], np.float32)
        check(lib.knnx_op_get_values(self.h, _np_ptr(out)))
        return out

    # stationary
    def spmv(self, x, y) -> None:
        check(lib.knnx_spmv_dev(self.h, _dev_ptr(x), _dev_ptr(y)))

    def spmv_repeat(self, n_steps: int, x, y, x_stride: int = 0, y_stride: int = 0) -> None:
        """n_steps applications in one CUDA-graph replay (knnx_spmv_batch_strided_dev);
        stride 0 = every step reads x / writes y (fixed charges)."""
        check(lib.knnx_spmv_batch_strided_dev(self.h, n_steps, _dev_ptr(x), x_stride, _dev_ptr(y),
                                              y_stride))

    def spmv_host(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty(self.n_rows, np.float32)
        check(lib.knnx_spmv_host(self.h, _np_ptr(x), _np_ptr(y)))
        return y

    # non-stationary
    def gauss_spmv(self, t, s, dim: int, h: float, x, y) -> None:
        check(lib.knnx_gauss_spmv_dev(self.h, _dev_ptr(t), t.shape[1], _dev_ptr(s), s.shape[1], dim,
                                      h, _dev_ptr(x), _dev_ptr(y)))

    def update_gaussian(self, t, s, dim: int, h: float) -> None:
        check(lib.knnx_update_gaussian_dev(self.h, _dev_ptr(t), t.shape[1], _dev_ptr(s), s.shape[1],
                                           dim, h))
        self.info["has_values"] = 1

    def meanshift(self, t_in, s, dim: int, h: float, t_out) -> None:
        check(lib.knnx_meanshift_dev(self.h, _dev_ptr(t_in), t_in.shape[1], _dev_ptr(s), s.shape[1],
                                     dim, h, _dev_ptr(t_out)))

    def meanshift_host(self, t_in: np.ndarray, s: np.ndarray, h: float) -> np.ndarray:
        t_in = np.ascontiguousarray(t_in, np.float32)
        s = np.ascontiguousarray(s, np.float32)
        out = np.empty_like(t_in)
        check(lib.knnx_meanshift_host(self.h, _np_ptr(t_in), _np_ptr(s), t_in.shape[1], h,
                                      _np_ptr(out)))
        return out

    def tsne(self, y, dim: int, f, store: bool = False, step: float = 0.0, y_out=None) -> None:
        check(lib.knnx_tsne_attr_dev(self.h, _dev_ptr(y), dim, _dev_ptr(f), 1 if store else 0,
                                     step, _dev_ptr(y_out)))

    def tsne_peers(self, y, dim: int, f, step: float, y_outs) -> None:
        """Forces of this shard's rows + y - step F stored into every replica
        in y_outs (device pointers or CUDA tensors valid in this process)."""
        ptrs = (C.c_void_p * len(y_outs))(*[p.data_ptr() if hasattr(p, "data_ptr") else int(p)
                                            for p in y_outs])
        check(lib.knnx_tsne_attr_peers_dev(self.h, _dev_ptr(y), dim, _dev_ptr(f), step, ptrs,
                                           len(y_outs)))

    def tsne_host(self, y: np.ndarray, store: bool = False) -> np.ndarray:
        y = np.ascontiguousarray(y, np.float32)
        f = np.empty_like(y)
        check(lib.knnx_tsne_attr_host(self.h, _np_ptr(y), y.shape[1], _np_ptr(f),
                                      1 if store else 0))
        return f


def to_device_points(points: np.ndarray, device="cuda", align: int = 4):
    """Upload an n x dim float array as a zero-padded n x ld CUDA tensor, ld the
    dim rounded up to `align` floats (4: 16-B rows for float4 loads; 32: 128-B
    rows, one cache line per 32 coordinates for the gather kernels)."""
    import torch
    n, dim = points.shape
    ld = (dim + align - 1) // align * align
    if ld == dim:  # nothing to pad: no staging copy (C5's 3.8 GB)
        return torch.from_numpy(np.ascontiguousarray(points, np.float32)).to(device)
    buf = np.zeros((n, ld), np.float32)
    buf[:, :dim] = points
    return torch.from_numpy(buf).to(device)
