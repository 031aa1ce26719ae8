"""ctypes binding of libknnx.so (include/knnx.h + include/knnx_host.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_1709_03671_b200``).  There is no fallback: if the library is
missing, importing this module raises, and every operator call goes to the
CUDA kernels or fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libknnx.so")

# patchord::errc names (proj/include/patchord/core.hpp:15-42), code = 1 + ordinal
ERRC_NAMES = [
    "OutOfBounds", "DuplicateEntry", "SizeMismatch", "DimMismatch", "KTooLarge", "NotSquare",
    "NonPositiveBandwidth", "DegenerateData", "DimTooHigh", "LevelOutOfRange", "EmptyPattern",
    "TooLarge", "NotDivisible", "TooWide", "TooMany", "SpanMismatch", "LocalIndexOverflow",
    "OrderingMismatch", "NonFiniteValue", "ZeroWeight", "MalformedRecord", "InconsistentDim",
    "EmptyFile", "IoError", "ChecksumMismatch", "InvalidArgument",
]
EXTRA_NAMES = {65: "CudaError", 66: "Unsupported"}


def code_name(code: int) -> str:
    if 1 <= code <= len(ERRC_NAMES):
        return ERRC_NAMES[code - 1]
    return EXTRA_NAMES.get(code, f"Error{code}")


class KnnxError(RuntimeError):
    """A failed libknnx call; ``code`` is 1 + the reference's errc ordinal."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.name = code_name(code)


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
        "(or __graft_entry__.build()); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

i32, i64, u64, f32, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_void_p
P = C.POINTER

_SIGS = {
    # knnx.h
    "knnx_abi_version": (C.c_int, []),
    "knnx_last_error": (C.c_char_p, []),
    "knnx_ctx_create": (C.c_int, [C.c_int, P(vp)]),
    "knnx_ctx_destroy": (C.c_int, [vp]),
    "knnx_ctx_set_stream": (C.c_int, [vp, vp]),
    "knnx_ctx_use_own_stream": (C.c_int, [vp]),
    "knnx_ctx_stream": (vp, [vp]),
    "knnx_ctx_sync": (C.c_int, [vp]),
    "knnx_ctx_launches": (i64, [vp]),
    "knnx_alloc": (C.c_int, [vp, i64, P(vp)]),
    "knnx_free": (C.c_int, [vp, vp]),
    "knnx_host_alloc": (C.c_int, [i64, P(vp)]),
    "knnx_host_free": (C.c_int, [vp]),
    "knnx_upload_points": (C.c_int, [vp, vp, i32, i32, i32, vp]),
    "knnx_download_points": (C.c_int, [vp, vp, i32, i32, i32, vp]),
    "knnx_op_create_csr": (C.c_int, [vp, i32, i32, i64, vp, vp, vp, i32, i32, P(vp)]),
    "knnx_op_create_csr_sched": (C.c_int, [vp, i32, i32, i64, vp, vp, vp, i32, i32, i32, i32, vp,
                                           P(vp)]),
    "knnx_op_create_csr_ex": (C.c_int, [vp, i32, i32, i64, vp, vp, vp, i32, i32, i32, i32, vp,
                                        i32, P(vp)]),
    "knnx_op_create_hier_leaves": (C.c_int, [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32, P(vp)]),
    "knnx_op_create_csr_dev": (C.c_int, [vp, i32, i32, i64, vp, vp, vp, i32, i32, vp, i32, P(vp)]),
    "knnx_op_slot_rows": (C.c_int, [vp, vp]),
    "knnx_op_destroy": (C.c_int, [vp]),
    "knnx_tsne_affinities_dev": (C.c_int, [vp, vp, vp, i32, i32, f64, f64, P(vp), P(vp), P(vp),
                                           P(i64)]),
    "knnx_copy_async": (C.c_int, [vp, vp, vp, i64]),
    "knnx_op_create_knn_dev": (C.c_int, [vp, vp, i32, i32, i32, P(vp)]),
    "knnx_hbm1_info": (C.c_int, [C.c_char_p, P(i32), P(i32), P(i64), P(i32)]),
    "knnx_op_load_hbm1": (C.c_int, [vp, C.c_char_p, i32, vp, vp, P(vp)]),
    "knnx_op_set_row_base": (C.c_int, [vp, i32]),
    "knnx_op_info": (C.c_int, [vp, vp]),
    "knnx_op_set_values": (C.c_int, [vp, vp]),
    "knnx_op_get_values": (C.c_int, [vp, vp]),
    "knnx_spmv_dev": (C.c_int, [vp, vp, vp]),
    "knnx_spmv_host": (C.c_int, [vp, vp, vp]),
    "knnx_spmv_batch_dev": (C.c_int, [vp, i32, vp, vp]),
    "knnx_spmv_batch_strided_dev": (C.c_int, [vp, i32, vp, i64, vp, i64]),
    "knnx_spmv_host_batch": (C.c_int, [vp, i32, vp, vp]),
    "knnx_gauss_spmv_dev": (C.c_int, [vp, vp, i32, vp, i32, i32, f64, vp, vp]),
    "knnx_update_gaussian_dev": (C.c_int, [vp, vp, i32, vp, i32, i32, f64]),
    "knnx_gauss_spmv_host": (C.c_int, [vp, vp, vp, i32, f64, vp, vp]),
    "knnx_update_gaussian_host": (C.c_int, [vp, vp, vp, i32, f64]),
    "knnx_permute_rows_host": (C.c_int, [vp, i32, i64, vp, vp, vp]),
    "knnx_meanshift_dev": (C.c_int, [vp, vp, i32, vp, i32, i32, f64, vp]),
    "knnx_meanshift_host": (C.c_int, [vp, vp, vp, i32, f64, vp]),
    "knnx_tsne_attr_dev": (C.c_int, [vp, vp, i32, vp, i32, f32, vp]),
    "knnx_tsne_attr_host": (C.c_int, [vp, vp, i32, vp, i32]),
    "knnx_permute_rows_dev": (C.c_int, [vp, i32, i64, vp, vp, vp]),
    "knnx_gather_rows_dev": (C.c_int, [vp, i32, i64, vp, vp, vp]),
    "knnx_knn_dev": (C.c_int, [vp, vp, i32, vp, i32, i32, i32, i32, i32, vp, vp]),
    "knnx_knn_wide_dev": (C.c_int, [vp, vp, i32, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp]),
    "knnx_gram_tf32_dev": (C.c_int, [vp, vp, i32, vp, i32, i32, i32, vp, i64]),
    "knnx_comm_unique_id": (C.c_int, [vp]),
    "knnx_comm_init_rank": (C.c_int, [vp, i32, i32, vp, P(vp)]),
    "knnx_comm_init_local": (C.c_int, [i32, vp, vp]),
    "knnx_comm_destroy": (C.c_int, [vp]),
    "knnx_comm_info": (C.c_int, [vp, P(i32), P(i32), P(i32)]),
    "knnx_allgather_rows_dev": (C.c_int, [vp, vp, i64, i64]),
    "knnx_allgather_rows_local": (C.c_int, [vp, i32, vp, i64, i64]),
    "knnx_comm_barrier": (C.c_int, [vp]),
    "knnx_comm_barrier_local": (C.c_int, [vp, i32]),
    "knnx_tsne_attr_peers_dev": (C.c_int, [vp, vp, i32, vp, f32, vp, i32]),
    "knnx_ipc_get_handle": (C.c_int, [vp, vp, vp]),
    "knnx_ipc_open": (C.c_int, [vp, vp, P(vp)]),
    "knnx_ipc_close": (C.c_int, [vp, vp]),
    # knnx_host.h
    "knnx_host_last_error": (C.c_char_p, []),
    "knnx_rng_u64": (C.c_int, [u64, i64, vp]),
    "knnx_rng_uniform01": (C.c_int, [u64, i64, vp]),
    "knnx_rng_normal": (C.c_int, [u64, i64, vp]),
    "knnx_order_scattered": (C.c_int, [i32, u64, vp]),
    "knnx_gen_points": (C.c_int, [i32, i32, i32, i32, f64, u64, vp]),
    "knnx_gen_uniform01": (C.c_int, [i64, u64, vp]),
    "knnx_median_distance": (C.c_int, [vp, i64, P(f64)]),
    "knnx_csr_from_knn": (C.c_int, [vp, i32, i32, i32, P(vp)]),
    "knnx_csr_from_arrays": (C.c_int, [i32, i32, i64, vp, vp, vp, P(vp)]),
    "knnx_csr_symmetrize": (C.c_int, [vp, P(vp)]),
    "knnx_csr_symmetrize_values": (C.c_int, [vp, f64, P(vp)]),
    "knnx_csr_row_normalize": (C.c_int, [vp]),
    "knnx_csr_permute": (C.c_int, [vp, vp, P(vp)]),
    "knnx_csr_row_block": (C.c_int, [vp, i32, i32, P(vp)]),
    "knnx_csr_locality_schedule": (C.c_int, [vp, i32, vp]),
    "knnx_csr_set_values": (C.c_int, [vp, vp]),
    "knnx_csr_shape": (C.c_int, [vp, P(i32), P(i32), P(i64), P(i32)]),
    "knnx_csr_export": (C.c_int, [vp, vp, vp, vp]),
    "knnx_csr_destroy": (None, [vp]),
    "knnx_order_tree": (C.c_int, [vp, i32, i32, i32, i32, i32, i32, P(vp), P(f64), P(i32)]),
    "knnx_tree_build": (C.c_int, [vp, i32, i32, i32, i32, P(vp)]),
    "knnx_tree_build_dev": (C.c_int, [vp, i32, i32, i32, i32, i32, P(vp)]),
    "knnx_tree_info": (C.c_int, [vp, P(i32), P(i32), P(i32)]),
    "knnx_tree_forward": (C.c_int, [vp, vp]),
    "knnx_tree_nodes": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "knnx_tree_level_blocking": (C.c_int, [vp, i32, vp, P(i32)]),
    "knnx_tree_destroy": (None, [vp]),
    "knnx_fit_pca": (C.c_int, [vp, i32, i32, i32, i32, vp, vp, vp, P(i32), P(i32), vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class OpInfo(C.Structure):
    _fields_ = [
        ("n_rows", i32), ("n_cols", i32), ("order", i32), ("tile_rows", i32),
        ("nnz", i64), ("stored", i64), ("n_tiles", i32), ("max_halo", i32),
        ("halo_total", i64), ("device_bytes", i64),
        ("has_values", i32), ("uniform_row_len", i32),
    ]


def check(rc: int, host: bool = False) -> None:
    """Raise KnnxError for a non-zero status."""
    if rc != 0:
        msg = (lib.knnx_host_last_error() if host else lib.knnx_last_error()) or b""
        raise KnnxError(rc, msg.decode(errors="replace"))


def exported_symbols() -> list[str]:
    return list(_SIGS)
