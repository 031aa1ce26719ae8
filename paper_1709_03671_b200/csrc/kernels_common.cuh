// Device-side view of an operator and the helpers every kernel file shares
// (kernels_spmv.cu, kernels_nonstat.cu, kernels_tsne.cu).
//
// Formats: every operator stores its entries SELL-32: rows
// are grouped in slices of 32 (one warp), and inside a slice entry q of lane
// r sits at slice_off[s] + 32 q + r, so a warp's q-th loads are one 128-byte
// line of values and one 64/128-byte line of indices.  Padding entries
// (q >= row_len) carry value 0 / index 0.
//  - KNNX_ORDER_ORIGINAL: int32 global columns (the spmv_flat path).
//  - KNNX_ORDER_CLUSTER : rows in tree order, cut into tiles of tile_rows
//    rows; each tile lists its sorted unique source columns (the halo) and
//    every entry stores a 16-bit index into it -- the GPU counterpart of the
//    reference's 16-bit cluster-local leaf payload (proj/include/patchord/
//    hier.hpp:15-24).
// Accumulation is fp32, per row in canonical (ascending column) order -- the
// order the reference accumulates in (proj/src/kernels.cpp:29,44-47).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "knnx_internal.cuh"

namespace knnx_dev {
namespace {

struct OpView {
  const int64_t* slice_off;
  const int32_t* slice_len;
  const int32_t* row_len;
  const int32_t* cols;
  const uint16_t* lidx;
  const int64_t* halo_off;
  const int32_t* halo_ids;
  float* vals;
  int n_rows, n_slices, tile_rows, row_base;
  const int32_t* slot_row;  // slot -> row (SELL-sigma); null = identity
};

inline OpView view_of(const knnx_operator& op) {
  return OpView{op.d_slice_off, op.d_slice_len, op.d_row_len, op.d_cols,  op.d_lidx,
                op.d_halo_off,  op.d_halo_ids,  op.d_vals,    op.n_rows,  op.n_slices,
                op.tile_rows,   op.row_base,    op.d_slot_row};
}

// only the t-SNE kernels read the relabelled / group-interleaved layouts
inline void require_plain(const knnx_operator& op) {
  if (!op.plain())
    throw knnx::error(knnx::errc::invalid_argument,
                      "relabelled / group-interleaved operators serve knnx_tsne_attr_* only");
}

// Kernels index entries by slot (a row's position in the SELL layout); the
// row a slot holds is the identity unless row lengths vary (SELL-sigma).
__device__ __forceinline__ int real_row(const OpView& v, int slot) {
  return v.slot_row ? __ldg(v.slot_row + slot) : slot;
}

__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const uint16_t* p) {
  return static_cast<int>(__ldcs(reinterpret_cast<const unsigned short*>(p)));
}

// global source column of a stored entry
template <bool kTiles>
__device__ __forceinline__ int entry_col(const OpView& v, int64_t pos, int64_t hbase) {
  if constexpr (kTiles)
    return __ldg(v.halo_ids + hbase + ld_stream(v.lidx + pos));
  else
    return ld_stream(v.cols + pos);
}


// ---------------------------------------------------------------------------
// masked float4 helpers for rows with dim % 4 != 0
__device__ __forceinline__ float sqdiff4(const float4 a, const float4 b, int c0, int dim) {
  float acc = 0.0f;
  const float d0 = (c0 + 0 < dim) ? a.x - b.x : 0.0f;
  const float d1 = (c0 + 1 < dim) ? a.y - b.y : 0.0f;
  const float d2 = (c0 + 2 < dim) ? a.z - b.z : 0.0f;
  const float d3 = (c0 + 3 < dim) ? a.w - b.w : 0.0f;
  acc = fmaf(d0, d0, acc);
  acc = fmaf(d1, d1, acc);
  acc = fmaf(d2, d2, acc);
  acc = fmaf(d3, d3, acc);
  return acc;
}

__device__ __forceinline__ void flag_error(int* flag, int code, int row) {
  atomicCAS(flag, 0, code);
  atomicMin(flag + 1, row);
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

inline int grid_for(int64_t threads, int block) {
  return static_cast<int>((threads + block - 1) / block);
}

}  // namespace
}  // namespace knnx_dev
