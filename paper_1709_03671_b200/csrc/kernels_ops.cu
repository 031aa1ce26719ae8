// sm_100a kernels for the kNN-interaction hot path.
//
// Formats: every operator stores its entries SELL-32:
// rows are grouped in slices of 32 (one warp), and inside a slice entry q of
// lane r sits at slice_off[s] + 32 q + r, so a warp's q-th loads are one
// 128-byte line of values and one 64/128-byte line of indices.  Padding
// entries (q >= row_len) carry value 0 / index 0.
//  - KNNX_ORDER_ORIGINAL: int32 global columns (the spmv_flat path).
//  - KNNX_ORDER_CLUSTER : rows in tree order, cut into tiles of tile_rows
//    rows; each tile lists its sorted unique source columns (the halo) and
//    every entry stores a 16-bit index into it -- the GPU counterpart of the
//    reference's 16-bit cluster-local leaf payload (proj/include/patchord/
//    hier.hpp:15-24).  The stationary kernel stages x[halo] in shared memory,
//    so every gather after the stage is a shared-memory load.
//
// Accumulation is fp32, per row in canonical (ascending column) order -- the
// order the reference accumulates in (proj/src/kernels.cpp:29,44-47).
#include <cuda_runtime.h>

#include <algorithm>
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
  int n_rows, n_slices, tile_rows;
};

OpView view_of(const knnx_operator& op) {
  return OpView{op.d_slice_off, op.d_slice_len, op.d_row_len, op.d_cols,  op.d_lidx,
                op.d_halo_off,  op.d_halo_ids,  op.d_vals,    op.n_rows,  op.n_slices,
                op.tile_rows};
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
// K2: stationary SpMV, original order (spmv_flat, proj/src/kernels.cpp:37-49)
__global__ void __launch_bounds__(256) spmv_orig_kernel(OpView v, const float* __restrict__ x,
                                                        float* __restrict__ y) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = row >> 5;
  if (s >= v.n_slices) return;
  const int64_t base = v.slice_off[s] + (row & 31);
  const int len = v.slice_len[s];
  float acc = 0.0f;
#pragma unroll 10
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    acc = fmaf(ld_stream(v.vals + p), __ldg(x + ld_stream(v.cols + p)), acc);
  }
  if (row < v.n_rows) y[row] = acc;
}

// K3: stationary SpMV, cluster tiles (spmv_hier / spmv_hier_parallel,
// proj/src/kernels.cpp:24-101).  One CTA per tile: stage x[halo] in shared
// memory, then thread-per-row accumulation from shared memory.
__global__ void __launch_bounds__(128) spmv_tiles_kernel(OpView v, const float* __restrict__ x,
                                                         float* __restrict__ y) {
  extern __shared__ float sx[];
  const int tile = blockIdx.x;
  const int64_t h0 = v.halo_off[tile];
  const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
  for (int i = threadIdx.x; i < H; i += blockDim.x) sx[i] = __ldg(x + __ldg(v.halo_ids + h0 + i));
  __syncthreads();
  const int row = tile * v.tile_rows + threadIdx.x;
  const int s = row >> 5;
  if (threadIdx.x >= v.tile_rows || s >= v.n_slices) return;
  const int64_t base = v.slice_off[s] + (row & 31);
  const int len = v.slice_len[s];
  float acc = 0.0f;
#pragma unroll 10
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    acc = fmaf(ld_stream(v.vals + p), sx[ld_stream(v.lidx + p)], acc);
  }
  if (row < v.n_rows) y[row] = acc;
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

// K4: Gaussian-recompute SpMV, thread per row, dim <= 4*NV
// (iterate_interactions + gaussian value_fn, proj/src/kernels.cpp:217-228;
// weight exp(-d^2/(2h^2)) evaluated as exp2(-d^2 * c2), c2 = log2(e)/(2h^2))
template <bool kTiles, int NV>
__global__ void __launch_bounds__(128) gauss_rows_kernel(OpView v, const float* __restrict__ t,
                                                         int ld_t, const float* __restrict__ s,
                                                         int ld_s, int dim, float c2,
                                                         const float* __restrict__ x,
                                                         float* __restrict__ y) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= v.n_rows) return;
  const int sl = row >> 5;
  const int64_t base = v.slice_off[sl] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  float4 ti[NV];
  const float4* tp = reinterpret_cast<const float4*>(t + static_cast<int64_t>(row) * ld_t);
#pragma unroll
  for (int c = 0; c < NV; ++c) ti[c] = __ldg(tp + c);
  float acc = 0.0f;
  for (int q = 0; q < len; ++q) {
    const int j = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q), hbase);
    const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
    float d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < NV; ++c) d2 += sqdiff4(ti[c], __ldg(sp + c), 4 * c, dim);
    acc = fmaf(exp2f(-d2 * c2), __ldg(x + j), acc);
  }
  y[row] = acc;
}

// K4 (wide rows): warp per row, lanes split the coordinates, dim <= 128*NVL
template <bool kTiles, int NVL>
__global__ void __launch_bounds__(256) gauss_warp_kernel(OpView v, const float* __restrict__ t,
                                                         int ld_t, const float* __restrict__ s,
                                                         int ld_s, int dim, float c2,
                                                         const float* __restrict__ x,
                                                         float* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= v.n_rows) return;
  const int64_t base = v.slice_off[row >> 5] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  const int nv4 = (dim + 3) >> 2;
  float4 ti[NVL];
  const float4* tp = reinterpret_cast<const float4*>(t + static_cast<int64_t>(row) * ld_t);
#pragma unroll
  for (int c = 0; c < NVL; ++c) {
    const int c4 = lane + 32 * c;
    ti[c] = c4 < nv4 ? __ldg(tp + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float acc = 0.0f;
  for (int q = 0; q < len; ++q) {
    const int j = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q), hbase);
    const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
    float d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < NVL; ++c) {
      const int c4 = lane + 32 * c;
      if (c4 < nv4) d2 += sqdiff4(ti[c], __ldg(sp + c4), 4 * c4, dim);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    acc = fmaf(exp2f(-d2 * c2), __ldg(x + j), acc);
  }
  if (lane == 0) y[row] = acc;
}

// update_values with the Gaussian model into the stored values
// (proj/src/hier.cpp:203-222); a non-finite weight raises NonFiniteValue
template <bool kTiles>
__global__ void __launch_bounds__(256) update_gauss_kernel(OpView v, const float* __restrict__ t,
                                                           int ld_t, const float* __restrict__ s,
                                                           int ld_s, int dim, float c2, int* flag) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= v.n_rows) return;
  const int64_t base = v.slice_off[row >> 5] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  const float* ti = t + static_cast<int64_t>(row) * ld_t;
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    const int j = entry_col<kTiles>(v, p, hbase);
    const float* sj = s + static_cast<int64_t>(j) * ld_s;
    float d2 = 0.0f;
    for (int c = 0; c < dim; ++c) {
      const float d = __ldg(ti + c) - __ldg(sj + c);
      d2 = fmaf(d, d, d2);
    }
    const float w = exp2f(-d2 * c2);
    if (!isfinite(w)) flag_error(flag, kFlagNonFinite, row);
    v.vals[p] = w;
  }
}

// ---------------------------------------------------------------------------
// K5: mean shift (meanshift_step, proj/src/kernels.cpp:184-208).  Weights
// are taken relative to the running nearest source (online rescale), which
// leaves sum(w s)/sum(w) unchanged but cannot underflow in fp32; ZeroWeight
// is raised when min d^2 / (2h^2) exceeds the fp64 underflow point, i.e.
// exactly when every reference weight is 0.
template <bool kTiles, int NV>
__global__ void __launch_bounds__(128) meanshift_rows_kernel(
    OpView v, const float* __restrict__ tin, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, float* __restrict__ tout, int* flag) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= v.n_rows) return;
  const int64_t base = v.slice_off[row >> 5] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  float4 ti[NV], acc[NV];
  const float4* tp = reinterpret_cast<const float4*>(tin + static_cast<int64_t>(row) * ld_t);
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    ti[c] = __ldg(tp + c);
    acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float m = INFINITY, tot = 0.0f;
  for (int q = 0; q < len; ++q) {
    const int j = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q), hbase);
    const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
    float4 sj[NV];
    float d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      sj[c] = __ldg(sp + c);
      d2 += sqdiff4(ti[c], sj[c], 4 * c, dim);
    }
    if (d2 < m) {
      const float sc = exp2f((d2 - m) * c2);
      tot *= sc;
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        acc[c].x *= sc; acc[c].y *= sc; acc[c].z *= sc; acc[c].w *= sc;
      }
      m = d2;
    }
    const float w = exp2f((m - d2) * c2);
    tot += w;
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      acc[c].x = fmaf(w, sj[c].x, acc[c].x);
      acc[c].y = fmaf(w, sj[c].y, acc[c].y);
      acc[c].z = fmaf(w, sj[c].z, acc[c].z);
      acc[c].w = fmaf(w, sj[c].w, acc[c].w);
    }
  }
  if (len == 0 || m > zero_thresh) flag_error(flag, kFlagZeroWeight, row);
  const float inv = 1.0f / tot;
  float4* op = reinterpret_cast<float4*>(tout + static_cast<int64_t>(row) * ld_t);
#pragma unroll
  for (int c = 0; c < NV; ++c)
    op[c] = make_float4(acc[c].x * inv, acc[c].y * inv, acc[c].z * inv, acc[c].w * inv);
}

// K5 (wide rows): warp per row
template <bool kTiles, int NVL>
__global__ void __launch_bounds__(256) meanshift_warp_kernel(
    OpView v, const float* __restrict__ tin, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, float* __restrict__ tout, int* flag) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= v.n_rows) return;
  const int64_t base = v.slice_off[row >> 5] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  const int nv4 = (dim + 3) >> 2;
  float4 ti[NVL], acc[NVL];
  const float4* tp = reinterpret_cast<const float4*>(tin + static_cast<int64_t>(row) * ld_t);
#pragma unroll
  for (int c = 0; c < NVL; ++c) {
    const int c4 = lane + 32 * c;
    ti[c] = c4 < nv4 ? __ldg(tp + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float m = INFINITY, tot = 0.0f;
  for (int q = 0; q < len; ++q) {
    const int j = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q), hbase);
    const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
    float4 sj[NVL];
    float d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < NVL; ++c) {
      const int c4 = lane + 32 * c;
      sj[c] = c4 < nv4 ? __ldg(sp + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (c4 < nv4) d2 += sqdiff4(ti[c], sj[c], 4 * c4, dim);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    if (d2 < m) {
      const float sc = exp2f((d2 - m) * c2);
      tot *= sc;
#pragma unroll
      for (int c = 0; c < NVL; ++c) {
        acc[c].x *= sc; acc[c].y *= sc; acc[c].z *= sc; acc[c].w *= sc;
      }
      m = d2;
    }
    const float w = exp2f((m - d2) * c2);
    tot += w;
#pragma unroll
    for (int c = 0; c < NVL; ++c) {
      acc[c].x = fmaf(w, sj[c].x, acc[c].x);
      acc[c].y = fmaf(w, sj[c].y, acc[c].y);
      acc[c].z = fmaf(w, sj[c].z, acc[c].z);
      acc[c].w = fmaf(w, sj[c].w, acc[c].w);
    }
  }
  if (lane == 0 && (len == 0 || m > zero_thresh)) flag_error(flag, kFlagZeroWeight, row);
  const float inv = 1.0f / tot;
  float4* op = reinterpret_cast<float4*>(tout + static_cast<int64_t>(row) * ld_t);
#pragma unroll
  for (int c = 0; c < NVL; ++c) {
    const int c4 = lane + 32 * c;
    if (c4 < nv4)
      op[c4] = make_float4(acc[c].x * inv, acc[c].y * inv, acc[c].z * inv, acc[c].w * inv);
  }
}

// ---------------------------------------------------------------------------
// K6: t-SNE attractive force (tsne_attractive_step, proj/src/kernels.cpp:103-136),
// computed directly as F_i = sum_j a_ij (y_i - y_j); optional in-place
// a_ij write-back (the reference's mutation) and fused y update.
template <bool kTiles, int DIM>
__global__ void __launch_bounds__(256) tsne_rows_kernel(OpView v, const float* __restrict__ y,
                                                        float* __restrict__ f, int store,
                                                        float step, float* __restrict__ y_out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= v.n_rows) return;
  const int64_t base = v.slice_off[row >> 5] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  float yi[DIM], acc[DIM];
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    yi[c] = __ldg(y + static_cast<int64_t>(row) * DIM + c);
    acc[c] = 0.0f;
  }
#pragma unroll 4
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    const int j = entry_col<kTiles>(v, p, hbase);
    const float pij = ld_stream(v.vals + p);
    float d[DIM], d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      d[c] = yi[c] - __ldg(y + static_cast<int64_t>(j) * DIM + c);
      d2 = fmaf(d[c], d[c], d2);
    }
    const float a = pij / (1.0f + d2);
    if (store) v.vals[p] = a;
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = fmaf(a, d[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    f[static_cast<int64_t>(row) * DIM + c] = acc[c];
    if (y_out) y_out[static_cast<int64_t>(row) * DIM + c] = yi[c] - step * acc[c];
  }
}

// ---------------------------------------------------------------------------
// K1: whole-row permutation copies (proj/src/core.cpp:141-148), bit-exact.
template <typename W>
__global__ void permute_kernel(int n, int words, const W* __restrict__ in,
                               const int32_t* __restrict__ idx, W* __restrict__ out, bool scatter) {
  const int64_t total = static_cast<int64_t>(n) * words;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / words);
    const int w = static_cast<int>(e - static_cast<int64_t>(i) * words);
    const int64_t other = static_cast<int64_t>(__ldg(idx + i)) * words + w;
    if (scatter)
      out[other] = in[e];
    else
      out[e] = in[other];
  }
}

int grid_for(int64_t threads, int block) {
  return static_cast<int>((threads + block - 1) / block);
}

}  // namespace

void launch_spmv(const knnx_operator& op, const float* x, float* y, cudaStream_t st) {
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  if (op.order == KNNX_ORDER_CLUSTER) {
    const size_t smem = static_cast<size_t>(op.max_halo) * sizeof(float);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(spmv_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    spmv_tiles_kernel<<<op.n_tiles, op.tile_rows, smem, st>>>(v, x, y);
  } else {
    spmv_orig_kernel<<<grid_for(static_cast<int64_t>(op.n_slices) * 32, 256), 256, 0, st>>>(v, x, y);
  }
}

#define KNNX_DISPATCH_NV(NVVAR, MACRO) \
  switch (NVVAR) {                     \
    case 1: MACRO(1); break;           \
    case 2: MACRO(2); break;           \
    case 3: MACRO(3); break;           \
    case 4: MACRO(4); break;           \
    case 5: MACRO(5); break;           \
    case 6: MACRO(6); break;           \
    case 7: MACRO(7); break;           \
    case 8: MACRO(8); break;           \
    case 9: MACRO(9); break;           \
    case 10: MACRO(10); break;         \
    case 11: MACRO(11); break;         \
    case 12: MACRO(12); break;         \
    case 13: MACRO(13); break;         \
    case 14: MACRO(14); break;         \
    case 15: MACRO(15); break;         \
    default: MACRO(16); break;         \
  }

#define KNNX_DISPATCH_NVL(NVVAR, MACRO) \
  switch (NVVAR) {                      \
    case 1: MACRO(1); break;            \
    case 2: MACRO(2); break;            \
    case 3: MACRO(3); break;            \
    case 4: MACRO(4); break;            \
    case 5: MACRO(5); break;            \
    case 6: MACRO(6); break;            \
    case 7: MACRO(7); break;            \
    default: MACRO(8); break;           \
  }

void launch_gauss_spmv(const knnx_operator& op, const float* t, int ld_t, const float* s,
                       int ld_s, int dim, float c2, const float* x, float* y, int* flag,
                       cudaStream_t st) {
  (void)flag;
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  const bool tiles = op.order == KNNX_ORDER_CLUSTER;
  const int nv = (dim + 3) / 4;
  if (nv <= 16) {
    const int grid = grid_for(op.n_rows, 128);
#define L(NV)                                                                                   \
  if (tiles)                                                                                    \
    gauss_rows_kernel<true, NV><<<grid, 128, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y);      \
  else                                                                                          \
    gauss_rows_kernel<false, NV><<<grid, 128, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y);
    KNNX_DISPATCH_NV(nv, L)
#undef L
  } else {
    const int nvl = (nv + 31) / 32;
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 32, 256);
#define L(NVL)                                                                                  \
  if (tiles)                                                                                    \
    gauss_warp_kernel<true, NVL><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y);     \
  else                                                                                          \
    gauss_warp_kernel<false, NVL><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y);
    KNNX_DISPATCH_NVL(nvl, L)
#undef L
  }
}

void launch_update_gaussian(const knnx_operator& op, const float* t, int ld_t, const float* s,
                            int ld_s, int dim, float c2, int* flag, cudaStream_t st) {
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  const int grid = grid_for(op.n_rows, 256);
  if (op.order == KNNX_ORDER_CLUSTER)
    update_gauss_kernel<true><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, flag);
  else
    update_gauss_kernel<false><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, flag);
}

void launch_meanshift(const knnx_operator& op, const float* t_in, int ld_t, const float* s,
                      int ld_s, int dim, float c2, float zero_thresh, float* t_out, int* flag,
                      cudaStream_t st) {
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  const bool tiles = op.order == KNNX_ORDER_CLUSTER;
  const int nv = (dim + 3) / 4;
  if (nv <= 16) {
    const int grid = grid_for(op.n_rows, 128);
#define L(NV)                                                                                  \
  if (tiles)                                                                                   \
    meanshift_rows_kernel<true, NV>                                                            \
        <<<grid, 128, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, t_out, flag);     \
  else                                                                                         \
    meanshift_rows_kernel<false, NV>                                                           \
        <<<grid, 128, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, t_out, flag);
    KNNX_DISPATCH_NV(nv, L)
#undef L
  } else {
    const int nvl = (nv + 31) / 32;
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 32, 256);
#define L(NVL)                                                                                 \
  if (tiles)                                                                                   \
    meanshift_warp_kernel<true, NVL>                                                           \
        <<<grid, 256, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, t_out, flag);     \
  else                                                                                         \
    meanshift_warp_kernel<false, NVL>                                                          \
        <<<grid, 256, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, t_out, flag);
    KNNX_DISPATCH_NVL(nvl, L)
#undef L
  }
}

void launch_tsne(const knnx_operator& op, const float* y, int dim, float* f, bool store,
                 float step, float* y_out, cudaStream_t st) {
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  const bool tiles = op.order == KNNX_ORDER_CLUSTER;
  const int grid = grid_for(op.n_rows, 256);
  const int st_flag = store ? 1 : 0;
#define L(D)                                                                                  \
  if (tiles)                                                                                  \
    tsne_rows_kernel<true, D><<<grid, 256, 0, st>>>(v, y, f, st_flag, step, y_out);           \
  else                                                                                        \
    tsne_rows_kernel<false, D><<<grid, 256, 0, st>>>(v, y, f, st_flag, step, y_out);
  switch (dim) {
    case 1: L(1); break;
    case 2: L(2); break;
    default: L(3); break;
  }
#undef L
}

void launch_permute(int n, int64_t row_bytes, const void* in, const int32_t* idx, void* out,
                    bool scatter, cudaStream_t st) {
  if (n == 0 || row_bytes == 0) return;
  if (row_bytes % 16 == 0) {
    const int words = static_cast<int>(row_bytes / 16);
    const int grid = std::min<int64_t>(grid_for(static_cast<int64_t>(n) * words, 256), 148 * 32);
    permute_kernel<uint4><<<grid, 256, 0, st>>>(n, words, static_cast<const uint4*>(in), idx,
                                                static_cast<uint4*>(out), scatter);
  } else {
    const int words = static_cast<int>(row_bytes / 4);
    const int grid = std::min<int64_t>(grid_for(static_cast<int64_t>(n) * words, 256), 148 * 32);
    permute_kernel<uint32_t><<<grid, 256, 0, st>>>(n, words, static_cast<const uint32_t*>(in), idx,
                                                   static_cast<uint32_t*>(out), scatter);
  }
}

}  // namespace knnx_dev
