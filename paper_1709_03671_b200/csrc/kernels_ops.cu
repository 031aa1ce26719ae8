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
#include <cstdlib>
#include <type_traits>

#include "knnx_internal.cuh"
#include "ptx.cuh"

#ifndef KNNX_TSNE_U
#define KNNX_TSNE_U 4
#endif

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

OpView view_of(const knnx_operator& op) {
  return OpView{op.d_slice_off, op.d_slice_len, op.d_row_len, op.d_cols,  op.d_lidx,
                op.d_halo_off,  op.d_halo_ids,  op.d_vals,    op.n_rows,  op.n_slices,
                op.tile_rows,   op.row_base,    op.d_slot_row};
}

// only the t-SNE kernels read the relabelled / group-interleaved layouts
void require_plain(const knnx_operator& op) {
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
  if (row < v.n_rows) y[real_row(v, row)] = acc;
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
  if (row < v.n_rows) y[real_row(v, row)] = acc;
}

// K3 (default): one CTA per tile like spmv_tiles_kernel, but the row's slice
// header is loaded before the stage and the x[halo] stage is unrolled kG-wide
// (kG independent id loads, then kG independent x gathers), so staging costs
// ~3 dependent memory latencies instead of two per halo id.
template <int kG, bool kPdl = false>
__global__ void __launch_bounds__(1024) spmv_tiles_g_kernel(OpView v, const float* __restrict__ x,
                                                            float* __restrict__ y) {
  extern __shared__ float sx[];
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int R = blockDim.x;  // == tile_rows
  const int row = tile * R + tid;
  const int s = row >> 5;
  const bool live = s < v.n_slices;
  const int64_t base = live ? v.slice_off[s] + (tid & 31) : 0;
  const int len = live ? v.slice_len[s] : 0;
  const int64_t h0 = v.halo_off[tile];
  const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
  if constexpr (kPdl) {
    // programmatic dependent launch: the header loads above overlap the
    // previous launch's tail; x (possibly produced by it) is read only after
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  for (int j0 = tid; j0 < H; j0 += R * kG) {
    int id[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) id[g] = j0 + R * g < H ? __ldg(v.halo_ids + h0 + j0 + R * g) : 0;
    float xv[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) xv[g] = __ldg(x + id[g]);
#pragma unroll
    for (int g = 0; g < kG; ++g)
      if (j0 + R * g < H) sx[j0 + R * g] = xv[g];
  }
  __syncthreads();
  if (!live) return;
  float acc = 0.0f;
#pragma unroll 10
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    acc = fmaf(ld_stream(v.vals + p), sx[ld_stream(v.lidx + p)], acc);
  }
  if (row < v.n_rows) y[real_row(v, row)] = acc;
}

// K3 (prefetching, one CTA per tile): before touching x, every thread issues
// the loads of its row's first kPF values/indices and of its share of the
// halo ids (all independent of x), so HBM streams while the dependent x[halo]
// gathers run; with programmatic dependent launch (kPdl) this prologue also
// overlaps the previous launch's tail -- griddepcontrol.wait sits right before
// the first read of x, so a kernel that produced x is complete by then.
template <int kPF, bool kPdl>
__global__ void __launch_bounds__(128) spmv_tiles_pf_kernel(OpView v, const float* __restrict__ x,
                                                            float* __restrict__ y) {
  extern __shared__ float sx[];
  constexpr int kG = 8;  // halo ids per thread per gather round
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t h0 = v.halo_off[tile];
  const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
  const int row = tile * 128 + tid;
  const int s = row >> 5;
  const bool live = s < v.n_slices;
  const int64_t base = live ? v.slice_off[s] + (tid & 31) : 0;
  const int len = live ? v.slice_len[s] : 0;
  float pv[kPF];
  int pl[kPF];
#pragma unroll
  for (int u = 0; u < kPF; ++u) {
    pv[u] = u < len ? ld_stream(v.vals + base + 32 * u) : 0.0f;
    pl[u] = u < len ? ld_stream(v.lidx + base + 32 * u) : 0;
  }
  int id[kG];
#pragma unroll
  for (int g = 0; g < kG; ++g) {
    const int j = tid + 128 * g;
    id[g] = j < H ? __ldg(v.halo_ids + h0 + j) : 0;
  }
  if constexpr (kPdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  float xv[kG];
#pragma unroll
  for (int g = 0; g < kG; ++g) xv[g] = tid + 128 * g < H ? __ldg(x + id[g]) : 0.0f;
#pragma unroll
  for (int g = 0; g < kG; ++g)
    if (tid + 128 * g < H) sx[tid + 128 * g] = xv[g];
  for (int j = tid + 128 * kG; j < H; j += 128) sx[j] = __ldg(x + __ldg(v.halo_ids + h0 + j));
  __syncthreads();
  if (!live) return;
  float acc = 0.0f;
#pragma unroll
  for (int u = 0; u < kPF; ++u)
    if (u < len) acc = fmaf(pv[u], sx[pl[u]], acc);
#pragma unroll 8
  for (int q = kPF; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    acc = fmaf(ld_stream(v.vals + p), sx[ld_stream(v.lidx + p)], acc);
  }
  if (row < v.n_rows) y[real_row(v, row)] = acc;
}

// K3 (pipelined, the default for tile_rows == 128): persistent CTAs walk
// their tiles t = blockIdx.x + i * gridDim.x through a 2-stage shared-memory
// ring.  One thread streams each tile's values, 16-bit indices and halo ids
// with TMA bulk copies (cp.async.bulk -> mbarrier complete_tx, L2 evict-first:
// they are read once) two tiles ahead; all threads gather x[halo] for tile
// i+1 into registers while computing tile i from shared memory, so neither
// the HBM stream nor the L2 gather latency sits on the critical path.
template <int GMAX>
__global__ void __launch_bounds__(128) spmv_tiles_tma_kernel(OpView v, const float* __restrict__ x,
                                                             float* __restrict__ y, int e_max,
                                                             int h_max) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lidx_bytes = (e_max * 2 + 15) / 16 * 16;
  const int stage_bytes = e_max * 4 + lidx_bytes + h_max * 4;
  float* sx = reinterpret_cast<float*>(smem + 2 * stage_bytes);  // [2][h_max]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sx + 2 * h_max);
  const int tid = threadIdx.x;
  const int tps = 4;  // slices per 128-row tile
  const int n_tiles = (v.n_slices + tps - 1) / tps;
  const int first = blockIdx.x, stride = gridDim.x;
  if (first >= n_tiles) return;

  auto stage_vals = [&](int s) { return reinterpret_cast<float*>(smem + s * stage_bytes); };
  auto stage_lidx = [&](int s) {
    return reinterpret_cast<uint16_t*>(smem + s * stage_bytes + e_max * 4);
  };
  auto stage_halo = [&](int s) {
    return reinterpret_cast<int32_t*>(smem + s * stage_bytes + e_max * 4 + lidx_bytes);
  };
  auto issue = [&](int t, int s, uint64_t pol) {
    const int s0 = t * tps, s1 = min(s0 + tps, v.n_slices);
    const int64_t e0 = v.slice_off[s0];
    const uint32_t cnt = static_cast<uint32_t>(v.slice_off[s1] - e0);
    const int64_t h0 = v.halo_off[t];
    const uint32_t hc = static_cast<uint32_t>(v.halo_off[t + 1] - h0);
    mbar_arrive_expect_tx(&bars[s], cnt * 6u + hc * 4u);
    if (cnt) {
      bulk_g2s(stage_vals(s), v.vals + e0, cnt * 4u, &bars[s], pol);
      bulk_g2s(stage_lidx(s), v.lidx + e0, cnt * 2u, &bars[s], pol);
    }
    if (hc) bulk_g2s(stage_halo(s), v.halo_ids + h0, hc * 4u, &bars[s], pol);
  };

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  if (tid == 0) {
    issue(first, 0, pol);
    if (first + stride < n_tiles) issue(first + stride, 1, pol);
  }

  float g[GMAX];
  auto gather = [&](int t, int s) {  // x[halo] of tile t (stage s) -> registers
    const int hc = static_cast<int>(v.halo_off[t + 1] - v.halo_off[t]);
    const int32_t* hs = stage_halo(s);
#pragma unroll
    for (int u = 0; u < GMAX; ++u) {
      const int j = tid + 128 * u;
      g[u] = j < hc ? __ldg(x + hs[j]) : 0.0f;
    }
  };
  auto park = [&](int t, float* dst) {
    const int hc = static_cast<int>(v.halo_off[t + 1] - v.halo_off[t]);
#pragma unroll
    for (int u = 0; u < GMAX; ++u) {
      const int j = tid + 128 * u;
      if (j < hc) dst[j] = g[u];
    }
  };

  mbar_wait(&bars[0], 0);
  gather(first, 0);
  park(first, sx);
  __syncthreads();

  int i = 0;
  for (int t = first; t < n_tiles; t += stride, ++i) {
    const int s = i & 1;
    const int tn = t + stride;
    if (tn < n_tiles) {  // prefetch the next tile's x[halo] into registers
      mbar_wait(&bars[s ^ 1], ((i + 1) >> 1) & 1);
      gather(tn, s ^ 1);
    }
    // compute tile t from stage s
    const int row = t * 128 + tid;
    const int sl = row >> 5;
    if (sl < v.n_slices) {
      const int64_t e0 = v.slice_off[t * tps];
      const int base = static_cast<int>(v.slice_off[sl] - e0) + (tid & 31);
      const int len = v.slice_len[sl];
      const float* vs = stage_vals(s);
      const uint16_t* ls = stage_lidx(s);
      const float* xs = sx + s * h_max;
      float acc = 0.0f;
#pragma unroll 6
      for (int q = 0; q < len; ++q) acc = fmaf(vs[base + 32 * q], xs[ls[base + 32 * q]], acc);
      if (row < v.n_rows) y[real_row(v, row)] = acc;
    }
    if (tn < n_tiles) park(tn, sx + (s ^ 1) * h_max);
    __syncthreads();  // stage s and sx[s] are free; sx[s^1] is complete
    if (tid == 0 && tn + stride < n_tiles) issue(tn + stride, s, pol);
  }
}

// K3 (bulk, one CTA per tile): thread 0 starts two TMA bulk copies at CTA
// entry -- the tile's halo ids (one mbarrier) and its values + 16-bit indices
// (another) -- so the value stream is in flight while the threads gather
// x[halo] (in place over the staged ids) and meet at the barrier.
__global__ void __launch_bounds__(128) spmv_tiles_bulk_kernel(OpView v, const float* __restrict__ x,
                                                              float* __restrict__ y, int e_max) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lidx_bytes = (e_max * 2 + 15) / 16 * 16;
  float* vs = reinterpret_cast<float*>(smem);
  uint16_t* ls = reinterpret_cast<uint16_t*>(smem + e_max * 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + e_max * 4 + lidx_bytes);
  int32_t* hx = reinterpret_cast<int32_t*>(bars + 2);  // halo ids, then x[halo] in place
  const int tid = threadIdx.x;
  const int t = blockIdx.x;
  const int s0 = t * 4, s1 = min(s0 + 4, v.n_slices);
  const int64_t e0 = v.slice_off[s0];
  const uint32_t cnt = static_cast<uint32_t>(v.slice_off[s1] - e0);
  const int64_t h0 = v.halo_off[t];
  const int hc = static_cast<int>(v.halo_off[t + 1] - h0);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&bars[0], static_cast<uint32_t>(hc) * 4u);
    if (hc) bulk_g2s(hx, v.halo_ids + h0, static_cast<uint32_t>(hc) * 4u, &bars[0], pol);
    mbar_arrive_expect_tx(&bars[1], cnt * 6u);
    if (cnt) {
      bulk_g2s(vs, v.vals + e0, cnt * 4u, &bars[1], pol);
      bulk_g2s(ls, v.lidx + e0, cnt * 2u, &bars[1], pol);
    }
  }
  __syncthreads();
  mbar_wait(&bars[0], 0);
  float* sx = reinterpret_cast<float*>(hx);
  for (int j = tid; j < hc; j += 128) sx[j] = __ldg(x + hx[j]);
  __syncthreads();
  mbar_wait(&bars[1], 0);
  const int row = t * 128 + tid;
  const int sl = row >> 5;
  if (sl >= v.n_slices) return;
  const int base = static_cast<int>(v.slice_off[sl] - e0) + (tid & 31);
  const int len = v.slice_len[sl];
  float acc = 0.0f;
#pragma unroll 6
  for (int q = 0; q < len; ++q) acc = fmaf(vs[base + 32 * q], sx[ls[base + 32 * q]], acc);
  if (row < v.n_rows) y[real_row(v, row)] = acc;
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

// ---------------------------------------------------------------------------
// K4/K5 on cluster tiles (default for dim <= 64): one CTA per tile, eight
// lanes (an "octet") per row.  The tile's halo source rows are staged in
// shared memory with cp.async (16-B LDGSTS), up to `cap` rows (the rest read
// from L2).  Inside an octet, lane l owns float4 chunks l, l+8 of every row,
// so one step of the neighbor loop reads 128 contiguous shared-memory bytes
// per row -- bank-conflict-free for any gather order -- and three xor
// shuffles finish |t_i - s_j|^2 in every lane.  Each source row is fetched
// from L2 once per tile instead of once per (row, neighbor).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int NC, bool kMeanShift>
__global__ void __launch_bounds__(1024) nonstat_octet_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, const float* __restrict__ x, float* __restrict__ out,
    int* flag, int cap, int e_max) {
  extern __shared__ __align__(16) float sh[];
  const int tile = blockIdx.x;
  const int R = v.tile_rows;
  const int tid = threadIdx.x;
  const int lane8 = tid & 7;
  const int nv4 = (dim + 3) >> 2;
  const int64_t h0 = v.halo_off[tile];
  const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
  const int Hs = min(H, cap);
  // shared layout: [cap x ld_s halo rows][e_max 16-bit indices][x[halo] (Gaussian only)]
  uint16_t* sl = reinterpret_cast<uint16_t*>(sh + static_cast<size_t>(cap) * ld_s);
  float* sxs = reinterpret_cast<float*>(sl + (e_max + 7) / 8 * 8);
  // stage the tile's halo rows, its 16-bit index stream and x[halo]
  const int s0 = tile * (R >> 5);
  const int64_t e0 = v.slice_off[s0];
  const int ecount = static_cast<int>(v.slice_off[min(s0 + (R >> 5), v.n_slices)] - e0);
  for (int e = tid; e < ecount / 8; e += blockDim.x)  // 8 indices per 16-B chunk
    cp_async16(sl + 8 * e, v.lidx + e0 + 8 * e);
  for (int e = tid; e < Hs * nv4; e += blockDim.x) {
    const int r = e / nv4, c = e - r * nv4;
    const int j = __ldg(v.halo_ids + h0 + r);
    cp_async16(sh + static_cast<size_t>(r) * ld_s + 4 * c, s + static_cast<int64_t>(j) * ld_s + 4 * c);
  }
  if constexpr (!kMeanShift)
    for (int r = tid; r < H; r += blockDim.x) sxs[r] = __ldg(x + __ldg(v.halo_ids + h0 + r));
  const int row_in_tile = tid >> 3;
  const int row = tile * R + row_in_tile;
  const bool live = row_in_tile < R && row < v.n_rows;
  float4 ti[NC], acc[NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = lane8 + 8 * u;
    ti[u] = (live && c < nv4) ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(real_row(v, row)) * ld_t) + c)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  cp_async_wait_all();
  __syncthreads();
  if (!live) return;
  const int base = static_cast<int>(v.slice_off[row >> 5] - e0) + (row & 31);
  const int len = v.row_len[row];
  float m = INFINITY, tot = 0.0f, accx = 0.0f;
#pragma unroll 2
  for (int q = 0; q < len; ++q) {
    const int l = sl[base + 32 * q];
    const float* sp = l < Hs ? sh + static_cast<size_t>(l) * ld_s
                             : s + static_cast<int64_t>(__ldg(v.halo_ids + h0 + l)) * ld_s;
    float4 sj[NC];
    float d2 = 0.0f;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int c = lane8 + 8 * u;
      if (c < nv4) {
        sj[u] = reinterpret_cast<const float4*>(sp)[c];
        d2 += sqdiff4(ti[u], sj[u], 4 * c, dim);
      } else {
        sj[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    d2 += __shfl_xor_sync(0xffffffffu, d2, 1);
    d2 += __shfl_xor_sync(0xffffffffu, d2, 2);
    d2 += __shfl_xor_sync(0xffffffffu, d2, 4);
    if constexpr (kMeanShift) {
      if (d2 < m) {
        const float sc = exp2f((d2 - m) * c2);
        tot *= sc;
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          acc[u].x *= sc; acc[u].y *= sc; acc[u].z *= sc; acc[u].w *= sc;
        }
        m = d2;
      }
      const float w = exp2f((m - d2) * c2);
      tot += w;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        acc[u].x = fmaf(w, sj[u].x, acc[u].x);
        acc[u].y = fmaf(w, sj[u].y, acc[u].y);
        acc[u].z = fmaf(w, sj[u].z, acc[u].z);
        acc[u].w = fmaf(w, sj[u].w, acc[u].w);
      }
    } else {
      const float xj = l < H ? sxs[l] : 0.0f;
      accx = fmaf(exp2f(-d2 * c2), xj, accx);
    }
  }
  if constexpr (kMeanShift) {
    if (lane8 == 0 && (len == 0 || m > zero_thresh)) flag_error(flag, kFlagZeroWeight, real_row(v, row));
    const float inv = 1.0f / tot;
    float4* op = reinterpret_cast<float4*>(out + static_cast<int64_t>(real_row(v, row)) * ld_t);
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int c = lane8 + 8 * u;
      if (c < nv4)
        op[c] = make_float4(acc[u].x * inv, acc[u].y * inv, acc[u].z * inv, acc[u].w * inv);
    }
  } else {
    if (lane8 == 0) out[real_row(v, row)] = accx;
  }
}

// K4/K5 octet variant without staging: 8 lanes per row read each source row
// as 128-B coalesced segments straight from L1/L2; the octet fetches the next
// 8 neighbor ids cooperatively (one index chain per lane) and broadcasts them
// by shuffle, so index latency is paid once per 8 neighbors.
template <bool kTiles, int NC, bool kMeanShift>
__global__ void __launch_bounds__(256) nonstat_octet_l1_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, const float* __restrict__ x, float* __restrict__ out,
    int* flag) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gt >> 3;  // slot
  const int lane8 = threadIdx.x & 7;
  if (row >= v.n_rows) return;  // whole octets exit together
  const unsigned mask = 0xffu << (threadIdx.x & 24);
  const int nv4 = (dim + 3) >> 2;
  const int rr = real_row(v, row);
  float4 ti[NC], acc[NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = lane8 + 8 * u;
    ti[u] = c < nv4 ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(rr) * ld_t) + c)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t base = v.slice_off[row >> 5] + (row & 31);
  const int len = v.row_len[row];
  const int64_t hbase = kTiles ? v.halo_off[row / v.tile_rows] : 0;
  float m = INFINITY, tot = 0.0f, accx = 0.0f;
  for (int q0 = 0; q0 < len; q0 += 8) {
    const int q = q0 + lane8;
    int jl = 0;
    float xl = 0.0f;
    if (q < len) {
      jl = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q), hbase);
      if constexpr (!kMeanShift) xl = __ldg(x + jl);
    }
    const int cnt = min(8, len - q0);
    for (int u8 = 0; u8 < cnt; ++u8) {
      const int j = __shfl_sync(mask, jl, u8, 8);
      const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
      float4 sj[NC];
      float d2 = 0.0f;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int c = lane8 + 8 * u;
        sj[u] = c < nv4 ? __ldg(sp + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        d2 += sqdiff4(ti[u], sj[u], 4 * c, dim);
      }
      d2 += __shfl_xor_sync(mask, d2, 1, 8);
      d2 += __shfl_xor_sync(mask, d2, 2, 8);
      d2 += __shfl_xor_sync(mask, d2, 4, 8);
      if constexpr (kMeanShift) {
        if (d2 < m) {
          const float sc = exp2f((d2 - m) * c2);
          tot *= sc;
#pragma unroll
          for (int u = 0; u < NC; ++u) {
            acc[u].x *= sc; acc[u].y *= sc; acc[u].z *= sc; acc[u].w *= sc;
          }
          m = d2;
        }
        const float w = exp2f((m - d2) * c2);
        tot += w;
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          acc[u].x = fmaf(w, sj[u].x, acc[u].x);
          acc[u].y = fmaf(w, sj[u].y, acc[u].y);
          acc[u].z = fmaf(w, sj[u].z, acc[u].z);
          acc[u].w = fmaf(w, sj[u].w, acc[u].w);
        }
      } else {
        accx = fmaf(exp2f(-d2 * c2), __shfl_sync(mask, xl, u8, 8), accx);
      }
    }
  }
  if constexpr (kMeanShift) {
    if (lane8 == 0 && (len == 0 || m > zero_thresh)) flag_error(flag, kFlagZeroWeight, rr);
    const float inv = 1.0f / tot;
    float4* op = reinterpret_cast<float4*>(out + static_cast<int64_t>(rr) * ld_t);
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int c = lane8 + 8 * u;
      if (c < nv4)
        op[c] = make_float4(acc[u].x * inv, acc[u].y * inv, acc[u].z * inv, acc[u].w * inv);
    }
  } else {
    if (lane8 == 0) out[rr] = accx;
  }
}

// K4/K5 lane-group variant (default, dim <= 64): G lanes per row, lane g
// owning float4 chunks g, g+G, ...; a source row is read as G*16-B contiguous
// segments.  Arithmetic runs on packed fp32x2 (FFMA2, sm_100): with per-lane
// masks m (1 for live components, 0 for padding) and tm = t*m precomputed,
// d = s*(-m) + tm and acc += d*d cost one FFMA2 each per two components.
// The whole warp iterates to the longest row it holds (lanes of shorter rows
// are predicated off), so every shuffle is full-warp.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

template <bool kTiles, int G, int NC, bool kMeanShift, bool kStore = false, int NB = 1>
__global__ void __launch_bounds__(256) nonstat_group_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, const float* __restrict__ x, float* __restrict__ out,
    int* flag) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gt / G;
  const int g = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const int gbase = lane - g;  // first lane of this row's group
  const bool live = slot < v.n_rows;
  const int nv4 = (dim + 3) >> 2;
  const int rr = live ? real_row(v, slot) : 0;
  float2 tm[2 * NC], nm[2 * NC], acc[2 * NC];
  bool has[NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = g + G * u;
    has[u] = c < nv4;
    const float4 tv = (live && has[u])
        ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(rr) * ld_t) + c)
        : make_float4(0.f, 0.f, 0.f, 0.f);
    const float m0 = 4 * c + 0 < dim ? 1.f : 0.f, m1 = 4 * c + 1 < dim ? 1.f : 0.f;
    const float m2 = 4 * c + 2 < dim ? 1.f : 0.f, m3 = 4 * c + 3 < dim ? 1.f : 0.f;
    tm[2 * u] = f2(tv.x * m0, tv.y * m1);
    tm[2 * u + 1] = f2(tv.z * m2, tv.w * m3);
    nm[2 * u] = f2(-m0, -m1);
    nm[2 * u + 1] = f2(-m2, -m3);
    acc[2 * u] = f2(0.f, 0.f);
    acc[2 * u + 1] = f2(0.f, 0.f);
  }
  const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int64_t hbase = (kTiles && live) ? v.halo_off[slot / v.tile_rows] : 0;
  const int wmax = __reduce_max_sync(0xffffffffu, len);
  float m = INFINITY, tot = 0.0f, accx = 0.0f;
  for (int q0 = 0; q0 < wmax; q0 += G) {
    const int qg = q0 + g;
    int jl = 0;
    float xl = 0.0f;
    if (qg < len) {
      jl = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(qg), hbase);
      if constexpr (!kMeanShift && !kStore) xl = __ldg(x + jl);
    }
    // neighbors in batches of NB: NB = 2 (default) keeps two source rows in
    // flight per lane at 64 registers, 7% faster than NB = 1 (variant 5) on
    // C3; NB = 4 was slower (89 registers, lower occupancy)
#pragma unroll
    for (int b0 = 0; b0 < G; b0 += NB) {
      float2 sj[NB][2 * NC];
      float d2[NB];
      bool ok[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = __shfl_sync(0xffffffffu, jl, gbase + b0 + b);
        ok[b] = q0 + b0 + b < len;
        const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float4 sv =
              (ok[b] && has[u]) ? __ldg(sp + g + G * u) : make_float4(0.f, 0.f, 0.f, 0.f);
          sj[b][2 * u] = f2(sv.x, sv.y);
          sj[b][2 * u + 1] = f2(sv.z, sv.w);
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float2 dd = f2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float2 d0 = __ffma2_rn(sj[b][2 * u], nm[2 * u], tm[2 * u]);
          const float2 d1 = __ffma2_rn(sj[b][2 * u + 1], nm[2 * u + 1], tm[2 * u + 1]);
          dd = __ffma2_rn(d0, d0, dd);
          dd = __ffma2_rn(d1, d1, dd);
        }
        d2[b] = dd.x + dd.y;
      }
#pragma unroll
      for (int o = 1; o < G; o <<= 1)
#pragma unroll
        for (int b = 0; b < NB; ++b) d2[b] += __shfl_xor_sync(0xffffffffu, d2[b], o);
      if constexpr (kMeanShift) {
        float mb = m;
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (ok[b]) mb = fminf(mb, d2[b]);
        if (mb < m) {
          const float sc = exp2f((mb - m) * c2);
          tot *= sc;
          const float2 sc2 = f2(sc, sc);
#pragma unroll
          for (int w = 0; w < 2 * NC; ++w) acc[w] = __fmul2_rn(acc[w], sc2);
          m = mb;
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (!ok[b]) continue;
          const float w = exp2f((m - d2[b]) * c2);
          tot += w;
          const float2 w2 = f2(w, w);
#pragma unroll
          for (int q = 0; q < 2 * NC; ++q) acc[q] = __ffma2_rn(w2, sj[b][q], acc[q]);
        }
      } else {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const float xj = __shfl_sync(0xffffffffu, xl, gbase + b0 + b);
          if constexpr (kStore) {  // update_values(Gaussian): store the weight
            if (ok[b] && g == b0 + b) {
              const float w = exp2f(-d2[b] * c2);
              if (!isfinite(w)) flag_error(flag, kFlagNonFinite, rr);
              v.vals[base + 32 * static_cast<int64_t>(q0 + b0 + b)] = w;
            }
          } else {
            if (ok[b]) accx = fmaf(exp2f(-d2[b] * c2), xj, accx);
          }
        }
      }
    }
  }
  if (!live) return;
  if constexpr (kMeanShift) {
    if (g == 0 && (len == 0 || m > zero_thresh)) flag_error(flag, kFlagZeroWeight, rr);
    const float inv = 1.0f / tot;
    float4* op = reinterpret_cast<float4*>(out + static_cast<int64_t>(rr) * ld_t);
#pragma unroll
    for (int u = 0; u < NC; ++u)
      if (has[u])
        op[g + G * u] = make_float4(acc[2 * u].x * inv, acc[2 * u].y * inv, acc[2 * u + 1].x * inv,
                                    acc[2 * u + 1].y * inv);
  } else if constexpr (!kStore) {
    if (g == 0) out[rr] = accx;
  }
}

// K5 mean shift, lean lane-group kernel (default for dim <= 64, variant 0):
// the lane-group layout of nonstat_group_kernel with the per-neighbour
// instruction count cut from ~58 to ~30 per lane (SASS-counted):
//  * no predicated loads: a lane whose float4 chunk lies past the row re-reads
//    the row's last chunk (same 128-B line) with zero masks, and a finished
//    row's slots read a valid source with weight exactly 0 (d2 = +inf), so
//    every load and FFMA2 issues unconditionally;
//  * the weight reference m (w = 2^((m - d2) c2), the result is normalised so
//    any m gives the same positions) moves only when a new distance is 2^64
//    below it, decided by one warp vote: the rescale branch is warp-uniform
//    and almost never taken after a row's first batch;
//  * ex2.approx.ftz (MUFU.EX2, ~2 ulp) for the weights.
// The exact minimum distance is still tracked for ZeroWeight (every fp64
// reference weight underflows, proj/src/kernels.cpp:204-206).
__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool kTiles, int NC, int kMinBlocks, int NB = 2, int G = 8>
__global__ void __launch_bounds__(256, kMinBlocks) meanshift_lane_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, float* __restrict__ out, int* flag) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gt / G;
  const int g = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const int gbase = lane - g;
  const bool live = slot < v.n_rows;
  const int nv4 = (dim + 3) >> 2;
  const int rr = live ? real_row(v, slot) : 0;
  // NC = ceil(ceil(dim/4) / 8): chunks g + 8u with u < NC - 1 are always
  // whole rows of 4 live components (no mask, no clamp: fewer registers);
  // only the last chunk index can be partial or past the row
  int cidx[NC];
  float2 tm[2 * NC], nm[2], acc[2 * NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = g + G * u;
    const bool last = u == NC - 1;
    const bool has = !last || c < nv4;
    cidx[u] = has ? c : nv4 - 1;
    const float4 tv =
        live ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(rr) * ld_t) + cidx[u])
             : make_float4(0.f, 0.f, 0.f, 0.f);
    if (last) {
      const float m0 = has && 4 * c + 0 < dim ? 1.f : 0.f, m1 = has && 4 * c + 1 < dim ? 1.f : 0.f;
      const float m2 = has && 4 * c + 2 < dim ? 1.f : 0.f, m3 = has && 4 * c + 3 < dim ? 1.f : 0.f;
      tm[2 * u] = f2(tv.x * m0, tv.y * m1);
      tm[2 * u + 1] = f2(tv.z * m2, tv.w * m3);
      nm[0] = f2(-m0, -m1);
      nm[1] = f2(-m2, -m3);
    } else {
      tm[2 * u] = f2(tv.x, tv.y);
      tm[2 * u + 1] = f2(tv.z, tv.w);
    }
    acc[2 * u] = f2(0.f, 0.f);
    acc[2 * u + 1] = f2(0.f, 0.f);
  }
  const float2 neg1 = f2(-1.f, -1.f);
  const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int64_t hbase = (kTiles && live) ? v.halo_off[slot / v.tile_rows] : 0;
  const int wmax = __reduce_max_sync(0xffffffffu, len);
  const float4* s4 = reinterpret_cast<const float4*>(s);
  const int ld4 = ld_s >> 2;
  float m = INFINITY, mc2 = INFINITY, dmin = INFINITY, tot = 0.0f;
  // neighbour ids one block of G ahead: the dependent id loads (16-bit halo
  // index, then halo id) of block q0 + G overlap block q0's arithmetic
  int jn = 0;  // a finished slot reads source 0 (valid) and weighs it 0
  if (g < len) jn = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(g), hbase);
  for (int q0 = 0; q0 < wmax; q0 += G) {
    const int jl = jn;
    const int qn = q0 + G + g;
    jn = 0;
    if (qn < len) jn = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(qn), hbase);
#pragma unroll
    for (int b0 = 0; b0 < G; b0 += NB) {
      if (q0 + b0 >= wmax) break;  // warp-uniform
      float2 sj[NB][2 * NC];
      float d2[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        // 32-bit element offsets (n_src * ld_s < 2^31 is checked by the launcher)
        const int j = __shfl_sync(0xffffffffu, jl, gbase + b0 + b);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float4 sv = __ldg(s4 + (j * ld4 + cidx[u]));
          sj[b][2 * u] = f2(sv.x, sv.y);
          sj[b][2 * u + 1] = f2(sv.z, sv.w);
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float2 dd = f2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float2 e0 = __ffma2_rn(sj[b][2 * u], u == NC - 1 ? nm[0] : neg1, tm[2 * u]);
          const float2 e1 = __ffma2_rn(sj[b][2 * u + 1], u == NC - 1 ? nm[1] : neg1, tm[2 * u + 1]);
          dd = __ffma2_rn(e0, e0, dd);
          dd = __ffma2_rn(e1, e1, dd);
        }
        d2[b] = dd.x + dd.y;
      }
#pragma unroll
      for (int o = 1; o < G; o <<= 1)
#pragma unroll
        for (int b = 0; b < NB; ++b) d2[b] += __shfl_xor_sync(0xffffffffu, d2[b], o);
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (q0 + b0 + b >= len) d2[b] = INFINITY;
      float mb = d2[0];
#pragma unroll
      for (int b = 1; b < NB; ++b) mb = fminf(mb, d2[b]);
      dmin = fminf(dmin, mb);
      const bool need = (m - mb) * c2 > 64.0f;
      if (__any_sync(0xffffffffu, need)) {  // rare after a row's first batch
        const float sc = need ? ex2_fast((mb - m) * c2) : 1.0f;
        tot *= sc;
        const float2 sc2 = f2(sc, sc);
#pragma unroll
        for (int w = 0; w < 2 * NC; ++w) acc[w] = __fmul2_rn(acc[w], sc2);
        m = need ? mb : m;
        mc2 = m * c2;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const float w = ex2_fast(fmaf(-d2[b], c2, mc2));  // d2 = +inf -> 0
        tot += w;
        const float2 w2 = f2(w, w);
#pragma unroll
        for (int q = 0; q < 2 * NC; ++q) acc[q] = __ffma2_rn(w2, sj[b][q], acc[q]);
      }
    }
  }
  if (!live) return;
  if (g == 0 && (len == 0 || dmin > zero_thresh)) flag_error(flag, kFlagZeroWeight, rr);
  const float inv = 1.0f / tot;
  float4* op = reinterpret_cast<float4*>(out + static_cast<int64_t>(rr) * ld_t);
#pragma unroll
  for (int u = 0; u < NC; ++u)
    if (g + G * u < nv4)
      op[g + G * u] = make_float4(acc[2 * u].x * inv, acc[2 * u].y * inv, acc[2 * u + 1].x * inv,
                                  acc[2 * u + 1].y * inv);
}

// K5 mean shift, neighbour-parallel mapping (variant 10): one
// warp per row, 8 groups of 4 lanes, group n takes neighbours n, n+8, ... of
// the row and lane c of a group owns the float4 chunks c, c+4, ... of the NF
// whole 16-float rounds, plus the tail past 16 NF: one scalar (element
// 16 NF + c, TAIL = 1, dim - 16 NF <= 4) or one masked float4 (TAIL = 2).
// The per-neighbour distance needs a 2-step butterfly (3 across 8 lanes in
// meanshift_lane_kernel) and each group keeps its own weight reference m; the
// groups are combined once per row (smallest reference, rescale, sum through
// shared memory).  Same weights and ZeroWeight rule as meanshift_lane_kernel
// (proj/src/kernels.cpp:184-215); only the fp32 summation order differs.
template <bool kTiles, int NF, int TAIL>
__global__ void __launch_bounds__(256, 4) meanshift_np_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, float* __restrict__ out, int* flag) {
  __shared__ __align__(16) float red[8][8][64];  // [warp][group][element]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * 8 + warp;
  if (slot >= v.n_rows) return;  // warp-uniform; only __syncwarp below
  const int n = lane >> 2, c = lane & 3;
  const int rr = real_row(v, slot);
  const float* trow = t + static_cast<int64_t>(rr) * ld_t;
  float2 tm[2 * NF + 2], acc[2 * NF + 2], nm[2];
  float tms = 0.f, accs = 0.f, nms = 0.f;
  const int te = 16 * NF + (TAIL == 1 ? c : 4 * c);  // first tail element of this lane
#pragma unroll
  for (int u = 0; u < NF; ++u) {
    const float4 tv = __ldg(reinterpret_cast<const float4*>(trow) + c + 4 * u);
    tm[2 * u] = f2(tv.x, tv.y);
    tm[2 * u + 1] = f2(tv.z, tv.w);
  }
#pragma unroll
  for (int r = 0; r < 2 * NF + 2; ++r) acc[r] = f2(0.f, 0.f);
  int tidx = 0;  // tail: clamped element (TAIL 1) / float4 chunk (TAIL 2) index
  if constexpr (TAIL == 1) {
    const bool has = te < dim;
    tidx = has ? te : dim - 1;
    nms = has ? -1.f : 0.f;
    tms = has ? __ldg(trow + tidx) : 0.f;
  } else if constexpr (TAIL == 2) {
    const int nv4 = (dim + 3) >> 2;
    const int ch = 4 * NF + c;
    tidx = ch < nv4 ? ch : nv4 - 1;
    const float4 tv = __ldg(reinterpret_cast<const float4*>(trow) + tidx);
    const float m0 = 4 * ch + 0 < dim ? 1.f : 0.f, m1 = 4 * ch + 1 < dim ? 1.f : 0.f;
    const float m2 = 4 * ch + 2 < dim ? 1.f : 0.f, m3 = 4 * ch + 3 < dim ? 1.f : 0.f;
    tm[2 * NF] = f2(tv.x * m0, tv.y * m1);
    tm[2 * NF + 1] = f2(tv.z * m2, tv.w * m3);
    nm[0] = f2(-m0, -m1);
    nm[1] = f2(-m2, -m3);
  }
  const float2 neg1 = f2(-1.f, -1.f);
  const int64_t base = v.slice_off[slot >> 5] + (slot & 31);
  const int len = v.row_len[slot];
  const int64_t hbase = kTiles ? v.halo_off[slot / v.tile_rows] : 0;
  const float4* s4 = reinterpret_cast<const float4*>(s);
  const int ld4 = ld_s >> 2;
  float m = INFINITY, mc2 = INFINITY, dmin = INFINITY, tot = 0.0f;
  // ids one round of 8 ahead; a slot past the row reads source 0, weight 0
  auto col_at = [&](int q) -> int {
    const int64_t pos = base + 32 * static_cast<int64_t>(q);
    if constexpr (kTiles)
      return __ldg(v.halo_ids + hbase + __ldg(reinterpret_cast<const unsigned short*>(v.lidx + pos)));
    else
      return __ldg(v.cols + pos);
  };
  int jn = n < len ? col_at(n) : 0;
  for (int q0 = 0; q0 < len; q0 += 8) {  // len is warp-uniform
    const int q = q0 + n;
    const int j = jn;
    jn = q + 8 < len ? col_at(q + 8) : 0;
    float2 sj[2 * NF + 2];
    float sjs = 0.f;
#pragma unroll
    for (int u = 0; u < NF; ++u) {
      const float4 sv = __ldg(s4 + (j * ld4 + c + 4 * u));
      sj[2 * u] = f2(sv.x, sv.y);
      sj[2 * u + 1] = f2(sv.z, sv.w);
    }
    if constexpr (TAIL == 1) sjs = __ldg(s + (j * ld_s + tidx));
    if constexpr (TAIL == 2) {
      const float4 sv = __ldg(s4 + (j * ld4 + tidx));
      sj[2 * NF] = f2(sv.x, sv.y);
      sj[2 * NF + 1] = f2(sv.z, sv.w);
    }
    float2 dd = f2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < NF; ++u) {
      const float2 e0 = __ffma2_rn(sj[2 * u], neg1, tm[2 * u]);
      const float2 e1 = __ffma2_rn(sj[2 * u + 1], neg1, tm[2 * u + 1]);
      dd = __ffma2_rn(e0, e0, dd);
      dd = __ffma2_rn(e1, e1, dd);
    }
    if constexpr (TAIL == 2) {
      const float2 e0 = __ffma2_rn(sj[2 * NF], nm[0], tm[2 * NF]);
      const float2 e1 = __ffma2_rn(sj[2 * NF + 1], nm[1], tm[2 * NF + 1]);
      dd = __ffma2_rn(e0, e0, dd);
      dd = __ffma2_rn(e1, e1, dd);
    }
    float d2 = dd.x + dd.y;
    if constexpr (TAIL == 1) {
      const float e = fmaf(sjs, nms, tms);
      d2 = fmaf(e, e, d2);
    }
    d2 += __shfl_xor_sync(0xffffffffu, d2, 1);
    d2 += __shfl_xor_sync(0xffffffffu, d2, 2);
    const bool in = q < len;
    if (!in) d2 = INFINITY;
    dmin = fminf(dmin, d2);
    const bool need = (m - d2) * c2 > 64.0f;  // false for d2 = +inf
    if (__any_sync(0xffffffffu, need)) {
      const float sc = need ? ex2_fast((d2 - m) * c2) : 1.0f;
      tot *= sc;
      accs *= sc;
      const float2 sc2 = f2(sc, sc);
#pragma unroll
      for (int r = 0; r < 2 * NF + 2; ++r) acc[r] = __fmul2_rn(acc[r], sc2);
      m = need ? d2 : m;
      mc2 = m * c2;
    }
    const float w = in ? ex2_fast(fmaf(-d2, c2, mc2)) : 0.0f;
    tot += w;
    const float2 w2 = f2(w, w);
#pragma unroll
    for (int r = 0; r < 2 * NF; ++r) acc[r] = __ffma2_rn(w2, sj[r], acc[r]);
    if constexpr (TAIL == 2) {
      acc[2 * NF] = __ffma2_rn(w2, sj[2 * NF], acc[2 * NF]);
      acc[2 * NF + 1] = __ffma2_rn(w2, sj[2 * NF + 1], acc[2 * NF + 1]);
    }
    if constexpr (TAIL == 1) accs = fmaf(w, sjs, accs);
  }
  // combine the 8 groups: common reference = the smallest group reference
  float ms = m;
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    ms = fminf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
    dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
  }
  const float sc = m == INFINITY ? 0.0f : ex2_fast((ms - m) * c2);  // group without neighbours: 0
  tot *= sc;
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  float* rw = red[warp][n];
#pragma unroll
  for (int u = 0; u < NF; ++u)
    *reinterpret_cast<float4*>(rw + 16 * u + 4 * c) = make_float4(
        acc[2 * u].x * sc, acc[2 * u].y * sc, acc[2 * u + 1].x * sc, acc[2 * u + 1].y * sc);
  if constexpr (TAIL == 1) rw[te] = te < dim ? accs * sc : 0.0f;  // te < 64: NF <= 3 here
  if constexpr (TAIL == 2)
    if (4 * NF + c < ((dim + 3) >> 2))
      *reinterpret_cast<float4*>(rw + te) =
          make_float4(acc[2 * NF].x * sc, acc[2 * NF].y * sc, acc[2 * NF + 1].x * sc, acc[2 * NF + 1].y * sc);
  __syncwarp();
  if (lane == 0 && (len == 0 || dmin > zero_thresh)) flag_error(flag, kFlagZeroWeight, rr);
  if (lane < ((dim + 3) >> 2)) {
    float4 a = *reinterpret_cast<const float4*>(&red[warp][0][4 * lane]);
#pragma unroll
    for (int g = 1; g < 8; ++g) {
      const float4 b = *reinterpret_cast<const float4*>(&red[warp][g][4 * lane]);
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    const float inv = 1.0f / tot;
    reinterpret_cast<float4*>(out + static_cast<int64_t>(rr) * ld_t)[lane] =
        make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
  }
}

// K4 Gaussian-recompute SpMV, lean lane-group kernel (D <= 64, default):
// iterate_interactions with the Gaussian value model (proj/src/kernels.cpp:
// 217-228 + knn.cpp:86-108), weights never stored.  The mean-shift kernel's
// structure: 8 lanes per row, unpredicated chunk loads (finished slots read
// source 0 and weigh it 0, lanes past the row re-read the last chunk with
// zero masks), masks only on the last chunk, neighbour ids and x[j] one block
// of 8 ahead, 64-register cap.  Weights are the reference's exp(-d2 / 2h^2)
// directly (no reference shift: y is not normalised).
// kStore: update_values(Gaussian) instead (proj/src/hier.cpp:203-222): the
// weight of entry q is stored in place by lane q % 8 of the row's group;
// a non-finite weight raises NonFiniteValue.
template <bool kTiles, int NC, bool kStore = false>
__global__ void __launch_bounds__(256, 4) gauss_lane_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, const float* __restrict__ x, float* __restrict__ y, int* flag = nullptr) {
  constexpr int G = 8, NB = 2;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gt / G;
  const int g = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const int gbase = lane - g;
  const bool live = slot < v.n_rows;
  const int nv4 = (dim + 3) >> 2;
  const int rr = live ? real_row(v, slot) : 0;
  int cidx[NC];
  float2 tm[2 * NC], nm[2];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = g + G * u;
    const bool last = u == NC - 1;
    const bool has = !last || c < nv4;
    cidx[u] = has ? c : nv4 - 1;
    const float4 tv =
        live ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(rr) * ld_t) + cidx[u])
             : make_float4(0.f, 0.f, 0.f, 0.f);
    if (last) {
      const float m0 = has && 4 * c + 0 < dim ? 1.f : 0.f, m1 = has && 4 * c + 1 < dim ? 1.f : 0.f;
      const float m2 = has && 4 * c + 2 < dim ? 1.f : 0.f, m3 = has && 4 * c + 3 < dim ? 1.f : 0.f;
      tm[2 * u] = f2(tv.x * m0, tv.y * m1);
      tm[2 * u + 1] = f2(tv.z * m2, tv.w * m3);
      nm[0] = f2(-m0, -m1);
      nm[1] = f2(-m2, -m3);
    } else {
      tm[2 * u] = f2(tv.x, tv.y);
      tm[2 * u + 1] = f2(tv.z, tv.w);
    }
  }
  const float2 neg1 = f2(-1.f, -1.f);
  const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int64_t hbase = (kTiles && live) ? v.halo_off[slot / v.tile_rows] : 0;
  const int wmax = __reduce_max_sync(0xffffffffu, len);
  const float4* s4 = reinterpret_cast<const float4*>(s);
  const int ld4 = ld_s >> 2;
  int jn = 0;
  float xn = 0.0f;
  if (g < len) {
    jn = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(g), hbase);
    if constexpr (!kStore) xn = __ldg(x + jn);
  }
  float acc = 0.0f;
  for (int q0 = 0; q0 < wmax; q0 += G) {
    const int jl = jn;
    const float xl = xn;
    const int qn = q0 + G + g;
    jn = 0;
    xn = 0.0f;
    if (qn < len) {
      jn = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(qn), hbase);
      if constexpr (!kStore) xn = __ldg(x + jn);
    }
#pragma unroll
    for (int b0 = 0; b0 < G; b0 += NB) {
      if (q0 + b0 >= wmax) break;  // warp-uniform
      float2 sj[NB][2 * NC];
      float d2[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = __shfl_sync(0xffffffffu, jl, gbase + b0 + b);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float4 sv = __ldg(s4 + (j * ld4 + cidx[u]));
          sj[b][2 * u] = f2(sv.x, sv.y);
          sj[b][2 * u + 1] = f2(sv.z, sv.w);
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float2 dd = f2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float2 e0 = __ffma2_rn(sj[b][2 * u], u == NC - 1 ? nm[0] : neg1, tm[2 * u]);
          const float2 e1 = __ffma2_rn(sj[b][2 * u + 1], u == NC - 1 ? nm[1] : neg1, tm[2 * u + 1]);
          dd = __ffma2_rn(e0, e0, dd);
          dd = __ffma2_rn(e1, e1, dd);
        }
        d2[b] = dd.x + dd.y;
      }
#pragma unroll
      for (int o = 1; o < G; o <<= 1)
#pragma unroll
        for (int b = 0; b < NB; ++b) d2[b] += __shfl_xor_sync(0xffffffffu, d2[b], o);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if constexpr (kStore) {
          if (q0 + b0 + b < len && g == b0 + b) {
            const float w = exp2f(-d2[b] * c2);
            if (!isfinite(w)) flag_error(flag, kFlagNonFinite, rr);
            v.vals[base + 32 * static_cast<int64_t>(q0 + b0 + b)] = w;
          }
        } else {
          const float xj = __shfl_sync(0xffffffffu, xl, gbase + b0 + b);
          if (q0 + b0 + b < len) acc = fmaf(exp2f(-d2[b] * c2), xj, acc);
        }
      }
    }
  }
  if constexpr (!kStore)
    if (live && g == 0) y[rr] = acc;
}

// variant 8: meanshift_lane_kernel with software-pipelined source loads
template <bool kTiles, int NC>
__global__ void __launch_bounds__(256) meanshift_pipe_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, float* __restrict__ out, int* flag) {
  constexpr int G = 8, NB = 2;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gt / G;
  const int g = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const int gbase = lane - g;
  const bool live = slot < v.n_rows;
  const int nv4 = (dim + 3) >> 2;
  const int rr = live ? real_row(v, slot) : 0;
  int cidx[NC];
  float2 tm[2 * NC], nm[2 * NC], acc[2 * NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = g + G * u;
    const bool has = c < nv4;
    cidx[u] = has ? c : nv4 - 1;
    const float4 tv =
        live ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(rr) * ld_t) + cidx[u])
             : make_float4(0.f, 0.f, 0.f, 0.f);
    const float m0 = has && 4 * c + 0 < dim ? 1.f : 0.f, m1 = has && 4 * c + 1 < dim ? 1.f : 0.f;
    const float m2 = has && 4 * c + 2 < dim ? 1.f : 0.f, m3 = has && 4 * c + 3 < dim ? 1.f : 0.f;
    tm[2 * u] = f2(tv.x * m0, tv.y * m1);
    tm[2 * u + 1] = f2(tv.z * m2, tv.w * m3);
    nm[2 * u] = f2(-m0, -m1);
    nm[2 * u + 1] = f2(-m2, -m3);
    acc[2 * u] = f2(0.f, 0.f);
    acc[2 * u + 1] = f2(0.f, 0.f);
  }
  const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int64_t hbase = (kTiles && live) ? v.halo_off[slot / v.tile_rows] : 0;
  const int wmax = __reduce_max_sync(0xffffffffu, len);
  const float4* s4 = reinterpret_cast<const float4*>(s);
  const int ld4 = ld_s >> 2;
  float m = INFINITY, mc2 = INFINITY, dmin = INFINITY, tot = 0.0f;
  // software-pipelined: the next batch's source rows are loaded before this
  // batch's arithmetic (two register buffers), ids one block of G ahead
  int jcur = 0, jnext = 0;  // a finished slot reads source 0 (valid) and weighs it 0
  if (g < len) jcur = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(g), hbase);
  if (G + g < len) jnext = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(G + g), hbase);
  float2 cur[NB][2 * NC], nxt[NB][2 * NC];
  auto load = [&](float2 (&dst)[NB][2 * NC], int src_ids, int first) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = __shfl_sync(0xffffffffu, src_ids, gbase + first + b);
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const float4 sv = __ldg(s4 + (j * ld4 + cidx[u]));
        dst[b][2 * u] = f2(sv.x, sv.y);
        dst[b][2 * u + 1] = f2(sv.z, sv.w);
      }
    }
  };
  load(cur, jcur, 0);
  for (int q0 = 0; q0 < wmax; q0 += G) {
#pragma unroll
    for (int b0 = 0; b0 < G; b0 += NB) {
      if (q0 + b0 >= wmax) break;  // warp-uniform
      if (b0 + NB < G) load(nxt, jcur, b0 + NB);
      else load(nxt, jnext, 0);
      float d2[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float2 dd = f2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float2 e0 = __ffma2_rn(cur[b][2 * u], nm[2 * u], tm[2 * u]);
          const float2 e1 = __ffma2_rn(cur[b][2 * u + 1], nm[2 * u + 1], tm[2 * u + 1]);
          dd = __ffma2_rn(e0, e0, dd);
          dd = __ffma2_rn(e1, e1, dd);
        }
        d2[b] = dd.x + dd.y;
      }
#pragma unroll
      for (int o = 1; o < G; o <<= 1)
#pragma unroll
        for (int b = 0; b < NB; ++b) d2[b] += __shfl_xor_sync(0xffffffffu, d2[b], o);
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (q0 + b0 + b >= len) d2[b] = INFINITY;
      float mb = d2[0];
#pragma unroll
      for (int b = 1; b < NB; ++b) mb = fminf(mb, d2[b]);
      dmin = fminf(dmin, mb);
      const bool need = (m - mb) * c2 > 64.0f;
      if (__any_sync(0xffffffffu, need)) {  // rare after a row's first batch
        const float sc = need ? ex2_fast((mb - m) * c2) : 1.0f;
        tot *= sc;
        const float2 sc2 = f2(sc, sc);
#pragma unroll
        for (int w = 0; w < 2 * NC; ++w) acc[w] = __fmul2_rn(acc[w], sc2);
        m = need ? mb : m;
        mc2 = m * c2;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const float w = ex2_fast(fmaf(-d2[b], c2, mc2));  // d2 = +inf -> 0
        tot += w;
        const float2 w2 = f2(w, w);
#pragma unroll
        for (int q = 0; q < 2 * NC; ++q) acc[q] = __ffma2_rn(w2, cur[b][q], acc[q]);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int q = 0; q < 2 * NC; ++q) cur[b][q] = nxt[b][q];
    }
    jcur = jnext;
    jnext = 0;
    if (q0 + 2 * G + g < len)
      jnext = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q0 + 2 * G + g), hbase);
  }
  if (!live) return;
  if (g == 0 && (len == 0 || dmin > zero_thresh)) flag_error(flag, kFlagZeroWeight, rr);
  const float inv = 1.0f / tot;
  float4* op = reinterpret_cast<float4*>(out + static_cast<int64_t>(rr) * ld_t);
#pragma unroll
  for (int u = 0; u < NC; ++u)
    if (g + G * u < nv4)
      op[g + G * u] = make_float4(acc[2 * u].x * inv, acc[2 * u].y * inv, acc[2 * u + 1].x * inv,
                                  acc[2 * u + 1].y * inv);
}

// K4/K5 staged (cluster order, variant 6): persistent CTAs (two per SM) walk
// the tiles; per tile one warp issues a TMA bulk copy per halo source row
// into shared memory (the whole halo, one mbarrier), then 8-lane groups run
// the lane-group arithmetic of nonstat_group_kernel with every source read a
// conflict-free 128-B shared-memory segment and no halo-id lookup.  A tile
// whose halo exceeds the buffer falls back to L1/L2 gathers.  Two CTAs per
// SM overlap one tile's copies with the other's arithmetic.
template <int NC, bool kMeanShift>
__global__ void __launch_bounds__(512, 2) nonstat_staged_kernel(
    OpView v, const float* __restrict__ t, int ld_t, const float* __restrict__ s, int ld_s,
    int dim, float c2, float zero_thresh, const float* __restrict__ x, float* __restrict__ out,
    int* flag, int cap, int n_tiles) {
  constexpr int G = 8, NB = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  float* sx = reinterpret_cast<float*>(smem_raw + 16);             // cap floats (x[halo])
  float* ssrc = reinterpret_cast<float*>(smem_raw + 16 + ((cap * 4 + 127) / 128) * 128);  // cap x ld_s
  const int tid = threadIdx.x;
  const int g = tid % G;
  const int lane = tid & 31;
  const int gbase = lane - g;
  const int nv4 = (dim + 3) >> 2;
  const uint32_t row_bytes = static_cast<uint32_t>(nv4) * 16;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  float2 nm[2 * NC];
  bool has[NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int c = g + G * u;
    has[u] = c < nv4;
    const float m0 = 4 * c + 0 < dim ? 1.f : 0.f, m1 = 4 * c + 1 < dim ? 1.f : 0.f;
    const float m2 = 4 * c + 2 < dim ? 1.f : 0.f, m3 = 4 * c + 3 < dim ? 1.f : 0.f;
    nm[2 * u] = f2(-m0, -m1);
    nm[2 * u + 1] = f2(-m2, -m3);
  }
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t h0 = v.halo_off[tile];
    const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
    const bool staged = H <= cap;
    __syncthreads();  // the previous tile's readers are done with the buffers
    if (staged) {
      if (tid < 32) {
        if (tid == 0) mbar_arrive_expect_tx(bar, row_bytes * static_cast<uint32_t>(H));
        __syncwarp();
        for (int e = tid; e < H; e += 32) {
          const int j = __ldg(v.halo_ids + h0 + e);
          bulk_g2s(ssrc + static_cast<int64_t>(e) * ld_s, s + static_cast<int64_t>(j) * ld_s, row_bytes, bar);
        }
      }
      if constexpr (!kMeanShift) {
        for (int e = tid; e < H; e += blockDim.x) sx[e] = __ldg(x + __ldg(v.halo_ids + h0 + e));
        __syncthreads();  // x[halo] written by every thread
      }
    }
    for (int r0 = 0; r0 < v.tile_rows; r0 += blockDim.x / G) {
      const int slot = tile * v.tile_rows + r0 + tid / G;
      const bool live = slot < v.n_rows && r0 + tid / G < v.tile_rows;
      const int rr = live ? real_row(v, slot) : 0;
      float2 tm[2 * NC], acc[2 * NC];
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int c = g + G * u;
        const float4 tv = (live && has[u])
            ? __ldg(reinterpret_cast<const float4*>(t + static_cast<int64_t>(rr) * ld_t) + c)
            : make_float4(0.f, 0.f, 0.f, 0.f);
        tm[2 * u] = f2(-tv.x * nm[2 * u].x, -tv.y * nm[2 * u].y);
        tm[2 * u + 1] = f2(-tv.z * nm[2 * u + 1].x, -tv.w * nm[2 * u + 1].y);
        acc[2 * u] = f2(0.f, 0.f);
        acc[2 * u + 1] = f2(0.f, 0.f);
      }
      const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
      const int len = live ? v.row_len[slot] : 0;
      const int wmax = __reduce_max_sync(0xffffffffu, len);
      if (staged && r0 == 0) mbar_wait(bar, phase);  // halo resident
      float m = INFINITY, tot = 0.0f, accx = 0.0f;
      for (int q0 = 0; q0 < wmax; q0 += G) {
        const int qg = q0 + g;
        int jl = 0;  // halo-local index when staged, global column otherwise
        float xl = 0.0f;
        if (qg < len) {
          const int l = ld_stream(v.lidx + base + 32 * static_cast<int64_t>(qg));
          jl = staged ? l : __ldg(v.halo_ids + h0 + l);
          if constexpr (!kMeanShift) xl = staged ? sx[l] : __ldg(x + jl);
        }
#pragma unroll
        for (int b0 = 0; b0 < G; b0 += NB) {
          float2 sj[NB][2 * NC];
          float d2[NB];
          bool ok[NB];
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const int j = __shfl_sync(0xffffffffu, jl, gbase + b0 + b);
            ok[b] = q0 + b0 + b < len;
#pragma unroll
            for (int u = 0; u < NC; ++u) {
              float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
              if (ok[b] && has[u])
                sv = staged ? reinterpret_cast<const float4*>(ssrc + static_cast<int64_t>(j) * ld_s)[g + G * u]
                            : __ldg(reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s) + g + G * u);
              sj[b][2 * u] = f2(sv.x, sv.y);
              sj[b][2 * u + 1] = f2(sv.z, sv.w);
            }
          }
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            float2 dd = f2(0.f, 0.f);
#pragma unroll
            for (int u = 0; u < NC; ++u) {
              const float2 d0 = __ffma2_rn(sj[b][2 * u], nm[2 * u], tm[2 * u]);
              const float2 d1 = __ffma2_rn(sj[b][2 * u + 1], nm[2 * u + 1], tm[2 * u + 1]);
              dd = __ffma2_rn(d0, d0, dd);
              dd = __ffma2_rn(d1, d1, dd);
            }
            d2[b] = dd.x + dd.y;
          }
#pragma unroll
          for (int o = 1; o < G; o <<= 1)
#pragma unroll
            for (int b = 0; b < NB; ++b) d2[b] += __shfl_xor_sync(0xffffffffu, d2[b], o);
          if constexpr (kMeanShift) {
            float mb = m;
#pragma unroll
            for (int b = 0; b < NB; ++b)
              if (ok[b]) mb = fminf(mb, d2[b]);
            if (mb < m) {
              const float sc = exp2f((mb - m) * c2);
              tot *= sc;
              const float2 sc2 = f2(sc, sc);
#pragma unroll
              for (int w = 0; w < 2 * NC; ++w) acc[w] = __fmul2_rn(acc[w], sc2);
              m = mb;
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              if (!ok[b]) continue;
              const float w = exp2f((m - d2[b]) * c2);
              tot += w;
              const float2 w2 = f2(w, w);
#pragma unroll
              for (int q = 0; q < 2 * NC; ++q) acc[q] = __ffma2_rn(w2, sj[b][q], acc[q]);
            }
          } else {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const float xj = __shfl_sync(0xffffffffu, xl, gbase + b0 + b);
              if (ok[b]) accx = fmaf(exp2f(-d2[b] * c2), xj, accx);
            }
          }
        }
      }
      if (live) {
        if constexpr (kMeanShift) {
          if (g == 0 && (len == 0 || m > zero_thresh)) flag_error(flag, kFlagZeroWeight, rr);
          const float inv = 1.0f / tot;
          float4* op = reinterpret_cast<float4*>(out + static_cast<int64_t>(rr) * ld_t);
#pragma unroll
          for (int u = 0; u < NC; ++u)
            if (has[u])
              op[g + G * u] = make_float4(acc[2 * u].x * inv, acc[2 * u].y * inv,
                                          acc[2 * u + 1].x * inv, acc[2 * u + 1].y * inv);
        } else {
          if (g == 0) out[rr] = accx;
        }
      }
    }
    if (staged) phase ^= 1;
  }
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
  const float4* tp = reinterpret_cast<const float4*>(t + static_cast<int64_t>(real_row(v, row)) * ld_t);
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
  y[real_row(v, row)] = acc;
}

// K4 (wide rows): warp per row, lanes split the coordinates (float4 c4 =
// lane + 32 c), dim <= 128*NVL.  The row's neighbour ids (two dependent loads
// each in the tile format) and x[j] are fetched up front, one neighbour per
// lane, and broadcast by shuffles, so the per-neighbour path holds only the
// coordinate loads; the squared differences run as packed FFMA2 pairs and
// only a trailing partial float4 (dim % 4 != 0) is masked.
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
  // NVL = ceil(nv4 / 32): every float4 with c < NVL-1 lies inside the row;
  // only the last one can be partial or past the end, and it is masked by
  // nm (-1 inside, 0 outside) in d = t + nm * s with t zeroed outside
  const int cl = lane + 32 * (NVL - 1);
  const int cl_ld = min(cl, nv4 - 1);
  float4 ti[NVL];
  const float4* tp = reinterpret_cast<const float4*>(t + static_cast<int64_t>(real_row(v, row)) * ld_t);
#pragma unroll
  for (int c = 0; c < NVL - 1; ++c) ti[c] = __ldg(tp + lane + 32 * c);
  float2 nm_lo, nm_hi;
  {
    const int e = 4 * cl;  // first coordinate of the last float4
    nm_lo = make_float2(e < dim ? -1.f : 0.f, e + 1 < dim ? -1.f : 0.f);
    nm_hi = make_float2(e + 2 < dim ? -1.f : 0.f, e + 3 < dim ? -1.f : 0.f);
    const float4 tl = __ldg(tp + cl_ld);
    ti[NVL - 1] = make_float4(-nm_lo.x * tl.x, -nm_lo.y * tl.y, -nm_hi.x * tl.z, -nm_hi.y * tl.w);
  }
  const float2 m1 = make_float2(-1.0f, -1.0f);
  float acc = 0.0f;
  for (int q0 = 0; q0 < len; q0 += 32) {
    const int qn = min(32, len - q0);
    int jl = 0;
    float xl = 0.0f;
    if (lane < qn) {
      jl = entry_col<kTiles>(v, base + 32 * static_cast<int64_t>(q0 + lane), hbase);
      xl = __ldg(x + jl);
    }
    for (int q = 0; q < qn; ++q) {
      const int j = __shfl_sync(0xffffffffu, jl, q);
      const float4* sp = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld_s);
      float4 sv[NVL];
#pragma unroll
      for (int c = 0; c < NVL; ++c) sv[c] = __ldg(sp + (c < NVL - 1 ? lane + 32 * c : cl_ld));
      float2 dd = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < NVL; ++c) {
        const float2 a = c < NVL - 1 ? m1 : nm_lo, b = c < NVL - 1 ? m1 : nm_hi;
        const float2 d0 = __ffma2_rn(make_float2(sv[c].x, sv[c].y), a, make_float2(ti[c].x, ti[c].y));
        const float2 d1 = __ffma2_rn(make_float2(sv[c].z, sv[c].w), b, make_float2(ti[c].z, ti[c].w));
        dd = __ffma2_rn(d0, d0, dd);
        dd = __ffma2_rn(d1, d1, dd);
      }
      float d2 = dd.x + dd.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
      acc = fmaf(exp2f(-d2 * c2), __shfl_sync(0xffffffffu, xl, q), acc);
    }
  }
  if (lane == 0) y[real_row(v, row)] = acc;
}

// K4 wide, source-streaming (C5; cluster tiles of 32 rows, rows <= 32
// entries).  Persistent CTAs: 16 consumer warps, each holding two of the
// tile's target rows in registers, plus one producer warp.  Each tile's halo
// (its sorted distinct source columns) streams once through a shared-memory
// ring of NBUF batches x B source rows filled by TMA bulk copies
// (cp.async.bulk -> mbarrier complete_tx); the producer runs ahead across the
// CTA's tiles, limited only by the ring (its halo-id loads are prefetched one
// batch ahead).  Consumers take the batches in order, evaluate only their
// rows' neighbours (16-bit halo indices ascend with the stream) and release
// each batch with one mbarrier arrival per warp.  A source row is read from L2
// once per tile instead of once per referencing row.  Halo padding ids
// (repeats of the last id) are not copied.
template <int NVL, int B, int NBUF>
__global__ void __launch_bounds__(544, 1) gauss_stream_kernel(OpView v, const float* __restrict__ t,
                                                              int ld_t, const float* __restrict__ s,
                                                              int ld_s, int dim, float c2,
                                                              const float* __restrict__ x,
                                                              float* __restrict__ y, int n_tiles) {
  constexpr int kConsumers = 16;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NBUF;
  float* ring = reinterpret_cast<float*>(smem_raw + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rowb = static_cast<uint32_t>(ld_s) * 4u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumers) {  // producer
    int tile = blockIdx.x, b = 0;
    // advance (tile, b) to the next batch that exists; false when done
    auto settle = [&](int& tl, int& bb) {
      while (tl < n_tiles &&
             bb * B >= static_cast<int>(v.halo_off[tl + 1] - v.halo_off[tl])) {
        tl += gridDim.x;
        bb = 0;
      }
      return tl < n_tiles;
    };
    auto fetch = [&](int tl, int bb, int& id, bool& real) {
      id = 0;
      real = false;
      if (tl < n_tiles && lane < B) {
        const int64_t h0 = v.halo_off[tl];
        const int H = static_cast<int>(v.halo_off[tl + 1] - h0);
        const int h = bb * B + lane;
        if (h < H) {
          id = __ldg(v.halo_ids + h0 + h);
          real = h == 0 || id != __ldg(v.halo_ids + h0 + h - 1);  // padding repeats the last id
        }
      }
    };
    settle(tile, b);
    int id, nid;
    bool real, nreal;
    fetch(tile, b, id, real);
    for (int gb = 0; tile < n_tiles; ++gb) {
      int ntile = tile, nb = b + 1;
      settle(ntile, nb);
      fetch(ntile, nb, nid, nreal);  // next batch's ids in flight during this one
      const int buf = gb % NBUF;
      if (gb >= NBUF) mbar_wait(&empty[buf], ((gb / NBUF) - 1) & 1);
      const unsigned m = __ballot_sync(0xffffffffu, real);
      if (lane == 0) mbar_arrive_expect_tx(&full[buf], __popc(m) * rowb);
      __syncwarp();
      if (real)
        bulk_g2s(ring + static_cast<int64_t>(buf * B + lane) * ld_s,
                 s + static_cast<int64_t>(id) * ld_s, rowb, &full[buf]);
      tile = ntile;
      b = nb;
      id = nid;
      real = nreal;
    }
    return;
  }

  const int nv4 = (dim + 3) >> 2;
  const int cl = lane + 32 * (NVL - 1);
  const int cl_ld = min(cl, nv4 - 1);
  float2 nm_lo, nm_hi;
  {
    const int e = 4 * cl;
    nm_lo = make_float2(e < dim ? -1.f : 0.f, e + 1 < dim ? -1.f : 0.f);
    nm_hi = make_float2(e + 2 < dim ? -1.f : 0.f, e + 3 < dim ? -1.f : 0.f);
  }
  const float2 m1 = make_float2(-1.0f, -1.0f);
  struct RowState {
    float4 ti[NVL];
    int li, want, ptr, len, rr;
    float xl, acc;
    bool live;
  };
  auto init_row = [&](RowState& r, int slot, int64_t h0) {
    r.live = slot < v.n_rows;
    r.len = r.live ? v.row_len[slot] : 0;
    const int64_t base = r.live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
    r.li = 0x7fffffff;
    r.xl = 0.0f;
    if (lane < r.len) {
      r.li = ld_stream(v.lidx + base + 32 * static_cast<int64_t>(lane));
      r.xl = __ldg(x + __ldg(v.halo_ids + h0 + r.li));
    }
    r.rr = r.live ? real_row(v, slot) : 0;
    const float4* tp = reinterpret_cast<const float4*>(t + static_cast<int64_t>(r.rr) * ld_t);
#pragma unroll
    for (int c = 0; c < NVL - 1; ++c)
      r.ti[c] = r.live ? __ldg(tp + lane + 32 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 tl = r.live ? __ldg(tp + cl_ld) : make_float4(0.f, 0.f, 0.f, 0.f);
    r.ti[NVL - 1] = make_float4(-nm_lo.x * tl.x, -nm_lo.y * tl.y, -nm_hi.x * tl.z, -nm_hi.y * tl.w);
    r.ptr = 0;
    r.want = __shfl_sync(0xffffffffu, r.li, 0);
    r.acc = 0.0f;
  };
  // this row's neighbours among batch items [lo, lo + B) in ring buffer buf
  auto consume = [&](RowState& r, int lo, int buf) {
    while (r.want < lo + B) {  // warp-uniform
      const float4* sp =
          reinterpret_cast<const float4*>(ring + static_cast<int64_t>(buf * B + r.want - lo) * ld_s);
      float2 dd = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < NVL; ++c) {
        const float4 sv = sp[c < NVL - 1 ? lane + 32 * c : cl_ld];
        const float2 a = c < NVL - 1 ? m1 : nm_lo, bb = c < NVL - 1 ? m1 : nm_hi;
        const float2 d0 = __ffma2_rn(make_float2(sv.x, sv.y), a, make_float2(r.ti[c].x, r.ti[c].y));
        const float2 d1 = __ffma2_rn(make_float2(sv.z, sv.w), bb, make_float2(r.ti[c].z, r.ti[c].w));
        dd = __ffma2_rn(d0, d0, dd);
        dd = __ffma2_rn(d1, d1, dd);
      }
      float d2 = dd.x + dd.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
      r.acc = fmaf(exp2f(-d2 * c2), __shfl_sync(0xffffffffu, r.xl, r.ptr), r.acc);
      ++r.ptr;
      r.want = __shfl_sync(0xffffffffu, r.li, r.ptr & 31);
      if (r.ptr >= r.len) r.want = 0x7fffffff;
    }
  };
  int gb = 0;
  RowState r0, r1;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t h0 = v.halo_off[tile];
    const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
    const int nb = (H + B - 1) / B;
    init_row(r0, tile * v.tile_rows + warp, h0);
    init_row(r1, tile * v.tile_rows + warp + kConsumers, h0);
    for (int b = 0; b < nb; ++b, ++gb) {
      const int buf = gb % NBUF;
      mbar_wait(&full[buf], (gb / NBUF) & 1);
      consume(r0, b * B, buf);
      consume(r1, b * B, buf);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[buf]);
    }
    if (lane == 0) {
      if (r0.live) y[r0.rr] = r0.acc;
      if (r1.live) y[r1.rr] = r1.acc;
    }
  }
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
  const float* ti = t + static_cast<int64_t>(real_row(v, row)) * ld_t;
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
    if (!isfinite(w)) flag_error(flag, kFlagNonFinite, real_row(v, row));
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
  const float4* tp = reinterpret_cast<const float4*>(tin + static_cast<int64_t>(real_row(v, row)) * ld_t);
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
  if (len == 0 || m > zero_thresh) flag_error(flag, kFlagZeroWeight, real_row(v, row));
  const float inv = 1.0f / tot;
  float4* op = reinterpret_cast<float4*>(tout + static_cast<int64_t>(real_row(v, row)) * ld_t);
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
  const float4* tp = reinterpret_cast<const float4*>(tin + static_cast<int64_t>(real_row(v, row)) * ld_t);
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
  if (lane == 0 && (len == 0 || m > zero_thresh)) flag_error(flag, kFlagZeroWeight, real_row(v, row));
  const float inv = 1.0f / tot;
  float4* op = reinterpret_cast<float4*>(tout + static_cast<int64_t>(real_row(v, row)) * ld_t);
#pragma unroll
  for (int c = 0; c < NVL; ++c) {
    const int c4 = lane + 32 * c;
    if (c4 < nv4)
      op[c4] = make_float4(acc[c].x * inv, acc[c].y * inv, acc[c].z * inv, acc[c].w * inv);
  }
}

// ---------------------------------------------------------------------------
// y_j of a DIM-wide embedding row (one 8-B load for the 2-D case)
// kYL: cache policy of the y_j gather (KNNX_TSNE_YLOAD, interleaved C4 kernel):
// 0 = ld.global.nc (L1 + L2), 1 = ld.global.cg (L2 only), 2 = ld.global.nc
// with L1::evict_last (keep the gathered embedding over the entry streams)
template <int DIM, int kYL = 0>
__device__ __forceinline__ void load_y(const float* __restrict__ y, int j, float (&out)[DIM]) {
  if constexpr (DIM == 2) {
    float2 v2;
    if constexpr (kYL == 1) {
      v2 = __ldcg(reinterpret_cast<const float2*>(y) + j);
    } else if constexpr (kYL == 2) {
      asm volatile("ld.global.nc.L1::evict_last.v2.f32 {%0, %1}, [%2];"
                   : "=f"(v2.x), "=f"(v2.y)
                   : "l"(reinterpret_cast<const float2*>(y) + j));
    } else {
      v2 = __ldg(reinterpret_cast<const float2*>(y) + j);
    }
    out[0] = v2.x;
    out[1] = v2.y;
  } else {
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = __ldg(y + static_cast<int64_t>(j) * DIM + c);
  }
}

// K6: t-SNE attractive force (tsne_attractive_step, proj/src/kernels.cpp:103-136),
// computed directly as F_i = sum_j a_ij (y_i - y_j); optional in-place
// a_ij write-back (the reference's mutation) and fused y update.
template <bool kTiles, int DIM, bool kStore>
__global__ void __launch_bounds__(256) tsne_rows_kernel(OpView v, const float* __restrict__ y,
                                                        const float* __restrict__ yg,
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
    yi[c] = __ldg(y + static_cast<int64_t>(v.row_base + real_row(v, row)) * DIM + c);
    acc[c] = 0.0f;
  }
#pragma unroll 8
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    const int j = entry_col<kTiles>(v, p, hbase);
    const float pij = ld_stream(v.vals + p);
    float d[DIM], d2 = 0.0f;
    float yj[DIM];
    load_y<DIM>(yg, j, yj);
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      d[c] = yi[c] - yj[c];
      d2 = fmaf(d[c], d[c], d2);
    }
    const float a = pij / (1.0f + d2);
    if constexpr (kStore) v.vals[p] = a;  // compile-time: no store, loads hoist freely
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = fmaf(a, d[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    f[static_cast<int64_t>(real_row(v, row)) * DIM + c] = acc[c];
    if (y_out) y_out[static_cast<int64_t>(real_row(v, row)) * DIM + c] = yi[c] - step * acc[c];
  }
}

// K6 on cluster tiles (default): one CTA per tile stages the embedding rows
// y[halo] in shared memory (kG-unrolled like the SpMV stage), then every slot
// streams its affinities and 16-bit indices and gathers y_j from shared
// memory.  Same arithmetic as tsne_rows_kernel.
template <int DIM, int kG, bool kStore>
__global__ void __launch_bounds__(1024) tsne_tiles_kernel(OpView v, const float* __restrict__ y,
                                                          const float* __restrict__ yg,
                                                          float* __restrict__ f, int store,
                                                          float step, float* __restrict__ y_out) {
  extern __shared__ float sy[];  // H x DIM
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int R = blockDim.x;
  const int slot = tile * R + tid;
  const bool live = slot < v.n_rows;
  const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int rr = live ? real_row(v, slot) : 0;
  const int64_t h0 = v.halo_off[tile];
  const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
  for (int j0 = tid; j0 < H; j0 += R * kG) {
    int id[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) id[g] = j0 + R * g < H ? __ldg(v.halo_ids + h0 + j0 + R * g) : 0;
    float yv[kG][DIM];
#pragma unroll
    for (int g = 0; g < kG; ++g)
#pragma unroll
      for (int c = 0; c < DIM; ++c) yv[g][c] = __ldg(yg + static_cast<int64_t>(id[g]) * DIM + c);
#pragma unroll
    for (int g = 0; g < kG; ++g)
      if (j0 + R * g < H)
#pragma unroll
        for (int c = 0; c < DIM; ++c) sy[(j0 + R * g) * DIM + c] = yv[g][c];
  }
  float yi[DIM], acc[DIM];
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    yi[c] = live ? __ldg(y + static_cast<int64_t>(v.row_base + rr) * DIM + c) : 0.0f;
    acc[c] = 0.0f;
  }
  __syncthreads();
  if (!live) return;
#pragma unroll 8
  for (int q = 0; q < len; ++q) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    const int l = ld_stream(v.lidx + p);
    const float pij = ld_stream(v.vals + p);
    float d[DIM], d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      d[c] = yi[c] - sy[l * DIM + c];
      d2 = fmaf(d[c], d[c], d2);
    }
    const float a = pij / (1.0f + d2);
    if constexpr (kStore) v.vals[p] = a;  // compile-time: no store, loads hoist freely
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = fmaf(a, d[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    f[static_cast<int64_t>(rr) * DIM + c] = acc[c];
    if (y_out) y_out[static_cast<int64_t>(rr) * DIM + c] = yi[c] - step * acc[c];
  }
}

// K6 for high-degree graphs (symmetrised k = 90: ~150 entries per row): G
// lanes per row split the row's entries (q = g, g+G, ...), so each row has G
// independent gather chains and the grid G times the warps; the G partial
// forces are combined with xor shuffles.  A warp's G-lane loads of one entry
// index q cover 32/G consecutive slots: one fully used 32-B sector each.
// kInter (KNNX_OPT_GROUP_INTERLEAVE, G = 8): entry q of a slot sits at
// slice_off + (q/8)*256 + (slot%32)*8 + q%8, so the 8 lanes of a group read
// one 32-B sector per step and a warp one 128-B line.
template <bool kTiles, int DIM, int G, bool kStore, bool kInter = false, int kMinB = 1, int kYL = 0>
__global__ void __launch_bounds__(256, kMinB) tsne_group_kernel(OpView v, const float* __restrict__ y,
                                                         const float* __restrict__ yg,
                                                         float* __restrict__ f, int store,
                                                         float step, float* __restrict__ y_out) {
  static_assert(!kInter || G == 8, "group interleave is laid out for 8-lane groups");
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = gt / G;
  const int g = threadIdx.x % G;
  const bool live = slot < v.n_rows;
  const int64_t base = live ? v.slice_off[slot >> 5] + (kInter ? (slot & 31) * 8 : (slot & 31)) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int rr = live ? real_row(v, slot) : 0;
  const int64_t hbase = (kTiles && live) ? v.halo_off[slot / v.tile_rows] : 0;
  float yi[DIM], acc[DIM];
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    yi[c] = live ? __ldg(y + static_cast<int64_t>(v.row_base + rr) * DIM + c) : 0.0f;
    acc[c] = 0.0f;
  }
  auto pos = [&](int q) -> int64_t {
    return kInter ? base + 256 * static_cast<int64_t>(q >> 3) + g : base + 32 * static_cast<int64_t>(q);
  };
  auto interact = [&](int64_t p, int j, float pij, const float (&yj)[DIM]) {
    float d[DIM], d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      d[c] = yi[c] - yj[c];
      d2 = fmaf(d[c], d[c], d2);
    }
    const float a = __fdividef(pij, 1.0f + d2);
    if constexpr (kStore) v.vals[p] = a;  // compile-time: no store, loads hoist freely
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = fmaf(a, d[c], acc[c]);
  };
  // blocks of U entries per lane: the U column / value loads are issued
  // together (and the next block's while this one computes), then the U
  // dependent y_j gathers together -- two memory latencies per block instead
  // of two per entry
  constexpr int U = KNNX_TSNE_U;
  int q = g;
  int jn[U];
  float pn[U];
  const bool first_full = q + (U - 1) * G < len;
  if (first_full) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      jn[u] = entry_col<kTiles>(v, pos(q + u * G), hbase);
      pn[u] = ld_stream(v.vals + pos(q + u * G));
    }
  }
  for (; q + (U - 1) * G < len; q += U * G) {
    int j[U];
    float pj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      j[u] = jn[u];
      pj[u] = pn[u];
    }
    const int qn = q + U * G;
    if (qn + (U - 1) * G < len) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        jn[u] = entry_col<kTiles>(v, pos(qn + u * G), hbase);
        pn[u] = ld_stream(v.vals + pos(qn + u * G));
      }
    }
    float yj[U][DIM];
#pragma unroll
    for (int u = 0; u < U; ++u) load_y<DIM, kYL>(yg, j[u], yj[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) interact(pos(q + u * G), j[u], pj[u], yj[u]);
  }
  for (; q < len; q += G) {
    const int64_t p = pos(q);
    const int j = entry_col<kTiles>(v, p, hbase);
    float yj[DIM];
    load_y<DIM, kYL>(yg, j, yj);
    interact(p, j, ld_stream(v.vals + p), yj);
  }
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int o = 1; o < G; o <<= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (!live || g != 0) return;
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    f[static_cast<int64_t>(rr) * DIM + c] = acc[c];
    if (y_out) y_out[static_cast<int64_t>(rr) * DIM + c] = yi[c] - step * acc[c];
  }
}

// K6 on small cluster tiles (tile_rows <= 64): one CTA per tile stages the
// embedding rows y[halo] in shared memory (a few KB), then G lanes per row
// stream the row's affinities and 16-bit halo indices and read y_j from
// shared memory.  The L1 then carries only the coalesced value / index
// streams: the per-entry y gathers (one 32-B sector each for 8 B) leave it.
template <int DIM, int G, bool kStore>
__global__ void __launch_bounds__(512) tsne_tiles_group_kernel(OpView v, const float* __restrict__ y,
                                                               const float* __restrict__ yg,
                                                               float* __restrict__ f, float step,
                                                               float* __restrict__ y_out) {
  extern __shared__ float sy[];  // H x DIM
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t h0 = v.halo_off[tile];
  const int H = static_cast<int>(v.halo_off[tile + 1] - h0);
  constexpr int U = 4;
  for (int e0 = tid; e0 < H; e0 += U * blockDim.x) {
    int id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      id[u] = e < H ? __ldg(v.halo_ids + h0 + e) : 0;
    }
    float yv[U][DIM];
#pragma unroll
    for (int u = 0; u < U; ++u) load_y<DIM>(yg, id[u], yv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < H)
#pragma unroll
        for (int c = 0; c < DIM; ++c) sy[e * DIM + c] = yv[u][c];
    }
  }
  const int slot = tile * v.tile_rows + tid / G;
  const int g = tid % G;
  const bool live = tid / G < v.tile_rows && slot < v.n_rows;
  const int64_t base = live ? v.slice_off[slot >> 5] + (slot & 31) : 0;
  const int len = live ? v.row_len[slot] : 0;
  const int rr = live ? real_row(v, slot) : 0;
  float yi[DIM], acc[DIM];
  if (live) load_y<DIM>(y, v.row_base + rr, yi);
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    if (!live) yi[c] = 0.0f;
    acc[c] = 0.0f;
  }
  __syncthreads();
#pragma unroll 4
  for (int q = g; q < len; q += G) {
    const int64_t p = base + 32 * static_cast<int64_t>(q);
    const int l = ld_stream(v.lidx + p);
    const float pij = ld_stream(v.vals + p);
    float d[DIM], d2 = 0.0f;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      d[c] = yi[c] - sy[l * DIM + c];
      d2 = fmaf(d[c], d[c], d2);
    }
    const float a = __fdividef(pij, 1.0f + d2);
    if constexpr (kStore) v.vals[p] = a;
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = fmaf(a, d[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int o = 1; o < G; o <<= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (!live || g != 0) return;
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    f[static_cast<int64_t>(rr) * DIM + c] = acc[c];
    if (y_out) y_out[static_cast<int64_t>(rr) * DIM + c] = yi[c] - step * acc[c];
  }
}

// ---------------------------------------------------------------------------
// K1: whole-row permutation copies (proj/src/core.cpp:141-148), bit-exact.
template <typename W>
__global__ void permute_kernel(int n, int words, const W* __restrict__ in,
                               const int32_t* __restrict__ idx, W* __restrict__ out, bool scatter) {
  // 4 independent (row, word) elements per thread, all loads before the
  // stores: four row gathers in flight per thread (32-bit element indices;
  // the launcher falls back to the 64-bit loop beyond 2^31 elements)
  constexpr int U = 4;
  const int total = n * words;
  const int stride = gridDim.x * blockDim.x;
  const int e0 = blockIdx.x * blockDim.x + threadIdx.x;
  W v[U];
  int dst[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int e = e0 + u * stride;
    dst[u] = -1;
    if (e < total) {
      const int i = e / words;
      const int w = e - i * words;
      const int other = __ldg(idx + i) * words + w;
      v[u] = scatter ? in[e] : in[other];
      dst[u] = scatter ? other : e;
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (dst[u] >= 0) out[dst[u]] = v[u];
}

template <typename W>
__global__ void permute_kernel_wide(int n, int words, const W* __restrict__ in,
                                    const int32_t* __restrict__ idx, W* __restrict__ out,
                                    bool scatter) {
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
  require_plain(op);
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  // variants: 0 default = unrolled-stage tiles + programmatic
  // dependent launch, 1 plain tiles, 2 TMA bulk tiles, 3/4 register prefetch
  // (+PDL), 5 persistent TMA ring, 6 unrolled stage x8, 8 = 0 without PDL
  if (op.order == KNNX_ORDER_CLUSTER && (op.spmv_variant == 8 || op.spmv_variant == 6)) {
    const size_t smem = static_cast<size_t>(op.max_halo) * sizeof(float);
    auto kernel = op.spmv_variant == 8 ? spmv_tiles_g_kernel<4> : spmv_tiles_g_kernel<8>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kernel<<<op.n_tiles, op.tile_rows, smem, st>>>(v, x, y);
  } else if (op.order == KNNX_ORDER_CLUSTER && (op.spmv_variant == 0 || op.spmv_variant == 7)) {
    const size_t smem = static_cast<size_t>(op.max_halo) * sizeof(float);
    auto kernel = spmv_tiles_g_kernel<4, true>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(op.n_tiles);
    cfg.blockDim = dim3(op.tile_rows);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, v, x, y);
  } else if (op.order == KNNX_ORDER_CLUSTER && op.tile_rows == 128 &&
             (op.spmv_variant == 3 || op.spmv_variant == 4)) {
    const size_t smem = static_cast<size_t>(op.max_halo) * sizeof(float);
    auto kernel = op.spmv_variant == 4 ? spmv_tiles_pf_kernel<16, true> : spmv_tiles_pf_kernel<16, false>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(op.n_tiles);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = op.spmv_variant == 4 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, v, x, y);
  } else if (op.order == KNNX_ORDER_CLUSTER && op.tile_rows == 128 && op.spmv_variant == 2) {
    const int e_max = static_cast<int>(op.max_tile_entries);
    const size_t smem = static_cast<size_t>(e_max) * 4 + (static_cast<size_t>(e_max) * 2 + 15) / 16 * 16 +
                        16 + static_cast<size_t>(op.max_halo) * 4;
    cudaFuncSetAttribute(spmv_tiles_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    spmv_tiles_bulk_kernel<<<op.n_tiles, 128, smem, st>>>(v, x, y, e_max);
  } else if (op.order == KNNX_ORDER_CLUSTER && op.tile_rows == 128 && op.max_halo <= 4096 &&
             op.spmv_variant == 5) {
    const int e_max = static_cast<int>(op.max_tile_entries), h_max = op.max_halo;
    const size_t stage = static_cast<size_t>(e_max) * 4 + (static_cast<size_t>(e_max) * 2 + 15) / 16 * 16 +
                         static_cast<size_t>(h_max) * 4;
    const size_t smem = 2 * stage + 2 * static_cast<size_t>(h_max) * 4 + 16;
    auto run = [&](auto kernel) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 128, smem);
      const int grid = std::max(1, std::min(op.n_tiles, op.ctx->n_sms * std::max(1, per_sm)));
      kernel<<<grid, 128, smem, st>>>(v, x, y, e_max, h_max);
    };
    if (h_max <= 1024)
      run(spmv_tiles_tma_kernel<8>);
    else if (h_max <= 2048)
      run(spmv_tiles_tma_kernel<16>);
    else
      run(spmv_tiles_tma_kernel<32>);
  } else if (op.order == KNNX_ORDER_CLUSTER) {
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

namespace {

// non-stationary kernel variants: 0 = lane group per row
// from L1/L2, 2 neighbours per batch (default, dim <= 64; mean shift runs
// meanshift_lane_kernel capped at 64 registers), 1 = thread per row, 2 =
// octet with the tile's halo staged in shared memory (cluster order,
// tile_rows <= 128), 3 = groups of 4 lanes, 4 = octet scalar arithmetic,
// 5 = default with 1 neighbour per batch, 6 = persistent TMA-staged halo,
// 7 = nonstat_group_kernel for mean shift (the previous default), 8 =
// meanshift_pipe_kernel (software-pipelined loads, 90 registers), 9 = lean
// kernel in 128-thread blocks, 10 = meanshift_np_kernel (warp per row)
// read per launch (a getenv, ~0.1 us) so A/B probes can switch in-process
int nonstat_variant() {
  const char* e = std::getenv("KNNX_NONSTAT_VARIANT");
  return e ? std::atoi(e) : 0;
}

bool octet_ok(const knnx_operator& op, int dim) {
  return nonstat_variant() == 2 && op.order == KNNX_ORDER_CLUSTER && dim <= 64 && op.tile_rows <= 128;
}

template <bool kMeanShift>
bool launch_octet_l1(const knnx_operator& op, const float* t, int ld_t, const float* s, int ld_s,
                     int dim, float c2, float zero_thresh, const float* x, float* out, int* flag,
                     cudaStream_t st) {
  const int var = nonstat_variant();
  if ((var != 0 && var != 3 && var != 4 && var != 5 && var != 6 && var != 7 &&
       var != 8 && var != 9 && var != 10) || dim > 64)
    return false;
  const OpView v = view_of(op);
  const bool tiles = op.order == KNNX_ORDER_CLUSTER;
  const int nv = (dim + 3) / 4;
  if (var == 4) {  // octet, scalar arithmetic (A/B reference)
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
#define L(T, NC)                                                                          \
  nonstat_octet_l1_kernel<T, NC, kMeanShift>                                              \
      <<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, zero_thresh, x, out, flag)
    if (tiles) {
      if (nv <= 8) L(true, 1); else L(true, 2);
    } else {
      if (nv <= 8) L(false, 1); else L(false, 2);
    }
#undef L
    return true;
  }
  if (var == 6 && tiles) {  // persistent, halo staged by TMA bulk copies
    const int cap = std::min(op.max_halo, (100 * 1024 - 16) / (4 * (ld_s + 1)));
    const size_t smem = 16 + static_cast<size_t>((cap * 4 + 127) / 128) * 128 +
                        static_cast<size_t>(cap) * ld_s * 4;
    const int grid = std::max(1, std::min(op.n_tiles, 2 * op.ctx->n_sms));
    auto go = [&](auto kernel) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kernel<<<grid, 512, smem, st>>>(v, t, ld_t, s, ld_s, dim, c2, zero_thresh, x, out, flag, cap,
                                      op.n_tiles);
    };
    if (nv <= 8) go(nonstat_staged_kernel<1, kMeanShift>);
    else go(nonstat_staged_kernel<2, kMeanShift>);
    return true;
  }
  if constexpr (kMeanShift) {
    // lean kernel (default; variant 7 = the previous default below); 32-bit
    // source offsets
    if (var == 10 && static_cast<int64_t>(op.n_cols) * ld_s < (int64_t{1} << 31)) {
      // neighbour-parallel: one warp (8 groups of 4 lanes) per row
      const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 32, 256);
      const int nf = dim / 16, rest = dim - 16 * nf;
      const int tail = rest == 0 ? 0 : rest <= 4 ? 1 : 2;
#define LNK(T, F, TL) meanshift_np_kernel<T, F, TL><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, zero_thresh, out, flag)
#define LNT(T, F) if (tail == 0) LNK(T, F, 0); else if (tail == 1) LNK(T, F, 1); else LNK(T, F, 2);
#define LN(T)                                                                    \
  switch (nf) {                                                                  \
    case 0: if (tail <= 1) LNK(T, 0, 1); else LNK(T, 0, 2); break;                   \
    case 1: LNT(T, 1) break;                                                     \
    case 2: LNT(T, 2) break;                                                     \
    case 3: LNT(T, 3) break;                                                     \
    default: LNK(T, 4, 0); break;                                                \
  }
      if (tiles) { LN(true) } else { LN(false) }
#undef LNK
#undef LNT
#undef LN
      return true;
    }
    if ((var == 0 || var == 8 || var == 9) &&
        static_cast<int64_t>(op.n_cols) * ld_s < (int64_t{1} << 31)) {
      const int blk = var == 9 ? 128 : 256;
      const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, blk);
#define LM(T, NC)                                                                          \
  if (var == 8)                                                                            \
    meanshift_pipe_kernel<T, NC><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2,       \
                                                       zero_thresh, out, flag);            \
  else                                                                                     \
    meanshift_lane_kernel<T, NC, 4><<<grid, blk, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2,    \
                                                          zero_thresh, out, flag)
      if (tiles) {
        if (nv <= 8) LM(true, 1); else LM(true, 2);
      } else {
        if (nv <= 8) LM(false, 1); else LM(false, 2);
      }
#undef LM
      return true;
    }
  }
  const int G = var == 3 ? 4 : 8;  // measured: G=8 fastest at D=49
  const int grid = grid_for(static_cast<int64_t>(op.n_rows) * G, 256);
#define L(T, GG, NC)                                                                      \
  if (var == 5)                                                                           \
    nonstat_group_kernel<T, GG, NC, kMeanShift, false, 1>                                 \
        <<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, zero_thresh, x, out, flag);  \
  else                                                                                    \
    nonstat_group_kernel<T, GG, NC, kMeanShift, false, 2>                                 \
        <<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, zero_thresh, x, out, flag)
#define LG(T)                                                                             \
  if (G == 8) {                                                                           \
    if (nv <= 8) L(T, 8, 1); else L(T, 8, 2);                                             \
  } else {                                                                                \
    if (nv <= 4) L(T, 4, 1); else if (nv <= 8) L(T, 4, 2); else if (nv <= 12) L(T, 4, 3); \
    else L(T, 4, 4);                                                                      \
  }
  if (tiles) {
    LG(true)
  } else {
    LG(false)
  }
#undef LG
#undef L
  return true;
}

template <bool kMeanShift>
void launch_octet(const knnx_operator& op, const float* t, int ld_t, const float* s, int ld_s,
                  int dim, float c2, float zero_thresh, const float* x, float* out, int* flag,
                  cudaStream_t st) {
  static const int budget_kb = [] {
    const char* e = std::getenv("KNNX_OCTET_SMEM_KB");
    return e ? std::atoi(e) : 200;
  }();
  const OpView v = view_of(op);
  const int e_max = static_cast<int>(op.max_tile_entries);
  const size_t fixed = (kMeanShift ? 0 : static_cast<size_t>(op.max_halo) * 4) +
                       static_cast<size_t>((e_max + 7) / 8 * 8) * 2;
  const size_t budget = static_cast<size_t>(budget_kb) * 1024;
  const size_t row_bytes = static_cast<size_t>(ld_s) * 4;
  int cap = static_cast<int>(std::min<size_t>(op.max_halo, (budget - std::min(budget, fixed)) / row_bytes));
  cap = std::max(cap, 1);
  const size_t smem = static_cast<size_t>(cap) * row_bytes + fixed;
  const int nv = (dim + 3) / 4;
  auto go = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kernel<<<op.n_tiles, op.tile_rows * 8, smem, st>>>(v, t, ld_t, s, ld_s, dim, c2, zero_thresh, x,
                                                        out, flag, cap, e_max);
  };
  if (nv <= 8)
    go(nonstat_octet_kernel<1, kMeanShift>);
  else
    go(nonstat_octet_kernel<2, kMeanShift>);
}

}  // namespace

void launch_gauss_spmv(const knnx_operator& op, const float* t, int ld_t, const float* s,
                       int ld_s, int dim, float c2, const float* x, float* y, int* flag,
                       cudaStream_t st) {
  require_plain(op);
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  if (octet_ok(op, dim)) {
    launch_octet<false>(op, t, ld_t, s, ld_s, dim, c2, 0.0f, x, y, flag, st);
    return;
  }
  if (dim <= 64 && nonstat_variant() == 0 &&
      static_cast<int64_t>(op.n_cols) * ld_s < (int64_t{1} << 31)) {  // lean kernel
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
    const bool tl = op.order == KNNX_ORDER_CLUSTER;
    const int nvv = (dim + 3) / 4;
#define LG2(T, NC) gauss_lane_kernel<T, NC><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y)
    if (tl) {
      if (nvv <= 8) LG2(true, 1); else LG2(true, 2);
    } else {
      if (nvv <= 8) LG2(false, 1); else LG2(false, 2);
    }
#undef LG2
    return;
  }
  if (launch_octet_l1<false>(op, t, ld_t, s, ld_s, dim, c2, 0.0f, x, y, flag, st)) return;
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
    // source-streaming kernel (experiment, KNNX_GAUSS_STREAM=1): cluster
    // tiles of 32 rows, rows <= 32 entries.  Measured at C5 5.7 ms vs 3.7 ms
    // for the warp kernel: 1.7x less L2 traffic, but 1.8x
    // the instructions and lockstep batches; off by default
    static const bool stream_on = [] {
      const char* e = std::getenv("KNNX_GAUSS_STREAM");
      return e && std::atoi(e) != 0;
    }();
    constexpr int kB = 8, kNBuf = 6;
    const size_t smem = 128 + static_cast<size_t>(kNBuf) * kB * ld_s * 4;
    if (stream_on && tiles && op.tile_rows == 32 && op.max_slice_len <= 32 && smem <= 227 * 1024 &&
        ld_s % 4 == 0 && nvl <= 8) {
      const int grid = std::min(op.n_tiles, op.ctx->n_sms);
#define L(NVL)                                                                                   \
  {                                                                                              \
    auto k = gauss_stream_kernel<NVL, kB, kNBuf>;                                                \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)); \
    k<<<grid, 544, smem, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y, op.n_tiles);                 \
  }
      KNNX_DISPATCH_NVL(nvl, L)
#undef L
      return;
    }
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
  require_plain(op);
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  if (dim <= 64 && nonstat_variant() == 0 &&
      static_cast<int64_t>(op.n_cols) * ld_s < (int64_t{1} << 31)) {  // lean kernel, weights stored
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
    const int nvv = (dim + 3) / 4;
    const bool tl = op.order == KNNX_ORDER_CLUSTER;
#define LU(T, NC) \
  gauss_lane_kernel<T, NC, true><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, nullptr, nullptr, flag)
    if (tl) {
      if (nvv <= 8) LU(true, 1); else LU(true, 2);
    } else {
      if (nvv <= 8) LU(false, 1); else LU(false, 2);
    }
#undef LU
    return;
  }
  if (dim <= 64 && nonstat_variant() != 1) {  // lane groups, weights stored
    const int nv = (dim + 3) / 4;
    const int g4 = grid_for(static_cast<int64_t>(op.n_rows) * 4, 256);
#define L(T, NC)                                                                           \
  nonstat_group_kernel<T, 4, NC, false, true>                                              \
      <<<g4, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, 0.0f, nullptr, nullptr, flag)
#define LG(T)                                                                              \
  if (nv <= 4) L(T, 1); else if (nv <= 8) L(T, 2); else if (nv <= 12) L(T, 3); else L(T, 4);
    if (op.order == KNNX_ORDER_CLUSTER) {
      LG(true)
    } else {
      LG(false)
    }
#undef LG
#undef L
    return;
  }
  const int grid = grid_for(op.n_rows, 256);
  if (op.order == KNNX_ORDER_CLUSTER)
    update_gauss_kernel<true><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, flag);
  else
    update_gauss_kernel<false><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, flag);
}

void launch_meanshift(const knnx_operator& op, const float* t_in, int ld_t, const float* s,
                      int ld_s, int dim, float c2, float zero_thresh, float* t_out, int* flag,
                      cudaStream_t st) {
  require_plain(op);
  const OpView v = view_of(op);
  if (op.n_rows == 0) return;
  if (octet_ok(op, dim)) {
    launch_octet<true>(op, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, nullptr, t_out, flag, st);
    return;
  }
  if (launch_octet_l1<true>(op, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, nullptr, t_out, flag, st))
    return;
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
  // relabelled columns: gather y into the operator's column numbering first
  const float* yg = y;
  if (op.d_col_order) {
    launch_permute(op.n_cols, static_cast<int64_t>(dim) * 4, y, op.d_col_order, op.d_gather_ws,
                   false, st);
    yg = op.d_gather_ws;
  }
  if (op.interleave) {
    const int g = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
    // register cap (KNNX_TSNE_MINB, read per launch): 6 CTAs per SM = 40
    // registers is the default (C4 N=4M, interleaved, bitwise equal results:
    // 1.60-1.63 ms vs 1.68-1.69 ms uncapped at 46 registers, 1.64-1.71 ms at
    // 32 registers with spills; scripts/probe_c4_minb.py); 1 = uncapped
    const char* mb = std::getenv("KNNX_TSNE_MINB");
    const int minb = mb ? std::atoi(mb) : 6;
    const char* ylenv = std::getenv("KNNX_TSNE_YLOAD");
    const int yl = ylenv ? std::atoi(ylenv) : 0;
#define LI(D)                                                                                  \
  do {                                                                                         \
    if (store) tsne_group_kernel<false, D, 8, true, true><<<g, 256, 0, st>>>(v, y, yg, f, 1, step, y_out); \
    else if (minb == 8) tsne_group_kernel<false, D, 8, false, true, 8><<<g, 256, 0, st>>>(v, y, yg, f, 0, step, y_out); \
    else if (minb == 6 && yl == 1) tsne_group_kernel<false, D, 8, false, true, 6, 1><<<g, 256, 0, st>>>(v, y, yg, f, 0, step, y_out); \
    else if (minb == 6 && yl == 2) tsne_group_kernel<false, D, 8, false, true, 6, 2><<<g, 256, 0, st>>>(v, y, yg, f, 0, step, y_out); \
    else if (minb == 6) tsne_group_kernel<false, D, 8, false, true, 6><<<g, 256, 0, st>>>(v, y, yg, f, 0, step, y_out); \
    else tsne_group_kernel<false, D, 8, false, true><<<g, 256, 0, st>>>(v, y, yg, f, 0, step, y_out);      \
  } while (0)
    switch (dim) {
      case 1: LI(1); break;
      case 2: LI(2); break;
      default: LI(3); break;
    }
#undef LI
    return;
  }
  const bool tiles = op.order == KNNX_ORDER_CLUSTER;
  const int grid = grid_for(op.n_rows, 256);
  const int st_flag = store ? 1 : 0;
  // variants: 0 tiles kG=8 (default), 1 rows, 2 tiles kG=4
  static const int variant = [] {
    const char* e = std::getenv("KNNX_TSNE_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  // variants: 0 auto (lane groups for long rows), 1 rows, 2/3 tiles kG=4/8,
  // 4/5 lane groups G=4/8
  const double avg_len = op.n_rows ? static_cast<double>(op.nnz) / op.n_rows : 0.0;
  // small cluster tiles with a small halo: y[halo] staged in shared memory
  const size_t tg_smem = static_cast<size_t>(op.max_halo) * dim * sizeof(float);
  if (tiles && (variant == 0 || variant == 6) && op.tile_rows <= 64 && tg_smem <= 64 * 1024 &&
      avg_len >= 16) {
    const int block = op.tile_rows * 8;
    auto go = [&](auto kernel) {
      if (tg_smem > 48 * 1024)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tg_smem));
      kernel<<<op.n_tiles, block, tg_smem, st>>>(v, y, yg, f, step, y_out);
    };
#define LTG(D)                                                             \
  do {                                                                     \
    if (store) go(tsne_tiles_group_kernel<D, 8, true>);                    \
    else go(tsne_tiles_group_kernel<D, 8, false>);                         \
  } while (0)
    switch (dim) {
      case 1: LTG(1); break;
      case 2: LTG(2); break;
      default: LTG(3); break;
    }
#undef LTG
    return;
  }
  int gsize = 0;
  if (variant == 4) gsize = 4;
  if (variant == 5) gsize = 8;
  if (variant == 0) gsize = avg_len >= 96 ? 8 : (avg_len >= 16 ? 4 : 0);
  if (gsize) {
    const int g = grid_for(static_cast<int64_t>(op.n_rows) * gsize, 256);
#define LT(T, D, GG)                                                                    \
  do {                                                                                  \
    if (store) tsne_group_kernel<T, D, GG, true><<<g, 256, 0, st>>>(v, y, yg, f, st_flag, step, y_out);  \
    else tsne_group_kernel<T, D, GG, false><<<g, 256, 0, st>>>(v, y, yg, f, st_flag, step, y_out);       \
  } while (0)
#define LD(T, GG)                          \
  switch (dim) {                           \
    case 1: LT(T, 1, GG); break;           \
    case 2: LT(T, 2, GG); break;           \
    default: LT(T, 3, GG); break;          \
  }
    if (tiles) {
      if (gsize == 8) { LD(true, 8) } else { LD(true, 4) }
    } else {
      if (gsize == 8) { LD(false, 8) } else { LD(false, 4) }
    }
#undef LD
#undef LT
    return;
  }
  if (tiles && (variant == 2 || variant == 3)) {
    const size_t smem = static_cast<size_t>(op.max_halo) * dim * sizeof(float);
    auto go = [&](auto kernel) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kernel<<<op.n_tiles, op.tile_rows, smem, st>>>(v, y, yg, f, st_flag, step, y_out);
    };
    if (variant == 2) {
      switch (dim) {
        case 1: (store ? go(tsne_tiles_kernel<1, 4, true>) : go(tsne_tiles_kernel<1, 4, false>)); break;
        case 2: (store ? go(tsne_tiles_kernel<2, 4, true>) : go(tsne_tiles_kernel<2, 4, false>)); break;
        default: (store ? go(tsne_tiles_kernel<3, 4, true>) : go(tsne_tiles_kernel<3, 4, false>)); break;
      }
    } else {
      switch (dim) {
        case 1: (store ? go(tsne_tiles_kernel<1, 8, true>) : go(tsne_tiles_kernel<1, 8, false>)); break;
        case 2: (store ? go(tsne_tiles_kernel<2, 8, true>) : go(tsne_tiles_kernel<2, 8, false>)); break;
        default: (store ? go(tsne_tiles_kernel<3, 8, true>) : go(tsne_tiles_kernel<3, 8, false>)); break;
      }
    }
    return;
  }
#define L(D)                                                                                  \
  if (tiles)                                                                                  \
    (store ? tsne_rows_kernel<true, D, true><<<grid, 256, 0, st>>>(v, y, yg, f, st_flag, step, y_out)       \
           : tsne_rows_kernel<true, D, false><<<grid, 256, 0, st>>>(v, y, yg, f, st_flag, step, y_out));   \
  else                                                                                        \
    (store ? tsne_rows_kernel<false, D, true><<<grid, 256, 0, st>>>(v, y, yg, f, st_flag, step, y_out)      \
           : tsne_rows_kernel<false, D, false><<<grid, 256, 0, st>>>(v, y, yg, f, st_flag, step, y_out));
  switch (dim) {
    case 1: L(1); break;
    case 2: L(2); break;
    default: L(3); break;
  }
#undef L
}

namespace {
// 16-B streaming copy; either side may be mapped pinned host memory (PCIe)
__global__ void __launch_bounds__(256) copy_kernel(uint4* __restrict__ dst,
                                                   const uint4* __restrict__ src, int64_t n) {
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcs(dst + i, __ldcs(src + i));
}
}  // namespace

void launch_copy(void* dst, const void* src, int64_t bytes, cudaStream_t st, int max_ctas) {
  const int64_t n = bytes / 16;
  if (n == 0) return;
  const int grid = static_cast<int>(std::min<int64_t>(grid_for(n, 256), max_ctas));
  copy_kernel<<<grid, 256, 0, st>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n);
}

void launch_permute(int n, int64_t row_bytes, const void* in, const int32_t* idx, void* out,
                    bool scatter, cudaStream_t st) {
  if (n == 0 || row_bytes == 0) return;
  auto go = [&](auto* tag, int64_t words) {
    using W = std::remove_pointer_t<decltype(tag)>;
    const int64_t total = static_cast<int64_t>(n) * words;
    if (total < (int64_t{1} << 31)) {
      const int grid = static_cast<int>(std::max<int64_t>(1, (total + 256 * 4 - 1) / (256 * 4)));
      permute_kernel<W><<<grid, 256, 0, st>>>(n, static_cast<int>(words), static_cast<const W*>(in),
                                              idx, static_cast<W*>(out), scatter);
    } else {
      const int grid = std::min<int64_t>(grid_for(total, 256), 148 * 32);
      permute_kernel_wide<W><<<grid, 256, 0, st>>>(n, static_cast<int>(words),
                                                   static_cast<const W*>(in), idx,
                                                   static_cast<W*>(out), scatter);
    }
  };
  if (row_bytes % 16 == 0)
    go(static_cast<uint4*>(nullptr), row_bytes / 16);
  else
    go(static_cast<uint32_t*>(nullptr), row_bytes / 4);
}

}  // namespace knnx_dev
