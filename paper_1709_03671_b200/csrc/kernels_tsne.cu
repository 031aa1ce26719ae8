// K6: the t-SNE attractive force (tsne_attractive_step,
// proj/src/kernels.cpp:103-136), computed directly as
// F_i = sum_j a_ij (y_i - y_j), a_ij = p_ij / (1 + |y_i - y_j|^2), with the
// optional in-place a_ij write-back (the reference's mutation of P) and the
// fused embedding update y_out = y - step * F.
//  tsne_group_kernel       -- G lanes per row (high-degree rows: C4's
//                             symmetrised k = 90 graph), optionally on the
//                             group-interleaved layout (KNNX_OPT_GROUP_INTERLEAVE)
//  tsne_tiles_group_kernel -- small cluster tiles, y[halo] in shared memory
//  tsne_rows_kernel        -- thread per row (short rows)
// The rejected variants (one CTA per 256-row tile with y[halo] staged,
// cache-policy A/B of the y gathers) were removed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels_common.cuh"

namespace knnx_dev {
namespace {

// ---------------------------------------------------------------------------
// fused update y_new = y - step F of one coordinate: into the local-row output
// and into every rank's replicated embedding (rows row_base + i) -- peer
// stores over NVLink when those buffers live on other GPUs, which replaces
// the all-gather after the kernel
__device__ __forceinline__ void store_y(const TsneOut& o, int row, int row_base, int c, int dim,
                                        float v) {
  if (o.local) o.local[static_cast<int64_t>(row) * dim + c] = v;
  const int64_t g = static_cast<int64_t>(row_base + row) * dim + c;
  // compile-time peer indices: the parameter struct stays in the constant bank
#pragma unroll
  for (int q = 0; q < kMaxPeers; ++q)
    if (q < o.n_peer) o.peer[q][g] = v;
}

// y_j of a DIM-wide embedding row (one 8-B load for the 2-D case)
template <int DIM>
__device__ __forceinline__ void load_y(const float* __restrict__ y, int j, float (&out)[DIM]) {
  if constexpr (DIM == 2) {
    const float2 v2 = __ldg(reinterpret_cast<const float2*>(y) + j);
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
                                                        float step, TsneOut y_out) {
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
    store_y(y_out, real_row(v, row), v.row_base, c, DIM, yi[c] - step * acc[c]);
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
template <bool kTiles, int DIM, int G, bool kStore, bool kInter = false, int kMinB = 1>
__global__ void __launch_bounds__(256, kMinB) tsne_group_kernel(OpView v, const float* __restrict__ y,
                                                         const float* __restrict__ yg,
                                                         float* __restrict__ f, int store,
                                                         float step, TsneOut y_out) {
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
  constexpr int U = 4;  // 8 per block: 362 vs 328 us at N=1M (registers)
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
    for (int u = 0; u < U; ++u) load_y<DIM>(yg, j[u], yj[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) interact(pos(q + u * G), j[u], pj[u], yj[u]);
  }
  for (; q < len; q += G) {
    const int64_t p = pos(q);
    const int j = entry_col<kTiles>(v, p, hbase);
    float yj[DIM];
    load_y<DIM>(yg, j, yj);
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
    store_y(y_out, rr, v.row_base, c, DIM, yi[c] - step * acc[c]);
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
                                                               TsneOut y_out) {
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
    store_y(y_out, rr, v.row_base, c, DIM, yi[c] - step * acc[c]);
  }
}

}  // namespace

void launch_permute(int n, int64_t row_bytes, const void* in, const int32_t* idx, void* out,
                    bool scatter, cudaStream_t st);

void launch_tsne(const knnx_operator& op, const float* y, int dim, float* f, bool store,
                 float step, const TsneOut& y_out, cudaStream_t st) {
  if (op.n_rows == 0) return;
  const OpView v = view_of(op);
  // relabelled columns: gather y into the operator's column numbering first
  const float* yg = y;
  if (op.d_col_order) {
    launch_permute(op.n_cols, static_cast<int64_t>(dim) * 4, y, op.d_col_order, op.d_gather_ws,
                   false, st);
    yg = op.d_gather_ws;
  }
  const int st_flag = store ? 1 : 0;
  if (op.interleave) {
    // 8-lane groups on the interleaved layout, capped at 40 registers (6 CTAs
    // per SM; C4 N=4M: 1.60-1.63 ms vs 1.68-1.69 ms uncapped, bitwise equal)
    const int g = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
#define LI(D)                                                                                      \
  do {                                                                                             \
    if (store)                                                                                     \
      tsne_group_kernel<false, D, 8, true, true, 6><<<g, 256, 0, st>>>(v, y, yg, f, 1, step, y_out); \
    else                                                                                           \
      tsne_group_kernel<false, D, 8, false, true, 6><<<g, 256, 0, st>>>(v, y, yg, f, 0, step, y_out); \
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
  const double avg_len = static_cast<double>(op.nnz) / op.n_rows;
  // small cluster tiles with a small halo: y[halo] staged in shared memory
  const size_t tg_smem = static_cast<size_t>(op.max_halo) * dim * sizeof(float);
  if (tiles && op.tile_rows <= 64 && tg_smem <= 64 * 1024 && avg_len >= 16) {
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
  // lane groups for long rows (8 lanes at >= 96 entries, 4 at >= 16)
  const int gsize = avg_len >= 96 ? 8 : (avg_len >= 16 ? 4 : 0);
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
  const int grid = grid_for(op.n_rows, 256);
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

}  // namespace knnx_dev
