// K4/K5: the non-stationary operators -- weights recomputed from the
// coordinates on every call, never stored.
//  K4 gauss_lane_kernel  -- iterate_interactions with the Gaussian value model
//                          (proj/src/kernels.cpp:217-228, knn.cpp:86-108),
//                          dim <= 64; kStore = update_values(Gaussian)
//                          (proj/src/hier.cpp:203-222)
//  K4 gauss_warp_kernel  -- the same for wide rows (C5, D = 960)
//  K5 meanshift_lane_kernel / meanshift_warp_kernel -- meanshift_step
//                          (proj/src/kernels.cpp:184-215)
//  update_gauss_kernel   -- update_values(Gaussian) for dim > 64
// The rejected variants (octets with shared-memory halos, thread per row,
// neighbour-parallel warps, software pipelining, TMA-staged halos and the C5
// source-streaming kernel; DESIGN.md §3.2/§3.3) were measured in round 1 and
// removed from the library.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels_common.cuh"

namespace knnx_dev {
namespace {

// float4 offset of chunk c of source row j: 32-bit arithmetic unless the
// source array spans 2^31 floats (checked by the launchers)
template <bool kOff64>
__device__ __forceinline__ auto src_off(int j, int ld4, int c) {
  if constexpr (kOff64)
    return static_cast<int64_t>(j) * ld4 + c;
  else
    return j * ld4 + c;
}

// K5 mean shift, lane-group kernel (dim <= 64): G = 8 lanes per row, lane g
// owns the float4 chunks g, g + 8 of every row, so a source row is read as
// 128-B contiguous segments; the per-neighbour instruction count is ~30 per
// lane (SASS-counted):
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
template <bool kTiles, int NC, bool kOff64, int kMinBlocks = 4, int NB = 2, int G = 8>
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
        const int j = __shfl_sync(0xffffffffu, jl, gbase + b0 + b);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          const float4 sv = __ldg(s4 + src_off<kOff64>(j, ld4, cidx[u]));
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
template <bool kTiles, int NC, bool kOff64, bool kStore = false>
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
          const float4 sv = __ldg(s4 + src_off<kOff64>(j, ld4, cidx[u]));
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

}  // namespace

namespace {
bool off64(const knnx_operator& op, int ld_s) {
  return static_cast<int64_t>(op.n_cols) * ld_s >= (int64_t{1} << 31);
}
}  // namespace

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

// the lane kernels by (order, chunks per lane, offset width)
#define KNNX_LANE_DISPATCH(TL, NC2, WIDE, LAUNCH) \
  if (TL) {                                       \
    if (NC2) {                                    \
      if (WIDE) LAUNCH(true, 2, true); else LAUNCH(true, 2, false);    \
    } else {                                      \
      if (WIDE) LAUNCH(true, 1, true); else LAUNCH(true, 1, false);    \
    }                                             \
  } else {                                        \
    if (NC2) {                                    \
      if (WIDE) LAUNCH(false, 2, true); else LAUNCH(false, 2, false);  \
    } else {                                      \
      if (WIDE) LAUNCH(false, 1, true); else LAUNCH(false, 1, false);  \
    }                                             \
  }

void launch_gauss_spmv(const knnx_operator& op, const float* t, int ld_t, const float* s,
                       int ld_s, int dim, float c2, const float* x, float* y, int* /*flag*/,
                       cudaStream_t st) {
  require_plain(op);
  if (op.n_rows == 0) return;
  const OpView v = view_of(op);
  const bool tl = op.order == KNNX_ORDER_CLUSTER;
  if (dim <= 64) {  // 8 lanes per row
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
#define L(T, NC, W) gauss_lane_kernel<T, NC, W><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y)
    KNNX_LANE_DISPATCH(tl, dim > 32, off64(op, ld_s), L)
#undef L
    return;
  }
  // wide rows: one warp per row
  const int nvl = ((dim + 3) / 4 + 31) / 32;
  const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 32, 256);
#define L(NVL)                                                                                  \
  if (tl)                                                                                       \
    gauss_warp_kernel<true, NVL><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y);     \
  else                                                                                          \
    gauss_warp_kernel<false, NVL><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, x, y);
  KNNX_DISPATCH_NVL(nvl, L)
#undef L
}

void launch_update_gaussian(const knnx_operator& op, const float* t, int ld_t, const float* s,
                            int ld_s, int dim, float c2, int* flag, cudaStream_t st) {
  require_plain(op);
  if (op.n_rows == 0) return;
  const OpView v = view_of(op);
  const bool tl = op.order == KNNX_ORDER_CLUSTER;
  if (dim <= 64) {  // the K4 lane kernel, weights stored in place
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
#define L(T, NC, W)                                                                              \
  gauss_lane_kernel<T, NC, W, true><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, nullptr, \
                                                          nullptr, flag)
    KNNX_LANE_DISPATCH(tl, dim > 32, off64(op, ld_s), L)
#undef L
    return;
  }
  const int grid = grid_for(op.n_rows, 256);
  if (tl)
    update_gauss_kernel<true><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, flag);
  else
    update_gauss_kernel<false><<<grid, 256, 0, st>>>(v, t, ld_t, s, ld_s, dim, c2, flag);
}

void launch_meanshift(const knnx_operator& op, const float* t_in, int ld_t, const float* s,
                      int ld_s, int dim, float c2, float zero_thresh, float* t_out, int* flag,
                      cudaStream_t st) {
  require_plain(op);
  if (op.n_rows == 0) return;
  const OpView v = view_of(op);
  const bool tl = op.order == KNNX_ORDER_CLUSTER;
  if (dim <= 64) {
    const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 8, 256);
#define L(T, NC, W)                                                                          \
  meanshift_lane_kernel<T, NC, W><<<grid, 256, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2,     \
                                                        zero_thresh, t_out, flag)
    KNNX_LANE_DISPATCH(tl, dim > 32, off64(op, ld_s), L)
#undef L
    return;
  }
  const int nvl = ((dim + 3) / 4 + 31) / 32;
  const int grid = grid_for(static_cast<int64_t>(op.n_rows) * 32, 256);
#define L(NVL)                                                                                 \
  if (tl)                                                                                      \
    meanshift_warp_kernel<true, NVL>                                                           \
        <<<grid, 256, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, t_out, flag);     \
  else                                                                                         \
    meanshift_warp_kernel<false, NVL>                                                          \
        <<<grid, 256, 0, st>>>(v, t_in, ld_t, s, ld_s, dim, c2, zero_thresh, t_out, flag);
  KNNX_DISPATCH_NVL(nvl, L)
#undef L
}

}  // namespace knnx_dev
