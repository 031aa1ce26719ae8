// kNN builder for wide points (D > 64; C5 has D = 960) on the 5th-generation
// tensor cores (the INPUT builder that replaces the
// O(N^2 D) brute force of proj/src/knn.cpp:9-62).  For wide rows the distance
// screen |q - s|^2 = |q|^2 + |s|^2 - 2 q.s over all (query, source) pairs is a
// real dense contraction, the one place on this path where tensor cores pay.
//
// Pipeline (all on the context stream):
//   1. column mean of the sources; centred copies of queries and sources
//      (less cancellation in the screen) with their squared norms, stored
//      K-chunk-major so that every TMA box is one contiguous run of HBM
//   2. per query tile (128 rows) and source tile (256 rows): centroid, radius,
//      and the squared lower bound (|c_q - c_s| - r_q - r_s)^2 of every
//      (query tile, source tile) pair
//   3. screen_kernel: one CTA per query tile.  Warp 0 = TMA producer (2-D
//      tiled tensor maps, 128-byte swizzle, 4-stage ring of 32-wide K chunks),
//      warp 1 = tcgen05.mma issuer (kind::tf32, 128 x 256 x 8, fp32
//      accumulators in TMEM, two accumulator buffers), warps 2-5 and 6-9 = one
//      epilogue set per accumulator (even / odd tiles, own candidate lists):
//      tcgen05.ld the accumulator, score = |s|^2 - 2 q.s, keep per row the
//      n_cand smallest scores (threshold + append, warp-cooperative radix
//      select when a row's list fills).  The producer walks the source tiles
//      outward from the closest one and skips every tile whose lower bound
//      exceeds the worst row's current n_cand-th distance (plus a rigorous
//      TF32 error bound), so cluster-ordered inputs touch only nearby tiles.
//   4. rerank_kernel: exact fp32 distances of the n_cand candidates per row,
//      the k smallest in ascending (distance, index) order.
//
// Measured on the B200 (profiles/r2_knn_wide_*): C5 (N = 1M, D = 960, k = 16)
// 3.6 s against 20.7 s for the cuBLAS TF32 + torch.topk tool it replaces; the
// screen runs the tensor pipe at 42 % with DRAM at 65 % of peak (the 3.8-KB
// rows make the 128 x 256 fp32 tiles HBM-latency bound at 192 KB in flight
// per SM; 256-query CTAs and co-scheduled groups were measured and are slower).
//
// The result equals fp32 brute force unless a true neighbour's TF32 score
// falls outside the n_cand best scores of its row.  Every row is certified
// against that (rerank_kernel); rows that fail -- clusters tight against
// their distance from the mean, where a TF32 product cannot rank -- are
// searched again by the exact SIMT kernel (dim <= 64) or screened again with
// 3xTF32 operands (kPrecise) and certified anew; the statistics report what
// is left, and the tests compare sampled rows with brute-force oracles.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <string>

#include "knnx_internal.cuh"
#include "knnx_rt.cuh"
#include "ptx.cuh"

using namespace knnx_rt;

namespace {

using knnx_dev::mbar_arrive;
using knnx_dev::mbar_arrive_expect_tx;
using knnx_dev::mbar_init;
using knnx_dev::mbar_wait;
using knnx_dev::smem_u32;

constexpr int kTM = 128;      // query rows per CTA (= TMEM lanes)
constexpr int kTN = 256;      // source rows per tile (= accumulator columns)
constexpr int kKC = 32;       // K per pipeline stage: 32 fp32 = one 128-byte swizzle row
constexpr int kStages = 4;        // TF32 screen: 4 stages of 48 KB
constexpr int kStagesPrecise = 2; // 3xTF32 screen: 2 stages of 96 KB (operands + their low parts)
constexpr int kMaxCand = 256; // candidates per row (list capacity 256 up to 128, 512 beyond)
constexpr int kThreads = 320; // producer warp, MMA warp, 2 sets of 4 epilogue warps (one per accumulator)
constexpr uint32_t kBytesA = kTM * kKC * 4, kBytesB = kTN * kKC * 4;
constexpr uint32_t kTmemCols = 512;  // two 256-column accumulators

// ---------------------------------------------------------------- prepasses

// partial column sums of rows [b * rows_per, ...): deterministic two-stage mean
__global__ void colsum_partial_kernel(const float* __restrict__ p, int n, int ld, int rows_per,
                                      float* __restrict__ part) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= ld) return;
  const int lo = blockIdx.x * rows_per, hi = min(n, lo + rows_per);
  float acc = 0.f;
  for (int i = lo; i < hi; ++i) acc += p[static_cast<int64_t>(i) * ld + c];
  part[static_cast<int64_t>(blockIdx.x) * ld + c] = acc;
}

__global__ void colsum_final_kernel(const float* __restrict__ part, int n_part, int ld, int dim,
                                    float inv_n, float* __restrict__ mean) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ld) return;
  float acc = 0.f;
  for (int b = 0; b < n_part; ++b) acc += part[static_cast<int64_t>(b) * ld + c];
  mean[c] = c < dim ? acc * inv_n : 0.f;
}

// The centred scratch copies are K-chunk-major: chunk c (32 columns = 128 B)
// of row r lives at ((c * n_pad + r) * 32) floats, so the 128- or 256-row box a
// TMA load fetches is one contiguous 16- or 32-KB run of HBM instead of 128-B
// pieces a row pitch apart.  Columns past dim and rows past n are zero.
__device__ __forceinline__ int64_t cm_off4(int row, int c4, int64_t n_pad) {
  return ((static_cast<int64_t>(c4 >> 3) * n_pad + row) << 5) + ((c4 & 7) << 2);
}

// out = in - mean in the chunk-major layout, norm2[i] = |out_i|^2; warp per row
// perm (may be null): scratch row p holds input row perm[p]; perm[p] < 0 marks
// the padding rows that align every pivot cell to a tile boundary
// lo (may be null): the part of every value the tensor core drops when it reads
// the fp32 word as TF32 (the low 13 mantissa bits), for the 3xTF32 screen
__global__ void center_kernel(const float* __restrict__ in, int n, int ld, int dim,
                              const float* __restrict__ mean, const int32_t* __restrict__ perm,
                              float* __restrict__ out, int64_t n_pad, float* __restrict__ norm2,
                              float* __restrict__ lo) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int src_row = perm ? perm[row] : row;
  if (src_row < 0) return;  // cell padding: the scratch row stays zero, its norm +inf
  const float4* src = reinterpret_cast<const float4*>(in + static_cast<int64_t>(src_row) * ld);
  const float4* mu = reinterpret_cast<const float4*>(mean);
  float acc = 0.f;
  for (int c = lane; c < ld / 4; c += 32) {
    float4 v = __ldg(src + c);
    const float4 m = __ldg(mu + c);
    v.x = 4 * c + 0 < dim ? v.x - m.x : 0.f;
    v.y = 4 * c + 1 < dim ? v.y - m.y : 0.f;
    v.z = 4 * c + 2 < dim ? v.z - m.z : 0.f;
    v.w = 4 * c + 3 < dim ? v.w - m.w : 0.f;
    *reinterpret_cast<float4*>(out + cm_off4(row, c, n_pad)) = v;
    if (lo) {
      float4 l;
      l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
      l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
      l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
      l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
      *reinterpret_cast<float4*>(lo + cm_off4(row, c, n_pad)) = l;
    }
    acc = fmaf(v.x, v.x, acc);
    acc = fmaf(v.y, v.y, acc);
    acc = fmaf(v.z, v.z, acc);
    acc = fmaf(v.w, v.w, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) norm2[row] = acc;
}

__global__ void fill_kernel(float* p, int n, float v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// per ball of `bs` rows of a chunk-major copy: centroid (ldc = 32 * n_chunks
// floats, row-major) and an outward-rounded radius over the rows that are not
// cell padding (perm[i] < 0); an empty ball gets radius -1.  256 threads.
__global__ void tile_stats_kernel(const float* __restrict__ p, int n, int64_t n_pad, int ldc, int bs,
                                  const int32_t* __restrict__ perm, float* __restrict__ ctr,
                                  float* __restrict__ rad) {
  const int b = blockIdx.x, lo = b * bs, hi = min(n, lo + bs);
  float* c = ctr + static_cast<int64_t>(b) * ldc;
  __shared__ int s_cnt;
  if (threadIdx.x == 0) {
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += (!perm || perm[i] >= 0) ? 1 : 0;
    s_cnt = cnt;
  }
  __syncthreads();
  const int cnt = s_cnt;
  // padding rows are zero in the scratch copy, so plain sums give the centroid
  const float inv = cnt > 0 ? 1.0f / static_cast<float>(cnt) : 0.f;
  for (int col = threadIdx.x; col < ldc; col += blockDim.x) {
    const float* base = p + ((static_cast<int64_t>(col >> 5) * n_pad) << 5) + (col & 31);
    float acc = 0.f;
    for (int i = lo; i < hi; ++i) acc += base[static_cast<int64_t>(i) << 5];
    c[col] = acc * inv;
  }
  __syncthreads();
  __shared__ float wmax[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, n_warps = blockDim.x >> 5;
  float mx = 0.f;
  for (int i = lo + warp; i < hi; i += n_warps) {
    if (perm && perm[i] < 0) continue;
    float acc = 0.f;
    for (int q = lane; q < ldc / 4; q += 32) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + cm_off4(i, q, n_pad)));
      const float4 m = reinterpret_cast<const float4*>(c)[q];
      const float e0 = v.x - m.x, e1 = v.y - m.y, e2 = v.z - m.z, e3 = v.w - m.w;
      acc = fmaf(e0, e0, acc);
      acc = fmaf(e1, e1, acc);
      acc = fmaf(e2, e2, acc);
      acc = fmaf(e3, e3, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    mx = fmaxf(mx, acc);
  }
  if (lane == 0) wmax[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < n_warps; ++w) mx = fmaxf(mx, wmax[w]);
    rad[b] = cnt > 0 ? sqrtf(mx) * 1.0001f + 1e-6f : -1.0f;
  }
}

// lb2[q][t] = min over the two 128-row balls h of source tile t of
// max(0, |c_q - c_h| - r_q - r_h)^2 (shrunk by 1e-4 against fp32 rounding;
// +inf when either side is empty).  One CTA per query tile, one warp per
// source ball in turn.
__global__ void tile_lb_kernel(const float* __restrict__ qc, const float* __restrict__ qr,
                               const float* __restrict__ sc, const float* __restrict__ sr, int n_sb,
                               int n_st, int ld, float* __restrict__ lb2) {
  extern __shared__ __align__(16) float qs[];
  const int qt = blockIdx.x;
  for (int c = threadIdx.x; c < ld; c += blockDim.x) qs[c] = qc[static_cast<int64_t>(qt) * ld + c];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, n_warps = blockDim.x >> 5;
  const float rq = qr[qt];
  for (int t = warp; t < n_st; t += n_warps) {
    float best = __int_as_float(0x7f800000);
    for (int h = 2 * t; h < min(n_sb, 2 * t + 2); ++h) {
      const float4* r = reinterpret_cast<const float4*>(sc + static_cast<int64_t>(h) * ld);
      float acc = 0.f;
      for (int q = lane; q < ld / 4; q += 32) {
        const float4 v = __ldg(r + q);
        const float4 m = reinterpret_cast<const float4*>(qs)[q];
        const float e0 = v.x - m.x, e1 = v.y - m.y, e2 = v.z - m.z, e3 = v.w - m.w;
        acc = fmaf(e0, e0, acc);
        acc = fmaf(e1, e1, acc);
        acc = fmaf(e2, e2, acc);
        acc = fmaf(e3, e3, acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const float rs = sr[h];
      if (rq >= 0.f && rs >= 0.f) {
        const float lb = (sqrtf(acc) - rq - rs) * 0.9999f;
        best = fminf(best, lb > 0.f ? lb * lb : 0.f);
      }
    }
    if (lane == 0) lb2[static_cast<int64_t>(qt) * n_st + t] = best;
  }
}

// ------------------------------------------------------------ screen kernel

// K-major operand tile, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B
// apart (SBO); LBO unused for swizzled K-major layouts
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// D fp32, A/B tf32, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) |
                            (static_cast<uint32_t>(kTN >> 3) << 17) |
                            (static_cast<uint32_t>(kTM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// order-preserving map float bits -> unsigned
__device__ __forceinline__ uint32_t f2key(uint32_t b) {
  return b ^ (static_cast<uint32_t>(static_cast<int32_t>(b) >> 31) | 0x80000000u);
}
__device__ __forceinline__ uint32_t key2f(uint32_t k) {
  return k ^ ((k & 0x80000000u) ? 0x80000000u : 0xFFFFFFFFu);
}

// Keeps the m smallest of the c (> m, <= kCap) entries of one row's list
// (score bits, id), all 32 lanes cooperating; returns the m-th smallest score.
template <int kCap>
__device__ float compact_row(uint2* base, int c, int m, int lane) {
  uint32_t key[kCap / 32], id[kCap / 32];
#pragma unroll
  for (int j = 0; j < kCap / 32; ++j) {
    const int idx = lane + 32 * j;
    key[j] = 0xFFFFFFFFu;
    id[j] = 0;
    if (idx < c) {
      const uint2 e = base[idx];
      key[j] = f2key(e.x);
      id[j] = e.y;
    }
  }
  __syncwarp();
  // smallest T with count(key <= T) >= m
  uint32_t lo = 0, hi = 0xFFFFFFFEu;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < kCap / 32; ++j) cnt += key[j] <= mid ? 1 : 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (cnt >= m) hi = mid; else lo = mid + 1;
  }
  const uint32_t thr = lo;
  const uint32_t below = (1u << lane) - 1u;
  int pos = 0;
#pragma unroll
  for (int j = 0; j < kCap / 32; ++j) {
    const bool f = key[j] < thr;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (f) base[pos + __popc(b & below)] = make_uint2(key2f(key[j]), id[j]);
    pos += __popc(b);
  }
#pragma unroll
  for (int j = 0; j < kCap / 32; ++j) {
    const bool f = key[j] == thr;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    const int my = pos + __popc(b & below);
    if (f && my < m) base[my] = make_uint2(key2f(key[j]), id[j]);
    pos += __popc(b);
  }
  __syncwarp();
  return __uint_as_float(key2f(thr));
}

struct ScreenArgs {
  int nq, ns, n_chunks, n_stiles, n_cand, self_set;
  int q_pad, s_pad;     // padded row counts of the chunk-major query / source copies
  const float* qnorm;   // [nq]
  const int32_t* qvalid; // null, or [nq] with < 0 on cell-padding rows
  const int32_t* qself;  // null (query row p is source p), or [nq]: the source position of query p itself
  const float* snorm;   // [n_stiles * kTN], +inf past ns
  const float* lb2;     // [n_qtiles][n_stiles]
  uint2* lists;         // [query tiles of this launch][2 epilogue sets][kTM][kCap]
  int qt_base;          // first query tile of this launch
  int32_t* cand;        // [nq][n_cand], -1 padded
  float* cand_score;    // [nq][n_cand]: the screen's squared distance of each candidate
  float* tau;           // [nq]: screen distance of the n_cand-th candidate (inf if fewer)
  unsigned long long* tiles_done;  // total source tiles multiplied (statistics)
};

// kPrecise: 3xTF32 -- every K step also multiplies the operands' dropped low
// parts (q.s ~ q_hi.s_hi + q_hi.s_lo + q_lo.s_hi, error ~2^-21 |q||s|), for the
// rows a plain TF32 screen cannot certify
template <int kCap, bool kPrecise>
__global__ void __launch_bounds__(kThreads, 1)
    screen_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_s,
                  const __grid_constant__ CUtensorMap map_qlo, const __grid_constant__ CUtensorMap map_slo,
                  const ScreenArgs a) {
  constexpr int kStages = kPrecise ? ::kStagesPrecise : ::kStages;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle
  unsigned char* ring = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* ring_a = ring;
  unsigned char* ring_b = ring + kStages * kBytesA;
  unsigned char* ring_alo = ring_b + kStages * kBytesB;      // used when kPrecise
  unsigned char* ring_blo = ring_alo + kStages * kBytesA;
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ volatile int stage_tile[kStages];
  __shared__ volatile int acc_tile[2];
  __shared__ volatile float warp_u[8];   // [set][quarter]
  __shared__ volatile float warp_qmax[4];
  __shared__ int cnt_b[kTM];             // set B's per-row results for the final merge
  __shared__ float tau_b[kTM];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = a.qt_base + blockIdx.x;
  const int m0 = qt * kTM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);
    }
    knnx_dev::fence_mbar_init();
  }
  if (threadIdx.x < 8) warp_u[threadIdx.x] = __int_as_float(0x7f800000);
  if (threadIdx.x < 4) warp_qmax[threadIdx.x] = 0.f;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------- producer: pick tiles, feed the ring with TMA
    const float* lbrow = a.lb2 + static_cast<int64_t>(qt) * a.n_stiles;
    float best = __int_as_float(0x7f800000);
    int bi = 0x7fffffff;
    for (int t = lane; t < a.n_stiles; t += 32) {
      const float v = lbrow[t];
      if (v < best) {
        best = v;
        bi = t;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (bi == 0x7fffffff) bi = 0;
    if (lane == 0) {
      uint32_t it = 0;
      unsigned long long n_done = 0;
      for (int d = 0; d < a.n_stiles; ++d) {
        for (int side = 0; side < (d == 0 ? 1 : 2); ++side) {
          const int t = side == 0 ? bi + d : bi - d;
          if (t < 0 || t >= a.n_stiles) continue;
          if (n_done > 0) {
            // every row's n_cand-th distance is bounded by either set's list
            const float u = fmaxf(fmaxf(fminf(warp_u[0], warp_u[4]), fminf(warp_u[1], warp_u[5])),
                                  fmaxf(fminf(warp_u[2], warp_u[6]), fminf(warp_u[3], warp_u[7])));
            const float qm = fmaxf(fmaxf(warp_qmax[0], warp_qmax[1]), fmaxf(warp_qmax[2], warp_qmax[3]));
            // TF32 operands are truncated: |err(q.s)| <= 2^-9 |q||s| and only
            // sources with |s| <= |q| + sqrt(u) matter; the score uses 2 q.s
            const float eps = 0.00390625f * qm * (qm + sqrtf(fmaxf(u, 0.f)));
            if (lbrow[t] > u + eps) continue;
          }
          ++n_done;
          for (int c = 0; c < a.n_chunks; ++c, ++it) {
            const int s = it % kStages;
            mbar_wait(&empty_bar[s], ((it / kStages) & 1) ^ 1);
            stage_tile[s] = t;
            mbar_arrive_expect_tx(&full_bar[s], (kBytesA + kBytesB) * (kPrecise ? 2 : 1));
            tma_load_2d(ring_a + s * kBytesA, &map_q, 0, c * a.q_pad + m0, &full_bar[s]);
            tma_load_2d(ring_b + s * kBytesB, &map_s, 0, c * a.s_pad + t * kTN, &full_bar[s]);
            if constexpr (kPrecise) {
              tma_load_2d(ring_alo + s * kBytesA, &map_qlo, 0, c * a.q_pad + m0, &full_bar[s]);
              tma_load_2d(ring_blo + s * kBytesB, &map_slo, 0, c * a.s_pad + t * kTN, &full_bar[s]);
            }
          }
        }
      }
      const int s = it % kStages;
      mbar_wait(&empty_bar[s], ((it / kStages) & 1) ^ 1);
      stage_tile[s] = -1;
      __threadfence_block();
      mbar_arrive(&full_bar[s]);
      if (a.tiles_done) atomicAdd(a.tiles_done, n_done);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      uint32_t tile_n = 0;
      for (uint32_t it = 0;; ++it) {
        const int s = it % kStages;
        mbar_wait(&full_bar[s], (it / kStages) & 1);
        const int t = stage_tile[s];
        const uint32_t acc = tile_n & 1;
        if (t < 0) {  // end of the stream: tell both epilogue sets
          for (uint32_t b = 0; b < 2; ++b) {
            const uint32_t uses = (tile_n + 1 - b) >> 1;  // tiles accumulator b has held
            mbar_wait(&tempty_bar[b], (uses & 1) ^ 1);
            acc_tile[b] = -1;
            __threadfence_block();
            mbar_arrive(&tfull_bar[b]);
          }
          break;
        }
        const int c = it % a.n_chunks;
        if (c == 0) {
          mbar_wait(&tempty_bar[acc], ((tile_n >> 1) & 1) ^ 1);
          acc_tile[acc] = t;
          __threadfence_block();
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t a0 = smem_u32(ring_a + s * kBytesA), b0 = smem_u32(ring_b + s * kBytesB);
#pragma unroll
        for (int ks = 0; ks < kKC / 8; ++ks) {
          mma_tf32(tmem + acc * kTN, umma_desc_sw128(a0 + ks * 32), umma_desc_sw128(b0 + ks * 32),
                   (c | ks) != 0 ? 1u : 0u);
          if constexpr (kPrecise) {
            const uint32_t al = smem_u32(ring_alo + s * kBytesA), bl = smem_u32(ring_blo + s * kBytesB);
            mma_tf32(tmem + acc * kTN, umma_desc_sw128(a0 + ks * 32), umma_desc_sw128(bl + ks * 32), 1u);
            mma_tf32(tmem + acc * kTN, umma_desc_sw128(al + ks * 32), umma_desc_sw128(b0 + ks * 32), 1u);
          }
        }
        umma_commit(&empty_bar[s]);  // frees the stage when these MMAs have read it
        if (c == a.n_chunks - 1) {
          umma_commit(&tfull_bar[acc]);
          ++tile_n;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: set A (warps 2-5) drains accumulator 0 (even
    // tiles), set B (warps 6-9) accumulator 1 (odd tiles); each set keeps its
    // own candidate list per row, merged at the end.  TMEM lanes (warp % 4) * 32 ..
    const int set = warp >= 6 ? 1 : 0;
    const int quarter = warp & 3;
    const int lrow = quarter * 32 + lane;
    const int row = m0 + lrow;
    const bool valid = row < a.nq && (a.qvalid == nullptr || a.qvalid[row] >= 0);
    const float qn = valid ? a.qnorm[row] : 0.f;
    const int self_col = (valid && a.qself) ? a.qself[row] : row;
    {
      float qm = valid ? sqrtf(qn) : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
      if (lane == 0 && set == 0) warp_qmax[quarter] = qm;
    }
    float tau = valid ? __int_as_float(0x7f800000) : -__int_as_float(0x7f800000);
    int cnt = 0;
    uint2* wlist = a.lists + ((static_cast<int64_t>(blockIdx.x) * 2 + set) * kTM + quarter * 32) * kCap;
    uint2* mylist = wlist + static_cast<int64_t>(lane) * kCap;
    for (uint32_t e = set;; e += 2) {
      const uint32_t acc = e & 1;
      mbar_wait(&tfull_bar[acc], (e >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int t = acc_tile[acc];
      if (t < 0) break;
      const int col0 = t * kTN;
#pragma unroll 1
      for (int c0 = 0; c0 < kTN; c0 += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kTN + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
            "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
            "%30, %31}, [%32];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
              "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
              "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const float4* sn4 = reinterpret_cast<const float4*>(a.snorm + col0 + c0);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 n4 = __ldg(sn4 + q4);
          const float nn[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float score = fmaf(-2.0f, __uint_as_float(r[4 * q4 + u]), nn[u]);
            if (score < tau) {
              const int col = col0 + c0 + 4 * q4 + u;
              if (!(a.self_set && col == self_col)) {
                mylist[cnt] = make_uint2(__float_as_uint(score), static_cast<uint32_t>(col));
                ++cnt;
              }
            }
          }
        }
        uint32_t fullm = __ballot_sync(0xffffffffu, cnt > kCap - 32);
        while (fullm) {
          const int l = __ffs(fullm) - 1;
          fullm &= fullm - 1;
          const int c = __shfl_sync(0xffffffffu, cnt, l);
          __syncwarp();
          const float nt = compact_row<kCap>(wlist + static_cast<int64_t>(l) * kCap, c, a.n_cand, lane);
          if (lane == l) {
            cnt = a.n_cand;
            tau = nt;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      float u = valid ? qn + tau : -__int_as_float(0x7f800000);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) u = fmaxf(u, __shfl_xor_sync(0xffffffffu, u, o));
      if (lane == 0) warp_u[set * 4 + quarter] = u;
    }
    // every list down to n_cand entries; tau = bound on the scores a set dropped
    __syncwarp();
    for (int l = 0; l < 32; ++l) {
      const int c = __shfl_sync(0xffffffffu, cnt, l);
      __syncwarp();
      if (c > a.n_cand) {
        const float nt = compact_row<kCap>(wlist + static_cast<int64_t>(l) * kCap, c, a.n_cand, lane);
        if (lane == l) {
          cnt = a.n_cand;
          tau = nt;
        }
      }
    }
    if (set == 1) {
      cnt_b[lrow] = cnt;
      tau_b[lrow] = tau;
    }
    // the two warps of a quarter meet (named barrier 1 + quarter, 64 threads);
    // set A then merges set B's list into its own and writes the row's output
    asm volatile("bar.sync %0, 64;\n" ::"r"(1 + quarter) : "memory");
    if (set == 0) {
      const uint2* blist = a.lists + ((static_cast<int64_t>(blockIdx.x) * 2 + 1) * kTM + quarter * 32) * kCap;
      for (int l = 0; l < 32; ++l) {
        const int r_out = m0 + quarter * 32 + l;
        if (r_out >= a.nq) break;
        const int ca = __shfl_sync(0xffffffffu, cnt, l);
        const int cb = cnt_b[quarter * 32 + l];
        uint2* base = wlist + static_cast<int64_t>(l) * kCap;
        const uint2* other = blist + static_cast<int64_t>(l) * kCap;
        float t_fin = fminf(__shfl_sync(0xffffffffu, tau, l), tau_b[quarter * 32 + l]);
        const float qn_l = __shfl_sync(0xffffffffu, qn, l);
        for (int i = lane; i < cb; i += 32) base[ca + i] = other[i];  // ca + cb <= 2 n_cand <= kCap
        __syncwarp();
        int c = ca + cb;
        if (c > a.n_cand) {
          t_fin = fminf(t_fin, compact_row<kCap>(base, c, a.n_cand, lane));
          c = a.n_cand;
        }
        for (int i = lane; i < a.n_cand; i += 32) {
          const uint2 e = i < c ? base[i] : make_uint2(0x7f800000u, 0xffffffffu);
          a.cand[static_cast<int64_t>(r_out) * a.n_cand + i] = static_cast<int32_t>(e.y);
          a.cand_score[static_cast<int64_t>(r_out) * a.n_cand + i] = qn_l + __uint_as_float(e.x);
        }
        if (lane == 0) a.tau[r_out] = qn_l + t_fin;
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
}

// ------------------------------------------------------------ exact re-rank

// warp per query row: exact fp32 squared distances of its candidates, then the
// k smallest in ascending (distance, index) order
__global__ void __launch_bounds__(256)
    rerank_kernel(const float* __restrict__ q, int nq, const float* __restrict__ s, int ld, int dim,
                  const int32_t* __restrict__ qperm, const int32_t* __restrict__ sperm,
                  const int32_t* __restrict__ cand, const float* __restrict__ cand_score, int n_cand, int k,
                  int32_t* __restrict__ ids, float* __restrict__ d2, const float* __restrict__ tau,
                  float* __restrict__ margin) {
  // the screen works on (optionally) re-partitioned copies: its row p is the
  // caller's query qperm[p] and its candidate c the caller's source sperm[c]
  const int prow = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (prow >= nq) return;
  const int row = qperm ? qperm[prow] : prow;
  if (row < 0) return;  // cell padding
  const float4* qv = reinterpret_cast<const float4*>(q + static_cast<int64_t>(row) * ld);
  const int nv = ld / 4;
  float dist[kMaxCand / 32];
  int cid[kMaxCand / 32];
#pragma unroll
  for (int j = 0; j < kMaxCand / 32; ++j) {
    dist[j] = FLT_MAX;
    cid[j] = 0x7fffffff;
  }
  // signed error (screen - exact squared distance) over this row's candidates:
  // TF32 truncates, so the errors share a bias (which does not change the
  // ranking) and spread around it
  float e_max = -FLT_MAX, e_min = FLT_MAX;
  for (int i0 = 0; i0 < n_cand; i0 += 32) {
    int mine = i0 + lane < n_cand ? cand[static_cast<int64_t>(prow) * n_cand + i0 + lane] : -1;
    const float approx = mine >= 0 ? cand_score[static_cast<int64_t>(prow) * n_cand + i0 + lane] : 0.f;
    if (mine >= 0 && sperm) mine = sperm[mine];
    float dmine = FLT_MAX;
    for (int i = 0; i < 32 && i0 + i < n_cand; ++i) {
      const int j = __shfl_sync(0xffffffffu, mine, i);
      if (j < 0) continue;
      const float4* sv = reinterpret_cast<const float4*>(s + static_cast<int64_t>(j) * ld);
      float p0 = 0.f, p1 = 0.f;
      for (int c = lane; c < nv; c += 32) {
        const float4 x = __ldg(qv + c), y = __ldg(sv + c);
        float e0 = x.x - y.x, e1 = x.y - y.y, e2 = x.z - y.z, e3 = x.w - y.w;
        if (4 * c + 3 >= dim) {
          if (4 * c + 1 >= dim) e1 = 0.f;
          if (4 * c + 2 >= dim) e2 = 0.f;
          e3 = 0.f;
        }
        p0 = fmaf(e0, e0, p0);
        p1 = fmaf(e1, e1, p1);
        p0 = fmaf(e2, e2, p0);
        p1 = fmaf(e3, e3, p1);
      }
      float acc = p0 + p1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == i) dmine = acc;
    }
    if (mine >= 0) {
      e_max = fmaxf(e_max, approx - dmine);
      e_min = fminf(e_min, approx - dmine);
    }
#pragma unroll
    for (int j = 0; j < kMaxCand / 32; ++j)
      if (j == i0 / 32) {
        dist[j] = mine >= 0 ? dmine : FLT_MAX;
        cid[j] = mine >= 0 ? mine : 0x7fffffff;
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e_max = fmaxf(e_max, __shfl_xor_sync(0xffffffffu, e_max, o));
    e_min = fminf(e_min, __shfl_xor_sync(0xffffffffu, e_min, o));
  }
  float kth = FLT_MAX;
  for (int r = 0; r < k; ++r) {
    float bd = FLT_MAX;
    int bi = 0x7fffffff, bj = 0;
#pragma unroll
    for (int j = 0; j < kMaxCand / 32; ++j)
      if (dist[j] < bd || (dist[j] == bd && cid[j] < bi)) {
        bd = dist[j];
        bi = cid[j];
        bj = j;
      }
    float wd = bd;
    int wi = bi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float od = __shfl_xor_sync(0xffffffffu, wd, o);
      const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
      if (od < wd || (od == wd && oi < wi)) {
        wd = od;
        wi = oi;
      }
    }
    if (wi == bi && wd == bd && bi != 0x7fffffff) {
#pragma unroll
      for (int j = 0; j < kMaxCand / 32; ++j)
        if (j == bj) {
          dist[j] = FLT_MAX;
          cid[j] = 0x7fffffff;
        }
    }
    if (lane == 0) {
      ids[static_cast<int64_t>(row) * k + r] = wi == 0x7fffffff ? -1 : wi;
      d2[static_cast<int64_t>(row) * k + r] = wd;
    }
    kth = wd;
  }
  // Certificate: every source the screen dropped had a screen distance above
  // tau, so its exact distance is above tau minus its screen error; that
  // error is bounded by the largest one seen on this row's own candidates
  // plus their whole spread as a safety margin.  margin > 0: no dropped
  // source can belong to the k nearest; rows with margin <= 0 are recomputed
  // exactly (dim <= 64) or reported.
  if (lane == 0 && margin)
    margin[row] = e_max >= e_min ? tau[prow] - (e_max + (e_max - e_min)) - kth : tau[prow] - kth;
}

// rows whose certificate failed, in any order
__global__ void select_uncertified_kernel(const float* __restrict__ margin, int n, int32_t* __restrict__ sel,
                                          int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(margin[i] > 0.f)) sel[atomicAdd(cnt, 1)] = i;
}

// exact rows (kk = k or k + 1 neighbours, self possibly among them) into the
// caller's arrays; those rows are exact, so their margin becomes +inf
__global__ void exact_rows_fixup_kernel(const int32_t* __restrict__ sel, int n_sel,
                                        const int32_t* __restrict__ ids_sub, const float* __restrict__ d2_sub,
                                        int kk, int k, bool self_set, int32_t* __restrict__ ids,
                                        float* __restrict__ d2, float* __restrict__ margin) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_sel) return;
  const int row = sel[r];
  int o = 0;
  for (int q = 0; q < kk && o < k; ++q) {
    const int j = ids_sub[static_cast<int64_t>(r) * kk + q];
    if (self_set && j == row) continue;
    ids[static_cast<int64_t>(row) * k + o] = j;
    d2[static_cast<int64_t>(row) * k + o] = d2_sub[static_cast<int64_t>(r) * kk + q];
    ++o;
  }
  margin[row] = __int_as_float(0x7f800000);
}

__global__ void inverse_perm_kernel(const int32_t* __restrict__ perm, int rows, int32_t* __restrict__ inv) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < rows && perm[p] >= 0) inv[perm[p]] = p;
}

// self position per scratch row of a re-partitioned subset
__global__ void remap_self_kernel(const int32_t* __restrict__ qperm, int rows, const int32_t* __restrict__ self_of,
                                  int32_t* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < rows) out[p] = qperm[p] >= 0 ? self_of[qperm[p]] : -1;
}

__global__ void scatter_rows_kernel(const int32_t* __restrict__ sel, int n_sel, const int32_t* __restrict__ ids_sub,
                                    const float* __restrict__ d2_sub, const float* __restrict__ margin_sub, int k,
                                    int32_t* __restrict__ ids, float* __restrict__ d2, float* __restrict__ margin) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_sel) return;
  const int row = sel[r];
  for (int q = 0; q < k; ++q) {
    ids[static_cast<int64_t>(row) * k + q] = ids_sub[static_cast<int64_t>(r) * k + q];
    d2[static_cast<int64_t>(row) * k + q] = d2_sub[static_cast<int64_t>(r) * k + q];
  }
  margin[row] = margin_sub[r];
}

__global__ void margin_stats_kernel(const float* __restrict__ margin, int n, float* __restrict__ out) {
  // out[0] = min margin, out[1] = number of rows with margin <= 0 (as float)
  __shared__ float smin[256];
  __shared__ int sneg[256];
  float mn = FLT_MAX;
  int neg = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = margin[i];
    mn = fminf(mn, v);
    neg += !(v > 0.f) ? 1 : 0;
  }
  smin[threadIdx.x] = mn;
  sneg[threadIdx.x] = neg;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < blockDim.x; ++t) {
      mn = fminf(mn, smin[t]);
      neg += sneg[t];
    }
    out[0] = mn;
    out[1] = static_cast<float>(neg);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// chunk-major copy seen as (n_chunks * n_pad) rows of 32 fp32; box = one
// chunk of box_rows rows, 128-byte swizzle
CUtensorMap make_map(const float* base, int64_t n_pad, int n_chunks, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  require(enc != nullptr, knnx::errc::unsupported, "cuTensorMapEncodeTiled is not available");
  CUtensorMap m;
  const cuuint64_t gdim[2] = {kKC, static_cast<cuuint64_t>(n_pad) * n_chunks};
  const cuuint64_t gstride[1] = {kKC * 4};
  const cuuint32_t box[2] = {kKC, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride,
                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, knnx::errc::invalid_argument,
          "cuTensorMapEncodeTiled failed with code " + std::to_string(static_cast<int>(r)));
  return m;
}

struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    check(cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), st), "cudaMallocAsync (kNN scratch)");
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};



__global__ void iota_kernel(int32_t* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

__global__ void pivot_rows_kernel(int32_t* p, int n_piv, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_piv) p[i] = static_cast<int32_t>(static_cast<int64_t>(i) * n / n_piv);
}

struct WideStats {
  float* margin = nullptr;            // [m], caller's row order
  unsigned long long* tiles = nullptr;
  double dense_tiles = 0;
};

// The screen + re-rank on the caller's points.  The screen works on scratch
// copies of m query rows and n source rows; qperm / sperm (device, may be
// null = identity) say which caller row each scratch row holds (< 0: padding).
// n_true = number of caller source rows (for the column mean).
// precise: the 3xTF32 screen.  qself (may be null): source scratch position of
// each query row's own point, for self exclusion when the queries are not the
// sources' scratch rows (the re-run of a subset of rows).
void knn_wide_core(knnx_ctx_t ctx, Scratch& ws, const float* t, int m, const float* s, int n, int n_true,
                   int ld, int dim, int k, int n_cand, bool self_set, bool same, const int32_t* qperm,
                   const int32_t* sperm, int32_t* ids, float* d2, WideStats* stats, bool precise = false,
                   const int32_t* qself = nullptr) {
  cudaStream_t st = ctx->stream;
  const int n_qt = (m + kTM - 1) / kTM, n_st = (n + kTN - 1) / kTN, n_sb = (n + kTM - 1) / kTM;
  const int n_chunks = (ld + kKC - 1) / kKC;

  // 1. column mean of the sources, centred copies, norms
  const int rows_per = 4096, n_part = (n_true + rows_per - 1) / rows_per;
  float* part = ws.get<float>(static_cast<size_t>(n_part) * ld);
  float* mean = ws.get<float>(ld);
  colsum_partial_kernel<<<dim3(n_part, (ld + 127) / 128), 128, 0, st>>>(s, n_true, ld, rows_per, part);
  colsum_final_kernel<<<(ld + 127) / 128, 128, 0, st>>>(part, n_part, ld, dim, 1.0f / n_true, mean);
  const int64_t s_pad = static_cast<int64_t>(n_st) * kTN, q_pad_own = static_cast<int64_t>(n_qt) * kTM;
  const int ldc = n_chunks * kKC;
  require(s_pad * n_chunks < (int64_t(1) << 31) && q_pad_own * n_chunks < (int64_t(1) << 31),
          knnx::errc::too_large, "wide kNN: rows x ceil(dim / 32) must stay below 2^31");
  float* sc = ws.get<float>(static_cast<size_t>(s_pad) * ldc);
  check(cudaMemsetAsync(sc, 0, sizeof(float) * static_cast<size_t>(s_pad) * ldc, st), "memset");
  float* snorm = ws.get<float>(static_cast<size_t>(n_st) * kTN);
  fill_kernel<<<(n_st * kTN + 255) / 256, 256, 0, st>>>(snorm, n_st * kTN, HUGE_VALF);
  float* sc_lo = nullptr;
  if (precise) {
    sc_lo = ws.get<float>(static_cast<size_t>(s_pad) * ldc);
    check(cudaMemsetAsync(sc_lo, 0, sizeof(float) * static_cast<size_t>(s_pad) * ldc, st), "memset");
  }
  center_kernel<<<(n + 7) / 8, 256, 0, st>>>(s, n, ld, dim, mean, sperm, sc, s_pad, snorm, sc_lo);
  float* qc = sc;
  float* qc_lo = sc_lo;
  float* qnorm = snorm;
  int64_t q_pad = s_pad;
  if (!same) {
    q_pad = q_pad_own;
    qc = ws.get<float>(static_cast<size_t>(q_pad) * ldc);
    check(cudaMemsetAsync(qc, 0, sizeof(float) * static_cast<size_t>(q_pad) * ldc, st), "memset");
    if (precise) {
      qc_lo = ws.get<float>(static_cast<size_t>(q_pad) * ldc);
      check(cudaMemsetAsync(qc_lo, 0, sizeof(float) * static_cast<size_t>(q_pad) * ldc, st), "memset");
    }
    qnorm = ws.get<float>(m);
    center_kernel<<<(m + 7) / 8, 256, 0, st>>>(t, m, ld, dim, mean, qperm, qc, q_pad, qnorm, qc_lo);
  }
  // 2. tile statistics and pair bounds
  float* q_ctr = ws.get<float>(static_cast<size_t>(n_qt) * ldc);
  float* q_rad = ws.get<float>(n_qt);
  float* s_ctr = ws.get<float>(static_cast<size_t>(n_sb) * ldc);
  float* s_rad = ws.get<float>(n_sb);
  tile_stats_kernel<<<n_qt, 256, 0, st>>>(qc, m, q_pad, ldc, kTM, qperm, q_ctr, q_rad);
  tile_stats_kernel<<<n_sb, 256, 0, st>>>(sc, n, s_pad, ldc, kTM, sperm, s_ctr, s_rad);
  float* lb2 = ws.get<float>(static_cast<size_t>(n_qt) * n_st);
  require(static_cast<size_t>(ldc) * 4 <= 48 * 1024, knnx::errc::dim_too_high,
          "wide kNN supports dim <= 12288");
  tile_lb_kernel<<<n_qt, 256, static_cast<size_t>(ldc) * 4, st>>>(q_ctr, q_rad, s_ctr, s_rad, n_sb, n_st, ldc,
                                                                  lb2);
  // 3. tensor-core screen
  ScreenArgs a{};
  a.nq = m;
  a.ns = n;
  a.n_chunks = n_chunks;
  a.n_stiles = n_st;
  a.n_cand = n_cand;
  a.self_set = self_set ? 1 : 0;
  a.qnorm = qnorm;
  a.qvalid = qperm;
  a.qself = qself;
  a.snorm = snorm;
  a.lb2 = lb2;
  // candidate lists hold 256 entries per row (n_cand <= 128) or 512; the
  // screen runs in launches of at most `batch` query tiles so the lists stay
  // around 1 GB whatever m is
  const int cap = n_cand <= 128 ? 256 : 512;
  const int batch = std::min(n_qt, (1 << 30) / (2 * kTM * cap * 8));
  a.lists = ws.get<uint2>(static_cast<size_t>(batch) * 2 * kTM * cap);  // one list per epilogue set
  a.cand = ws.get<int32_t>(static_cast<size_t>(m) * n_cand);
  a.cand_score = ws.get<float>(static_cast<size_t>(m) * n_cand);
  a.tau = ws.get<float>(m);
  a.tiles_done = stats ? stats->tiles : nullptr;
  a.q_pad = static_cast<int>(q_pad);
  a.s_pad = static_cast<int>(s_pad);
  const CUtensorMap map_q = make_map(qc, q_pad, n_chunks, kTM);
  const CUtensorMap map_s = make_map(sc, s_pad, n_chunks, kTN);
  const CUtensorMap map_qlo = precise ? make_map(qc_lo, q_pad, n_chunks, kTM) : map_q;
  const CUtensorMap map_slo = precise ? make_map(sc_lo, s_pad, n_chunks, kTN) : map_s;
  const size_t smem = (precise ? kStagesPrecise * 2 : kStages) * (kBytesA + kBytesB) + 1024;
  auto launch = [&](auto kernel, int grid) {
    check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
          "smem attribute");
    kernel<<<grid, kThreads, smem, st>>>(map_q, map_s, map_qlo, map_slo, a);
  };
  int n_launch = 0;
  for (int q0 = 0; q0 < n_qt; q0 += batch, ++n_launch) {
    a.qt_base = q0;
    const int g = std::min(batch, n_qt - q0);
    if (cap == 256) {
      if (precise) launch(screen_kernel<256, true>, g); else launch(screen_kernel<256, false>, g);
    } else {
      if (precise) launch(screen_kernel<512, true>, g); else launch(screen_kernel<512, false>, g);
    }
  }
  // 4. exact re-rank on the caller's (uncentred) points
  rerank_kernel<<<(m + 7) / 8, 256, 0, st>>>(t, m, s, ld, dim, qperm, sperm, a.cand, a.cand_score, n_cand, k,
                                             ids, d2, a.tau, stats ? stats->margin : nullptr);
  launched(ctx, "knn_wide", (same ? 8 : 9) + n_launch);
  if (stats) stats->dense_tiles = static_cast<double>(n_qt) * n_st;
}

__global__ void cell_count_kernel(const int32_t* __restrict__ cell, int n, int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[cell[i]], 1);
}

// ustart = exclusive scan of the cell sizes, off = the same with every cell
// rounded up to a multiple of kTM rows; total[0] = padded row count
__global__ void cell_scan_kernel(const int32_t* __restrict__ cnt, int n_piv, int32_t* __restrict__ ustart,
                                 int32_t* __restrict__ off, int32_t* __restrict__ total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int u = 0, o = 0;
  for (int c = 0; c < n_piv; ++c) {
    ustart[c] = u;
    off[c] = o;
    u += cnt[c];
    o += (cnt[c] + kTM - 1) / kTM * kTM;
  }
  total[0] = o;
}

__global__ void cell_place_kernel(const int32_t* __restrict__ cell_sorted, const int32_t* __restrict__ idx_sorted,
                                  int n, const int32_t* __restrict__ ustart, const int32_t* __restrict__ off,
                                  int32_t* __restrict__ perm) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int c = cell_sorted[j];
  perm[off[c] + (j - ustart[c])] = idx_sorted[j];
}

struct Partition {
  int32_t* perm = nullptr;  // [rows]: caller row of each scratch row, -1 = padding
  int rows = 0;
};

// Spatial partition for the pruning: every point is assigned to the nearest of
// n_piv pivot points (the same screen with k = 1) and laid out cell by cell,
// every cell padded to a multiple of 128 rows, so each of the screen's 128-row
// balls lies inside one cell whatever order the caller's points come in.
Partition partition_points(knnx_ctx_t ctx, Scratch& ws, const float* pts, int n, const float* piv,
                           int n_piv, int ld, int dim) {
  cudaStream_t st = ctx->stream;
  int32_t* cell = ws.get<int32_t>(n);
  {
    Scratch inner(st);
    float* cd2 = inner.get<float>(n);
    knn_wide_core(ctx, inner, pts, n, piv, n_piv, n_piv, ld, dim, 1, 64 < n_piv ? 64 : n_piv, false, false,
                  nullptr, nullptr, cell, cd2, nullptr);
  }
  int32_t* idx = ws.get<int32_t>(n);
  int32_t* cell_sorted = ws.get<int32_t>(n);
  int32_t* idx_sorted = ws.get<int32_t>(n);
  iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(idx, n);
  size_t tmp_bytes = 0;
  int bits = 1;
  while ((1 << bits) < n_piv) ++bits;
  check(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, cell, cell_sorted, idx, idx_sorted, n, 0, bits, st),
        "radix sort size");
  void* tmp = ws.get<unsigned char>(tmp_bytes);
  check(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, cell, cell_sorted, idx, idx_sorted, n, 0, bits, st),
        "radix sort");
  int32_t* cnt = ws.get<int32_t>(n_piv);
  int32_t* ustart = ws.get<int32_t>(n_piv);
  int32_t* off = ws.get<int32_t>(n_piv);
  int32_t* total = ws.get<int32_t>(1);
  check(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n_piv, st), "memset");
  cell_count_kernel<<<(n + 255) / 256, 256, 0, st>>>(cell, n, cnt);
  cell_scan_kernel<<<1, 32, 0, st>>>(cnt, n_piv, ustart, off, total);
  int h_total = 0;
  check(cudaMemcpyAsync(&h_total, total, sizeof(int), cudaMemcpyDeviceToHost, st), "partition size");
  check(cudaStreamSynchronize(st), "partition sync");
  Partition part;
  part.rows = (h_total + kTN - 1) / kTN * kTN;
  part.perm = ws.get<int32_t>(part.rows);
  check(cudaMemsetAsync(part.perm, 0xFF, sizeof(int32_t) * part.rows, st), "memset");
  cell_place_kernel<<<(n + 255) / 256, 256, 0, st>>>(cell_sorted, idx_sorted, n, ustart, off, part.perm);
  ctx->launches += 6;
  return part;
}

}  // namespace

extern "C" int knnx_knn_wide_dev(knnx_ctx_t ctx, const float* t, int32_t m, const float* s, int32_t n,
                                 int32_t ld, int32_t dim, int32_t k, int32_t n_cand, int32_t self_set,
                                 int32_t* ids, float* d2, double* stats) {
  return guard([&] {
    require(ctx != nullptr && t && s && ids && d2, knnx::errc::invalid_argument, "null argument");
    require(m >= 1 && n >= 1 && dim >= 1 && ld >= dim && ld % 4 == 0, knnx::errc::invalid_argument,
            "need m, n, dim >= 1 and a leading dimension that is a multiple of 4 and >= dim");
    require((reinterpret_cast<uintptr_t>(t) & 15) == 0 && (reinterpret_cast<uintptr_t>(s) & 15) == 0,
            knnx::errc::invalid_argument, "point arrays must be 16-byte aligned");
    require(k >= 1, knnx::errc::invalid_argument, "k must be >= 1");
    require(k <= (self_set ? n - 1 : n), knnx::errc::k_too_large,
            "k = " + std::to_string(k) + " with " + std::to_string(n) + " sources");
    if (n_cand <= 0) n_cand = 4 * k < 64 ? 64 : 4 * k;
    if (n_cand > kMaxCand) n_cand = kMaxCand;
    require(k <= n_cand, knnx::errc::too_large, "wide kNN supports k <= 256");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = ctx->stream;
    Scratch ws(st);
    const bool same = t == s && m == n;
    // pivot cells of about 512 points once the source set is large enough to
    // prune (self exclusion between two different arrays compares caller
    // indices, which a re-partitioned screen does not have)
    const int32_t* sperm = nullptr;
    const int32_t* qperm = nullptr;
    int m_rows = m, n_rows = n, n_piv = 0;
    float* piv = nullptr;
    if (n >= 16384 && (same || !self_set)) {
      n_piv = std::min(8192, n / 512);
      int32_t* prow = ws.get<int32_t>(n_piv);
      pivot_rows_kernel<<<(n_piv + 255) / 256, 256, 0, st>>>(prow, n_piv, n);
      piv = ws.get<float>(static_cast<size_t>(n_piv) * ld);
      knnx_dev::launch_permute(n_piv, static_cast<int64_t>(ld) * 4, s, prow, piv, false, st);
      const Partition ps = partition_points(ctx, ws, s, n, piv, n_piv, ld, dim);
      sperm = ps.perm;
      n_rows = ps.rows;
      if (same) {
        qperm = sperm;
        m_rows = n_rows;
      } else {
        const Partition pq = partition_points(ctx, ws, t, m, piv, n_piv, ld, dim);
        qperm = pq.perm;
        m_rows = pq.rows;
      }
    }
    WideStats wst;
    wst.margin = ws.get<float>(m);
    wst.tiles = ws.get<unsigned long long>(1);
    check(cudaMemsetAsync(wst.tiles, 0, sizeof(unsigned long long), st), "memset");
    knn_wide_core(ctx, ws, t, m_rows, s, n_rows, n, ld, dim, k, n_cand, self_set != 0, same, qperm, sperm,
                  ids, d2, &wst);
    float* out = ws.get<float>(2);
    float h_out[2];
    auto margin_stats = [&] {
      margin_stats_kernel<<<1, 256, 0, st>>>(wst.margin, m, out);
      check(cudaMemcpyAsync(h_out, out, sizeof(h_out), cudaMemcpyDeviceToHost, st), "stats copy");
      check(cudaStreamSynchronize(st), "stats sync");
      ctx->launches += 1;
    };
    margin_stats();
    // rows the certificate does not cover (the TF32 screen is too coarse for
    // them: tight clusters far from the mean) are searched again exactly
    // with the SIMT kernel when it applies (dim <= 64)
    // the rows whose certificate failed, ascending (deterministic, and the
    // gathered targets keep the caller's locality)
    auto select_rows = [&](int count) {
      int32_t* sel = ws.get<int32_t>(count);
      int* d_cnt = ws.get<int>(1);
      check(cudaMemsetAsync(d_cnt, 0, sizeof(int), st), "memset");
      select_uncertified_kernel<<<(m + 255) / 256, 256, 0, st>>>(wst.margin, m, sel, d_cnt);
      int32_t* sorted = ws.get<int32_t>(count);
      size_t tmp_bytes = 0;
      check(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, sel, sorted, count, 0, 32, st), "sort size");
      void* tmp = ws.get<unsigned char>(tmp_bytes);
      check(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, sel, sorted, count, 0, 32, st), "sort");
      return sorted;
    };
    int n_redone = 0, n_precise = 0;
    const int n_bad = static_cast<int>(h_out[1]);
    const int kk = k + (self_set ? 1 : 0);
    if (n_bad > 0 && dim <= 64 && kk <= 192 && kk <= n) {
      const int32_t* sel = select_rows(n_bad);
      float* t_sub = ws.get<float>(static_cast<size_t>(n_bad) * ld);
      knnx_dev::launch_permute(n_bad, static_cast<int64_t>(ld) * 4, t, sel, t_sub, false, st);
      int32_t* ids_sub = ws.get<int32_t>(static_cast<size_t>(n_bad) * kk);
      float* d2_sub = ws.get<float>(static_cast<size_t>(n_bad) * kk);
      // self exclusion by index cannot be used on the gathered rows: ask for
      // one neighbour more and drop the row's own index afterwards
      knnx_dev::launch_knn(t_sub, n_bad, s, n, ld, dim, kk, false, ids_sub, d2_sub, st);
      exact_rows_fixup_kernel<<<(n_bad + 255) / 256, 256, 0, st>>>(sel, n_bad, ids_sub, d2_sub, kk, k,
                                                                  self_set != 0, ids, d2, wst.margin);
      launched(ctx, "knn_wide exact rows", 6);
      n_redone = n_bad;
      margin_stats();
    } else if (n_bad > 0) {
      // no exact SIMT search for these shapes: screen the failed rows again
      // with 3xTF32 operands (error ~2^-21 |q||s| instead of ~2^-10) and
      // certify them anew
      const int32_t* sel = select_rows(n_bad);
      float* t_sub = ws.get<float>(static_cast<size_t>(n_bad) * ld);
      knnx_dev::launch_permute(n_bad, static_cast<int64_t>(ld) * 4, t, sel, t_sub, false, st);
      const int32_t* qself = nullptr;
      if (self_set) {
        int32_t* qs = ws.get<int32_t>(n_bad);
        if (same && sperm) {
          int32_t* sinv = ws.get<int32_t>(n);
          inverse_perm_kernel<<<(n_rows + 255) / 256, 256, 0, st>>>(sperm, n_rows, sinv);
          knnx_dev::launch_permute(n_bad, 4, sinv, sel, qs, false, st);
        } else {
          check(cudaMemcpyAsync(qs, sel, sizeof(int32_t) * n_bad, cudaMemcpyDeviceToDevice, st), "copy");
        }
        qself = qs;
      }
      // the failed rows get their own pivot-cell layout (the caller's order
      // need not be spatial), with the self positions carried along
      const int32_t* qperm_sub = nullptr;
      int sub_rows = n_bad;
      if (piv != nullptr && n_bad >= 1024) {
        const Partition pq = partition_points(ctx, ws, t_sub, n_bad, piv, n_piv, ld, dim);
        qperm_sub = pq.perm;
        sub_rows = pq.rows;
        if (qself) {
          int32_t* qs2 = ws.get<int32_t>(sub_rows);
          remap_self_kernel<<<(sub_rows + 255) / 256, 256, 0, st>>>(qperm_sub, sub_rows, qself, qs2);
          qself = qs2;
        }
      }
      int32_t* ids_sub = ws.get<int32_t>(static_cast<size_t>(n_bad) * k);
      float* d2_sub = ws.get<float>(static_cast<size_t>(n_bad) * k);
      WideStats wst2;
      wst2.margin = ws.get<float>(n_bad);
      wst2.tiles = wst.tiles;
      knn_wide_core(ctx, ws, t_sub, sub_rows, s, n_rows, n, ld, dim, k, n_cand, self_set != 0, false,
                    qperm_sub, sperm, ids_sub, d2_sub, &wst2, /*precise=*/true, qself);
      scatter_rows_kernel<<<(n_bad + 255) / 256, 256, 0, st>>>(sel, n_bad, ids_sub, d2_sub, wst2.margin, k, ids,
                                                              d2, wst.margin);
      launched(ctx, "knn_wide precise rows", 4);
      n_precise = n_bad;
      margin_stats();
    }
    // a caller that does not read the statistics must not get uncertified
    // rows silently (wide points have no exact device fallback): DegenerateData
    require(stats != nullptr || h_out[1] == 0.0f, knnx::errc::degenerate_data,
            std::to_string(static_cast<long long>(h_out[1])) +
                " rows could not be certified by the TF32 distance screen (clusters tight against their "
                "distance from the mean); pass a stats array to accept them or use the exact search");
    if (stats) {
      unsigned long long h_tiles = 0;
      check(cudaMemcpyAsync(&h_tiles, wst.tiles, sizeof(h_tiles), cudaMemcpyDeviceToHost, st), "stats copy");
      check(cudaStreamSynchronize(st), "stats sync");
      stats[0] = h_out[0];                      // min certificate margin (squared-distance units)
      stats[1] = h_out[1];                      // rows left without a certificate
      stats[2] = static_cast<double>(h_tiles);  // source tiles multiplied
      stats[3] = wst.dense_tiles;               // tiles of the dense screen
      stats[4] = n_redone;                      // rows recomputed by the exact SIMT search
      stats[5] = n_precise;                     // rows screened again with 3xTF32 operands
    }
    return KNNX_OK;
  });
}
