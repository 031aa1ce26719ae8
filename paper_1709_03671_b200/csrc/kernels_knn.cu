// Exact fp32 kNN on the device (replaces the
// O(N^2 D) brute force of proj/src/knn.cpp:9-62 as the INPUT builder).
//
// Block-pruned exhaustive search.  Targets are cut into blocks of kTB and
// sources into blocks of kSB consecutive points; every block gets a center and
// an (outward-rounded) radius.  A source block whose bound
//   |c_t - c_s| - rho_t - rho_s
// exceeds the current k-th distance of every target in the target block
// provably holds no neighbor (triangle inequality) and is skipped.  Targets
// first scan the source blocks around their own index range (tight thresholds
// when the points are cluster-ordered), then, in ascending block order, every
// block the bound cannot exclude.  The result equals fp32 brute force for ANY
// point order: candidates are ranked by (fp32 squared distance, index), a
// total order, and no block that can hold a point below the final threshold is
// skipped (1e-3 relative slack against fp32 rounding).  Locality only changes
// how many blocks are visited.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>

#include "knnx_internal.cuh"

namespace knnx_dev {

namespace {

constexpr int kTB = 128;  // targets per CTA (thread per target)
constexpr int kSB = 64;   // sources per staged block
constexpr int kWin = 3;   // source blocks scanned first on each side of the home range

__device__ __forceinline__ float sqdiff4m(const float4 a, const float4 b, int c0, int dim) {
  const float d0 = (c0 + 0 < dim) ? a.x - b.x : 0.0f;
  const float d1 = (c0 + 1 < dim) ? a.y - b.y : 0.0f;
  const float d2 = (c0 + 2 < dim) ? a.z - b.z : 0.0f;
  const float d3 = (c0 + 3 < dim) ? a.w - b.w : 0.0f;
  float acc = d0 * d0;
  acc = fmaf(d1, d1, acc);
  acc = fmaf(d2, d2, acc);
  acc = fmaf(d3, d3, acc);
  return acc;
}

// squared distance with the last float4 masked (dim > 4*(NV-1) always)
template <int NV>
__device__ __forceinline__ float dist2(const float4 (&a)[NV], const float4* b, int dim) {
  float p0 = 0.f, p1 = 0.f;
#pragma unroll
  for (int c = 0; c < NV - 1; ++c) {
    const float4 v = b[c];
    const float e0 = a[c].x - v.x, e1 = a[c].y - v.y, e2 = a[c].z - v.z, e3 = a[c].w - v.w;
    p0 = fmaf(e0, e0, p0);
    p1 = fmaf(e1, e1, p1);
    p0 = fmaf(e2, e2, p0);
    p1 = fmaf(e3, e3, p1);
  }
  return p0 + p1 + sqdiff4m(a[NV - 1], b[NV - 1], 4 * (NV - 1), dim);
}

// per block of `bs` points: center (ld floats, padding zeroed) and radius
template <int NV>
__global__ void block_stats_kernel(const float* __restrict__ p, int n, int ld, int dim, int bs,
                                   float* __restrict__ centers, float* __restrict__ radius) {
  const int b = blockIdx.x;
  const int lo = b * bs, hi = min(n, lo + bs);
  __shared__ float4 ctr[NV];
  __shared__ float red[128];
  if (threadIdx.x < NV) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = lo; i < hi; ++i) {
      const float4 v = reinterpret_cast<const float4*>(p + static_cast<int64_t>(i) * ld)[threadIdx.x];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const float inv = 1.0f / static_cast<float>(hi - lo);
    acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
    const int c0 = 4 * threadIdx.x;
    if (c0 + 0 >= dim) acc.x = 0.f;
    if (c0 + 1 >= dim) acc.y = 0.f;
    if (c0 + 2 >= dim) acc.z = 0.f;
    if (c0 + 3 >= dim) acc.w = 0.f;
    ctr[threadIdx.x] = acc;
    reinterpret_cast<float4*>(centers + static_cast<int64_t>(b) * ld)[threadIdx.x] = acc;
  }
  __syncthreads();
  float d2 = 0.0f;
  const int i = lo + threadIdx.x;
  if (i < hi) {
    const float4* pv = reinterpret_cast<const float4*>(p + static_cast<int64_t>(i) * ld);
    for (int c = 0; c < NV; ++c) d2 += sqdiff4m(pv[c], ctr[c], 4 * c, dim);
  }
  red[threadIdx.x] = d2;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.f;
    for (int q = 0; q < bs; ++q) mx = fmaxf(mx, red[q]);
    radius[b] = sqrtf(mx) * 1.0001f + 1e-6f;
  }
}

template <int NV, int kP>
__global__ void __launch_bounds__(kTB) knn_block_kernel(
    const float* __restrict__ t, int m, const float* __restrict__ s, int n, int ld, int dim, int k,
    int self_set, const float* __restrict__ t_ctr, const float* __restrict__ t_rad,
    const float* __restrict__ s_ctr, const float* __restrict__ s_rad, int n_sblocks,
    int32_t* __restrict__ ids_out, float* __restrict__ d2_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  float4* sblk = reinterpret_cast<float4*>(smem);                                // kSB * NV
  float* ldist = reinterpret_cast<float*>(sblk + kSB * NV);                      // k * kTB
  int* lid = reinterpret_cast<int*>(ldist + static_cast<size_t>(k) * kTB);       // k * kTB
  __shared__ int cand[kTB];
  __shared__ int warp_cnt[kTB / 32];
  __shared__ float thr_max;
  __shared__ float4 tctr[NV];

  const int tb = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = tb * kTB + tid;
  const bool active = row < m;
  float4 ti[NV];
  const float4* tp = reinterpret_cast<const float4*>(t + static_cast<int64_t>(active ? row : 0) * ld);
#pragma unroll
  for (int c = 0; c < NV; ++c) ti[c] = tp[c];
  for (int q = 0; q < k; ++q) {
    ldist[q * kTB + tid] = FLT_MAX;
    lid[q * kTB + tid] = INT_MAX;
  }
  float thr = FLT_MAX;
  int thr_id = INT_MAX;
  if (tid < NV) tctr[tid] = reinterpret_cast<const float4*>(t_ctr + static_cast<int64_t>(tb) * ld)[tid];
  const float rho_t = t_rad[tb];

  // accepted candidates wait in a register buffer of kP entries and are
  // merged into the sorted shared-memory list kP at a time (one backward
  // merge instead of kP insertion shifts through the list; k = 90 at C4)
  float pd[kP];
  int pi[kP];
  int npend = 0;
  auto better = [](float d, int i, float e, int j) { return d < e || (d == e && i < j); };
  auto flush = [&]() {
    if (npend == 0) return;
#pragma unroll
    for (int q = 0; q < kP; ++q)
      if (q >= npend) {
        pd[q] = FLT_MAX;
        pi[q] = INT_MAX;
      }
    // sort the buffer ascending (odd-even transposition, static indices)
#pragma unroll
    for (int r = 0; r < kP; ++r)
#pragma unroll
      for (int q = r & 1; q + 1 < kP; q += 2)
        if (better(pd[q + 1], pi[q + 1], pd[q], pi[q])) {
          const float td = pd[q];
          const int ti2 = pi[q];
          pd[q] = pd[q + 1];
          pi[q] = pi[q + 1];
          pd[q + 1] = td;
          pi[q + 1] = ti2;
        }
    // backward merge of list (k) and buffer (npend): the k smallest stay
    int ia = k - 1, ib = npend - 1, out = k + npend - 1;
    float bd = 0.f;
    int bi = 0;
#pragma unroll
    for (int q = 0; q < kP; ++q)
      if (q == ib) {
        bd = pd[q];
        bi = pi[q];
      }
    while (ib >= 0) {
      const float ad = ia >= 0 ? ldist[ia * kTB + tid] : -FLT_MAX;
      const int ai = ia >= 0 ? lid[ia * kTB + tid] : INT_MIN;
      if (ia >= 0 && better(bd, bi, ad, ai)) {  // list element is larger
        if (out < k) {
          ldist[out * kTB + tid] = ad;
          lid[out * kTB + tid] = ai;
        }
        --ia;
      } else {
        if (out < k) {
          ldist[out * kTB + tid] = bd;
          lid[out * kTB + tid] = bi;
        }
        --ib;
#pragma unroll
        for (int q = 0; q < kP; ++q)
          if (q == ib) {
            bd = pd[q];
            bi = pi[q];
          }
      }
      --out;
    }
    thr = ldist[(k - 1) * kTB + tid];
    thr_id = lid[(k - 1) * kTB + tid];
    npend = 0;
  };

  auto scan_block = [&](int sb) {
    __syncthreads();
    const int s0 = sb * kSB;
    const int cnt = min(kSB, n - s0);
    for (int e = tid; e < cnt * NV; e += kTB) {
      const int r = e / NV, c = e - r * NV;
      sblk[e] = reinterpret_cast<const float4*>(s + static_cast<int64_t>(s0 + r) * ld)[c];
    }
    __syncthreads();
    if (!active) return;
    for (int r = 0; r < cnt; ++r) {
      const int j = s0 + r;
      const float d2 = dist2<NV>(ti, sblk + r * NV, dim);
      if (self_set && j == row) continue;
      if (d2 < thr || (d2 == thr && j < thr_id)) {
#pragma unroll
        for (int q = 0; q < kP; ++q)
          if (q == npend) {
            pd[q] = d2;
            pi[q] = j;
          }
        if (++npend == kP) flush();
      }
    }
    // no flush here: a threshold that has not yet seen the buffered
    // candidates is only larger, so the block bound below stays conservative
  };

  auto block_lb2 = [&](int sb) {
    const float d2 = dist2<NV>(tctr, reinterpret_cast<const float4*>(s_ctr + static_cast<int64_t>(sb) * ld), dim);
    const float lb = sqrtf(d2) - rho_t - s_rad[sb];
    return lb > 0.0f ? lb * lb : 0.0f;
  };

  auto refresh_thr = [&]() {
    __syncthreads();
    if (tid == 0) thr_max = 0.0f;
    __syncthreads();
    if (active) atomicMax(reinterpret_cast<int*>(&thr_max), __float_as_int(thr));
    __syncthreads();
  };

  // 1. the source blocks around this target block's index range
  const int r_lo = min(tb * kTB, n - 1), r_hi = min(tb * kTB + kTB - 1, n - 1);
  const int w_lo = max(0, r_lo / kSB - kWin), w_hi = min(n_sblocks - 1, r_hi / kSB + kWin);
  for (int sb = w_lo; sb <= w_hi; ++sb) scan_block(sb);
  refresh_thr();

  // 2. every other block the bound cannot exclude, in ascending order
  for (int c0 = 0; c0 < n_sblocks; c0 += kTB) {
    const int sb = c0 + tid;
    const bool pass = sb < n_sblocks && (sb < w_lo || sb > w_hi) &&
                      block_lb2(sb) <= thr_max * 1.001f;
    const unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (lane == 0) warp_cnt[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < kTB / 32; ++w) {
      before += w < warp ? warp_cnt[w] : 0;
      total += warp_cnt[w];
    }
    if (pass) cand[before + __popc(bal & ((1u << lane) - 1u))] = sb;
    __syncthreads();
    for (int q = 0; q < total; ++q) {
      const int cb = cand[q];
      if (block_lb2(cb) <= thr_max * 1.001f) scan_block(cb);
    }
    refresh_thr();
  }

  if (active) flush();
  if (active)
    for (int q = 0; q < k; ++q) {
      ids_out[static_cast<int64_t>(row) * k + q] = lid[q * kTB + tid];
      d2_out[static_cast<int64_t>(row) * k + q] = ldist[q * kTB + tid];
    }
}

}  // namespace

void launch_knn(const float* t, int m, const float* s, int n, int ld, int dim, int k,
                bool self_set, int32_t* ids, float* d2, cudaStream_t st) {
  if (m == 0) return;
  const int nv = (dim + 3) / 4;
  const int n_tb = (m + kTB - 1) / kTB, n_sb = (n + kSB - 1) / kSB;
  float *t_ctr = nullptr, *t_rad = nullptr, *s_ctr = nullptr, *s_rad = nullptr;
  cudaMallocAsync(&t_ctr, sizeof(float) * static_cast<size_t>(n_tb) * ld, st);
  cudaMallocAsync(&t_rad, sizeof(float) * n_tb, st);
  cudaMallocAsync(&s_ctr, sizeof(float) * static_cast<size_t>(n_sb) * ld, st);
  cudaMallocAsync(&s_rad, sizeof(float) * n_sb, st);
  const size_t smem =
      sizeof(float4) * kSB * nv + (sizeof(float) + sizeof(int)) * static_cast<size_t>(k) * kTB;
#define L(NV)                                                                                    \
  do {                                                                                           \
    block_stats_kernel<NV><<<n_tb, 128, 0, st>>>(t, m, ld, dim, kTB, t_ctr, t_rad);              \
    block_stats_kernel<NV><<<n_sb, 128, 0, st>>>(s, n, ld, dim, kSB, s_ctr, s_rad);              \
    if (k > 32) {                                                                                \
      cudaFuncSetAttribute(knn_block_kernel<NV, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           static_cast<int>(smem));                                              \
      knn_block_kernel<NV, 8><<<n_tb, kTB, smem, st>>>(t, m, s, n, ld, dim, k, self_set ? 1 : 0, \
                                                      t_ctr, t_rad, s_ctr, s_rad, n_sb, ids, d2); \
    } else {                                                                                     \
      cudaFuncSetAttribute(knn_block_kernel<NV, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           static_cast<int>(smem));                                              \
      knn_block_kernel<NV, 1><<<n_tb, kTB, smem, st>>>(t, m, s, n, ld, dim, k, self_set ? 1 : 0, \
                                                      t_ctr, t_rad, s_ctr, s_rad, n_sb, ids, d2); \
    }                                                                                            \
  } while (0)
  switch (nv) {
    case 1: L(1); break;
    case 2: L(2); break;
    case 3: L(3); break;
    case 4: L(4); break;
    case 5: L(5); break;
    case 6: L(6); break;
    case 7: L(7); break;
    case 8: L(8); break;
    case 9: L(9); break;
    case 10: L(10); break;
    case 11: L(11); break;
    case 12: L(12); break;
    case 13: L(13); break;
    case 14: L(14); break;
    case 15: L(15); break;
    default: L(16); break;
  }
#undef L
  cudaFreeAsync(t_ctr, st);
  cudaFreeAsync(t_rad, st);
  cudaFreeAsync(s_ctr, st);
  cudaFreeAsync(s_rad, st);
}

}  // namespace knnx_dev
