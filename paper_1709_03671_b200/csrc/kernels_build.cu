// GPU construction of the cluster-tile format from device kNN rows
// (the host path is csr_from_knn + build_cluster_tiles,
// the counterpart of the reference's permute/csr_from_coo sort and build_hier
// bucketing, proj/src/core.cpp:75-92,130-139, proj/src/hier.cpp:84-155).
//
// Uniform-k rows (kNN graphs before symmetrisation).  Pass 1: one CTA per
// tile radix-sorts the tile's k*R neighbor ids (CUB block sort), marks unique
// ids and counts the halo.  A device scan of the 4-padded counts gives the
// halo offsets.  Pass 2 repeats the sort, writes the halo, sorts every row's k
// ids (canonical ascending-column order) and stores each entry's 16-bit halo
// index (binary search in shared memory) in the SELL-32 layout.  The result is
// byte-identical to the host builder's (tests/test_gpu_build.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <vector>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "knnx_internal.cuh"

namespace knnx_dev {

namespace {

constexpr int kThreads = 256;

template <int KP>  // KP: padded items per thread (k rounded up), tile = kThreads rows
struct TileSort {
  using Sort = cub::BlockRadixSort<int, kThreads, KP>;
  using Scan = cub::BlockScan<int, kThreads>;
  union Storage {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  };
};

// sorted unique ids of tile t into halo[] (shared); returns H
template <int KP>
__device__ int tile_halo(const int32_t* __restrict__ ids, int m, int k, int t,
                         typename TileSort<KP>::Storage& tmp, int* halo, int* total) {
  const int tid = threadIdx.x;
  const int row = t * kThreads + tid;
  int keys[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q)
    keys[q] = (row < m && q < k) ? __ldg(ids + static_cast<int64_t>(row) * k + q) : INT_MAX;
  typename TileSort<KP>::Sort(tmp.sort).Sort(keys);  // blocked arrangement
  __syncthreads();
  // unique flags: key differs from its predecessor in the blocked order
  __shared__ int last_of[kThreads];
  last_of[tid] = keys[KP - 1];
  __syncthreads();
  const int prev = tid > 0 ? last_of[tid - 1] : INT_MIN;
  int flags = 0;
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int before = q == 0 ? prev : keys[q - 1];
    flags += (keys[q] != before && keys[q] != INT_MAX) ? 1 : 0;
  }
  int offset = 0;
  typename TileSort<KP>::Scan(tmp.scan).ExclusiveSum(flags, offset, *total);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int before = q == 0 ? prev : keys[q - 1];
    if (keys[q] != before && keys[q] != INT_MAX) halo[offset++] = keys[q];
  }
  __syncthreads();
  return *total;
}

template <int KP>
__global__ void __launch_bounds__(kThreads) halo_count_kernel(const int32_t* __restrict__ ids, int m,
                                                              int k, int64_t* __restrict__ counts) {
  __shared__ typename TileSort<KP>::Storage tmp;
  extern __shared__ int halo[];
  __shared__ int total;
  const int H = tile_halo<KP>(ids, m, k, blockIdx.x, tmp, halo, &total);
  if (threadIdx.x == 0) counts[blockIdx.x + 1] = (H + 3) / 4 * 4;  // 16-B padded
}

template <int KP>
__global__ void __launch_bounds__(kThreads) tile_fill_kernel(const int32_t* __restrict__ ids, int m,
                                                             int k, const int64_t* __restrict__ halo_off,
                                                             int32_t* __restrict__ halo_ids,
                                                             uint16_t* __restrict__ lidx) {
  __shared__ typename TileSort<KP>::Storage tmp;
  extern __shared__ int halo[];
  __shared__ int total;
  const int t = blockIdx.x;
  const int H = tile_halo<KP>(ids, m, k, t, tmp, halo, &total);
  const int64_t h0 = halo_off[t];
  const int Hp = static_cast<int>(halo_off[t + 1] - h0);
  for (int j = threadIdx.x; j < Hp; j += kThreads)
    halo_ids[h0 + j] = j < H ? halo[j] : (H ? halo[H - 1] : 0);  // pad repeats the last id
  const int row = t * kThreads + threadIdx.x;
  if (row >= m) return;
  // this row's ids, ascending (insertion sort in registers; k <= KP)
  int r[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) r[q] = q < k ? __ldg(ids + static_cast<int64_t>(row) * k + q) : INT_MAX;
#pragma unroll
  for (int a = 1; a < KP; ++a)
#pragma unroll
    for (int b = a; b > 0; --b)
      if (r[b] < r[b - 1]) {
        const int tmpv = r[b];
        r[b] = r[b - 1];
        r[b - 1] = tmpv;
      }
  const int64_t base = static_cast<int64_t>(row >> 5) * 32 * k + (row & 31);
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    if (q >= k) break;
    int lo = 0, hi = H;  // lower_bound of r[q] in halo[0, H)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (halo[mid] < r[q]) lo = mid + 1; else hi = mid;
    }
    lidx[base + 32 * static_cast<int64_t>(q)] = static_cast<uint16_t>(lo);
  }
}

}  // namespace

// Fills op's device tile arrays from device ids (m x k, uniform k <= 64,
// tile_rows == 256).  Allocates halo_off / halo_ids / lidx on the stream.
void build_tiles_from_knn(const int32_t* ids, int m, int k, int64_t** d_halo_off,
                          int32_t** d_halo_ids, uint16_t** d_lidx, int64_t* halo_total,
                          int* max_halo, cudaStream_t st) {
  const int n_tiles = (m + kThreads - 1) / kThreads;
  const size_t smem = sizeof(int) * static_cast<size_t>(kThreads) * 32;  // k <= 32
  int64_t* off = nullptr;
  cudaMallocAsync(&off, sizeof(int64_t) * (n_tiles + 1), st);
  cudaMemsetAsync(off, 0, sizeof(int64_t) * (n_tiles + 1), st);
  auto count = halo_count_kernel<32>;
  cudaFuncSetAttribute(count, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  count<<<n_tiles, kThreads, smem, st>>>(ids, m, k, off);
  // max halo (before the scan turns counts into offsets)
  std::vector<int64_t> h_cnt(n_tiles + 1);
  cudaMemcpyAsync(h_cnt.data(), off, sizeof(int64_t) * (n_tiles + 1), cudaMemcpyDeviceToHost, st);
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, off, off, n_tiles + 1, st);
  cudaMallocAsync(&tmp, tmp_bytes, st);
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, off, off, n_tiles + 1, st);
  cudaFreeAsync(tmp, st);
  int64_t total = 0;
  cudaMemcpyAsync(&total, off + n_tiles, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  int mh = 0;
  for (int t = 1; t <= n_tiles; ++t) mh = std::max<int>(mh, static_cast<int>(h_cnt[t]));
  int32_t* hids = nullptr;
  uint16_t* lx = nullptr;
  cudaMallocAsync(&hids, sizeof(int32_t) * std::max<int64_t>(1, total), st);
  cudaMallocAsync(&lx, sizeof(uint16_t) * std::max<int64_t>(1, static_cast<int64_t>(m + 31) / 32 * 32 * k), st);
  auto fill = tile_fill_kernel<32>;
  cudaFuncSetAttribute(fill, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  fill<<<n_tiles, kThreads, smem, st>>>(ids, m, k, off, hids, lx);
  *d_halo_off = off;
  *d_halo_ids = hids;
  *d_lidx = lx;
  *halo_total = total;
  *max_halo = mh;
}

}  // namespace knnx_dev
