// GPU construction of the t-SNE joint affinities (C4's P; SURVEY.md §8f next
// #2).  The host path is pattern_from_knn + symmetrize (proj/src/knn.cpp:
// 64-84) with values, i.e. csr_from_coo's sort of every (i, j) and (j, i)
// entry (proj/src/core.cpp:75-92) -- at C4 ~7.2e8 entries through host sorts.
// Here, from the device kNN rows (ids, squared distances):
//   1. conditional p_j|i = exp(-d2_ij / (2 h^2)) / sum_j (one warp per row);
//   2. both orientations of every entry as 64-bit keys row << 32 | col;
//   3. one device radix sort of (key, value) pairs (CUB), then a reduce by
//      key: entries present in both directions add (p_j|i + p_i|j);
//   4. scale, column decode and row pointers (row histogram + scan).
// The result is a canonical CSR (rows ascending, columns strictly ascending)
// in device buffers the caller releases with knnx_free.
#include <cuda_runtime.h>

#include <cstdint>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "knnx_internal.cuh"
#include "knnx_rt.cuh"

using namespace knnx_rt;

namespace {

// conditional affinities of one row per warp (k entries, lanes strided)
__global__ void __launch_bounds__(256) cond_affinity_kernel(const float* __restrict__ d2, int n,
                                                            int k, float c2, float* __restrict__ w) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* d = d2 + static_cast<int64_t>(row) * k;
  float* o = w + static_cast<int64_t>(row) * k;
  float sum = 0.0f;
  for (int q = lane; q < k; q += 32) sum += exp2f(-__ldg(d + q) * c2);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
  const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
  for (int q = lane; q < k; q += 32) o[q] = exp2f(-__ldg(d + q) * c2) * inv;
}

// entry e = (row, q): (row, id) and (id, row), both with the weight
__global__ void __launch_bounds__(256) both_orientations_kernel(const int32_t* __restrict__ ids,
                                                                const float* __restrict__ w,
                                                                int64_t nk, int k,
                                                                uint64_t* __restrict__ keys,
                                                                float* __restrict__ vals) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= nk) return;
  const uint64_t i = static_cast<uint64_t>(e / k);
  const uint64_t j = static_cast<uint64_t>(static_cast<uint32_t>(__ldg(ids + e)));
  const float v = __ldg(w + e);
  keys[e] = (i << 32) | j;
  vals[e] = v;
  keys[nk + e] = (j << 32) | i;
  vals[nk + e] = v;
}

__global__ void __launch_bounds__(256) decode_kernel(const uint64_t* __restrict__ keys,
                                                     const float* __restrict__ sums,
                                                     const int64_t* __restrict__ n_unique, float scale,
                                                     int32_t* __restrict__ cols,
                                                     float* __restrict__ vals,
                                                     int64_t* __restrict__ row_count) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= *n_unique) return;
  const uint64_t key = keys[e];
  cols[e] = static_cast<int32_t>(key & 0xffffffffu);
  vals[e] = sums[e] * scale;
  atomicAdd(reinterpret_cast<unsigned long long*>(row_count + (key >> 32)), 1ull);
}

int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

}  // namespace

extern "C" int knnx_tsne_affinities_dev(knnx_ctx_t ctx, const int32_t* ids, const float* d2,
                                        int32_t n, int32_t k, double h, double scale,
                                        int64_t** row_ptr_out, int32_t** cols_out,
                                        float** vals_out, int64_t* nnz_out) {
  return guard([&] {
    require(ctx != nullptr && row_ptr_out && cols_out && vals_out && nnz_out,
            knnx::errc::invalid_argument, "null argument");
    require(n >= 1 && k >= 1 && ids != nullptr && d2 != nullptr, knnx::errc::invalid_argument,
            "need n >= 1, k >= 1 and the kNN rows");
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t nk = static_cast<int64_t>(n) * k, m = 2 * nk;
    // scratch: conditional weights, keys / values (double buffers), sums
    float* w = nullptr;
    uint64_t *k0 = nullptr, *k1 = nullptr;
    float *v0 = nullptr, *v1 = nullptr;
    int64_t* n_unique = nullptr;
    void* tmp = nullptr;
    auto release = [&] {
      for (void* p : {static_cast<void*>(w), static_cast<void*>(k0), static_cast<void*>(k1),
                      static_cast<void*>(v0), static_cast<void*>(v1), static_cast<void*>(n_unique),
                      tmp})
        if (p) cudaFreeAsync(p, st);
    };
    int64_t* row_ptr = nullptr;
    int32_t* cols = nullptr;
    float* vals = nullptr;
    try {
      check(cudaMallocAsync(&w, sizeof(float) * nk, st), "alloc");
      check(cudaMallocAsync(&k0, sizeof(uint64_t) * m, st), "alloc");
      check(cudaMallocAsync(&k1, sizeof(uint64_t) * m, st), "alloc");
      check(cudaMallocAsync(&v0, sizeof(float) * m, st), "alloc");
      check(cudaMallocAsync(&v1, sizeof(float) * m, st), "alloc");
      check(cudaMallocAsync(&n_unique, sizeof(int64_t), st), "alloc");
      const float c2 = static_cast<float>(1.4426950408889634 / (2.0 * h * h));
      cond_affinity_kernel<<<static_cast<int>((static_cast<int64_t>(n) * 32 + 255) / 256), 256, 0,
                             st>>>(d2, n, k, c2, w);
      both_orientations_kernel<<<static_cast<int>((nk + 255) / 256), 256, 0, st>>>(ids, w, nk, k,
                                                                                  k0, v0);
      launched(ctx, "affinities", 2);
      // sort by (row, col): the key bits that can be set
      const int end_bit = 32 + bits_for(static_cast<uint64_t>(n));
      cub::DoubleBuffer<uint64_t> kb(k0, k1);
      cub::DoubleBuffer<float> vb(v0, v1);
      size_t sort_bytes = 0, red_bytes = 0;
      check(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, m, 0, end_bit, st), "sort size");
      uint64_t* uk = kb.Alternate();  // the reduce writes into the spare buffers
      float* us = vb.Alternate();
      check(cub::DeviceReduce::ReduceByKey(nullptr, red_bytes, kb.Current(), uk, vb.Current(), us,
                                           n_unique, cub::Sum(), m, st),
            "reduce size");
      check(cudaMallocAsync(&tmp, std::max(sort_bytes, red_bytes), st), "alloc");
      check(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, kb, vb, m, 0, end_bit, st), "sort");
      uk = kb.Alternate();
      us = vb.Alternate();
      check(cub::DeviceReduce::ReduceByKey(tmp, red_bytes, kb.Current(), uk, vb.Current(), us,
                                           n_unique, cub::Sum(), m, st),
            "reduce");
      int64_t nnz = 0;
      check(cudaMemcpyAsync(&nnz, n_unique, sizeof nnz, cudaMemcpyDeviceToHost, st), "nnz");
      check(cudaStreamSynchronize(st), "sync");
      check(cudaMalloc(&row_ptr, sizeof(int64_t) * (static_cast<size_t>(n) + 1)), "alloc");
      check(cudaMalloc(&cols, sizeof(int32_t) * std::max<int64_t>(1, nnz)), "alloc");
      check(cudaMalloc(&vals, sizeof(float) * std::max<int64_t>(1, nnz)), "alloc");
      int64_t* count = reinterpret_cast<int64_t*>(kb.Current());  // sorted keys no longer needed
      check(cudaMemsetAsync(count, 0, sizeof(int64_t) * (static_cast<size_t>(n) + 1), st), "memset");
      decode_kernel<<<static_cast<int>((nnz + 255) / 256), 256, 0, st>>>(
          uk, us, n_unique, static_cast<float>(scale), cols, vals, count);
      launched(ctx, "affinities decode");
      size_t scan_bytes = 0;
      check(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, count, row_ptr, n + 1, st), "scan size");
      void* scan_tmp = nullptr;
      check(cudaMallocAsync(&scan_tmp, scan_bytes, st), "alloc");
      check(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, count, row_ptr, n + 1, st), "scan");
      check(cudaFreeAsync(scan_tmp, st), "free");
      release();
      check(cudaStreamSynchronize(st), "sync");
      ctx->launches += 4;  // radix sort, reduce and scan passes (counted once each)
      *row_ptr_out = row_ptr;
      *cols_out = cols;
      *vals_out = vals;
      *nnz_out = nnz;
    } catch (...) {
      release();
      cudaStreamSynchronize(st);
      if (row_ptr) cudaFree(row_ptr);
      if (cols) cudaFree(cols);
      if (vals) cudaFree(vals);
      throw;
    }
    return KNNX_OK;
  });
}
