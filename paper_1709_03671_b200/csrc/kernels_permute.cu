// K1: whole-row permutation copies (permute(PointSet) proj/src/core.cpp:141-148,
// the charge / checksum permutes proj/src/pipeline.cpp:67-71,189-191), bit-exact,
// and the SM-driven streaming copy the host-buffer entry points use.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "kernels_common.cuh"

namespace knnx_dev {
namespace {

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
