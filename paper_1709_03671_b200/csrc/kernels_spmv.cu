// K2/K3: the stationary operator y = A x.
//  K2 spmv_orig_kernel   -- original order, int32 columns (spmv_flat,
//                           proj/src/kernels.cpp:37-49)
//  K3 spmv_tiles_g_kernel -- cluster order (spmv_hier / spmv_hier_parallel,
//                           proj/src/kernels.cpp:24-101): one CTA per row
//                           tile stages x[halo] in shared memory, then
//                           thread-per-row streaming accumulation.
// The rejected K3 variants (TMA bulk copies, persistent TMA ring, register
// prefetch) were measured in round 1 and removed from the
// library; the table in DESIGN.md keeps their numbers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels_common.cuh"

namespace knnx_dev {
namespace {

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


// K3: one CTA per tile; the row's slice header is loaded before the stage and
// the x[halo] stage is unrolled kG-wide
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

}  // namespace

void launch_spmv(const knnx_operator& op, const float* x, float* y, cudaStream_t st) {
  require_plain(op);
  if (op.n_rows == 0) return;
  const OpView v = view_of(op);
  if (op.order != KNNX_ORDER_CLUSTER) {
    // the random x gathers make this L2-sector bound (30M x 32-B sectors at
    // C2); explicit 8 / 15 / 30-entry batches measured identical (116.6-117 us,
    // profiles/r2_c2_orig_probe.log)
    spmv_orig_kernel<<<grid_for(static_cast<int64_t>(op.n_slices) * 32, 256), 256, 0, st>>>(v, x, y);
    return;
  }
  // one CTA per tile (blockDim = tile_rows), x[halo] staged in shared memory;
  // programmatic dependent launch lets this launch's slice-header loads
  // overlap the previous kernel on the stream (33.8 vs 36.5 us
  // at C2 back to back)
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
}

}  // namespace knnx_dev
