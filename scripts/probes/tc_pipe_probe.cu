// What bounds the kNN screen's pipeline on one SM?  The screen's loop
// (TMA 2-D loads with 128-byte swizzle into a ring of 32-wide K chunks,
// tcgen05.mma kind::tf32 128 x 256 x 8 into TMEM) with either side switched
// off: mode 0 = both, 1 = TMA only (the MMA thread releases stages without
// multiplying), 2 = MMA only (stages are never refilled).  One CTA per SM,
// `tiles` source tiles of 30 chunks each; sources either one shared tile
// (L2 hits) or a distinct tile per step (HBM).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tc_pipe_probe.cu -o tc_pipe_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kTM = 128, kKC = 32;
constexpr uint32_t kBytesA = kTM * kKC * 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

template <int TN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    pipe_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_s, int mode,
                int tiles, int n_chunks, int n_stiles, int q_pad, int s_pad, int distinct, float* sink) {
  constexpr uint32_t kBytesB = TN * kKC * 4;
  constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(TN >> 3) << 17) |
                              (static_cast<uint32_t>(kTM >> 4) << 24);
  extern __shared__ unsigned char smem_raw[];
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* ring_a = ring;
  unsigned char* ring_b = ring + STAGES * kBytesA;
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], done_bar;
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  const uint32_t total = static_cast<uint32_t>(tiles) * n_chunks;
  const int m0 = (blockIdx.x % (q_pad / kTM)) * kTM;
  if (warp == 0 && lane == 0) {
    for (uint32_t it = 0; it < total; ++it) {
      const int s = it % STAGES;
      mbar_wait(&empty_bar[s], ((it / STAGES) & 1) ^ 1);
      const int c = it % n_chunks;
      const int t = distinct ? static_cast<int>((blockIdx.x * 977u + (it / n_chunks) * 131u) % n_stiles) : 0;
      if (mode == 2 && it >= STAGES) {
        mbar_arrive(&full_bar[s]);
        continue;
      }
      mbar_arrive_expect_tx(&full_bar[s], kBytesA + kBytesB);
      tma_load_2d(ring_a + s * kBytesA, &map_q, 0, c * q_pad + m0, &full_bar[s]);
      tma_load_2d(ring_b + s * kBytesB, &map_s, 0, c * s_pad + t * TN, &full_bar[s]);
    }
  } else if (warp == 1 && lane == 0) {
    for (uint32_t it = 0; it < total; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full_bar[s], (it / STAGES) & 1);
      if (mode == 1) {
        mbar_arrive(&empty_bar[s]);
        continue;
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a0 = smem_u32(ring_a + s * kBytesA), b0 = smem_u32(ring_b + s * kBytesB);
      const int c = it % n_chunks;
#pragma unroll
      for (int ks = 0; ks < kKC / 8; ++ks) {
        const uint32_t acc = (c | ks) != 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + ((it / n_chunks) & 1) * TN),
            "l"(desc_sw128(a0 + ks * 32)), "l"(desc_sw128(b0 + ks * 32)), "r"(kIdesc), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&empty_bar[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(&done_bar))
                 : "memory");
    mbar_wait(&done_bar, 0);
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2 && mode != 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t r0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r0) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (sink && __uint_as_float(r0) == 123.456f) sink[0] = 1.f;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncodeTiledFn enc, float* base, int64_t n_pad, int n_chunks, int box_rows) {
  CUtensorMap m;
  const cuuint64_t gdim[2] = {kKC, static_cast<cuuint64_t>(n_pad) * n_chunks};
  const cuuint64_t gstride[1] = {kKC * 4};
  const cuuint32_t box[2] = {kKC, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::printf("encode failed %d\n", static_cast<int>(r));
    std::exit(1);
  }
  return m;
}

template <int TN, int STAGES>
static void run(EncodeTiledFn enc, float* q, float* s, int q_pad, int s_pad, int n_chunks, int tiles) {
  const CUtensorMap mq = make_map(enc, q, q_pad, n_chunks, kTM), ms = make_map(enc, s, s_pad, n_chunks, TN);
  const size_t smem = STAGES * (kBytesA + TN * kKC * 4) + 1024;
  cudaFuncSetAttribute(pipe_kernel<TN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  float* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int distinct = 0; distinct < 2; ++distinct)
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        pipe_kernel<TN, STAGES><<<148, 192, smem>>>(mq, ms, mode, tiles, n_chunks, s_pad / TN, q_pad, s_pad, distinct, sink);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) {
          std::printf("kernel failed: %s\n", cudaGetErrorString(cudaGetLastError()));
          std::exit(1);
        }
        float ms_;
        cudaEventElapsedTime(&ms_, e0, e1);
        best = ms_ < best ? ms_ : best;
      }
      const double flops = 148.0 * tiles * n_chunks * 2.0 * kTM * TN * kKC;
      const double bytes = 148.0 * tiles * n_chunks * (kBytesA + TN * kKC * 4.0);
      std::printf("TN=%d stages=%d %s sources, %s: %.3f ms, %.0f TFLOP/s, %.2f TB/s into shared memory, %.2f us per tile\n", TN,
                  STAGES, distinct ? "distinct (HBM)" : "one shared tile (L2)",
                  mode == 0 ? "TMA + MMA" : mode == 1 ? "TMA only " : "MMA only ", best, mode == 1 ? 0.0 : flops / best * 1e-9,
                  mode == 2 ? 0.0 : bytes / best * 1e-9, best * 1e3 / tiles);
    }
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  const int n_chunks = 30, q_pad = 148 * kTM, s_pad = 1 << 20, tiles = 200;
  float *q, *s;
  cudaMalloc(&q, sizeof(float) * static_cast<size_t>(q_pad) * n_chunks * kKC);
  cudaMalloc(&s, sizeof(float) * static_cast<size_t>(s_pad) * n_chunks * kKC);
  cudaMemset(q, 0, sizeof(float) * static_cast<size_t>(q_pad) * n_chunks * kKC);
  cudaMemset(s, 0, sizeof(float) * static_cast<size_t>(s_pad) * n_chunks * kKC);
  run<256, 4>(enc, q, s, q_pad, s_pad, n_chunks, tiles);
  run<128, 6>(enc, q, s, q_pad, s_pad, n_chunks, tiles);
  run<256, 3>(enc, q, s, q_pad, s_pad, n_chunks, tiles);
  return 0;
}
