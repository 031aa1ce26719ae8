// 5th-generation tensor cores (tcgen05 + TMEM) for the one dense contraction
// near the hot path: the Gram block C = A B^T of point rows (SURVEY.md §8f
// next #1, the exact kNN builder's distance screen for D > 64, where
// |a - b|^2 = |a|^2 + |b|^2 - 2 a.b over all pairs is a real dense GEMM).
//
// One CTA per 128 x 256 output tile, kind::tf32 (fp32 operands read as TF32,
// fp32 accumulation in TMEM).  Operands are staged in shared memory in the
// canonical K-major no-swizzle UMMA layout: element (r, k) of an R-row tile at
// byte ((k / 4) * R + r) * 16 + (k % 4) * 4, i.e. 8-row x 16-byte core
// matrices, 128 B apart along rows (SBO) and R * 16 B apart along K (LBO).
// One elected thread issues the MMAs (4 per 32-wide K chunk), commits them to
// an mbarrier, and the four warps read the accumulator back with tcgen05.ld
// (warp w owns TMEM lanes 32w .. 32w + 31 = output rows).  Two K-chunk stages
// let the loads of chunk c + 1 overlap the MMAs of chunk c.
#include <cuda_runtime.h>

#include <cstdint>

#include "knnx_internal.cuh"
#include "knnx_rt.cuh"

using namespace knnx_rt;

namespace {

constexpr int kTM = 128, kTN = 256, kKC = 32;  // tile rows, tile cols, K per chunk
constexpr int kThreads = 128;
constexpr uint32_t kTmemCols = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no swizzle: LBO = stride between the two 16-byte core matrices of
// one K=8 step, SBO = stride between 8-row groups (both in bytes)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  return d;                             // base offset 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor: D fp32, A/B tf32, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kTN >> 3) << 17) |
                            (static_cast<uint32_t>(kTM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(phase));
}

// stage a kRows x kKC chunk of row-major fp32 rows (leading dim ld) into the
// canonical layout; rows past `rows` are zero
template <int kRows>
__device__ __forceinline__ void stage_chunk(float* dst, const float* __restrict__ src, int rows,
                                            int ld, int k0) {
  constexpr int kVec = kRows * (kKC / 4);  // float4 per chunk
#pragma unroll 4
  for (int v = threadIdx.x; v < kVec; v += kThreads) {
    const int r = v % kRows, c = v / kRows;  // consecutive threads: consecutive rows
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < rows) val = __ldg(reinterpret_cast<const float4*>(src + static_cast<int64_t>(r) * ld + k0) + c);
    reinterpret_cast<float4*>(dst)[c * kRows + r] = val;
  }
}

__global__ void __launch_bounds__(kThreads, 1) gram_tf32_kernel(const float* __restrict__ a, int m,
                                                                const float* __restrict__ b, int n,
                                                                int ld, int k, float* __restrict__ c,
                                                                int64_t ldc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sa[2] = {reinterpret_cast<float*>(smem), reinterpret_cast<float*>(smem) + kTM * kKC};
  float* sb[2] = {reinterpret_cast<float*>(smem) + 2 * kTM * kKC,
                  reinterpret_cast<float*>(smem) + 2 * kTM * kKC + kTN * kKC};
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kTM, n0 = blockIdx.y * kTN;
  const float* ab = a + static_cast<int64_t>(m0) * ld;
  const float* bb = b + static_cast<int64_t>(n0) * ld;
  const int mr = min(kTM, m - m0), nr = min(kTN, n - n0);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;

  const int n_chunks = k / kKC;
  uint32_t phase[2] = {0, 0};
  stage_chunk<kTM>(sa[0], ab, mr, ld, 0);
  stage_chunk<kTN>(sb[0], bb, nr, ld, 0);
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int s = ch & 1;
    // make this chunk's generic-proxy smem stores visible to the tensor core
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a0 = smem_u32(sa[s]), b0 = smem_u32(sb[s]);
#pragma unroll
      for (int ks = 0; ks < kKC / 8; ++ks) {
        const uint64_t da = umma_desc(a0 + ks * 2 * kTM * 16, kTM * 16, 128);
        const uint64_t db = umma_desc(b0 + ks * 2 * kTN * 16, kTN * 16, 128);
        mma_tf32(tmem, da, db, (ch | ks) != 0 ? 1u : 0u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&mbar[s]))
                   : "memory");
    }
    // stage the next chunk into the other buffers while these MMAs run; that
    // buffer's previous MMAs (chunk ch - 1) must have completed first
    if (ch + 1 < n_chunks) {
      if (ch >= 1) {
        mbar_wait(smem_u32(&mbar[s ^ 1]), phase[s ^ 1]);
        phase[s ^ 1] ^= 1;
      }
      stage_chunk<kTM>(sa[s ^ 1], ab, mr, ld, (ch + 1) * kKC);
      stage_chunk<kTN>(sb[s ^ 1], bb, nr, ld, (ch + 1) * kKC);
    }
  }
  // the last chunk's MMAs (and with them every earlier one) are complete when
  // its barrier flips
  {
    const int s = (n_chunks - 1) & 1;
    mbar_wait(smem_u32(&mbar[s]), phase[s]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // epilogue: warp w reads rows 32w .. 32w + 31 (TMEM lanes), 32 columns at a time
  const int row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < kTN; c0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0);
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
    if (row < m) {
      float* out = c + static_cast<int64_t>(row) * ldc + n0 + c0;
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (n0 + c0 + q < n) out[q] = __uint_as_float(r[q]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(kTmemCols));
}

}  // namespace

extern "C" int knnx_gram_tf32_dev(knnx_ctx_t ctx, const float* a, int32_t m, const float* b,
                                  int32_t n, int32_t ld, int32_t k, float* c, int64_t ldc) {
  return guard([&] {
    require(ctx != nullptr && a && b && c, knnx::errc::invalid_argument, "null argument");
    require(m >= 1 && n >= 1 && k >= kKC && k % kKC == 0, knnx::errc::invalid_argument,
            "need m, n >= 1 and k a multiple of 32");
    require(ld >= k && ld % 4 == 0 && ldc >= n, knnx::errc::invalid_argument, "bad leading dimensions");
    DeviceGuard dg(ctx->device);
    const size_t smem = sizeof(float) * 2 * (kTM + kTN) * kKC;
    check(cudaFuncSetAttribute(gram_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)),
          "smem attribute");
    const dim3 grid((m + kTM - 1) / kTM, (n + kTN - 1) / kTN);
    gram_tf32_kernel<<<grid, kThreads, smem, ctx->stream>>>(a, m, b, n, ld, k, c, ldc);
    launched(ctx, "gram_tf32");
    return KNNX_OK;
  });
}
