// Bit-exact PCA covariance action on the device.
//
// The subspace iteration of proj/src/pca.cpp:194-216 computes
//   b_i[a]  = sum_r xc[i][r] * v[r][a]   (r ascending, per row i)
//   out[r][a] = sum_i xc[i][r] * b_i[a]  (i ascending, per (r, a))
// with separately rounded fp64 multiplies and adds (no FMA in the canonical
// x86-64 build).  Both are reproduced exactly: __dmul_rn / __dadd_rn forbid
// contraction, every sum keeps the reference's order, and only independent
// sums run in parallel (rows for b; the D*p (r, a) chains for out).  The
// result is bit-identical to the host loop, so the ordering permutation is
// unchanged (tests/test_host_ordering.py, -m gpu).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/host.hpp"
#include "ptx.cuh"

namespace knnx_dev {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw knnx::error(knnx::errc::cuda_error, std::string(what) + ": " + cudaGetErrorString(e));
}

template <int P>
__global__ void xv_kernel(const double* __restrict__ xc, int n, int D, const double* __restrict__ v,
                          double* __restrict__ b) {
  extern __shared__ double sv[];  // D * P
  for (int e = threadIdx.x; e < D * P; e += blockDim.x) sv[e] = v[e];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* row = xc + static_cast<int64_t>(i) * D;
  double acc[P];
#pragma unroll
  for (int a = 0; a < P; ++a) acc[a] = 0.0;
  for (int r = 0; r < D; ++r) {
    const double x = __ldg(row + r);
#pragma unroll
    for (int a = 0; a < P; ++a) acc[a] = __dadd_rn(acc[a], __dmul_rn(x, sv[r * P + a]));
  }
#pragma unroll
  for (int a = 0; a < P; ++a) b[static_cast<int64_t>(i) * P + a] = acc[a];
}

// one thread per (r, a) chain, i ascending; loads run ahead of the add chain
template <int P>
__global__ void __launch_bounds__(32) xtb_kernel(const double* __restrict__ xc, int n, int D,
                                                 const double* __restrict__ b,
                                                 double* __restrict__ out) {
  const int chain = blockIdx.x * blockDim.x + threadIdx.x;
  if (chain >= D * P) return;
  const int r = chain / P, a = chain - r * P;
  double acc = 0.0;
  constexpr int U = 16;
  int i = 0;
  for (; i + U <= n; i += U) {
    double xs[U], bs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xs[u] = __ldg(xc + static_cast<int64_t>(i + u) * D + r);
      bs[u] = __ldg(b + static_cast<int64_t>(i + u) * P + a);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(xs[u], bs[u]));
  }
  for (; i < n; ++i)
    acc = __dadd_rn(acc, __dmul_rn(__ldg(xc + static_cast<int64_t>(i) * D + r),
                                   __ldg(b + static_cast<int64_t>(i) * P + a)));
  out[static_cast<int64_t>(r) * P + a] = acc;
}

// The chains run in CTAs of a few columns each: rows stream through a ring of
// shared-memory stages filled by TMA bulk copies, so the only critical path
// left is the chains' dependent fp64 adds (~12 cycles per row; one CTA running
// all D * P chains of a 49-column input spent 41).  Zero padding rows (n
// rounded up to kCh) leave every sum bit-identical: acc + (+-0.0) == acc for
// acc != -0.0, and an accumulator that starts at +0.0 never becomes -0.0 in
// round-to-nearest.
constexpr int kCh = 32;      // row padding granule
constexpr int kStages = 10;

// The columns are cut into blocks of `dblk`, re-laid out once so every block
// is contiguous (xcb[block][row][col]), and one CTA per block runs its
// dblk * P chains over its own TMA-staged row stream.  Every chain keeps the
// reference's summation order.
__global__ void relayout_blocks_kernel(const double* __restrict__ xc, int n_pad, int D, int dblk,
                                       double* __restrict__ xcb) {
  const int64_t total = static_cast<int64_t>(n_pad) * ((D + dblk - 1) / dblk) * dblk;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t blk = e / (static_cast<int64_t>(n_pad) * dblk);
    const int64_t rem = e - blk * n_pad * dblk;
    const int64_t i = rem / dblk;
    const int c = static_cast<int>(blk * dblk + (rem - i * dblk));
    xcb[e] = c < D ? xc[i * D + c] : 0.0;
  }
}

// blockDim = the block's dblk * P chains rounded up to a warp; `ch` rows per
// staged chunk (a multiple of 32; the last chunk may be shorter)
template <int P>
__global__ void __launch_bounds__(512) xtb_blocked_kernel(const double* __restrict__ xcb, int n_pad,
                                                          int D, int dblk, int ch, int stages,
                                                          const double* __restrict__ b,
                                                          double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int xbytes = ch * dblk * 8, bbytes = ch * P * 8;
  const int stage_bytes = xbytes + bbytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  const double* xblk = xcb + static_cast<int64_t>(blockIdx.x) * n_pad * dblk;
  const int c0 = blockIdx.x * dblk;
  const int tid = threadIdx.x;
  const int n_chunks = (n_pad + ch - 1) / ch;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % stages;
    const int rows = min(ch, n_pad - c * ch);
    unsigned char* st = smem + s * stage_bytes;
    mbar_arrive_expect_tx(&full[s], rows * (dblk + P) * 8);
    bulk_g2s(st, xblk + static_cast<int64_t>(c) * ch * dblk, rows * dblk * 8, &full[s]);
    bulk_g2s(st + xbytes, b + static_cast<int64_t>(c) * ch * P, rows * P * 8, &full[s]);
  };
  if (tid == 0)
    for (int c = 0; c < stages && c < n_chunks; ++c) issue(c);
  const bool chain = tid < dblk * P;
  const int r = chain ? tid / P : 0, a = chain ? tid - (tid / P) * P : 0;
  double acc = 0.0;
  for (int c = 0; c < n_chunks; ++c) {
    const int s = c % stages;
    mbar_wait(&full[s], (c / stages) & 1);
    if (chain) {
      const double* sx = reinterpret_cast<const double*>(smem + s * stage_bytes);
      const double* sb = reinterpret_cast<const double*>(smem + s * stage_bytes + xbytes);
      const int rows = min(ch, n_pad - c * ch);
#pragma unroll 8
      for (int rr = 0; rr < rows; ++rr) acc = __dadd_rn(acc, __dmul_rn(sx[rr * dblk + r], sb[rr * P + a]));
    }
    __syncthreads();
    if (tid == 0 && c + stages < n_chunks) issue(c + stages);
  }
  if (chain && c0 + r < D) out[static_cast<int64_t>(c0 + r) * P + a] = acc;
}

class DeviceCovariance final : public knnx::CovarianceOp {
 public:
  DeviceCovariance(const std::vector<double>& xc, int n, int D, int device)
      : n_(n), D_(D), n_pad_((n + kCh - 1) / kCh * kCh) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
    const size_t xbytes = sizeof(double) * static_cast<size_t>(n_pad_) * D;
    ck(cudaMalloc(&d_xc_, xbytes), "alloc xc");
    ck(cudaMemsetAsync(d_xc_, 0, xbytes, st_), "zero xc");
    ck(cudaMemcpyAsync(d_xc_, xc.data(), sizeof(double) * xc.size(), cudaMemcpyHostToDevice, st_),
       "upload xc");
    ck(cudaMalloc(&d_b_, sizeof(double) * static_cast<size_t>(n_pad_) * 8), "alloc b");
    ck(cudaMemsetAsync(d_b_, 0, sizeof(double) * static_cast<size_t>(n_pad_) * 8, st_), "zero b");
    ck(cudaMalloc(&d_v_, sizeof(double) * static_cast<size_t>(D) * 8), "alloc v");
    ck(cudaMalloc(&d_out_, sizeof(double) * static_cast<size_t>(D) * 8), "alloc out");
  }
  ~DeviceCovariance() override {
    cudaStreamSynchronize(st_);
    cudaFree(d_xc_);
    cudaFree(d_b_);
    cudaFree(d_v_);
    cudaFree(d_out_);
    cudaFree(d_xcb_);
    cudaStreamDestroy(st_);
  }

  void xv(const std::vector<double>& v, std::vector<double>& b, int p) override {
    run_xv(v, p);
    b.resize(static_cast<size_t>(n_) * p);
    ck(cudaMemcpyAsync(b.data(), d_b_, sizeof(double) * b.size(), cudaMemcpyDeviceToHost, st_), "d2h b");
    ck(cudaStreamSynchronize(st_), "sync");
  }

  void apply(const std::vector<double>& in, std::vector<double>& out, int p) override {
    run_xv(in, p);
    const int chains = D_ * p;
    const int grid = (chains + 31) / 32;
    if (p <= 5) {
      // column-blocked: every chain is N dependent fp64 adds, so the time is
      // set by how many chains run side by side, not by bandwidth -- blocks
      // of >= 8 columns sized to spread the D columns over up to 148 SMs
      // (D = 960: 120 CTAs of 40 chains; round 1 ran 10 CTAs of 510 chains,
      // 41 ms per action instead of the ~8 ms of the add chain)
      const int dblk = std::max(8, 2 * ((D_ + 2 * 148 - 1) / (2 * 148)));
      if (dblk != dblk_) relayout(dblk);
      const int ch = 128;
      const size_t stage_bytes = static_cast<size_t>(ch) * (dblk + p) * 8;
      const int stages = static_cast<int>(std::min<size_t>(kStages, (200 * 1024) / stage_bytes));
      const size_t smem = stages * stage_bytes + stages * 8;
      const int nblk = (D_ + dblk - 1) / dblk;
      const int threads = (dblk * p + 31) / 32 * 32;
      auto run = [&](auto kernel) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kernel<<<nblk, threads, smem, st_>>>(d_xcb_, n_pad_, D_, dblk, ch, stages, d_b_, d_out_);
      };
      switch (p) {
        case 1: run(xtb_blocked_kernel<1>); break;
        case 2: run(xtb_blocked_kernel<2>); break;
        case 3: run(xtb_blocked_kernel<3>); break;
        case 4: run(xtb_blocked_kernel<4>); break;
        default: run(xtb_blocked_kernel<5>); break;
      }
    } else switch (p) {
      case 1: xtb_kernel<1><<<grid, 32, 0, st_>>>(d_xc_, n_, D_, d_b_, d_out_); break;
      case 2: xtb_kernel<2><<<grid, 32, 0, st_>>>(d_xc_, n_, D_, d_b_, d_out_); break;
      case 3: xtb_kernel<3><<<grid, 32, 0, st_>>>(d_xc_, n_, D_, d_b_, d_out_); break;
      case 4: xtb_kernel<4><<<grid, 32, 0, st_>>>(d_xc_, n_, D_, d_b_, d_out_); break;
      case 5: xtb_kernel<5><<<grid, 32, 0, st_>>>(d_xc_, n_, D_, d_b_, d_out_); break;
      default: throw knnx::error(knnx::errc::unsupported, "device PCA supports block sizes <= 5");
    }
    ck(cudaGetLastError(), "xtb_kernel");
    out.resize(static_cast<size_t>(D_) * p);
    ck(cudaMemcpyAsync(out.data(), d_out_, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, st_),
       "d2h out");
    ck(cudaStreamSynchronize(st_), "sync");
  }

 private:
  void relayout(int dblk) {
    if (d_xcb_) cudaFree(d_xcb_);
    const int nblk = (D_ + dblk - 1) / dblk;
    ck(cudaMalloc(&d_xcb_, sizeof(double) * static_cast<size_t>(n_pad_) * nblk * dblk), "alloc xcb");
    relayout_blocks_kernel<<<4 * 148, 256, 0, st_>>>(d_xc_, n_pad_, D_, dblk, d_xcb_);
    ck(cudaGetLastError(), "relayout");
    dblk_ = dblk;
  }

  void run_xv(const std::vector<double>& v, int p) {
    ck(cudaMemcpyAsync(d_v_, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, st_), "h2d v");
    const int grid = (n_ + 255) / 256;
    const size_t smem = sizeof(double) * static_cast<size_t>(D_) * p;
    switch (p) {
      case 1: xv_kernel<1><<<grid, 256, smem, st_>>>(d_xc_, n_, D_, d_v_, d_b_); break;
      case 2: xv_kernel<2><<<grid, 256, smem, st_>>>(d_xc_, n_, D_, d_v_, d_b_); break;
      case 3: xv_kernel<3><<<grid, 256, smem, st_>>>(d_xc_, n_, D_, d_v_, d_b_); break;
      case 4: xv_kernel<4><<<grid, 256, smem, st_>>>(d_xc_, n_, D_, d_v_, d_b_); break;
      case 5: xv_kernel<5><<<grid, 256, smem, st_>>>(d_xc_, n_, D_, d_v_, d_b_); break;
      default: throw knnx::error(knnx::errc::unsupported, "device PCA supports block sizes <= 5");
    }
    ck(cudaGetLastError(), "xv_kernel");
  }

  int n_, D_, n_pad_, dblk_ = 0;
  cudaStream_t st_ = nullptr;
  double *d_xc_ = nullptr, *d_b_ = nullptr, *d_v_ = nullptr, *d_out_ = nullptr, *d_xcb_ = nullptr;
};

}  // namespace

knnx::CovarianceOp* make_device_covariance(const std::vector<double>& xc, int n, int D, int device) {
  if (D > 6000) throw knnx::error(knnx::errc::unsupported, "device PCA: dim too large for the v stage");
  return new DeviceCovariance(xc, n, D, device);
}

}  // namespace knnx_dev
