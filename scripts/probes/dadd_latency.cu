// Dependent fp64 add latency on sm_100a (the bit-exact PCA covariance action is
// N such adds per chain): one warp, a chain of 4096 DADDs, clock64 around it;
// then the same with the DMUL feeding it from shared memory as in xtb_blocked_kernel.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, const double* in, long long* cyc) {
  double acc = in[threadIdx.x];
  const double x = in[32 + threadIdx.x];
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) acc = __dadd_rn(acc, x);
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_mul(double* out, const double* in, long long* cyc) {
  __shared__ double sx[2048], sb[2048];
  for (int i = threadIdx.x; i < 2048; i += 32) { sx[i] = in[i & 63]; sb[i] = in[(i + 7) & 63]; }
  __syncwarp();
  double acc = 0.0;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < 4096; ++i) acc = __dadd_rn(acc, __dmul_rn(sx[i & 2047], sb[(i + threadIdx.x) & 2047]));
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
// does the fp64 pipe's time per warp instruction shrink with fewer active lanes?
__global__ void chain_lanes(double* out, const double* in, long long* cyc, int lanes, int slot) {
  __shared__ double sx[2048], sb[2048];
  for (int i = threadIdx.x; i < 2048; i += 32) { sx[i] = in[i & 63]; sb[i] = in[(i + 7) & 63]; }
  __syncwarp();
  if (threadIdx.x >= lanes) return;
  double acc = 0.0;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < 4096; ++i) acc = __dadd_rn(acc, __dmul_rn(sx[i & 2047], sb[(i + threadIdx.x) & 2047]));
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[slot] = t1 - t0;
}
// the same chain software-pipelined by hand: the product of row r + 8 and the
// loads of row r + 16 are issued between the dependent adds
__global__ void chain_pipe(double* out, const double* in, long long* cyc) {
  __shared__ double sx[2048], sb[2048];
  for (int i = threadIdx.x; i < 2048; i += 32) { sx[i] = in[i & 63]; sb[i] = in[(i + 7) & 63]; }
  __syncwarp();
  const double* sbr = sb + threadIdx.x;
  double acc = 0.0, xv[8], bv[8], pv[8];
  long long t0 = clock64();
  for (int rep = 0; rep < 2; ++rep) {
    const int rows = 2048 - 32;
#pragma unroll
    for (int i = 0; i < 8; ++i) { xv[i] = sx[i]; bv[i] = sbr[i]; }
#pragma unroll
    for (int i = 0; i < 8; ++i) pv[i] = __dmul_rn(xv[i], bv[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) { xv[i] = sx[8 + i]; bv[i] = sbr[8 + i]; }
    for (int base = 0; base < rows; base += 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc = __dadd_rn(acc, pv[i]);
        if (base + 8 < rows) pv[i] = __dmul_rn(xv[i], bv[i]);
        if (base + 16 < rows) { xv[i] = sx[base + 16 + i]; bv[i] = sbr[base + 16 + i]; }
      }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
int main() {
  double *in, *out; long long* cyc;
  cudaMalloc(&in, 64 * 8); cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 64);
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 1e-3;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) { chain<<<1, 32>>>(out, in, cyc); chain_mul<<<1, 32>>>(out, in, cyc); chain_pipe<<<1, 32>>>(out, in, cyc); chain_lanes<<<1, 32>>>(out, in, cyc, 16, 3); chain_lanes<<<1, 32>>>(out, in, cyc, 8, 4); chain_lanes<<<1, 32>>>(out, in, cyc, 4, 5); chain_lanes<<<1, 32>>>(out, in, cyc, 1, 6); }
  long long c[8]; cudaMemcpy(c, cyc, 64, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.2f cycles each; DADD(acc, DMUL(lds, lds)) chain: %.2f cycles per step; hand-pipelined: %.2f\n",
         c[0] / 4096.0, c[1] / 4096.0, c[2] / (2.0 * (2048 - 32)));
  printf("mul+add chain with 16 / 8 / 4 / 1 active lanes: %.2f / %.2f / %.2f / %.2f cycles per step\n", c[3] / 4096.0,
         c[4] / 4096.0, c[5] / 4096.0, c[6] / 4096.0);
  return 0;
}
