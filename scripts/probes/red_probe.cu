// Scattered float2 RED throughput into an L2-resident array (C4 symmetric
// pair-once feasibility): E reductions into n float2 slots,
// targets row +- window (graph-local, like cluster-ordered kNN columns) or
// uniformly random.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int MODE>  // 0 = float2 RED, 1 = two scalar RED, 2 = float2 load (no atomic)
__global__ void red_kernel(float2* f, int n, long long e_total, int per_row, int window,
                           float* sink) {
  float acc = 0.f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e_total;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e / per_row);
    const unsigned h = hash32((unsigned)e);
    int j = window > 0 ? row + (int)(h % (2u * window + 1)) - window : (int)(h % (unsigned)n);
    j = j < 0 ? 0 : (j >= n ? n - 1 : j);
    if (MODE == 0) atomicAdd(f + j, make_float2(1e-3f, -1e-3f));
    else if (MODE == 1) { atomicAdd(&f[j].x, 1e-3f); atomicAdd(&f[j].y, -1e-3f); }
    else { const float2 v = __ldg(f + j); acc += v.x + v.y; }
  }
  if (MODE == 2 && acc == 12345.f) sink[0] = acc;
}
int main() {
  const int n = 4000000; const long long E = 302000000LL; const int per_row = 75;
  float2* f; float* sink;
  cudaMalloc(&f, n * sizeof(float2)); cudaMalloc(&sink, 4);
  cudaMemset(f, 0, n * sizeof(float2));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int windows[] = {2048, 65536, 0};
  for (int mode = 0; mode < 3; ++mode)
    for (int wi = 0; wi < 3; ++wi) {
      auto run = [&] {
        if (mode == 0) red_kernel<0><<<148 * 16, 256>>>(f, n, E, per_row, windows[wi], sink);
        if (mode == 1) red_kernel<1><<<148 * 16, 256>>>(f, n, E, per_row, windows[wi], sink);
        if (mode == 2) red_kernel<2><<<148 * 16, 256>>>(f, n, E, per_row, windows[wi], sink);
      };
      run(); cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
      printf("{\"mode\": \"%s\", \"window\": %d, \"ms\": %.3f, \"ops_per_s\": %.3e}\n",
             mode == 0 ? "float2_red" : mode == 1 ? "2x_scalar_red" : "float2_load", windows[wi], ms,
             E / (ms * 1e-3));
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
