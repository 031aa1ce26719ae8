// tests/cpp/test_multi.cpp -- two ranks driven through the C ABI only
// (include/knnx.h), the multi-device generalisation of the reference's
// spmv_hier_parallel worker model (proj/src/kernels.cpp:63-101) whose
// results must not depend on the worker count (proj/tests/test_kernels.cpp:
// 158-177).  On a one-GPU box both ranks share device 0 (local transport);
// with two GPUs the ranks sit on devices 0 and 1 (NCCL + peer stores).
//
// Checks, all bitwise against one rank holding the whole operator:
//   * row-block sharded y = A x (cluster tiles) and its all-gather;
//   * 5 t-SNE steps whose embedding exchange is fused into the force kernel
//     (knnx_tsne_attr_peers_dev: peer stores into every rank's replica) with
//     a stream-ordered barrier between steps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "knnx.h"

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                                  \
  do {                                                                            \
    if (c) ++g_pass;                                                              \
    else { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); }   \
  } while (0)
#define OK(call)                                                                   \
  do {                                                                             \
    const int rc_ = (call);                                                        \
    if (rc_ != 0) {                                                                \
      std::printf("FAIL %s:%d  %s -> %d (%s)\n", __FILE__, __LINE__, #call, rc_,   \
                  knnx_last_error());                                              \
      ++g_fail;                                                                    \
      return;                                                                      \
    }                                                                              \
  } while (0)

namespace {

template <typename T>
T* dev_copy(const std::vector<T>& h) {
  T* d = nullptr;
  cudaMalloc(&d, sizeof(T) * std::max<size_t>(1, h.size()));
  cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice);
  return d;
}

template <typename T>
std::vector<T> host_copy(const T* d, size_t n) {
  std::vector<T> h(n);
  cudaDeviceSynchronize();
  cudaMemcpy(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost);
  return h;
}

// a symmetric pattern with exactly k entries per row (each row i: i +- offsets)
struct Csr {
  int32_t n = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> cols;
  std::vector<float> vals;
};

Csr make_problem(int32_t n, int32_t half_k, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<int32_t> offs;
  while (static_cast<int32_t>(offs.size()) < half_k) {
    const int32_t o = 1 + static_cast<int32_t>(rng() % 400);
    if (std::find(offs.begin(), offs.end(), o) == offs.end()) offs.push_back(o);
  }
  Csr a;
  a.n = n;
  a.rp.push_back(0);
  std::uniform_real_distribution<float> u(0.1f, 1.1f);
  for (int32_t i = 0; i < n; ++i) {
    std::vector<int32_t> row;
    for (int32_t o : offs) {
      row.push_back((i + o) % n);
      row.push_back((i - o + n) % n);
    }
    std::sort(row.begin(), row.end());
    for (int32_t c : row) {
      a.cols.push_back(c);
      // symmetric values: a function of the unordered pair
      const uint64_t key = static_cast<uint64_t>(std::min(i, c)) * 1000003ull + std::max(i, c);
      a.vals.push_back(1e-6f * (1.0f + static_cast<float>(key % 997) / 997.0f));
    }
    a.rp.push_back(static_cast<int64_t>(a.cols.size()));
  }
  (void)u;
  return a;
}

Csr row_block(const Csr& a, int32_t r0, int32_t r1) {
  Csr b;
  b.n = r1 - r0;
  b.rp.push_back(0);
  for (int32_t i = r0; i < r1; ++i) {
    for (int64_t e = a.rp[i]; e < a.rp[i + 1]; ++e) {
      b.cols.push_back(a.cols[e]);
      b.vals.push_back(a.vals[e]);
    }
    b.rp.push_back(static_cast<int64_t>(b.cols.size()));
  }
  return b;
}

void run() {
  int n_dev = 0;
  cudaGetDeviceCount(&n_dev);
  const int dev1 = n_dev > 1 ? 1 : 0;
  const int32_t n = 4096 + 512, half_k = 12;  // 24 entries per row
  const Csr a = make_problem(n, half_k, 7);
  const int32_t rows_per_rank = 2304;          // tile-aligned (9 x 256) equal blocks
  const int32_t cuts[3] = {0, rows_per_rank, n};

  knnx_ctx_t ctx[2];
  OK(knnx_ctx_create(0, &ctx[0]));
  OK(knnx_ctx_create(dev1, &ctx[1]));
  knnx_comm_t comm[2];
  OK(knnx_comm_init_local(2, ctx, comm));
  int32_t nr = 0, rk = -1, tr = 0;
  OK(knnx_comm_info(comm[1], &nr, &rk, &tr));
  CHECK(nr == 2 && rk == 1 && (tr == KNNX_COMM_LOCAL || tr == KNNX_COMM_NCCL));
  std::printf("transport: %s (devices 0, %d)\n", tr == KNNX_COMM_NCCL ? "nccl" : "local", dev1);

  // ---- one rank, whole operator
  knnx_op_t full = nullptr;
  OK(knnx_op_create_csr(ctx[0], n, n, static_cast<int64_t>(a.cols.size()), a.rp.data(),
                        a.cols.data(), a.vals.data(), KNNX_ORDER_CLUSTER, 256, &full));
  std::vector<float> x(n);
  std::mt19937 rng(3);
  std::uniform_real_distribution<float> u01(0.f, 1.f);
  for (float& v : x) v = u01(rng);
  cudaSetDevice(0);
  float* dx = dev_copy(x);
  float* dy = nullptr;
  cudaMalloc(&dy, sizeof(float) * n);
  OK(knnx_spmv_dev(full, dx, dy));
  OK(knnx_ctx_sync(ctx[0]));
  const std::vector<float> y_full = host_copy(dy, n);

  // ---- two ranks: row blocks, x replicated, all-gather of y into padded buffers
  knnx_op_t shard[2];
  float* xr[2];
  float* yr[2];  // each rank: 2 * rows_per_rank floats, own block filled by the multiply
  for (int r = 0; r < 2; ++r) {
    const Csr b = row_block(a, cuts[r], cuts[r + 1]);
    OK(knnx_op_create_csr(ctx[r], b.n, n, static_cast<int64_t>(b.cols.size()), b.rp.data(),
                          b.cols.data(), b.vals.data(), KNNX_ORDER_CLUSTER, 256, &shard[r]));
    OK(knnx_op_set_row_base(shard[r], cuts[r]));
    cudaSetDevice(ctx[r] == ctx[0] ? 0 : dev1);
    xr[r] = dev_copy(x);
    cudaMalloc(&yr[r], sizeof(float) * 2 * rows_per_rank);
    cudaMemset(yr[r], 0, sizeof(float) * 2 * rows_per_rank);
  }
  for (int r = 0; r < 2; ++r)
    OK(knnx_spmv_dev(shard[r], xr[r], yr[r] + static_cast<int64_t>(r) * rows_per_rank));
  void* bufs[2] = {yr[0], yr[1]};
  OK(knnx_allgather_rows_local(comm, 2, bufs, rows_per_rank, sizeof(float)));
  for (int r = 0; r < 2; ++r) OK(knnx_ctx_sync(ctx[r]));
  for (int r = 0; r < 2; ++r) {
    const std::vector<float> g = host_copy(yr[r], 2 * rows_per_rank);
    CHECK(std::memcmp(g.data(), y_full.data(), sizeof(float) * n) == 0);
  }

  // ---- t-SNE, 5 steps with the fused embedding update
  const int32_t dim = 2, steps = 5;
  const float eta = 0.5f * n;
  std::vector<float> y0(static_cast<size_t>(n) * dim);
  std::normal_distribution<float> nd(0.f, 1e-2f);
  for (float& v : y0) v = nd(rng);
  // one rank: y <- y - eta F via knnx_tsne_attr_dev's fused update
  cudaSetDevice(0);
  float* ya = dev_copy(y0);
  float* yb = dev_copy(y0);
  float* f = nullptr;
  cudaMalloc(&f, sizeof(float) * n * dim);
  for (int s = 0; s < steps; ++s) {
    OK(knnx_tsne_attr_dev(full, ya, dim, f, 0, eta, yb));
    std::swap(ya, yb);
  }
  OK(knnx_ctx_sync(ctx[0]));
  const std::vector<float> y_one = host_copy(ya, static_cast<size_t>(n) * dim);
  // two ranks: each holds a replicated embedding pair; the kernel of rank r
  // stores its rows into both ranks' "next" replicas, then a barrier
  float* cur[2];
  float* nxt[2];
  float* fr[2];
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(r == 0 ? 0 : dev1);
    cur[r] = dev_copy(y0);
    nxt[r] = dev_copy(y0);
    cudaMalloc(&fr[r], sizeof(float) * (cuts[r + 1] - cuts[r]) * dim);
  }
  for (int s = 0; s < steps; ++s) {
    for (int r = 0; r < 2; ++r) OK(knnx_tsne_attr_peers_dev(shard[r], cur[r], dim, fr[r], eta, nxt, 2));
    OK(knnx_comm_barrier_local(comm, 2));
    std::swap(cur[0], nxt[0]);
    std::swap(cur[1], nxt[1]);
  }
  for (int r = 0; r < 2; ++r) OK(knnx_ctx_sync(ctx[r]));
  for (int r = 0; r < 2; ++r) {
    const std::vector<float> g = host_copy(cur[r], static_cast<size_t>(n) * dim);
    CHECK(std::memcmp(g.data(), y_one.data(), sizeof(float) * n * dim) == 0);
  }
  // the fused path and the plain one agree on the forces of the last step
  {
    std::vector<float> fs;
    for (int r = 0; r < 2; ++r) {
      const std::vector<float> g = host_copy(fr[r], static_cast<size_t>(cuts[r + 1] - cuts[r]) * dim);
      fs.insert(fs.end(), g.begin(), g.end());
    }
    const std::vector<float> fo = host_copy(f, static_cast<size_t>(n) * dim);
    CHECK(std::memcmp(fs.data(), fo.data(), sizeof(float) * n * dim) == 0);
  }

  // ---- argument checks
  CHECK(knnx_allgather_rows_dev(comm[0], yr[0], rows_per_rank, 4) == KNNX_ERR_INVALID_ARGUMENT);
  knnx_comm_t wrong[2] = {comm[1], comm[0]};
  CHECK(knnx_comm_barrier_local(wrong, 2) == KNNX_ERR_INVALID_ARGUMENT);
  CHECK(knnx_tsne_attr_peers_dev(shard[0], cur[0], dim, fr[0], eta, nxt, 9) ==
        KNNX_ERR_INVALID_ARGUMENT);

  for (int r = 0; r < 2; ++r) {
    knnx_op_destroy(shard[r]);
    knnx_comm_destroy(comm[r]);
  }
  knnx_op_destroy(full);
  knnx_ctx_destroy(ctx[0]);
  knnx_ctx_destroy(ctx[1]);
}

}  // namespace

int main() {
  run();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
