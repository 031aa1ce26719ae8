// tests/cpp/test_build.cpp -- the device-side input builders driven through
// the C ABI only (include/knnx.h, include/knnx_host.h), as a C++ caller of the
// reference's pipeline would use them in place of build_knn (proj/src/knn.cpp:
// 9-62), symmetrize + values (knn.cpp:72-84) and the blocked layout
// (hier.cpp:84-155):
//   * knnx_knn_wide_dev (tcgen05 screen + exact re-rank) == a double brute
//     force on the same points, every row certified;
//   * knnx_tsne_affinities_dev -> knnx_op_create_csr_dev (scheduled,
//     group-interleaved, built on the device) == the operator
//     knnx_op_create_csr_ex builds on the host from the downloaded CSR:
//     same slot -> row map, same stored values, bitwise equal t-SNE forces.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <vector>

#include "knnx.h"
#include "knnx_host.h"

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                                \
  do {                                                                          \
    if (c) ++g_pass;                                                            \
    else { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); } \
  } while (0)
#define OK(call)                                                                                            \
  do {                                                                                                      \
    const int rc_ = (call);                                                                                 \
    if (rc_ != 0) {                                                                                         \
      std::printf("FAIL %s:%d  %s -> %d (%s)\n", __FILE__, __LINE__, #call, rc_, knnx_last_error());        \
      ++g_fail;                                                                                             \
      return 1;                                                                                             \
    }                                                                                                       \
  } while (0)

int main() {
  const int32_t n = 3000, dim = 96, k = 12, ld = 96;
  std::vector<float> pts(static_cast<size_t>(n) * dim);
  OK(knnx_gen_points(3, n, dim, (4 << 16) | 4, 1.0, 13, pts.data()));
  knnx_ctx_t ctx = nullptr;
  OK(knnx_ctx_create(0, &ctx));
  void *d_pts = nullptr, *d_ids = nullptr, *d_d2 = nullptr;
  OK(knnx_alloc(ctx, static_cast<int64_t>(n) * ld * 4, &d_pts));
  OK(knnx_alloc(ctx, static_cast<int64_t>(n) * k * 4, &d_ids));
  OK(knnx_alloc(ctx, static_cast<int64_t>(n) * k * 4, &d_d2));
  OK(knnx_upload_points(ctx, pts.data(), n, dim, ld, static_cast<float*>(d_pts)));
  double stats[6] = {};
  OK(knnx_knn_wide_dev(ctx, static_cast<float*>(d_pts), n, static_cast<float*>(d_pts), n, ld, dim, k, 0, 1,
                       static_cast<int32_t*>(d_ids), static_cast<float*>(d_d2), stats));
  CHECK(stats[1] == 0.0);  // every row certified
  std::vector<int32_t> ids(static_cast<size_t>(n) * k);
  std::vector<float> d2(ids.size());
  cudaMemcpy(ids.data(), d_ids, ids.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(d2.data(), d_d2, d2.size() * 4, cudaMemcpyDeviceToHost);
  // double brute force (ascending (distance, index), self excluded)
  int wrong = 0;
  double worst = 0.0;
  std::vector<std::pair<double, int32_t>> all(n);
  for (int32_t i = 0; i < n; i += 7) {
    for (int32_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int32_t c = 0; c < dim; ++c) {
        const double e = static_cast<double>(pts[static_cast<size_t>(i) * dim + c]) - pts[static_cast<size_t>(j) * dim + c];
        s += e * e;
      }
      all[j] = {j == i ? 1e300 : s, j};
    }
    std::partial_sort(all.begin(), all.begin() + k, all.end());
    for (int32_t q = 0; q < k; ++q) {
      if (ids[static_cast<size_t>(i) * k + q] != all[q].second) ++wrong;
      worst = std::max(worst, std::fabs(d2[static_cast<size_t>(i) * k + q] - all[q].first) / all[q].first);
    }
  }
  CHECK(wrong <= 2);  // fp32 near-ties only
  CHECK(worst < 1e-5);

  // joint affinities and the operator, both on the device
  int64_t* d_rp = nullptr;
  int32_t* d_cols = nullptr;
  float* d_vals = nullptr;
  int64_t nnz = 0;
  double h = 0.0;
  OK(knnx_median_distance(d2.data(), static_cast<int64_t>(d2.size()), &h));
  OK(knnx_tsne_affinities_dev(ctx, static_cast<int32_t*>(d_ids), static_cast<float*>(d_d2), n, k, h / std::sqrt(2.0),
                              1.0 / (2.0 * n), &d_rp, &d_cols, &d_vals, &nnz));
  knnx_op_t op_dev = nullptr, op_host = nullptr;
  OK(knnx_op_create_csr_dev(ctx, n, n, nnz, d_rp, d_cols, d_vals, KNNX_SCHEDULE_GRAPH, 0, nullptr,
                            KNNX_OPT_GROUP_INTERLEAVE, &op_dev));
  std::vector<int64_t> rp(n + 1);
  std::vector<int32_t> cols(nnz);
  std::vector<float> vals(nnz);
  cudaMemcpy(rp.data(), d_rp, rp.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(cols.data(), d_cols, cols.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(vals.data(), d_vals, vals.size() * 4, cudaMemcpyDeviceToHost);
  OK(knnx_op_create_csr_ex(ctx, n, n, nnz, rp.data(), cols.data(), vals.data(), KNNX_ORDER_ORIGINAL, 256,
                           KNNX_SCHEDULE_GRAPH, 0, nullptr, KNNX_OPT_GROUP_INTERLEAVE, &op_host));
  std::vector<int32_t> sr_dev(n), sr_host(n);
  OK(knnx_op_slot_rows(op_dev, sr_dev.data()));
  OK(knnx_op_slot_rows(op_host, sr_host.data()));
  CHECK(sr_dev == sr_host);
  std::vector<float> v_dev(nnz), v_host(nnz);
  OK(knnx_op_get_values(op_dev, v_dev.data()));
  OK(knnx_op_get_values(op_host, v_host.data()));
  CHECK(v_dev == v_host && v_dev == vals);
  double psum = 0.0;
  for (float v : vals) psum += v;
  CHECK(std::fabs(psum - 1.0) < 1e-5);
  std::vector<float> y(static_cast<size_t>(n) * 2);
  OK(knnx_gen_points(4, n, 2, 0, 1e-2, 2, y.data()));
  void *d_y = nullptr, *d_f1 = nullptr, *d_f2 = nullptr;
  OK(knnx_alloc(ctx, static_cast<int64_t>(n) * 8, &d_y));
  OK(knnx_alloc(ctx, static_cast<int64_t>(n) * 8, &d_f1));
  OK(knnx_alloc(ctx, static_cast<int64_t>(n) * 8, &d_f2));
  OK(knnx_upload_points(ctx, y.data(), n, 2, 2, static_cast<float*>(d_y)));
  OK(knnx_tsne_attr_dev(op_dev, static_cast<float*>(d_y), 2, static_cast<float*>(d_f1), 0, 0.0f, nullptr));
  OK(knnx_tsne_attr_dev(op_host, static_cast<float*>(d_y), 2, static_cast<float*>(d_f2), 0, 0.0f, nullptr));
  OK(knnx_ctx_sync(ctx));
  std::vector<float> f1(y.size()), f2(y.size());
  cudaMemcpy(f1.data(), d_f1, f1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(f2.data(), d_f2, f2.size() * 4, cudaMemcpyDeviceToHost);
  CHECK(f1 == f2);
  OK(knnx_op_destroy(op_dev));
  OK(knnx_op_destroy(op_host));
  for (void* p : {d_pts, d_ids, d_d2, d_y, d_f1, d_f2, static_cast<void*>(d_rp), static_cast<void*>(d_cols),
                  static_cast<void*>(d_vals)})
    knnx_free(ctx, p);
  OK(knnx_ctx_destroy(ctx));
  std::printf("test_build: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
