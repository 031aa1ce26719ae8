// The call path INTEGRATION.md gives a patchord maintainer, timed end to end:
// reference types in (SparseMatrix / ChargeVector, std::vector<double>),
// gpu::Operator::spmv out (PotentialVector), i.e. per call an fp64 -> fp32
// conversion of x, a pageable 4-MB upload, the multiply, a pageable download
// and the fp32 -> fp64 widening of y.  Synthetic banded kNN-like matrix at the
// C2 shape (N rows, 30 neighbours each); the result is checked against the
// reference's own spmv_flat.  Prints one JSON line.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "patchord/core.hpp"
#include "patchord/kernels.hpp"
#include "patchord_gpu.hpp"

using namespace patchord;

int main(int argc, char** argv) {
  const index_t n = argc > 1 ? std::atoi(argv[1]) : 1000000, k = 30, calls = argc > 2 ? std::atoi(argv[2]) : 20;
  SparseMatrix m;
  m.pattern.n_rows = n;
  m.pattern.n_cols = n;
  m.pattern.entries.reserve(static_cast<std::size_t>(n) * k);
  m.values.reserve(static_cast<std::size_t>(n) * k);
  Rng rng(5);
  for (index_t i = 0; i < n; ++i) {
    const index_t lo = std::min(std::max<index_t>(i - k / 2, 0), n - k - 1);
    for (index_t j = lo; j <= lo + k; ++j) {
      if (j == i) continue;
      m.pattern.entries.emplace_back(i, j);
      m.values.push_back(static_cast<float>(0.25 + 0.5 * rng.uniform01()));
    }
  }
  ChargeVector x;
  x.values.resize(n);
  for (double& v : x.values) v = static_cast<float>(rng.uniform01());
  gpu::Device dev(0);
  const auto t_up0 = std::chrono::steady_clock::now();
  gpu::Operator op(dev, m);
  const double upload_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_up0).count();
  PotentialVector y;
  for (int w = 0; w < 3; ++w) y = op.spmv(x);
  const auto t0 = std::chrono::steady_clock::now();
  for (index_t c = 0; c < calls; ++c) y = op.spmv(x);
  const double per_call = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / calls;
  // drop-in free function: uploads the matrix on every call, like the reference signature implies
  const auto t1 = std::chrono::steady_clock::now();
  const PotentialVector y2 = gpu::spmv_flat(m, x);
  const double free_call = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  const auto t2 = std::chrono::steady_clock::now();
  const PotentialVector want = spmv_flat(m, x);
  const double ref_call = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
  double scale = 0.0, err = 0.0;
  for (index_t i = 0; i < n; ++i) {
    scale = std::max(scale, std::fabs(want.values[i]));
    err = std::max(err, std::max(std::fabs(want.values[i] - y.values[i]), std::fabs(want.values[i] - y2.values[i])));
  }
  const double nnz = static_cast<double>(m.nnz());
  std::printf("{\"bench\": \"patchord::gpu shim, std::vector<double> in / out\", \"n\": %d, \"nnz\": %.0f, "
              "\"operator_spmv_ms\": %.3f, \"operator_spmv_interactions_per_s\": %.4g, "
              "\"operator_upload_s\": %.3f, \"free_function_spmv_flat_s\": %.3f, "
              "\"reference_spmv_flat_s\": %.4f, \"reference_interactions_per_s\": %.4g, \"rel_err\": %.2e}\n",
              n, nnz, per_call * 1e3, nnz / per_call, upload_s, free_call, ref_call, nnz / ref_call, err / scale);
  return err / scale <= 1e-5 ? 0 : 1;
}
