// Rng transforms and the synthetic workload generators (BASELINE.json configs).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <numbers>
#include <thread>

#include "host.hpp"

namespace knnx {

const char* errc_name(errc c) {
  switch (c) {
    case errc::out_of_bounds: return "OutOfBounds";
    case errc::duplicate_entry: return "DuplicateEntry";
    case errc::size_mismatch: return "SizeMismatch";
    case errc::dim_mismatch: return "DimMismatch";
    case errc::k_too_large: return "KTooLarge";
    case errc::not_square: return "NotSquare";
    case errc::non_positive_bandwidth: return "NonPositiveBandwidth";
    case errc::degenerate_data: return "DegenerateData";
    case errc::dim_too_high: return "DimTooHigh";
    case errc::level_out_of_range: return "LevelOutOfRange";
    case errc::empty_pattern: return "EmptyPattern";
    case errc::too_large: return "TooLarge";
    case errc::not_divisible: return "NotDivisible";
    case errc::too_wide: return "TooWide";
    case errc::too_many: return "TooMany";
    case errc::span_mismatch: return "SpanMismatch";
    case errc::local_index_overflow: return "LocalIndexOverflow";
    case errc::ordering_mismatch: return "OrderingMismatch";
    case errc::non_finite_value: return "NonFiniteValue";
    case errc::zero_weight: return "ZeroWeight";
    case errc::malformed_record: return "MalformedRecord";
    case errc::inconsistent_dim: return "InconsistentDim";
    case errc::empty_file: return "EmptyFile";
    case errc::io_error: return "IoError";
    case errc::checksum_mismatch: return "ChecksumMismatch";
    case errc::invalid_argument: return "InvalidArgument";
    case errc::cuda_error: return "CudaError";
    case errc::unsupported: return "Unsupported";
  }
  return "UnknownError";
}

// Box-Muller with one cached spare; u1, u2 in (0,1) (proj/src/core.cpp:186-199)
double Rng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  const double u1 = (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53;
  const double u2 = (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * std::numbers::pi * u2;
  spare_ = r * std::sin(a);
  has_spare_ = true;
  return r * std::cos(a);
}

std::vector<float> gen_mixture_c1(index_t n, index_t dim, index_t n_clusters, double sigma,
                                  std::uint64_t seed) {
  if (n <= 0 || dim <= 0 || n_clusters <= 0 || !(sigma > 0.0))
    throw error(errc::invalid_argument, "mixture parameters must be positive");
  Rng rng(seed);
  std::vector<double> centers(static_cast<std::size_t>(n_clusters) * dim);
  for (double& c : centers) c = -10.0 + 20.0 * rng.uniform01();
  std::vector<float> out(static_cast<std::size_t>(n) * dim);
  for (index_t p = 0; p < n; ++p) {
    const double* c = centers.data() + static_cast<std::size_t>(p % n_clusters) * dim;
    for (index_t a = 0; a < dim; ++a)
      out[static_cast<std::size_t>(p) * dim + a] = static_cast<float>(c[a] + sigma * rng.normal());
  }
  return out;
}

std::vector<float> gen_mixture_3level(index_t n, index_t dim, double noise, std::uint64_t seed) {
  if (n <= 0 || dim <= 0 || !(noise > 0.0))
    throw error(errc::invalid_argument, "mixture parameters must be positive");
  constexpr index_t kFan = 16;
  const double scales[3] = {10.0, 2.0, 0.5};
  Rng rng(seed);
  std::vector<double> lvl1(static_cast<std::size_t>(kFan) * dim);
  for (double& c : lvl1) c = scales[0] * rng.normal();
  std::vector<double> lvl2(static_cast<std::size_t>(kFan * kFan) * dim);
  for (index_t s = 0; s < kFan * kFan; ++s)
    for (index_t a = 0; a < dim; ++a)
      lvl2[static_cast<std::size_t>(s) * dim + a] =
          lvl1[static_cast<std::size_t>(s / kFan) * dim + a] + scales[1] * rng.normal();
  std::vector<double> lvl3(static_cast<std::size_t>(kFan * kFan * kFan) * dim);
  for (index_t s = 0; s < kFan * kFan * kFan; ++s)
    for (index_t a = 0; a < dim; ++a)
      lvl3[static_cast<std::size_t>(s) * dim + a] =
          lvl2[static_cast<std::size_t>(s / kFan) * dim + a] + scales[2] * rng.normal();
  std::vector<float> out(static_cast<std::size_t>(n) * dim);
  for (index_t p = 0; p < n; ++p) {
    const index_t leaf = static_cast<index_t>(rng.bounded(kFan * kFan * kFan));
    const double* c = lvl3.data() + static_cast<std::size_t>(leaf) * dim;
    for (index_t a = 0; a < dim; ++a)
      out[static_cast<std::size_t>(p) * dim + a] = static_cast<float>(c[a] + noise * rng.normal());
  }
  return out;
}

std::vector<float> gen_mixture_aniso(index_t n, index_t dim, index_t n_top, index_t n_sub,
                                     std::uint64_t seed) {
  if (n <= 0 || dim <= 0 || n_top <= 0 || n_sub <= 0)
    throw error(errc::invalid_argument, "mixture parameters must be positive");
  constexpr int kReflections = 3;
  Rng rng(seed);
  // per top cluster: center ~ N(0, 3^2), sqrt-eigenvalues, 3 unit Householder vectors
  std::vector<double> top(static_cast<std::size_t>(n_top) * dim), sd(top.size());
  std::vector<double> house(static_cast<std::size_t>(n_top) * kReflections * dim);
  for (double& c : top) c = 3.0 * rng.normal();
  for (double& s : sd) s = std::sqrt(std::pow(10.0, -2.0 + 2.0 * rng.uniform01()));
  for (index_t t = 0; t < n_top * kReflections; ++t) {
    double* h = house.data() + static_cast<std::size_t>(t) * dim;
    double nrm = 0.0;
    for (index_t a = 0; a < dim; ++a) {
      h[a] = rng.normal();
      nrm += h[a] * h[a];
    }
    nrm = std::sqrt(nrm);
    for (index_t a = 0; a < dim; ++a) h[a] /= nrm;
  }
  std::vector<double> sub(static_cast<std::size_t>(n_top) * n_sub * dim);
  for (index_t s = 0; s < n_top * n_sub; ++s)
    for (index_t a = 0; a < dim; ++a)
      sub[static_cast<std::size_t>(s) * dim + a] =
          top[static_cast<std::size_t>(s / n_sub) * dim + a] + 1.0 * rng.normal();
  // Points: block b of kPointBlock points draws from its own substream
  // Rng(seed ^ golden * (b + 1)), so the result is independent of how the
  // blocks are spread over host threads (1M x 960 is ~1e9 normals).
  constexpr index_t kPointBlock = 8192;
  std::vector<float> out(static_cast<std::size_t>(n) * dim);
  const index_t n_blocks = (n + kPointBlock - 1) / kPointBlock;
  std::atomic<index_t> next{0};
  auto worker = [&] {
    std::vector<double> z(dim);
    for (index_t b = next++; b < n_blocks; b = next++) {
      Rng prng(seed ^ (0x9E3779B97F4A7C15ULL * static_cast<std::uint64_t>(b + 1)));
      const index_t hi = std::min(n, (b + 1) * kPointBlock);
      for (index_t p = b * kPointBlock; p < hi; ++p) {
        const index_t s =
            static_cast<index_t>(prng.bounded(static_cast<std::uint64_t>(n_top) * n_sub));
        const index_t t = s / n_sub;
        const double* sdt = sd.data() + static_cast<std::size_t>(t) * dim;
        for (index_t a = 0; a < dim; ++a) z[a] = sdt[a] * prng.normal();
        for (int r = 0; r < kReflections; ++r) {  // z <- (I - 2 h h^T) z
          const double* h = house.data() + (static_cast<std::size_t>(t) * kReflections + r) * dim;
          double dot = 0.0;
          for (index_t a = 0; a < dim; ++a) dot += h[a] * z[a];
          for (index_t a = 0; a < dim; ++a) z[a] -= 2.0 * dot * h[a];
        }
        const double* c = sub.data() + static_cast<std::size_t>(s) * dim;
        for (index_t a = 0; a < dim; ++a)
          out[static_cast<std::size_t>(p) * dim + a] = static_cast<float>(c[a] + z[a]);
      }
    }
  };
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned w = 1; w < hw && w < static_cast<unsigned>(n_blocks); ++w) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return out;
}

std::vector<float> gen_uniform01(std::int64_t n, std::uint64_t seed) {
  Rng rng(seed);
  std::vector<float> out(static_cast<std::size_t>(n));
  for (float& v : out) v = static_cast<float>(rng.uniform01());
  return out;
}

std::vector<float> gen_normal(std::int64_t n, double sigma, std::uint64_t seed) {
  Rng rng(seed);
  std::vector<float> out(static_cast<std::size_t>(n));
  for (float& v : out) v = static_cast<float>(sigma * rng.normal());
  return out;
}

double median_distance(const float* d2, std::int64_t count) {
  if (count <= 0) throw error(errc::invalid_argument, "no distances");
  std::vector<double> d(static_cast<std::size_t>(count));
  for (std::int64_t i = 0; i < count; ++i) d[i] = std::sqrt(static_cast<double>(d2[i]));
  const std::size_t mid = d.size() / 2;
  std::nth_element(d.begin(), d.begin() + mid, d.end());
  double m = d[mid];
  if (d.size() % 2 == 0) {
    const double lo = *std::max_element(d.begin(), d.begin() + mid);
    m = 0.5 * (lo + m);
  }
  return m;
}

}  // namespace knnx
