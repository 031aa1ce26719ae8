// extern "C" veneer over the host-side C++ (include/knnx_host.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/knnx_host.h"
#include "host.hpp"

namespace knnx_dev {
knnx::CovarianceOp* make_device_covariance(const std::vector<double>& xc, int n, int D, int device);
knnx::PartitionTree build_tree_device(const double* emb, int n, int dim, int leaf_capacity, int max_depth,
                                      int device);
}

struct knnx_csr {
  knnx::Csr a;
};
struct knnx_tree {
  knnx::PartitionTree t;
};

namespace {

thread_local std::string g_host_error;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const knnx::error& e) {
    g_host_error = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::bad_alloc&) {
    g_host_error = "TooLarge: host allocation failed";
    return 1 + static_cast<int>(knnx::errc::too_large);
  } catch (const std::exception& e) {
    g_host_error = e.what();
    return 1 + static_cast<int>(knnx::errc::invalid_argument);
  }
}

void need(bool c, const char* msg) {
  if (!c) throw knnx::error(knnx::errc::invalid_argument, msg);
}

std::function<knnx::CovarianceOp*(const std::vector<double>&, knnx::index_t, knnx::index_t)>
covariance_factory(int32_t device) {
  if (device < 0) return nullptr;
  return [device](const std::vector<double>& xc, knnx::index_t n, knnx::index_t dim) {
    return knnx_dev::make_device_covariance(xc, n, dim, device);
  };
}

}  // namespace

extern "C" {

const char* knnx_host_last_error(void) { return g_host_error.c_str(); }

int knnx_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  return guard([&] {
    knnx::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next();
  });
}
int knnx_rng_uniform01(uint64_t seed, int64_t n, double* out) {
  return guard([&] {
    knnx::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform01();
  });
}
int knnx_rng_normal(uint64_t seed, int64_t n, double* out) {
  return guard([&] {
    knnx::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
  });
}
int knnx_order_scattered(int32_t n, uint64_t seed, int32_t* forward) {
  return guard([&] {
    need(n >= 1, "n must be >= 1");
    std::vector<int32_t> f(n);
    for (int32_t i = 0; i < n; ++i) f[i] = i;
    knnx::Rng r(seed);
    r.shuffle(f);
    std::copy(f.begin(), f.end(), forward);
  });
}

int knnx_gen_points(int32_t kind, int32_t n, int32_t dim, int32_t n_clusters, double p0,
                    uint64_t seed, float* out) {
  return guard([&] {
    std::vector<float> v;
    switch (kind) {
      case 1: v = knnx::gen_mixture_c1(n, dim, n_clusters, p0, seed); break;
      case 2: v = knnx::gen_mixture_3level(n, dim, p0, seed); break;
      case 3: v = knnx::gen_mixture_aniso(n, dim, n_clusters >> 16, n_clusters & 0xffff, seed); break;
      case 4: v = knnx::gen_normal(static_cast<int64_t>(n) * dim, p0, seed); break;
      default: throw knnx::error(knnx::errc::invalid_argument, "unknown generator kind");
    }
    std::copy(v.begin(), v.end(), out);
  });
}
int knnx_gen_uniform01(int64_t n, uint64_t seed, float* out) {
  return guard([&] {
    const std::vector<float> v = knnx::gen_uniform01(n, seed);
    std::copy(v.begin(), v.end(), out);
  });
}
int knnx_median_distance(const float* d2, int64_t count, double* out) {
  return guard([&] { *out = knnx::median_distance(d2, count); });
}

int knnx_csr_from_knn(const int32_t* ids, int32_t m, int32_t n, int32_t k, knnx_csr_t* out) {
  return guard([&] {
    auto h = std::make_unique<knnx_csr>();
    h->a = knnx::csr_from_knn(ids, m, n, k);
    *out = h.release();
  });
}
int knnx_csr_from_arrays(int32_t m, int32_t n, int64_t nnz, const int64_t* row_ptr,
                         const int32_t* cols, const float* vals, knnx_csr_t* out) {
  return guard([&] {
    need(m >= 0 && n >= 0 && nnz >= 0 && row_ptr, "bad CSR arrays");
    need(row_ptr[0] == 0 && row_ptr[m] == nnz, "row_ptr does not span nnz");
    auto h = std::make_unique<knnx_csr>();
    h->a.n_rows = m;
    h->a.n_cols = n;
    h->a.row_ptr.assign(row_ptr, row_ptr + m + 1);
    h->a.cols.assign(cols, cols + nnz);
    if (vals) h->a.vals.assign(vals, vals + nnz);
    for (int32_t i = 0; i < m; ++i)
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        if (cols[e] < 0 || cols[e] >= n)
          throw knnx::error(knnx::errc::out_of_bounds, "column out of range");
        if (e > row_ptr[i] && cols[e - 1] >= cols[e])
          throw knnx::error(knnx::errc::duplicate_entry, "row not strictly ascending");
      }
    *out = h.release();
  });
}
int knnx_csr_symmetrize(knnx_csr_t a, knnx_csr_t* out) {
  return guard([&] {
    need(a && out, "null handle");
    auto h = std::make_unique<knnx_csr>();
    h->a = knnx::symmetrize(a->a);
    *out = h.release();
  });
}
int knnx_csr_symmetrize_values(knnx_csr_t a, double scale, knnx_csr_t* out) {
  return guard([&] {
    need(a && out, "null handle");
    auto h = std::make_unique<knnx_csr>();
    h->a = knnx::symmetrize_values(a->a, scale);
    *out = h.release();
  });
}
int knnx_csr_row_normalize(knnx_csr_t a) {
  return guard([&] {
    need(a != nullptr && !a->a.vals.empty(), "row_normalize needs stored values");
    for (int32_t i = 0; i < a->a.n_rows; ++i) {
      double s = 0.0;
      for (int64_t e = a->a.row_ptr[i]; e < a->a.row_ptr[i + 1]; ++e) s += a->a.vals[e];
      if (s > 0.0)
        for (int64_t e = a->a.row_ptr[i]; e < a->a.row_ptr[i + 1]; ++e)
          a->a.vals[e] = static_cast<float>(a->a.vals[e] / s);
    }
  });
}
int knnx_csr_permute(knnx_csr_t a, const int32_t* forward, knnx_csr_t* out) {
  return guard([&] {
    need(a && forward && out, "null argument");
    if (a->a.n_rows != a->a.n_cols) throw knnx::error(knnx::errc::not_square, "permute needs a square matrix");
    std::vector<int32_t> f(forward, forward + a->a.n_rows);
    auto h = std::make_unique<knnx_csr>();
    h->a = knnx::permute(a->a, f, f);
    *out = h.release();
  });
}
int knnx_csr_locality_schedule(knnx_csr_t a, int32_t col_base, int32_t* out) {
  return guard([&] {
    need(a && (out || a->a.n_rows == 0), "null argument");
    const std::vector<int32_t> s = knnx::locality_schedule(a->a, col_base);
    std::copy(s.begin(), s.end(), out);
  });
}

int knnx_csr_row_block(knnx_csr_t a, int32_t r0, int32_t r1, knnx_csr_t* out) {
  return guard([&] {
    need(a && out && r0 >= 0 && r0 <= r1 && r1 <= a->a.n_rows, "bad row range");
    auto h = std::make_unique<knnx_csr>();
    const knnx::Csr& s = a->a;
    h->a.n_rows = r1 - r0;
    h->a.n_cols = s.n_cols;
    h->a.row_ptr.resize(static_cast<size_t>(r1 - r0) + 1);
    for (int32_t i = r0; i <= r1; ++i) h->a.row_ptr[i - r0] = s.row_ptr[i] - s.row_ptr[r0];
    h->a.cols.assign(s.cols.begin() + s.row_ptr[r0], s.cols.begin() + s.row_ptr[r1]);
    if (!s.vals.empty()) h->a.vals.assign(s.vals.begin() + s.row_ptr[r0], s.vals.begin() + s.row_ptr[r1]);
    *out = h.release();
  });
}
int knnx_csr_set_values(knnx_csr_t a, const float* vals) {
  return guard([&] {
    need(a != nullptr, "null handle");
    if (!vals) {
      a->a.vals.clear();
      return;
    }
    a->a.vals.assign(vals, vals + a->a.nnz());
  });
}
int knnx_csr_shape(knnx_csr_t a, int32_t* m, int32_t* n, int64_t* nnz, int32_t* has_values) {
  return guard([&] {
    need(a != nullptr, "null handle");
    *m = a->a.n_rows;
    *n = a->a.n_cols;
    *nnz = a->a.nnz();
    *has_values = a->a.vals.empty() ? 0 : 1;
  });
}
int knnx_csr_export(knnx_csr_t a, int64_t* row_ptr, int32_t* cols, float* vals) {
  return guard([&] {
    need(a != nullptr, "null handle");
    if (row_ptr) std::copy(a->a.row_ptr.begin(), a->a.row_ptr.end(), row_ptr);
    if (cols) std::copy(a->a.cols.begin(), a->a.cols.end(), cols);
    if (vals && !a->a.vals.empty()) std::copy(a->a.vals.begin(), a->a.vals.end(), vals);
  });
}
void knnx_csr_destroy(knnx_csr_t a) { delete a; }

int knnx_order_tree(const double* pts, int32_t n, int32_t dim, int32_t d, int32_t leaf_capacity,
                    int32_t max_depth, int32_t pca_device, knnx_tree_t* out,
                    double* captured_ratio, int32_t* pca_iterations) {
  return guard([&] {
    need(pts && out, "null argument");
    auto h = std::make_unique<knnx_tree>();
    double ratio = 1.0;
    if (dim <= d) {
      h->t = knnx::build_tree(pts, n, dim, leaf_capacity, max_depth);
      if (pca_iterations) *pca_iterations = 0;
    } else {
      const knnx::Embedding e =
          knnx::fit_pca(pts, n, dim, d, 1e-9, 1000, 1, covariance_factory(pca_device));
      double s = 0.0;
      for (double sv : e.singular_values) s += sv * sv;
      ratio = std::clamp(s / e.total_sq_norm, 0.0, 1.0);
      const std::vector<double> emb = e.projected.empty() ? knnx::project(pts, n, dim, e) : e.projected;
      h->t = (pca_device >= 0 && max_depth <= 21)
                 ? knnx_dev::build_tree_device(emb.data(), n, d, leaf_capacity, max_depth, pca_device)
                 : knnx::build_tree(emb.data(), n, d, leaf_capacity, max_depth);
      if (pca_iterations) *pca_iterations = e.iterations;
    }
    if (captured_ratio) *captured_ratio = ratio;
    *out = h.release();
  });
}
int knnx_tree_build_dev(const double* emb, int32_t n, int32_t dim, int32_t leaf_capacity,
                        int32_t max_depth, int32_t device, knnx_tree_t* out) {
  return guard([&] {
    need(emb && out, "null argument");
    auto h = std::make_unique<knnx_tree>();
    h->t = knnx_dev::build_tree_device(emb, n, dim, leaf_capacity, max_depth, device);
    *out = h.release();
  });
}
int knnx_tree_build(const double* emb, int32_t n, int32_t dim, int32_t leaf_capacity,
                    int32_t max_depth, knnx_tree_t* out) {
  return guard([&] {
    need(emb && out, "null argument");
    auto h = std::make_unique<knnx_tree>();
    h->t = knnx::build_tree(emb, n, dim, leaf_capacity, max_depth);
    *out = h.release();
  });
}
int knnx_tree_info(knnx_tree_t t, int32_t* n_nodes, int32_t* depth, int32_t* n_points) {
  return guard([&] {
    need(t != nullptr, "null handle");
    *n_nodes = static_cast<int32_t>(t->t.nodes.size());
    *depth = t->t.depth();
    *n_points = t->t.n_points;
  });
}
int knnx_tree_forward(knnx_tree_t t, int32_t* forward) {
  return guard([&] {
    need(t && forward, "null argument");
    std::copy(t->t.forward.begin(), t->t.forward.end(), forward);
  });
}
int knnx_tree_nodes(knnx_tree_t t, int32_t* begin, int32_t* end, int32_t* depth, int32_t* parent,
                    int32_t* is_leaf) {
  return guard([&] {
    need(t != nullptr, "null handle");
    for (size_t i = 0; i < t->t.nodes.size(); ++i) {
      const knnx::TreeNode& nd = t->t.nodes[i];
      begin[i] = nd.begin;
      end[i] = nd.end;
      depth[i] = nd.depth;
      parent[i] = nd.parent;
      is_leaf[i] = nd.is_leaf ? 1 : 0;
    }
  });
}
int knnx_tree_level_blocking(knnx_tree_t t, int32_t level, int32_t* offsets, int32_t* count) {
  return guard([&] {
    need(t && offsets && count, "null argument");
    const std::vector<int32_t> o = knnx::level_blocking(t->t, level);
    std::copy(o.begin(), o.end(), offsets);
    *count = static_cast<int32_t>(o.size());
  });
}
void knnx_tree_destroy(knnx_tree_t t) { delete t; }

int knnx_fit_pca(const double* pts, int32_t n, int32_t dim, int32_t d, int32_t pca_device,
                 double* mean, double* axes, double* singular_values, int32_t* iterations,
                 int32_t* converged, double* projected) {
  return guard([&] {
    need(pts != nullptr, "null points");
    const knnx::Embedding e =
        knnx::fit_pca(pts, n, dim, d, 1e-9, 1000, 1, covariance_factory(pca_device));
    if (mean) std::copy(e.mean.begin(), e.mean.end(), mean);
    if (axes) std::copy(e.axes.begin(), e.axes.end(), axes);
    if (singular_values) std::copy(e.singular_values.begin(), e.singular_values.end(), singular_values);
    if (iterations) *iterations = e.iterations;
    if (converged) *converged = e.converged ? 1 : 0;
    if (projected) {
      const std::vector<double> p = e.projected.empty() ? knnx::project(pts, n, dim, e) : e.projected;
      std::copy(p.begin(), p.end(), projected);
    }
  });
}

}  // extern "C"
