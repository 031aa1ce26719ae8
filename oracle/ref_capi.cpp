// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" veneer over the UNMODIFIED reference library (patchord,
// /root/reference/proj/src/*.cpp), so the pytest suite and bench.py's CPU
// baseline can call the reference itself through ctypes.  Nothing here is
// product code: the product path (paper_1709_03671_b200/) never links it.
// Built by oracle/Makefile into oracle/_ref/libpatchord_ref.so together with
// the reference sources, compiled where they lie (never copied).
//
// Every entry point returns 0 on success, or 1 + (int)patchord::errc on a
// reference error (the message is kept for ref_last_error()), or -1 on any
// other exception.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "patchord/core.hpp"
#include "patchord/hier.hpp"
#include "patchord/kernels.hpp"
#include "patchord/knn.hpp"
#include "patchord/orderings.hpp"
#include "patchord/pca.hpp"
#include "patchord/pipeline.hpp"
#include "patchord/synth.hpp"
#include "patchord/tree.hpp"

using namespace patchord;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

PointSet points_from(const double* p, index_t n, index_t d) {
  return make_point_set(n, d, std::vector<double>(p, p + static_cast<std::size_t>(n) * d));
}

SparseMatrix matrix_from(index_t n_rows, index_t n_cols, std::int64_t nnz, const std::int32_t* rows,
                         const std::int32_t* cols, const double* vals) {
  std::vector<std::tuple<index_t, index_t, double>> e;
  e.reserve(static_cast<std::size_t>(nnz));
  for (std::int64_t q = 0; q < nnz; ++q) e.emplace_back(rows[q], cols[q], vals ? vals[q] : 1.0);
  return csr_from_coo(e, n_rows, n_cols);
}

struct RefHier {
  HierBlockMatrix h;
};

struct RefTree {
  PartitionTree t;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- Rng streams (proj/include/patchord/core.hpp:124-149) ----
int ref_rng_u64(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
  return guard([&] {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.next();
  });
}
int ref_rng_uniform01(std::uint64_t seed, std::int64_t n, double* out) {
  return guard([&] {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.uniform01();
  });
}
int ref_rng_normal(std::uint64_t seed, std::int64_t n, double* out) {
  return guard([&] {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.normal();
  });
}
int ref_rng_bounded(std::uint64_t seed, std::uint64_t bound, std::int64_t n, std::uint64_t* out) {
  return guard([&] {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.bounded(bound);
  });
}
int ref_order_scattered(std::int32_t n, std::uint64_t seed, std::int32_t* forward) {
  return guard([&] {
    const Permutation p = order_scattered(n, seed);
    std::copy(p.forward.begin(), p.forward.end(), forward);
  });
}

// ---- generators (proj/src/synth.cpp:60-74) ----
int ref_gen_gaussian_mixture(std::int32_t n, std::int32_t dim, std::int32_t n_clusters,
                             double spread, double sigma, std::uint64_t seed, double* out) {
  return guard([&] {
    const PointSet p = gen_gaussian_mixture(n, dim, n_clusters, spread, sigma, seed);
    std::copy(p.coords.begin(), p.coords.end(), out);
  });
}

// ---- kNN (proj/src/knn.cpp:9-62) ----
int ref_build_knn(const double* targets, std::int32_t m, const double* sources, std::int32_t n,
                  std::int32_t dim, std::int32_t k, int self_set, std::int32_t* ids,
                  double* dists) {
  return guard([&] {
    const PointSet t = points_from(targets, m, dim);
    KnnGraph g;
    if (self_set) {
      g = build_knn(t, t, k);
    } else {
      const PointSet s = points_from(sources, n, dim);
      g = build_knn(t, s, k);
    }
    std::copy(g.neighbor_ids.begin(), g.neighbor_ids.end(), ids);
    std::copy(g.neighbor_dists.begin(), g.neighbor_dists.end(), dists);
  });
}

// value at (i, j) = exp(-|t_i - s_j|^2 / (2 h^2))  (proj/src/knn.cpp:86-108)
int ref_gaussian_values(std::int32_t m, std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                        const std::int32_t* cols, const double* targets, const double* sources,
                        std::int32_t dim, double h, double* out_vals) {
  return guard([&] {
    std::vector<std::pair<index_t, index_t>> e(static_cast<std::size_t>(nnz));
    for (std::int64_t q = 0; q < nnz; ++q) e[q] = {rows[q], cols[q]};
    const SparsePattern p = make_pattern(m, n, std::move(e));
    const SparseMatrix v = gaussian_values(p, points_from(targets, m, dim),
                                           points_from(sources, n, dim), h);
    std::copy(v.values.begin(), v.values.end(), out_vals);
  });
}

// ---- stationary operator, original order (proj/src/kernels.cpp:37-49) ----
int ref_spmv_flat(std::int32_t m, std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                  const std::int32_t* cols, const double* vals, const double* x, double* y) {
  return guard([&] {
    const SparseMatrix a = matrix_from(m, n, nnz, rows, cols, vals);
    const PotentialVector out = spmv_flat(a, ChargeVector{std::vector<double>(x, x + n), ""});
    std::copy(out.values.begin(), out.values.end(), y);
  });
}

// Median-of-reps timing of spmv_flat, the bench_spmv method (proj/src/pipeline.cpp:296-312).
int ref_bench_spmv_flat(std::int32_t m, std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                        const std::int32_t* cols, const double* vals, const double* x,
                        std::int32_t reps, std::int64_t* times_ns, double* y) {
  return guard([&] {
    const SparseMatrix a = matrix_from(m, n, nnz, rows, cols, vals);
    const ChargeVector xv{std::vector<double>(x, x + n), ""};
    spmv_flat(a, xv);  // warm-up
    PotentialVector out;
    for (std::int32_t r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      out = spmv_flat(a, xv);
      times_ns[r] = std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - t0)
                        .count();
    }
    std::copy(out.values.begin(), out.values.end(), y);
  });
}

// ---- ordering (proj/src/pipeline.cpp:91-129) ----
int ref_make_ordering(const char* scheme, std::int32_t n, std::int32_t dim, const double* pts,
                      std::int32_t leaf_capacity, std::int32_t max_depth, std::uint64_t seed,
                      std::int32_t* forward, double* captured_ratio) {
  return guard([&] {
    SparsePattern p;
    p.n_rows = p.n_cols = n;
    const OrderingResult r = make_ordering(scheme, p, points_from(pts, n, dim), 32, leaf_capacity,
                                           max_depth, seed, captured_ratio);
    std::copy(r.row_perm.forward.begin(), r.row_perm.forward.end(), forward);
  });
}

int ref_fit_pca(const double* pts, std::int32_t n, std::int32_t dim, std::int32_t d,
                double* mean, double* axes, double* singular_values, std::int32_t* iterations,
                int* converged, double* projected) {
  return guard([&] {
    const PointSet ps = points_from(pts, n, dim);
    const Embedding e = fit_pca(ps, d);
    std::copy(e.mean.begin(), e.mean.end(), mean);
    std::copy(e.axes.begin(), e.axes.end(), axes);
    std::copy(e.singular_values.begin(), e.singular_values.end(), singular_values);
    *iterations = e.iterations;
    *converged = e.converged ? 1 : 0;
    if (projected) {
      const PointSet pr = project(ps, e);
      std::copy(pr.coords.begin(), pr.coords.end(), projected);
    }
  });
}

int ref_tree_create(const double* emb, std::int32_t n, std::int32_t dim,
                    std::int32_t leaf_capacity, std::int32_t max_depth, void** out) {
  return guard([&] {
    auto t = std::make_unique<RefTree>();
    t->t = build_tree(points_from(emb, n, dim), leaf_capacity, max_depth);
    *out = t.release();
  });
}
void ref_tree_destroy(void* t) { delete static_cast<RefTree*>(t); }
std::int32_t ref_tree_n_nodes(void* t) {
  return static_cast<std::int32_t>(static_cast<RefTree*>(t)->t.nodes.size());
}
std::int32_t ref_tree_depth(void* t) { return static_cast<RefTree*>(t)->t.depth(); }
// per node: begin, end, depth, parent, is_leaf, n_children; lo/hi (3 doubles each)
int ref_tree_nodes(void* tp, std::int32_t* begin, std::int32_t* end, std::int32_t* depth,
                   std::int32_t* parent, std::int32_t* is_leaf, double* lo, double* hi) {
  return guard([&] {
    const PartitionTree& t = static_cast<RefTree*>(tp)->t;
    for (std::size_t i = 0; i < t.nodes.size(); ++i) {
      const TreeNode& nd = t.nodes[i];
      begin[i] = nd.begin;
      end[i] = nd.end;
      depth[i] = nd.depth;
      parent[i] = nd.parent;
      is_leaf[i] = nd.is_leaf ? 1 : 0;
      for (int a = 0; a < 3; ++a) {
        lo[3 * i + a] = nd.lo[a];
        hi[3 * i + a] = nd.hi[a];
      }
    }
  });
}
int ref_tree_forward(void* tp, std::int32_t* forward) {
  return guard([&] {
    const PartitionTree& t = static_cast<RefTree*>(tp)->t;
    std::copy(t.leaf_order.forward.begin(), t.leaf_order.forward.end(), forward);
  });
}
// offsets has room for n_nodes + 1 entries; returns the count through *count
int ref_tree_level_blocking(void* tp, std::int32_t level, std::int32_t* offsets,
                            std::int32_t* count) {
  return guard([&] {
    const std::vector<index_t> o = level_blocking(static_cast<RefTree*>(tp)->t, level);
    std::copy(o.begin(), o.end(), offsets);
    *count = static_cast<std::int32_t>(o.size());
  });
}

int ref_permute_points(const double* pts, std::int32_t n, std::int32_t dim,
                       const std::int32_t* forward, double* out) {
  return guard([&] {
    const PointSet moved =
        permute(points_from(pts, n, dim), make_permutation(std::vector<index_t>(forward, forward + n)));
    std::copy(moved.coords.begin(), moved.coords.end(), out);
  });
}

// COO (any order) -> canonical permuted COO (proj/src/core.cpp:130-139)
int ref_permute_matrix(std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                       const std::int32_t* cols, const double* vals, const std::int32_t* forward,
                       std::int32_t* out_rows, std::int32_t* out_cols, double* out_vals) {
  return guard([&] {
    const SparseMatrix a = matrix_from(n, n, nnz, rows, cols, vals);
    const Permutation p = make_permutation(std::vector<index_t>(forward, forward + n));
    const SparseMatrix b = permute(a, p, p);
    for (std::size_t e = 0; e < b.values.size(); ++e) {
      out_rows[e] = b.pattern.entries[e].first;
      out_cols[e] = b.pattern.entries[e].second;
      out_vals[e] = b.values[e];
    }
  });
}

int ref_symmetrize(std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                   const std::int32_t* cols, std::int64_t* out_nnz, std::int32_t* out_rows,
                   std::int32_t* out_cols) {
  return guard([&] {
    std::vector<std::pair<index_t, index_t>> e(static_cast<std::size_t>(nnz));
    for (std::int64_t q = 0; q < nnz; ++q) e[q] = {rows[q], cols[q]};
    const SparsePattern s = symmetrize(make_pattern(n, n, std::move(e)));
    *out_nnz = s.nnz();
    if (out_rows)
      for (std::size_t q = 0; q < s.entries.size(); ++q) {
        out_rows[q] = s.entries[q].first;
        out_cols[q] = s.entries[q].second;
      }
  });
}

// ---- blocked operator, cluster order (proj/src/hier.cpp:40-163, kernels.cpp:51-136) ----
// The matrix is given in ORIGINAL order with an embedded point set; the tree
// is built over the embedding, the matrix permuted into its leaf order and
// blocked at cut_level (-1 = auto).  forward receives the leaf order.
int ref_hier_create(std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                    const std::int32_t* cols, const double* vals, const double* emb,
                    std::int32_t emb_dim, std::int32_t leaf_capacity, std::int32_t max_depth,
                    std::int32_t cut_level, std::int32_t* forward, void** out) {
  return guard([&] {
    const SparseMatrix a = matrix_from(n, n, nnz, rows, cols, vals);
    const OrderingResult ord = order_tree(points_from(emb, n, emb_dim), leaf_capacity, max_depth);
    const SparseMatrix ap = permute(a, ord.row_perm, ord.col_perm);
    auto h = std::make_unique<RefHier>();
    h->h = build_hier(ap, ord.row_tree, ord.col_tree, cut_level);
    h->h.row_tag = h->h.col_tag = ord.scheme;
    if (forward) std::copy(ord.row_perm.forward.begin(), ord.row_perm.forward.end(), forward);
    *out = h.release();
  });
}

// Already-permuted matrix under caller-supplied single-cluster trees (build_hier_flat).
int ref_hier_create_flat(std::int32_t m, std::int32_t n, std::int64_t nnz, const std::int32_t* rows,
                         const std::int32_t* cols, const double* vals, void** out) {
  return guard([&] {
    auto h = std::make_unique<RefHier>();
    h->h = build_hier_flat(matrix_from(m, n, nnz, rows, cols, vals));
    *out = h.release();
  });
}

void ref_hier_destroy(void* h) { delete static_cast<RefHier*>(h); }

// dump_hbm1 (proj/src/hier.cpp:291-323)
int ref_hier_dump(void* hp, const char* path) {
  return guard([&] { dump_hbm1(static_cast<RefHier*>(hp)->h, path); });
}

int ref_hier_info(void* hp, std::int32_t* cut_level, std::int32_t* n_blocks,
                  std::int32_t* n_leaf_blocks, std::int32_t* n_top_blocks, std::int64_t* nnz) {
  return guard([&] {
    const HierBlockMatrix& h = static_cast<RefHier*>(hp)->h;
    *cut_level = h.cut_level;
    *n_blocks = static_cast<std::int32_t>(h.blocks.size());
    std::int32_t leaves = 0;
    for (const HierBlock& b : h.blocks) leaves += b.is_leaf ? 1 : 0;
    *n_leaf_blocks = leaves;
    *n_top_blocks = static_cast<std::int32_t>(h.top_blocks.size());
    *nnz = h.nnz;
  });
}

// canonical COO of the blocked matrix (proj/src/hier.cpp:182-191)
int ref_hier_flatten(void* hp, std::int32_t* rows, std::int32_t* cols, double* vals) {
  return guard([&] {
    const SparseMatrix f = flatten(static_cast<RefHier*>(hp)->h);
    for (std::size_t e = 0; e < f.values.size(); ++e) {
      rows[e] = f.pattern.entries[e].first;
      cols[e] = f.pattern.entries[e].second;
      vals[e] = f.values[e];
    }
  });
}

int ref_hier_spmv(void* hp, const double* x, double* y, std::int32_t workers) {
  return guard([&] {
    const HierBlockMatrix& h = static_cast<RefHier*>(hp)->h;
    const ChargeVector xv{std::vector<double>(x, x + h.n_cols), ""};
    const PotentialVector out = workers <= 0 ? spmv_hier(h, xv) : spmv_hier_parallel(h, xv, workers);
    std::copy(out.values.begin(), out.values.end(), y);
  });
}

int ref_hier_bench(void* hp, const double* x, std::int32_t workers, std::int32_t reps,
                   std::int64_t* times_ns, double* y) {
  return guard([&] {
    const HierBlockMatrix& h = static_cast<RefHier*>(hp)->h;
    const ChargeVector xv{std::vector<double>(x, x + h.n_cols), ""};
    auto once = [&] { return workers <= 0 ? spmv_hier(h, xv) : spmv_hier_parallel(h, xv, workers); };
    once();  // warm-up
    PotentialVector out;
    for (std::int32_t r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      out = once();
      times_ns[r] = std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - t0)
                        .count();
    }
    std::copy(out.values.begin(), out.values.end(), y);
  });
}

// update_values with the Gaussian value model (proj/src/hier.cpp:203-222 with
// the knn.cpp:97-106 kernel); coordinates are in the matrix (tree) order.
int ref_hier_update_gaussian(void* hp, const double* targets, const double* sources,
                             std::int32_t dim, double h_bw, std::int32_t* updated) {
  return guard([&] {
    HierBlockMatrix& h = static_cast<RefHier*>(hp)->h;
    const double inv = 1.0 / (2.0 * h_bw * h_bw);
    const index_t cnt = update_values(h, [&](index_t i, index_t j, double) {
      const double* t = targets + static_cast<std::size_t>(i) * dim;
      const double* s = sources + static_cast<std::size_t>(j) * dim;
      double acc = 0.0;
      for (index_t d = 0; d < dim; ++d) {
        const double diff = t[d] - s[d];
        acc += diff * diff;
      }
      return std::exp(-acc * inv);
    });
    if (updated) *updated = cnt;
  });
}

// iterate_interactions with a Gaussian value_fn over K charge vectors
// (proj/src/kernels.cpp:217-228).  xs, ys: K x n_cols / K x n_rows.
int ref_hier_iterate_gaussian(void* hp, const double* targets, const double* sources,
                              std::int32_t dim, double h_bw, std::int32_t n_steps, const double* xs,
                              double* ys, std::int64_t* times_ns) {
  return guard([&] {
    HierBlockMatrix& h = static_cast<RefHier*>(hp)->h;
    const double inv = 1.0 / (2.0 * h_bw * h_bw);
    auto value_fn = [&](index_t) {
      return [&](index_t i, index_t j, double) {
        const double* t = targets + static_cast<std::size_t>(i) * dim;
        const double* s = sources + static_cast<std::size_t>(j) * dim;
        double acc = 0.0;
        for (index_t d = 0; d < dim; ++d) {
          const double diff = t[d] - s[d];
          acc += diff * diff;
        }
        return std::exp(-acc * inv);
      };
    };
    for (std::int32_t kappa = 0; kappa < n_steps; ++kappa) {
      const std::vector<ChargeVector> one{
          ChargeVector{std::vector<double>(xs + static_cast<std::size_t>(kappa) * h.n_cols,
                                           xs + static_cast<std::size_t>(kappa + 1) * h.n_cols),
                       ""}};
      const auto t0 = std::chrono::steady_clock::now();
      const auto out = iterate_interactions(
          h, [&](index_t) { return std::function<double(index_t, index_t, double)>(value_fn(kappa)); },
          one);
      if (times_ns)
        times_ns[kappa] = std::chrono::duration_cast<std::chrono::nanoseconds>(
                              std::chrono::steady_clock::now() - t0)
                              .count();
      std::copy(out[0].values.begin(), out[0].values.end(),
                ys + static_cast<std::size_t>(kappa) * h.n_rows);
    }
  });
}

// tsne_attractive_step (proj/src/kernels.cpp:103-136); mutates the stored
// affinities exactly like the reference.  Y, F: n x dim_out.
int ref_hier_tsne(void* hp, const double* y, std::int32_t dim_out, double* f) {
  return guard([&] {
    HierBlockMatrix& h = static_cast<RefHier*>(hp)->h;
    const PointSet yp = points_from(y, h.n_rows, dim_out);
    const PointSet out = tsne_attractive_step(h, yp, dim_out);
    std::copy(out.coords.begin(), out.coords.end(), f);
  });
}

// One meanshift_step (proj/src/kernels.cpp:184-215) over a caller-supplied
// kNN graph: the state is assembled directly and its refresh pushed past the
// step, so the reference's own step loop runs on exactly these neighbor rows.
int ref_meanshift_step(const double* sources, std::int32_t n_src, const double* targets,
                       std::int32_t n_tgt, std::int32_t dim, const std::int32_t* ids,
                       std::int32_t k, double bandwidth, double* targets_out) {
  return guard([&] {
    if (!(bandwidth > 0.0)) throw error(errc::non_positive_bandwidth, "bandwidth must be positive");
    MeanShiftState s;
    s.sources = points_from(sources, n_src, dim);
    s.targets = points_from(targets, n_tgt, dim);
    s.bandwidth = bandwidth;
    s.k = k;
    s.knn.k = k;
    s.knn.n_targets = n_tgt;
    s.knn.n_sources = n_src;
    s.knn.neighbor_ids.assign(ids, ids + static_cast<std::size_t>(n_tgt) * k);
    s.knn.neighbor_dists.assign(static_cast<std::size_t>(n_tgt) * k, 0.0);
    s.refresh_period = 1 << 30;
    s = meanshift_step(std::move(s));
    std::copy(s.targets.coords.begin(), s.targets.coords.end(), targets_out);
  });
}

// Times `reps` calls of the reference's meanshift_step on the same state
// (the state is copied outside the timed region; times_ns per call).
int ref_meanshift_bench(const double* sources, std::int32_t n_src, const double* targets,
                        std::int32_t n_tgt, std::int32_t dim, const std::int32_t* ids,
                        std::int32_t k, double bandwidth, std::int32_t reps,
                        std::int64_t* times_ns) {
  return guard([&] {
    MeanShiftState s0;
    s0.sources = points_from(sources, n_src, dim);
    s0.targets = points_from(targets, n_tgt, dim);
    s0.bandwidth = bandwidth;
    s0.k = k;
    s0.knn.k = k;
    s0.knn.n_targets = n_tgt;
    s0.knn.n_sources = n_src;
    s0.knn.neighbor_ids.assign(ids, ids + static_cast<std::size_t>(n_tgt) * k);
    s0.knn.neighbor_dists.assign(static_cast<std::size_t>(n_tgt) * k, 0.0);
    s0.refresh_period = 1 << 30;
    for (std::int32_t r = 0; r < reps; ++r) {
      MeanShiftState s = s0;
      const auto t0 = std::chrono::steady_clock::now();
      s = meanshift_step(std::move(s));
      const auto t1 = std::chrono::steady_clock::now();
      times_ns[r] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    }
  });
}

// meanshift_init + steps exactly as the reference runs them (kNN built by the
// reference, refresh every refresh_period).  targets_out: final positions.
int ref_meanshift_run(const double* sources, std::int32_t n_src, const double* targets,
                      std::int32_t n_tgt, std::int32_t dim, std::int32_t k, double bandwidth,
                      std::int32_t refresh_period, std::int32_t steps, double* targets_out,
                      std::int32_t* ids_out) {
  return guard([&] {
    MeanShiftState s = meanshift_init(points_from(sources, n_src, dim),
                                      points_from(targets, n_tgt, dim), bandwidth, k,
                                      refresh_period, false);
    if (ids_out && steps == 0)
      std::copy(s.knn.neighbor_ids.begin(), s.knn.neighbor_ids.end(), ids_out);
    for (std::int32_t q = 0; q < steps; ++q) {
      if (ids_out && q == steps - 1)
        std::copy(s.knn.neighbor_ids.begin(), s.knn.neighbor_ids.end(), ids_out);
      s = meanshift_step(std::move(s));
    }
    std::copy(s.targets.coords.begin(), s.targets.coords.end(), targets_out);
  });
}

// machine_descriptor (proj/src/pipeline.cpp:75-89): "<cpu model>, <n> hardware threads"
int ref_machine_descriptor(char* buf, std::int32_t len) {
  return guard([&] {
    const std::string d = machine_descriptor();
    if (len > 0) {
      const std::size_t n = std::min<std::size_t>(d.size(), static_cast<std::size_t>(len - 1));
      std::memcpy(buf, d.data(), n);
      buf[n] = 0;
    }
  });
}

std::int32_t ref_hardware_threads() {
  return static_cast<std::int32_t>(std::thread::hardware_concurrency());
}

}  // extern "C"
