// Host-side C++ of the B200 kNN-interaction framework: the ☆ rows of
// SURVEY.md §2 that stay on the CPU (bit-exact ordering, input formats) and
// the inputs generators.  Everything here is deterministic; the ordering code
// restates the reference algorithm operation by operation so the permutation
// is bit-identical to patchord's (checked against the reference library in
// tests/test_host_ordering.py).  Compiled with -ffp-contract=off and without
// -march, like the reference's canonical build.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace knnx {

using index_t = std::int32_t;

// Error codes mirror patchord::errc (proj/include/patchord/core.hpp:15-42);
// the C ABI returns 1 + ordinal.
enum class errc : int {
  out_of_bounds,
  duplicate_entry,
  size_mismatch,
  dim_mismatch,
  k_too_large,
  not_square,
  non_positive_bandwidth,
  degenerate_data,
  dim_too_high,
  level_out_of_range,
  empty_pattern,
  too_large,
  not_divisible,
  too_wide,
  too_many,
  span_mismatch,
  local_index_overflow,
  ordering_mismatch,
  non_finite_value,
  zero_weight,
  malformed_record,
  inconsistent_dim,
  empty_file,
  io_error,
  checksum_mismatch,
  invalid_argument,
  // beyond the reference's set
  cuda_error = 64,
  unsupported = 65,
};

const char* errc_name(errc c);

class error : public std::runtime_error {
 public:
  error(errc code, const std::string& msg)
      : std::runtime_error(std::string(errc_name(code)) + ": " + msg), code_(code) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

// Deterministic generator: std::mt19937_64 (standard-specified, so identical
// across libraries) with the reference's hand-rolled transforms
// (proj/include/patchord/core.hpp:124-149, proj/src/core.cpp:186-199).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t next() { return eng_(); }
  double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t bounded(std::uint64_t n) { return next() % n; }
  double normal();
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[bounded(i)]);
  }

 private:
  std::mt19937_64 eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ---- synthetic workloads (BASELINE.json configs) ----
// Points are generated in double from Rng and rounded to fp32 (the GPU's
// storage type); the oracle receives the same fp32 values widened.
// C1: 64-component mixture, means U[-10,10]^dim, sigma 1, point p in cluster p mod 64.
std::vector<float> gen_mixture_c1(index_t n, index_t dim, index_t n_clusters, double sigma,
                                  std::uint64_t seed);
// C2/C3: 3-level mixture (16 x 16 x 16 clusters, scales 10/2/0.5, point noise
// `noise`); every point picks a uniformly random leaf cluster.
std::vector<float> gen_mixture_3level(index_t n, index_t dim, double noise, std::uint64_t seed);
// C5: 2-level mixture, n_top x n_sub clusters, anisotropic: per top cluster a
// random rotation of diag(sqrt(lambda)), lambda log-uniform [0.01, 1].
std::vector<float> gen_mixture_aniso(index_t n, index_t dim, index_t n_top, index_t n_sub,
                                     std::uint64_t seed);
std::vector<float> gen_uniform01(std::int64_t n, std::uint64_t seed);
std::vector<float> gen_normal(std::int64_t n, double sigma, std::uint64_t seed);

// ---- PCA (restates proj/src/pca.cpp:133-282 operation by operation) ----
struct Embedding {
  index_t dim_in = 0, dim_out = 0;
  std::vector<double> mean, axes, singular_values;
  double total_sq_norm = 0.0;
  bool converged = false;
  index_t iterations = 0;
  // n x dim_out projection of the fitted points, filled when fit_pca ran with a
  // device covariance hook (the same sums as project(), row by row, on the
  // centred copy the device already holds); empty otherwise
  std::vector<double> projected;
};

// Covariance action hook: out(D x p) = Xc^T (Xc in) with the reference's
// summation order.  The default runs on the host; the GPU library installs a
// bit-exact device version (knnx_pca_device in the C ABI).
struct CovarianceOp {
  virtual ~CovarianceOp() = default;
  // b (n x p) = Xc in, out (D x p) = Xc^T b
  virtual void apply(const std::vector<double>& in, std::vector<double>& out, index_t p) = 0;
  // b (n x p) = Xc v only
  virtual void xv(const std::vector<double>& v, std::vector<double>& b, index_t p) = 0;
};

Embedding fit_pca(const double* pts, index_t n, index_t dim, index_t d, double tol = 1e-9,
                  index_t max_iter = 1000, std::uint64_t seed = 1,
                  std::function<CovarianceOp*(const std::vector<double>& xc, index_t n,
                                              index_t dim)> make_op = nullptr);
std::vector<double> project(const double* pts, index_t n, index_t dim, const Embedding& e);

// ---- partition tree (restates proj/src/tree.cpp:15-124) ----
struct TreeNode {
  std::array<double, 3> lo{}, hi{};
  index_t begin = 0, end = 0, depth = 0, parent = -1;
  bool is_leaf = false;
  std::vector<index_t> children;
};
struct PartitionTree {
  index_t dim = 0, leaf_capacity = 0, max_depth = 0, n_points = 0;
  std::vector<TreeNode> nodes;
  std::vector<index_t> forward;  // forward[original] = leaf-order position
  index_t depth() const;
};
PartitionTree build_tree(const double* emb, index_t n, index_t dim, index_t leaf_capacity,
                         index_t max_depth);
std::vector<index_t> level_blocking(const PartitionTree& t, index_t level);

// make_ordering for the tree schemes (proj/src/pipeline.cpp:91-129 with
// embed_points :40-45): PCA to d = 2|3 when dim > d, then the tree.
PartitionTree order_tree_scheme(const double* pts, index_t n, index_t dim, index_t d,
                                index_t leaf_capacity, index_t max_depth, double* captured_ratio,
                                std::function<CovarianceOp*(const std::vector<double>&, index_t,
                                                            index_t)> make_op = nullptr);

// ---- sparse formats ----
struct Csr {
  index_t n_rows = 0, n_cols = 0;
  std::vector<std::int64_t> row_ptr;
  std::vector<index_t> cols;
  std::vector<float> vals;  // empty for pattern-only matrices
  std::int64_t nnz() const { return static_cast<std::int64_t>(cols.size()); }
};
// kNN rows -> canonical CSR (pattern_from_knn, proj/src/knn.cpp:64-70: every
// row sorted by column)
Csr csr_from_knn(const index_t* ids, index_t m, index_t n, index_t k);
// structural union with the transpose (proj/src/knn.cpp:72-84)
Csr symmetrize(const Csr& a);
// union pattern with values scale * (a_ij + a_ji) (t-SNE P = (P_cond + P_cond^T) / 2N)
Csr symmetrize_values(const Csr& a, double scale);
// rows and columns renumbered by forward, each row re-sorted by column
// (proj/src/core.cpp:130-139 -> csr_from_coo :75-92); values follow
Csr permute(const Csr& a, const std::vector<index_t>& row_fwd, const std::vector<index_t>& col_fwd);

// Cluster-order tile format: rows cut into tiles
// of `tile_rows` consecutive rows; per tile the sorted unique source columns
// (halo) and, per entry, a 16-bit index into that halo; entries laid out
// slice-major (32 rows per slice, column-major inside a slice, padded to the
// slice's longest row with (halo 0, value 0)).
struct ClusterTiles {
  index_t n_rows = 0, n_cols = 0, tile_rows = 0, n_tiles = 0;
  std::int64_t nnz = 0, stored = 0;  // true and padded entry counts
  std::vector<std::int64_t> halo_off;  // n_tiles + 1
  std::vector<index_t> halo_ids;
  std::vector<std::int64_t> slice_off;  // n_slices + 1, offsets into lidx/vals
  std::vector<index_t> slice_len;       // n_slices: padded row length
  std::vector<index_t> row_len;         // n_rows: true row length, by slot
  std::vector<index_t> slot_row;        // slot -> row (empty: identity, uniform rows)
  std::vector<std::uint16_t> lidx;
  std::vector<float> vals;             // empty when the source has no values
  index_t max_halo = 0;
};
// schedule: optional row processing order (slot p holds row schedule[p]);
// null = tree order.  Results per row do not depend on it.
// with_halos = false (original order): SELL slices + values only, no per-tile
// halo / 16-bit local indices (and so no LocalIndexOverflow)
ClusterTiles build_cluster_tiles(const Csr& a, index_t tile_rows, const index_t* schedule = nullptr,
                                 bool with_halos = true);

// Graph-locality row schedule: breadth-first over the kNN graph (rows visited
// from the lowest unvisited row, neighbours in column order; column c is row
// c - col_base).  Rows that share sources end up adjacent, so their source
// reads hit L2 together even when the given ordering does not group them.
std::vector<index_t> locality_schedule(const Csr& a, index_t col_base);

// HBM1 dump of a HierBlockMatrix (proj/docs/hbm1-format.md): leaf payload in
// arena order with cluster offsets, plus both trees' leaf orders
struct Hbm1 {
  index_t n_rows = 0, n_cols = 0, cut_level = 0;
  std::int64_t nnz = 0;
  std::vector<index_t> row_offset, col_offset, row_forward, col_forward;
  std::vector<std::int64_t> block_ptr;  // leaf blocks + 1
  std::vector<std::uint16_t> lr, lc;
  std::vector<float> vals;
};
Hbm1 read_hbm1(const std::string& path);

// median of sqrt(d2) over all neighbor distances (BASELINE bandwidth rule)
double median_distance(const float* d2, std::int64_t count);

}  // namespace knnx
