// Bit-exact ordering: PCA by blocked subspace iteration (restating
// proj/src/pca.cpp:14-282) and the adaptive 2^d partition tree (restating
// proj/src/tree.cpp:15-124).  Operation order and rounding match the
// reference's canonical build (separate multiply / add, no contraction), so the
// resulting permutation is bit-identical; tests/test_host_ordering.py checks it
// against the reference library itself.
#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>

#include "host.hpp"

namespace knnx {

namespace {

// cyclic Jacobi (pca.cpp:14-62)
void jacobi_eig(std::vector<double> a, index_t p, std::vector<double>& evals,
                std::vector<double>& evecs) {
  std::vector<double> v(static_cast<std::size_t>(p) * p, 0.0);
  for (index_t i = 0; i < p; ++i) v[i * p + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (index_t i = 0; i < p; ++i)
      for (index_t j = 0; j < p; ++j) {
        const double sq = a[i * p + j] * a[i * p + j];
        if (i == j) diag += sq; else off += sq;
      }
    if (off <= 1e-30 * (diag + 1e-300)) break;
    for (index_t i = 0; i < p - 1; ++i)
      for (index_t j = i + 1; j < p; ++j) {
        const double apq = a[i * p + j];
        if (apq == 0.0) continue;
        const double theta = (a[j * p + j] - a[i * p + i]) / (2.0 * apq);
        const double t =
            (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        for (index_t r = 0; r < p; ++r) {
          const double ari = a[r * p + i], arj = a[r * p + j];
          a[r * p + i] = c * ari - s * arj;
          a[r * p + j] = s * ari + c * arj;
        }
        for (index_t r = 0; r < p; ++r) {
          const double air = a[i * p + r], ajr = a[j * p + r];
          a[i * p + r] = c * air - s * ajr;
          a[j * p + r] = s * air + c * ajr;
        }
        for (index_t r = 0; r < p; ++r) {
          const double vri = v[r * p + i], vrj = v[r * p + j];
          v[r * p + i] = c * vri - s * vrj;
          v[r * p + j] = s * vri + c * vrj;
        }
      }
  }
  std::vector<index_t> rank(p);
  std::iota(rank.begin(), rank.end(), 0);
  std::stable_sort(rank.begin(), rank.end(),
                   [&](index_t x, index_t y) { return a[x * p + x] > a[y * p + y]; });
  evals.resize(p);
  evecs.assign(static_cast<std::size_t>(p) * p, 0.0);
  for (index_t o = 0; o < p; ++o) {
    evals[o] = a[rank[o] * p + rank[o]];
    for (index_t r = 0; r < p; ++r) evecs[r * p + o] = v[r * p + rank[o]];
  }
}

// two-pass modified Gram-Schmidt with rng refill (pca.cpp:70-98)
void orthonormalize(std::vector<double>& m, index_t dim, index_t p, Rng& rng) {
  for (index_t a = 0; a < p; ++a) {
    for (int attempt = 0; attempt < 8; ++attempt) {
      double norm0 = 0.0;
      for (index_t r = 0; r < dim; ++r) norm0 += m[r * p + a] * m[r * p + a];
      norm0 = std::sqrt(norm0);
      double norm = 0.0;
      if (norm0 > 0.0) {
        for (int pass = 0; pass < 2; ++pass)
          for (index_t b = 0; b < a; ++b) {
            double dot = 0.0;
            for (index_t r = 0; r < dim; ++r) dot += m[r * p + a] * m[r * p + b];
            for (index_t r = 0; r < dim; ++r) m[r * p + a] -= dot * m[r * p + b];
          }
        for (index_t r = 0; r < dim; ++r) norm += m[r * p + a] * m[r * p + a];
        norm = std::sqrt(norm);
      }
      if (norm > 1e-12 * norm0 && norm > 1e-150) {
        for (index_t r = 0; r < dim; ++r) m[r * p + a] /= norm;
        break;
      }
      for (index_t r = 0; r < dim; ++r) m[r * p + a] = rng.normal();
    }
  }
}

// smallest singular value of the d x d cross-Gramian (pca.cpp:102-120)
double min_cross_singular(const std::vector<double>& u, const std::vector<double>& w, index_t dim,
                          index_t p, index_t d) {
  std::vector<double> g(static_cast<std::size_t>(d) * d, 0.0);
  for (index_t a = 0; a < d; ++a)
    for (index_t b = 0; b < d; ++b) {
      double dot = 0.0;
      for (index_t r = 0; r < dim; ++r) dot += u[r * p + a] * w[r * p + b];
      g[a * d + b] = dot;
    }
  std::vector<double> gtg(static_cast<std::size_t>(d) * d, 0.0);
  for (index_t a = 0; a < d; ++a)
    for (index_t b = 0; b < d; ++b) {
      double dot = 0.0;
      for (index_t r = 0; r < d; ++r) dot += g[r * d + a] * g[r * d + b];
      gtg[a * d + b] = dot;
    }
  std::vector<double> evals, evecs;
  jacobi_eig(gtg, d, evals, evecs);
  return std::sqrt(std::max(0.0, evals[d - 1]));
}

void fix_axis_signs(Embedding& e) {
  for (index_t a = 0; a < e.dim_out; ++a) {
    double* ax = e.axes.data() + static_cast<std::size_t>(a) * e.dim_in;
    index_t arg = 0;
    for (index_t r = 1; r < e.dim_in; ++r)
      if (std::abs(ax[r]) > std::abs(ax[arg])) arg = r;
    if (ax[arg] < 0.0)
      for (index_t r = 0; r < e.dim_in; ++r) ax[r] = -ax[r];
  }
}

// host covariance action with the reference's loop order (pca.cpp:194-216)
class HostCovariance final : public CovarianceOp {
 public:
  HostCovariance(const std::vector<double>& xc, index_t n, index_t dim) : xc_(xc), n_(n), dim_(dim) {}
  void xv(const std::vector<double>& v, std::vector<double>& b, index_t p) override {
    b.assign(static_cast<std::size_t>(n_) * p, 0.0);
    for (index_t i = 0; i < n_; ++i) {
      const double* row = xc_.data() + static_cast<std::size_t>(i) * dim_;
      double* bi = b.data() + static_cast<std::size_t>(i) * p;
      for (index_t r = 0; r < dim_; ++r) {
        const double x = row[r];
        const double* vr = v.data() + static_cast<std::size_t>(r) * p;
        for (index_t a = 0; a < p; ++a) bi[a] += x * vr[a];
      }
    }
  }
  void apply(const std::vector<double>& in, std::vector<double>& out, index_t p) override {
    xv(in, b_, p);
    out.assign(static_cast<std::size_t>(dim_) * p, 0.0);
    for (index_t i = 0; i < n_; ++i) {
      const double* row = xc_.data() + static_cast<std::size_t>(i) * dim_;
      const double* bi = b_.data() + static_cast<std::size_t>(i) * p;
      for (index_t r = 0; r < dim_; ++r) {
        double* wr = out.data() + static_cast<std::size_t>(r) * p;
        const double x = row[r];
        for (index_t a = 0; a < p; ++a) wr[a] += x * bi[a];
      }
    }
  }

 private:
  const std::vector<double>& xc_;
  index_t n_, dim_;
  std::vector<double> b_;
};

}  // namespace

Embedding fit_pca(const double* pts, index_t n, index_t D, index_t d, double tol, index_t max_iter,
                  std::uint64_t seed,
                  std::function<CovarianceOp*(const std::vector<double>&, index_t, index_t)> make_op) {
  if (d < 1 || d > std::min(D, n))
    throw error(errc::invalid_argument, "d must be in [1, min(dim, n_points)]");
  if (!(tol > 0.0)) throw error(errc::invalid_argument, "tol must be positive");
  Embedding e;
  e.dim_in = D;
  e.dim_out = d;
  e.mean.assign(D, 0.0);
  for (index_t i = 0; i < n; ++i) {
    const double* x = pts + static_cast<std::size_t>(i) * D;
    for (index_t r = 0; r < D; ++r) e.mean[r] += x[r];
  }
  for (index_t r = 0; r < D; ++r) e.mean[r] /= static_cast<double>(n);

  std::vector<double> xc(static_cast<std::size_t>(n) * D);
  double total = 0.0;
  for (index_t i = 0; i < n; ++i) {
    const double* x = pts + static_cast<std::size_t>(i) * D;
    double* row = xc.data() + static_cast<std::size_t>(i) * D;
    for (index_t r = 0; r < D; ++r) {
      row[r] = x[r] - e.mean[r];
      total += row[r] * row[r];
    }
  }
  e.total_sq_norm = total;
  if (total == 0.0) throw error(errc::degenerate_data, "all points identical; axes undefined");

  if (d == D) {  // exact identity-minus-centering case (pca.cpp:160-180)
    std::vector<double> colsq(D, 0.0);
    for (index_t i = 0; i < n; ++i) {
      const double* row = xc.data() + static_cast<std::size_t>(i) * D;
      for (index_t r = 0; r < D; ++r) colsq[r] += row[r] * row[r];
    }
    std::vector<index_t> rank(D);
    std::iota(rank.begin(), rank.end(), 0);
    std::stable_sort(rank.begin(), rank.end(), [&](index_t x, index_t y) { return colsq[x] > colsq[y]; });
    e.axes.assign(static_cast<std::size_t>(D) * D, 0.0);
    e.singular_values.resize(D);
    for (index_t a = 0; a < D; ++a) {
      e.axes[static_cast<std::size_t>(a) * D + rank[a]] = 1.0;
      e.singular_values[a] = std::sqrt(colsq[rank[a]]);
    }
    e.converged = true;
    e.iterations = 0;
    return e;
  }

  const index_t p = std::min<index_t>(D, d + 2);
  Rng rng(seed);
  std::vector<double> v(static_cast<std::size_t>(D) * p);
  for (double& x : v) x = rng.normal();
  orthonormalize(v, D, p, rng);

  std::unique_ptr<CovarianceOp> op(make_op ? make_op(xc, n, D) : new HostCovariance(xc, n, D));
  std::vector<double> w(static_cast<std::size_t>(D) * p);
  e.converged = false;
  for (index_t it = 1; it <= max_iter; ++it) {
    op->apply(v, w, p);
    orthonormalize(w, D, p, rng);
    const double cos_angle = min_cross_singular(v, w, D, p, d);
    v.swap(w);
    e.iterations = it;
    if (std::acos(std::clamp(cos_angle, 0.0, 1.0)) < tol) {
      e.converged = true;
      break;
    }
  }

  // Rayleigh-Ritz (pca.cpp:230-262)
  std::vector<double> b;
  op->xv(v, b, p);
  std::vector<double> gram(static_cast<std::size_t>(p) * p, 0.0);
  for (index_t i = 0; i < n; ++i) {
    const double* bi = b.data() + static_cast<std::size_t>(i) * p;
    for (index_t a = 0; a < p; ++a)
      for (index_t c = 0; c < p; ++c) gram[a * p + c] += bi[a] * bi[c];
  }
  std::vector<double> evals, evecs;
  jacobi_eig(gram, p, evals, evecs);
  e.axes.assign(static_cast<std::size_t>(d) * D, 0.0);
  e.singular_values.resize(d);
  for (index_t a = 0; a < d; ++a) {
    e.singular_values[a] = std::sqrt(std::max(0.0, evals[a]));
    double* ax = e.axes.data() + static_cast<std::size_t>(a) * D;
    for (index_t r = 0; r < D; ++r) {
      double acc = 0.0;
      for (index_t c = 0; c < p; ++c) acc += v[r * p + c] * evecs[c * p + a];
      ax[r] = acc;
    }
  }
  fix_axis_signs(e);
  if (make_op) {  // y_i[a] = sum_r xc[i][r] * axes[a][r], r ascending: project() on the device
    std::vector<double> vt(static_cast<std::size_t>(D) * d);
    for (index_t a = 0; a < d; ++a)
      for (index_t r = 0; r < D; ++r) vt[static_cast<std::size_t>(r) * d + a] = e.axes[static_cast<std::size_t>(a) * D + r];
    op->xv(vt, e.projected, d);
  }
  return e;
}

std::vector<double> project(const double* pts, index_t n, index_t dim, const Embedding& e) {
  if (dim != e.dim_in) throw error(errc::dim_mismatch, "point dim does not match the embedding");
  std::vector<double> out(static_cast<std::size_t>(n) * e.dim_out);
  for (index_t i = 0; i < n; ++i) {
    const double* x = pts + static_cast<std::size_t>(i) * dim;
    double* y = out.data() + static_cast<std::size_t>(i) * e.dim_out;
    for (index_t a = 0; a < e.dim_out; ++a) {
      const double* ax = e.axes.data() + static_cast<std::size_t>(a) * dim;
      double acc = 0.0;
      for (index_t r = 0; r < dim; ++r) acc += (x[r] - e.mean[r]) * ax[r];
      y[a] = acc;
    }
  }
  return out;
}

// ---------------------------------------------------------------------------
// partition tree

index_t PartitionTree::depth() const {
  index_t d = 0;
  for (const TreeNode& nd : nodes) d = std::max(d, nd.depth);
  return d;
}

namespace {

// Recursive restatement (the depth is bounded by max_depth <= a few dozen).
void split(const double* pts, PartitionTree& tree, std::vector<index_t>& order,
           std::vector<index_t>& scratch, index_t node_id, index_t lo, index_t hi, index_t depth) {
  tree.nodes[node_id].begin = lo;
  tree.nodes[node_id].end = hi;
  tree.nodes[node_id].depth = depth;
  if (hi - lo <= tree.leaf_capacity || depth >= tree.max_depth) {
    tree.nodes[node_id].is_leaf = true;
    return;
  }
  const index_t dim = tree.dim;
  const index_t n_orth = index_t{1} << dim;
  std::array<double, 3> center{};
  for (index_t a = 0; a < dim; ++a)
    center[a] = 0.5 * (tree.nodes[node_id].lo[a] + tree.nodes[node_id].hi[a]);
  auto orthant = [&](index_t original) {
    const double* x = pts + static_cast<std::size_t>(original) * dim;
    index_t code = 0;
    for (index_t a = 0; a < dim; ++a)
      if (x[a] >= center[a]) code |= index_t{1} << a;
    return code;
  };
  std::array<index_t, 9> start{};
  for (index_t i = lo; i < hi; ++i) ++start[orthant(order[i]) + 1];
  for (index_t c = 0; c < n_orth; ++c) start[c + 1] += start[c];
  std::array<index_t, 9> fill = start;
  for (index_t i = lo; i < hi; ++i) scratch[lo + fill[orthant(order[i])]++] = order[i];
  std::copy(scratch.begin() + lo, scratch.begin() + hi, order.begin() + lo);
  const std::array<double, 3> plo = tree.nodes[node_id].lo, phi = tree.nodes[node_id].hi;
  for (index_t code = 0; code < n_orth; ++code) {
    const index_t c_lo = lo + start[code], c_hi = lo + start[code + 1];
    if (c_lo == c_hi) continue;
    const index_t child_id = static_cast<index_t>(tree.nodes.size());
    tree.nodes.emplace_back();
    TreeNode& child = tree.nodes.back();
    child.parent = node_id;
    for (index_t a = 0; a < dim; ++a) {
      const bool high = (code >> a) & 1;
      child.lo[a] = high ? center[a] : plo[a];
      child.hi[a] = high ? phi[a] : center[a];
    }
    tree.nodes[node_id].children.push_back(child_id);
    split(pts, tree, order, scratch, child_id, c_lo, c_hi, depth + 1);
  }
}

}  // namespace

PartitionTree build_tree(const double* emb, index_t n, index_t dim, index_t leaf_capacity,
                         index_t max_depth) {
  if (dim < 1 || dim > 3)
    throw error(errc::dim_too_high, "partition tree supports dim 1..3, got " + std::to_string(dim));
  if (leaf_capacity < 1) throw error(errc::invalid_argument, "leaf_capacity must be >= 1");
  if (max_depth < 1) throw error(errc::invalid_argument, "max_depth must be >= 1");
  PartitionTree tree;
  tree.dim = dim;
  tree.leaf_capacity = leaf_capacity;
  tree.max_depth = max_depth;
  tree.n_points = n;
  tree.nodes.emplace_back();
  std::array<double, 3> lo{}, hi{};
  for (index_t a = 0; a < dim; ++a) {
    lo[a] = n > 0 ? emb[a] : 0.0;
    hi[a] = lo[a];
  }
  for (index_t i = 1; i < n; ++i) {
    const double* x = emb + static_cast<std::size_t>(i) * dim;
    for (index_t a = 0; a < dim; ++a) {
      lo[a] = std::min(lo[a], x[a]);
      hi[a] = std::max(hi[a], x[a]);
    }
  }
  double side = 0.0;
  for (index_t a = 0; a < dim; ++a) side = std::max(side, hi[a] - lo[a]);
  for (index_t a = 0; a < dim; ++a) {
    const double center = 0.5 * (lo[a] + hi[a]);
    tree.nodes[0].lo[a] = center - 0.5 * side;
    tree.nodes[0].hi[a] = center + 0.5 * side;
  }
  std::vector<index_t> order(n), scratch(n);
  std::iota(order.begin(), order.end(), 0);
  split(emb, tree, order, scratch, 0, 0, n, 0);
  tree.forward.assign(n, 0);
  for (index_t pos = 0; pos < n; ++pos) tree.forward[order[pos]] = pos;
  return tree;
}

std::vector<index_t> level_blocking(const PartitionTree& t, index_t level) {
  if (level < 0 || level > t.depth())
    throw error(errc::level_out_of_range, "level " + std::to_string(level) +
                                              " exceeds tree depth " + std::to_string(t.depth()));
  std::vector<index_t> offsets;
  for (const TreeNode& nd : t.nodes)
    if (nd.depth == level || (nd.is_leaf && nd.depth < level)) offsets.push_back(nd.begin);
  offsets.push_back(t.n_points);
  std::sort(offsets.begin(), offsets.end());
  return offsets;
}

PartitionTree order_tree_scheme(const double* pts, index_t n, index_t dim, index_t d,
                                index_t leaf_capacity, index_t max_depth, double* captured_ratio,
                                std::function<CovarianceOp*(const std::vector<double>&, index_t,
                                                            index_t)> make_op) {
  if (d < 2 || d > 3) throw error(errc::invalid_argument, "tree schemes are tree2 and tree3");
  if (captured_ratio) *captured_ratio = 1.0;
  if (dim <= d) return build_tree(pts, n, dim, leaf_capacity, max_depth);
  const Embedding e = fit_pca(pts, n, dim, d, 1e-9, 1000, 1, make_op);
  if (captured_ratio) {  // variance_ratio (pca.cpp:284-290)
    double s = 0.0;
    for (double sv : e.singular_values) s += sv * sv;
    *captured_ratio = std::clamp(s / e.total_sq_norm, 0.0, 1.0);
  }
  const std::vector<double> emb = e.projected.empty() ? project(pts, n, dim, e) : e.projected;
  return build_tree(emb.data(), n, d, leaf_capacity, max_depth);
}

}  // namespace knnx
