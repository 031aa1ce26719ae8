// paper_1709_03671_b200/shim/patchord_gpu.cpp -- implementation of
// include/patchord_gpu.hpp: patchord's interaction kernels on the B200 via the
// knnx C ABI.  Compiled against the reference's headers (it is integration
// code meant to live in the reference tree).
#include "patchord_gpu.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>

#include "knnx.h"
#include "patchord/knn.hpp"
#include "patchord/orderings.hpp"
#include "patchord/pca.hpp"

namespace patchord::gpu {

namespace {

// knnx status -> patchord::error with the reference's errc (code = 1 + ordinal)
void ok(int rc) {
  if (rc == KNNX_OK) return;
  std::string msg = knnx_last_error();
  const auto colon = msg.find(": ");
  if (colon != std::string::npos && colon < 32) msg = msg.substr(colon + 2);  // drop "Name: "
  if (rc >= 1 && rc <= static_cast<int>(errc::invalid_argument) + 1)
    throw error(static_cast<errc>(rc - 1), msg);
  throw error(errc::invalid_argument, "device error " + std::to_string(rc) + ": " + msg);
}

void check_tag(const std::string& vec_tag, const std::string& mat_tag, const char* side) {
  if (!vec_tag.empty() && !mat_tag.empty() && vec_tag != mat_tag)
    throw error(errc::ordering_mismatch, std::string(side) + " vector is laid out under '" +
                                             vec_tag + "' but the matrix expects '" + mat_tag + "'");
}

std::vector<float> to_f32(const std::vector<double>& v) { return {v.begin(), v.end()}; }

// canonical (row, col) order of the leaf payload: position -> (block, entry)
struct LeafIndex {
  std::vector<std::pair<index_t, std::size_t>> where;  // canonical position -> (block id, entry)
};

LeafIndex leaf_index(const HierBlockMatrix& h) {
  std::vector<std::tuple<index_t, index_t, index_t, std::size_t>> all;
  all.reserve(static_cast<std::size_t>(h.nnz));
  for (index_t b = 0; b < static_cast<index_t>(h.blocks.size()); ++b) {
    const HierBlock& blk = h.blocks[b];
    if (!blk.is_leaf) continue;
    for (std::size_t e = 0; e < blk.vals.size(); ++e)
      all.emplace_back(blk.row_offset + blk.lr[e], blk.col_offset + blk.lc[e], b, e);
  }
  std::sort(all.begin(), all.end());
  LeafIndex li;
  li.where.reserve(all.size());
  for (const auto& [r, c, b, e] : all) li.where.emplace_back(b, e);
  return li;
}

std::vector<float> flat_coords(const PointSet& p) { return to_f32(p.coords); }

}  // namespace

// ---------------------------------------------------------------------------
// PointBuffer

namespace {
index_t ld_for(index_t dim, bool padded) { return padded ? (dim + 3) / 4 * 4 : dim; }
}  // namespace

PointBuffer::PointBuffer(Device& dev, index_t n, index_t dim, bool padded)
    : dev_(&dev), n_(n), dim_(dim), ld_(ld_for(dim, padded)) {
  if (n < 0 || dim < 1) throw error(errc::invalid_argument, "point buffer shape");
  void* p = nullptr;
  ok(knnx_alloc(dev.handle(), static_cast<int64_t>(n) * ld_ * 4, &p));
  d_ = static_cast<float*>(p);
  const std::vector<float> zero(static_cast<std::size_t>(n) * dim, 0.0f);
  ok(knnx_upload_points(dev.handle(), zero.data(), n, dim, ld_, d_));
}

PointBuffer::PointBuffer(Device& dev, const PointSet& p, bool padded)
    : PointBuffer(dev, p.n_points, p.dim, padded) {
  upload(p);
}

PointBuffer::PointBuffer(PointBuffer&& o) noexcept
    : dev_(o.dev_), d_(o.d_), n_(o.n_), dim_(o.dim_), ld_(o.ld_) {
  o.d_ = nullptr;
}

PointBuffer::~PointBuffer() {
  if (d_) knnx_free(dev_->handle(), d_);
}

void PointBuffer::upload(const PointSet& p) {
  if (p.n_points != n_ || p.dim != dim_)
    throw error(errc::dim_mismatch, "point set shape does not match the buffer");
  const std::vector<float> f(p.coords.begin(), p.coords.end());
  ok(knnx_upload_points(dev_->handle(), f.data(), n_, dim_, ld_, d_));
}

PointSet PointBuffer::download() const {
  std::vector<float> f(static_cast<std::size_t>(n_) * dim_);
  ok(knnx_download_points(dev_->handle(), d_, n_, dim_, ld_, f.data()));
  return make_point_set(n_, dim_, std::vector<double>(f.begin(), f.end()));
}

Device::Device(int device) { ok(knnx_ctx_create(device, &ctx_)); }
Device::~Device() { knnx_ctx_destroy(ctx_); }
Device& Device::default_device() {
  static Device dev(0);
  return dev;
}

Operator::Operator(Device& dev, const SparseMatrix& m)
    : dev_(&dev), n_rows_(m.pattern.n_rows), n_cols_(m.pattern.n_cols) {
  const std::vector<index_t> rp32 = row_pointers(m.pattern);
  const std::vector<int64_t> rp(rp32.begin(), rp32.end());
  std::vector<int32_t> cols(m.pattern.entries.size());
  for (std::size_t e = 0; e < cols.size(); ++e) cols[e] = m.pattern.entries[e].second;
  const std::vector<float> vals = to_f32(m.values);
  ok(knnx_op_create_csr(dev.handle(), n_rows_, n_cols_, static_cast<int64_t>(cols.size()), rp.data(),
                        cols.data(), vals.data(), KNNX_ORDER_ORIGINAL, 0, &op_));
}

Operator::Operator(Device& dev, const HierBlockMatrix& h)
    : dev_(&dev), n_rows_(h.n_rows), n_cols_(h.n_cols), row_tag_(h.row_tag), col_tag_(h.col_tag),
      hier_(true) {
  std::vector<int32_t> ro, co;
  std::vector<int64_t> ptr{0};
  std::vector<uint16_t> lr, lc;
  std::vector<float> vals;
  for (const HierBlock& b : h.blocks) {  // leaf payload in traversal-independent order
    if (!b.is_leaf) continue;
    ro.push_back(b.row_offset);
    co.push_back(b.col_offset);
    lr.insert(lr.end(), b.lr.begin(), b.lr.end());
    lc.insert(lc.end(), b.lc.begin(), b.lc.end());
    for (double v : b.vals) vals.push_back(static_cast<float>(v));
    ptr.push_back(static_cast<int64_t>(lr.size()));
  }
  ok(knnx_op_create_hier_leaves(dev.handle(), n_rows_, n_cols_, static_cast<int32_t>(ro.size()),
                                ro.data(), co.data(), ptr.data(), lr.data(), lc.data(),
                                vals.data(), 0, &op_));
}

Operator::~Operator() {
  knnx_op_destroy(op_);
  knnx_host_free(x_stage_);
  knnx_host_free(y_stage_);
}

namespace {

// fn(lo, hi) over [0, n) on a few threads (the fp64 <-> fp32 conversions of
// million-entry vectors are memory-bound loops worth splitting)
template <typename Fn>
void split_range(std::size_t n, Fn&& fn) {
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < (std::size_t{1} << 18) || hw == 1) {
    fn(std::size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const std::size_t step = (n + hw - 1) / hw;
  for (unsigned w = 0; w < hw; ++w) {
    const std::size_t lo = std::min(n, w * step), hi = std::min(n, lo + step);
    if (lo < hi) pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : pool) t.join();
}

}  // namespace

PotentialVector Operator::spmv(const ChargeVector& x) const {
  if (static_cast<index_t>(x.values.size()) != n_cols_)
    throw error(errc::dim_mismatch, "charge vector length " + std::to_string(x.values.size()) +
                                        " vs " + std::to_string(n_cols_) + " columns");
  if (hier_) check_tag(x.ordering, col_tag_, "charge");
  if (!x_stage_) ok(knnx_host_alloc(static_cast<int64_t>(n_cols_) * 4, reinterpret_cast<void**>(&x_stage_)));
  if (!y_stage_) ok(knnx_host_alloc(static_cast<int64_t>(n_rows_) * 4, reinterpret_cast<void**>(&y_stage_)));
  const double* xv = x.values.data();
  float* xs = x_stage_;
  split_range(static_cast<std::size_t>(n_cols_), [xv, xs](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) xs[i] = static_cast<float>(xv[i]);
  });
  ok(knnx_spmv_host(op_, x_stage_, y_stage_));
  PotentialVector y;
  y.values.resize(n_rows_);
  double* yv = y.values.data();
  const float* ys = y_stage_;
  split_range(static_cast<std::size_t>(n_rows_), [yv, ys](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) yv[i] = static_cast<double>(ys[i]);
  });
  y.ordering = hier_ ? row_tag_ : x.ordering;
  return y;
}

void Operator::set_values(const std::vector<double>& canonical_vals) {
  const std::vector<float> v = to_f32(canonical_vals);
  ok(knnx_op_set_values(op_, v.data()));
}

std::vector<double> Operator::values() const {
  knnx_op_info_t info{};
  ok(knnx_op_info(op_, &info));
  std::vector<float> v(static_cast<std::size_t>(info.nnz));
  ok(knnx_op_get_values(op_, v.data()));
  return {v.begin(), v.end()};
}

PotentialVector Operator::gauss_spmv(const PointBuffer& targets, const PointBuffer& sources,
                                     double bandwidth, const ChargeVector& x) const {
  if (!(bandwidth > 0.0)) throw error(errc::non_positive_bandwidth, "bandwidth must be positive");
  if (targets.dim() != sources.dim()) throw error(errc::dim_mismatch, "target and source dims differ");
  if (targets.n_points() != n_rows_ || sources.n_points() != n_cols_ ||
      static_cast<index_t>(x.values.size()) != n_cols_)
    throw error(errc::dim_mismatch, "pattern shape does not match point / charge counts");
  if (hier_) check_tag(x.ordering, col_tag_, "charge");
  PointBuffer xd(*dev_, make_point_set(n_cols_, 1, x.values), false);
  PointBuffer yd(*dev_, n_rows_, 1, false);
  ok(knnx_gauss_spmv_dev(op_, targets.data(), targets.ld(), sources.data(), sources.ld(),
                         targets.dim(), bandwidth, xd.data(), yd.data()));
  PotentialVector y;
  y.values = yd.download().coords;
  y.ordering = hier_ ? row_tag_ : x.ordering;
  return y;
}

void Operator::meanshift(const PointBuffer& t_in, const PointBuffer& sources, double bandwidth,
                         PointBuffer& t_out) const {
  if (!(bandwidth > 0.0)) throw error(errc::non_positive_bandwidth, "bandwidth must be positive");
  if (t_in.dim() != sources.dim() || t_out.dim() != t_in.dim() || t_out.ld() != t_in.ld())
    throw error(errc::dim_mismatch, "target and source dims differ");
  if (t_in.n_points() != n_rows_ || t_out.n_points() != n_rows_ || sources.n_points() != n_cols_)
    throw error(errc::dim_mismatch, "pattern shape does not match point counts");
  ok(knnx_meanshift_dev(op_, t_in.data(), t_in.ld(), sources.data(), sources.ld(), t_in.dim(),
                        bandwidth, t_out.data()));
}

void Operator::tsne(const PointBuffer& y, PointBuffer& forces, double step, PointBuffer* y_out) const {
  if (n_rows_ != n_cols_) throw error(errc::not_square, "affinity matrix is not square");
  if (y.n_points() != n_rows_ || forces.n_points() != n_rows_ || y.ld() != y.dim() ||
      forces.dim() != y.dim() || forces.ld() != y.dim() ||
      (y_out && (y_out->n_points() != n_rows_ || y_out->ld() != y.dim())))
    throw error(errc::dim_mismatch, "embedding buffers must be n x dim_out, unpadded");
  ok(knnx_tsne_attr_dev(op_, y.data(), y.dim(), forces.data(), 0, static_cast<float>(step),
                        y_out ? y_out->data() : nullptr));
}

// ---------------------------------------------------------------------------

PotentialVector spmv_flat(const SparseMatrix& m, const ChargeVector& x) {
  if (static_cast<index_t>(x.values.size()) != m.pattern.n_cols)
    throw error(errc::dim_mismatch, "charge vector length " + std::to_string(x.values.size()) +
                                        " vs " + std::to_string(m.pattern.n_cols) + " columns");
  return Operator(Device::default_device(), m).spmv(x);
}

PotentialVector spmv_hier(const HierBlockMatrix& h, const ChargeVector& x) {
  if (static_cast<index_t>(x.values.size()) != h.n_cols)
    throw error(errc::dim_mismatch, "charge vector length " + std::to_string(x.values.size()) +
                                        " vs " + std::to_string(h.n_cols) + " columns");
  check_tag(x.ordering, h.col_tag, "charge");
  return Operator(Device::default_device(), h).spmv(x);
}

PotentialVector spmv_hier_parallel(const HierBlockMatrix& h, const ChargeVector& x,
                                   index_t workers) {
  if (workers < 1) throw error(errc::invalid_argument, "workers must be >= 1");
  return gpu::spmv_hier(h, x);
}

PointSet tsne_attractive_step(HierBlockMatrix& h, const PointSet& y, index_t dim_out) {
  if (h.n_rows != h.n_cols) throw error(errc::not_square, "affinity matrix is not square");
  if (y.n_points != h.n_rows)
    throw error(errc::dim_mismatch, "embedding has " + std::to_string(y.n_points) +
                                        " points for an order-" + std::to_string(h.n_rows) +
                                        " matrix");
  if (y.dim != dim_out)
    throw error(errc::dim_mismatch, "embedding dimension " + std::to_string(y.dim) + " vs " +
                                        std::to_string(dim_out));
  if (dim_out < 1 || dim_out > 3)
    throw error(errc::dim_mismatch, "device t-SNE supports embedding dimensions 1..3");
  Operator op(Device::default_device(), h);
  const std::vector<float> yf = flat_coords(y);
  std::vector<float> f(yf.size());
  ok(knnx_tsne_attr_host(op.handle(), yf.data(), dim_out, f.data(), /*store_affinities=*/1));
  // write a_ij back into the leaf payload, as the reference does in place
  const std::vector<double> a = op.values();
  const LeafIndex li = leaf_index(h);
  for (std::size_t q = 0; q < a.size(); ++q) h.blocks[li.where[q].first].vals[li.where[q].second] = a[q];
  return make_point_set(y.n_points, dim_out, std::vector<double>(f.begin(), f.end()));
}

namespace {

// build_knn(targets, sources, k) for the mean-shift refresh (distinct
// objects: no self exclusion, proj/src/knn.cpp:10): exact fp32 kNN on the
// device (ascending (distance, index)): knnx_knn_dev for dim <= 64, the
// tcgen05 distance screen + exact re-rank knnx_knn_wide_dev beyond (k <= 128).
// Near-ties can order differently from the fp64 reference; distances are the
// device's squared distances widened.
KnnGraph refresh_knn(const PointSet& targets, const PointSet& sources, index_t k) {
  const bool wide = targets.dim > 64;
  if (k > (wide ? 128 : 256)) return build_knn(targets, sources, k);
  if (targets.dim != sources.dim)
    throw error(errc::dim_mismatch, "target dim " + std::to_string(targets.dim) +
                                        " != source dim " + std::to_string(sources.dim));
  if (k < 1) throw error(errc::invalid_argument, "k must be >= 1");
  if (k > sources.n_points)
    throw error(errc::k_too_large, "k = " + std::to_string(k) + " with " +
                                       std::to_string(sources.n_points) + " sources");
  Device& dev = Device::default_device();
  const PointBuffer t(dev, targets), s(dev, sources);
  const index_t m = targets.n_points;
  void *ids = nullptr, *d2 = nullptr;
  ok(knnx_alloc(dev.handle(), static_cast<int64_t>(m) * k * 4, &ids));
  ok(knnx_alloc(dev.handle(), static_cast<int64_t>(m) * k * 4, &d2));
  const int rc =
      wide ? knnx_knn_wide_dev(dev.handle(), t.data(), m, s.data(), sources.n_points, t.ld(),
                               targets.dim, k, 0, 0, static_cast<int32_t*>(ids),
                               static_cast<float*>(d2), nullptr)
           : knnx_knn_dev(dev.handle(), t.data(), m, s.data(), sources.n_points, t.ld(), targets.dim,
                          k, 0, static_cast<int32_t*>(ids), static_cast<float*>(d2));
  std::vector<float> hi(static_cast<std::size_t>(m) * k), hd(hi.size());
  if (rc == KNNX_OK) {
    ok(knnx_download_points(dev.handle(), static_cast<const float*>(ids), m * k, 1, 1, hi.data()));
    ok(knnx_download_points(dev.handle(), static_cast<const float*>(d2), m * k, 1, 1, hd.data()));
  }
  knnx_free(dev.handle(), ids);
  knnx_free(dev.handle(), d2);
  // wide points whose neighbour distances the TF32 screen cannot certify: the
  // reference's own (host) search, as for every dim > 64 before round 2
  if (wide && rc == 1 + static_cast<int>(errc::degenerate_data)) return build_knn(targets, sources, k);
  ok(rc);
  KnnGraph g;
  g.k = k;
  g.n_targets = m;
  g.n_sources = sources.n_points;
  g.neighbor_ids.resize(hi.size());
  std::memcpy(g.neighbor_ids.data(), hi.data(), sizeof(float) * hi.size());  // int32 bits
  g.neighbor_dists.assign(hd.begin(), hd.end());
  return g;
}

}  // namespace

MeanShiftState meanshift_step(MeanShiftState state) {
  const index_t m = state.targets.n_points, k = state.knn.k, dim = state.targets.dim;
  // neighbor rows -> canonical pattern (columns sorted; accumulation order is
  // immaterial at fp32 tolerance)
  std::vector<int64_t> rp(static_cast<std::size_t>(m) + 1);
  std::vector<int32_t> cols(static_cast<std::size_t>(m) * k);
  for (index_t i = 0; i <= m; ++i) rp[i] = static_cast<int64_t>(i) * k;
  for (index_t i = 0; i < m; ++i) {
    std::copy(state.knn.ids(i), state.knn.ids(i) + k, cols.begin() + static_cast<std::size_t>(i) * k);
    std::sort(cols.begin() + static_cast<std::size_t>(i) * k,
              cols.begin() + static_cast<std::size_t>(i + 1) * k);
  }
  knnx_op_t op = nullptr;
  ok(knnx_op_create_csr(Device::default_device().handle(), m, state.sources.n_points,
                        static_cast<int64_t>(cols.size()), rp.data(), cols.data(), nullptr,
                        KNNX_ORDER_ORIGINAL, 0, &op));
  const std::vector<float> t = flat_coords(state.targets), s = flat_coords(state.sources);
  std::vector<float> out(t.size());
  const int rc = knnx_meanshift_host(op, t.data(), s.data(), dim, state.bandwidth, out.data());
  knnx_op_destroy(op);
  ok(rc);
  state.targets.coords.assign(out.begin(), out.end());
  ++state.iteration;
  if (state.iteration % state.refresh_period == 0) {  // proj/src/kernels.cpp:209-213
    state.knn = refresh_knn(state.targets, state.sources, state.k);
    if (state.reorder_on_refresh) {  // reorder_targets, proj/src/kernels.cpp:162-180
      const index_t d_view = std::min<index_t>(3, state.targets.dim);
      PointSet view = state.targets;
      if (state.targets.dim > 3) view = project(state.targets, fit_pca(state.targets, d_view));
      const OrderingResult ord = order_tree(view, 128, 12);
      state.targets = gpu::permute(state.targets, ord.row_perm);
      KnnGraph moved = state.knn;
      for (index_t q = 0; q < state.knn.n_targets; ++q) {
        const index_t pos = ord.row_perm.forward[q];
        std::copy(state.knn.ids(q), state.knn.ids(q) + k,
                  moved.neighbor_ids.begin() + static_cast<std::size_t>(pos) * k);
        std::copy(state.knn.dists(q), state.knn.dists(q) + k,
                  moved.neighbor_dists.begin() + static_cast<std::size_t>(pos) * k);
      }
      state.knn = std::move(moved);
    }
  }
  return state;
}

std::vector<PotentialVector> iterate_interactions(
    HierBlockMatrix& h,
    const std::function<std::function<double(index_t, index_t, double)>(index_t)>& value_fn,
    const std::vector<ChargeVector>& x_seq) {
  Operator op(Device::default_device(), h);
  const LeafIndex li = leaf_index(h);
  std::vector<std::size_t> canon_of;  // (block, entry) -> canonical position
  std::vector<std::size_t> block_base(h.blocks.size() + 1, 0);
  for (std::size_t b = 0; b < h.blocks.size(); ++b) block_base[b + 1] = block_base[b] + h.blocks[b].vals.size();
  canon_of.assign(block_base.back(), 0);
  for (std::size_t q = 0; q < li.where.size(); ++q)
    canon_of[block_base[li.where[q].first] + li.where[q].second] = q;
  std::vector<PotentialVector> out;
  out.reserve(x_seq.size());
  std::vector<double> canon(li.where.size());
  for (std::size_t kappa = 0; kappa < x_seq.size(); ++kappa) {
    // the user's value_fn is host code: evaluated in the reference's
    // pre-order traversal (hier.cpp:195-222), then the multiply runs on the GPU
    const auto f = value_fn(static_cast<index_t>(kappa));
    std::function<void(index_t)> visit = [&](index_t id) {
      HierBlock& b = h.blocks[id];
      if (b.is_leaf)
        for (std::size_t e = 0; e < b.vals.size(); ++e) {
          const double v = f(b.row_offset + b.lr[e], b.col_offset + b.lc[e], b.vals[e]);
          if (!std::isfinite(v))
            throw error(errc::non_finite_value,
                        "update produced a non-finite value at (" +
                            std::to_string(b.row_offset + b.lr[e]) + "," +
                            std::to_string(b.col_offset + b.lc[e]) + ")");
          b.vals[e] = v;
          canon[canon_of[block_base[id] + e]] = v;
        }
      for (index_t c : b.children) visit(c);
    };
    for (index_t top : h.top_blocks) visit(top);
    op.set_values(canon);
    out.push_back(op.spmv(x_seq[kappa]));
  }
  return out;
}

std::vector<PotentialVector> iterate_interactions_gaussian(const HierBlockMatrix& h,
                                                           const PointSet& targets,
                                                           const PointSet& sources,
                                                           double bandwidth,
                                                           const std::vector<ChargeVector>& x_seq) {
  if (!(bandwidth > 0.0)) throw error(errc::non_positive_bandwidth, "bandwidth must be positive");
  if (targets.dim != sources.dim) throw error(errc::dim_mismatch, "target and source dims differ");
  if (targets.n_points != h.n_rows || sources.n_points != h.n_cols)
    throw error(errc::dim_mismatch, "pattern shape does not match point counts");
  Operator op(Device::default_device(), h);
  const std::vector<float> t = flat_coords(targets), s = flat_coords(sources);
  std::vector<PotentialVector> out;
  for (const ChargeVector& x : x_seq) {
    if (static_cast<index_t>(x.values.size()) != h.n_cols)
      throw error(errc::dim_mismatch, "charge vector length mismatch");
    check_tag(x.ordering, h.col_tag, "charge");
    const std::vector<float> xf = to_f32(x.values);
    std::vector<float> y(h.n_rows);
    ok(knnx_gauss_spmv_host(op.handle(), t.data(), s.data(), targets.dim, bandwidth, xf.data(),
                            y.data()));
    out.push_back(PotentialVector{std::vector<double>(y.begin(), y.end()), h.row_tag});
  }
  return out;
}

index_t update_values_gaussian(HierBlockMatrix& h, const PointSet& targets, const PointSet& sources,
                               double bandwidth) {
  if (!(bandwidth > 0.0)) throw error(errc::non_positive_bandwidth, "bandwidth must be positive");
  if (targets.dim != sources.dim) throw error(errc::dim_mismatch, "target and source dims differ");
  Operator op(Device::default_device(), h);
  const std::vector<float> t = flat_coords(targets), s = flat_coords(sources);
  ok(knnx_update_gaussian_host(op.handle(), t.data(), s.data(), targets.dim, bandwidth));
  const std::vector<double> a = op.values();
  const LeafIndex li = leaf_index(h);
  for (std::size_t q = 0; q < a.size(); ++q) h.blocks[li.where[q].first].vals[li.where[q].second] = a[q];
  return static_cast<index_t>(a.size());
}

PointSet permute(const PointSet& pts, const Permutation& p) {
  if (p.size() != pts.n_points)
    throw error(errc::size_mismatch, "permutation size does not match point count");
  PointSet out = pts;
  ok(knnx_permute_rows_host(Device::default_device().handle(), pts.n_points,
                            static_cast<int64_t>(pts.dim) * 8, pts.coords.data(), p.forward.data(),
                            out.coords.data()));
  return out;
}

}  // namespace patchord::gpu
