// tests/cpp/test_shim.cpp -- the reference's own kernel tests
// (proj/tests/test_kernels.cpp), restated against the drop-in GPU shim
// patchord::gpu (include/patchord_gpu.hpp) with fp32 tolerances.  Linked with
// the reference library objects (for the types and the double oracles) and
// libknnx.so.  Run by tests/test_gpu_shim.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>
#include <string>

#include "patchord/kernels.hpp"
#include "patchord/orderings.hpp"
#include "patchord/pca.hpp"
#include "patchord_gpu.hpp"

using namespace patchord;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                               \
  do {                                                                         \
    if (c) ++g_pass;                                                           \
    else { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); } \
  } while (0)

template <typename Fn>
static void expect_errc(errc want, Fn&& fn, const char* what) {
  try {
    fn();
    ++g_fail;
    std::printf("FAIL no error: %s\n", what);
  } catch (const error& e) {
    if (e.code() == want) ++g_pass;
    else { ++g_fail; std::printf("FAIL wrong errc for %s: %s\n", what, e.what()); }
  }
}

namespace {

SparseMatrix random_matrix(index_t n, index_t target_nnz, std::uint64_t seed, bool symmetric = false) {
  Rng rng(seed);
  std::set<std::pair<index_t, index_t>> seen;
  std::vector<std::tuple<index_t, index_t, double>> entries;
  while (static_cast<index_t>(seen.size()) < target_nnz) {
    const index_t i = static_cast<index_t>(rng.bounded(n)), j = static_cast<index_t>(rng.bounded(n));
    const double v = rng.uniform01() + 0.1;
    if (symmetric) {
      if (i == j) continue;
      if (seen.insert({i, j}).second && seen.insert({j, i}).second) {
        entries.emplace_back(i, j, v);
        entries.emplace_back(j, i, v);
      }
    } else if (seen.insert({i, j}).second) {
      entries.emplace_back(i, j, v);
    }
  }
  return csr_from_coo(entries, n, n);
}

std::shared_ptr<const PartitionTree> random_tree(index_t n, index_t dim, index_t cap, std::uint64_t seed) {
  Rng rng(seed);
  std::vector<double> c(static_cast<std::size_t>(n) * dim);
  for (double& v : c) v = rng.normal();
  return std::make_shared<PartitionTree>(build_tree(make_point_set(n, dim, c), cap, 12));
}

ChargeVector random_charge(index_t n, std::uint64_t seed, std::string tag = "") {
  Rng rng(seed);
  ChargeVector x;
  x.values.resize(n);
  for (double& v : x.values) v = rng.normal();
  x.ordering = std::move(tag);
  return x;
}

// SURVEY.md §8d scale-aware metric
double rel(const std::vector<double>& g, const std::vector<double>& r) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < g.size(); ++i) {
    num = std::max(num, std::abs(g[i] - r[i]));
    den = std::max(den, std::abs(r[i]));
  }
  return den > 0 ? num / den : num;
}

constexpr double kTol = 1e-5;

}  // namespace

int main() {
  {  // test_kernels.cpp:65-71
    const SparseMatrix eye = csr_from_coo({{0, 0, 1.0}, {1, 1, 1.0}, {2, 2, 1.0}}, 3, 3);
    const PotentialVector y = gpu::spmv_flat(eye, {{0.5, -2.0, 7.25}, "natural"});
    CHECK((y.values == std::vector<double>{0.5, -2.0, 7.25}));
    CHECK(y.ordering == "natural");
  }
  {  // :73-77
    const SparseMatrix m = csr_from_coo({{0, 0, 1.0}, {0, 1, 2.0}, {1, 1, 3.0}}, 2, 2);
    CHECK((gpu::spmv_flat(m, {{1.0, 1.0}, ""}).values == std::vector<double>{3.0, 3.0}));
  }
  {  // :79-91 dense oracle (the reference's spmv_flat in double)
    const SparseMatrix m = random_matrix(64, 900, 3);
    const ChargeVector x = random_charge(64, 4);
    CHECK(rel(gpu::spmv_flat(m, x).values, spmv_flat(m, x).values) < kTol);
  }
  expect_errc(errc::dim_mismatch,
              [] { gpu::spmv_flat(csr_from_coo({{0, 0, 1.0}}, 2, 2), {{1.0}, ""}); },
              "spmv_flat short charge");  // :93-101
  {  // :103-110 flat degenerate case
    const SparseMatrix m = random_matrix(50, 400, 5);
    const ChargeVector x = random_charge(50, 6);
    CHECK(rel(gpu::spmv_hier(build_hier_flat(m), x).values, spmv_flat(m, x).values) < kTol);
  }
  {  // :129-139 across random trees and cut levels
    const SparseMatrix m = random_matrix(96, 1200, 11);
    const auto rt = random_tree(96, 3, 8, 12), ct = random_tree(96, 3, 8, 13);
    const ChargeVector x = random_charge(96, 14);
    for (index_t cut : std::vector<index_t>{0, 1, 2, kAutoCutLevel, rt->depth()}) {
      const HierBlockMatrix h = build_hier(m, rt, ct, cut);
      CHECK(rel(gpu::spmv_hier(h, x).values, spmv_hier(h, x).values) < kTol);
    }
  }
  {  // :141-156 ordering tags
    HierBlockMatrix h = build_hier_flat(random_matrix(20, 80, 15));
    h.row_tag = h.col_tag = "tree2";
    expect_errc(errc::ordering_mismatch, [&] { gpu::spmv_hier(h, random_charge(20, 16, "scattered")); },
                "tag mismatch");
    const PotentialVector y = gpu::spmv_hier(h, random_charge(20, 16));
    CHECK(y.ordering == "tree2");
    CHECK(gpu::spmv_hier(h, random_charge(20, 16, "tree2")).values == y.values);
  }
  {  // :158-177 identical for any worker count
    const SparseMatrix m = random_matrix(200, 3000, 17);
    const auto t = random_tree(200, 3, 16, 18);
    const HierBlockMatrix h = build_hier(m, t, t);
    const ChargeVector x = random_charge(200, 19);
    const PotentialVector seq = gpu::spmv_hier(h, x);
    for (index_t w : {1, 2, 4, 8}) CHECK(gpu::spmv_hier_parallel(h, x, w).values == seq.values);
    expect_errc(errc::invalid_argument, [&] { gpu::spmv_hier_parallel(h, x, 0); }, "0 workers");
  }
  {  // :179-190 two-point t-SNE, stored values rescaled in place
    const SparseMatrix p = csr_from_coo({{0, 1, 0.5}, {1, 0, 0.5}}, 2, 2);
    HierBlockMatrix h = build_hier_flat(p);
    const PointSet f = gpu::tsne_attractive_step(h, make_point_set(2, 2, {0.0, 0.0, 1.0, 0.0}), 2);
    CHECK(f.point(0)[0] == -0.25 && f.point(0)[1] == 0.0);
    CHECK(f.point(1)[0] == 0.25 && f.point(1)[1] == 0.0);
    for (double v : flatten(h).values) CHECK(v == 0.25);
  }
  {  // :192-204 coincident points
    const SparseMatrix p = random_matrix(10, 40, 23, true);
    HierBlockMatrix h = build_hier_flat(p);
    const PointSet f0 = gpu::tsne_attractive_step(h, make_point_set(10, 3, std::vector<double>(30, 0.0)), 3);
    std::vector<double> p32;
    for (double v : p.values) p32.push_back(static_cast<float>(v));
    CHECK(flatten(h).values == p32);  // 1 + 0 leaves every (fp32) affinity intact
    for (double v : f0.coords) CHECK(v == 0.0);
  }
  {  // :206-232 dense oracle at N = 64, d = 2, 3 (vs the reference step)
    for (index_t d : {2, 3}) {
      const SparseMatrix p = random_matrix(64, 700, 25 + d, true);
      Rng rng(27 + d);
      std::vector<double> c(static_cast<std::size_t>(64) * d);
      for (double& v : c) v = static_cast<float>(rng.normal());
      const PointSet y = make_point_set(64, d, c);
      HierBlockMatrix hg = build_hier_flat(p), hr = build_hier_flat(p);
      CHECK(rel(gpu::tsne_attractive_step(hg, y, d).coords, tsne_attractive_step(hr, y, d).coords) < 1e-4);
      CHECK(rel(flatten(hg).values, flatten(hr).values) < kTol);
    }
  }
  expect_errc(errc::not_square,
              [] {
                HierBlockMatrix rect = build_hier_flat(csr_from_coo({{0, 1, 1.0}}, 2, 3));
                gpu::tsne_attractive_step(rect, make_point_set(2, 2, {0.0, 0.0, 1.0, 1.0}), 2);
              },
              "tsne rectangular");  // :256-265
  {  // :277-285 single source
    MeanShiftState s = meanshift_init(make_point_set(1, 2, {3.0, -1.0}),
                                      make_point_set(1, 2, {10.0, 10.0}), 5.0, 1);
    s = gpu::meanshift_step(std::move(s));
    CHECK(s.targets.point(0)[0] == 3.0 && s.targets.point(0)[1] == -1.0);
    CHECK(s.iteration == 1);
  }
  {  // :287-293 symmetric sources
    MeanShiftState s = meanshift_init(make_point_set(2, 1, {-1.0, 1.0}), make_point_set(1, 1, {0.0}), 1.0, 2);
    s = gpu::meanshift_step(std::move(s));
    CHECK(s.targets.point(0)[0] == 0.0);
  }
  {  // :303-354 kNN-restricted oracle over 12 steps with refresh every 5
    Rng rng(37);
    std::vector<double> src, tgt;
    const double cx[3] = {0.0, 20.0, -15.0}, cy[3] = {0.0, 5.0, 18.0};
    for (index_t i = 0; i < 120; ++i) {
      src.push_back(cx[i % 3] + rng.normal());
      src.push_back(cy[i % 3] + rng.normal());
    }
    for (index_t i = 0; i < 40; ++i) {
      tgt.push_back(cx[i % 3] + 2.0 * rng.normal());
      tgt.push_back(cy[i % 3] + 2.0 * rng.normal());
    }
    for (double& v : src) v = static_cast<float>(v);
    for (double& v : tgt) v = static_cast<float>(v);
    MeanShiftState s = meanshift_init(make_point_set(120, 2, src), make_point_set(40, 2, tgt), 2.0, 8, 5);
    for (int step = 0; step < 12; ++step) {
      MeanShiftState want = meanshift_step(s);  // the reference step on the same state
      s = gpu::meanshift_step(std::move(s));
      CHECK(rel(s.targets.coords, want.targets.coords) < kTol);
      if (s.iteration % 5 == 0) {  // refreshed on the device: the reference's rows
        const KnnGraph g = build_knn(s.targets, s.sources, s.k);
        CHECK(s.knn.neighbor_ids == g.neighbor_ids);
        CHECK(rel(s.knn.neighbor_dists, g.neighbor_dists) < kTol);
      }
      for (double& v : s.targets.coords) v = static_cast<float>(v);
    }
    CHECK(s.iteration == 12);
  }
  {  // the same with wide points (dim = 96): the refresh runs on the tensor-core
     // kNN (knnx_knn_wide_dev) and must reproduce the reference's rows
    Rng rng(41);
    const index_t ns = 300, nt = 70, d = 96;
    std::vector<double> src(static_cast<std::size_t>(ns) * d), tgt(static_cast<std::size_t>(nt) * d);
    for (index_t i = 0; i < ns; ++i)
      for (index_t c = 0; c < d; ++c) src[i * d + c] = static_cast<float>(6.0 * ((i % 4) == (c % 4)) + rng.normal());
    for (index_t i = 0; i < nt; ++i)
      for (index_t c = 0; c < d; ++c) tgt[i * d + c] = static_cast<float>(6.0 * ((i % 4) == (c % 4)) + 1.5 * rng.normal());
    MeanShiftState s = meanshift_init(make_point_set(ns, d, src), make_point_set(nt, d, tgt), 12.0, 10, 2);
    for (int step = 0; step < 4; ++step) {
      MeanShiftState want = meanshift_step(s);
      s = gpu::meanshift_step(std::move(s));
      CHECK(rel(s.targets.coords, want.targets.coords) < kTol);
      if (s.iteration % 2 == 0) {
        const KnnGraph g = build_knn(s.targets, s.sources, s.k);
        CHECK(s.knn.neighbor_ids == g.neighbor_ids);
        CHECK(rel(s.knn.neighbor_dists, g.neighbor_dists) < kTol);
      }
      for (double& v : s.targets.coords) v = static_cast<float>(v);
    }
  }
  {  // :356-368 zero weight names the target
    MeanShiftState s = meanshift_init(make_point_set(1, 1, {1e6}), make_point_set(1, 1, {0.0}), 1.0, 1);
    try {
      gpu::meanshift_step(std::move(s));
      CHECK(false);
    } catch (const error& e) {
      CHECK(e.code() == errc::zero_weight);
      CHECK(e.message().find("target 0") != std::string::npos);
    }
  }
  {  // :433-447 iterate_interactions hand values
    const SparseMatrix m = csr_from_coo({{0, 0, 0.0}, {0, 1, 0.0}, {1, 0, 0.0}, {1, 1, 0.0}}, 2, 2);
    HierBlockMatrix h = build_hier_flat(m);
    auto value_fn = [](index_t kappa) {
      return [kappa](index_t i, index_t j, double) { return static_cast<double>((kappa + 1) * (1 + 2 * i + j)); };
    };
    const auto out = gpu::iterate_interactions(h, value_fn, {{{1.0, 1.0}, ""}, {{1.0, -1.0}, ""}});
    CHECK((out[0].values == std::vector<double>{3.0, 7.0}));
    CHECK((out[1].values == std::vector<double>{-2.0, -2.0}));
  }
  {  // Gaussian value model on the device == reference update_values + spmv_hier
    const index_t n = 300, d = 5;
    Rng rng(51);
    std::vector<double> c(static_cast<std::size_t>(n) * d);
    for (double& v : c) v = static_cast<float>(3.0 * rng.normal());
    const PointSet pts = make_point_set(n, d, c);
    const SparsePattern pat = pattern_from_knn(build_knn(pts, pts, 7));
    const OrderingResult ord = order_tree(pts.dim <= 3 ? pts : project(pts, fit_pca(pts, 3)), 16, 12);
    const SparseMatrix m0 = permute(gaussian_values(pat, pts, pts, 1.5), ord.row_perm, ord.col_perm);
    const PointSet pp = permute(pts, ord.row_perm);
    CHECK(gpu::permute(pts, ord.row_perm).coords == pp.coords);  // bit-exact
    HierBlockMatrix h = build_hier(m0, ord.row_tree, ord.col_tree);
    const std::vector<ChargeVector> xs{random_charge(n, 52), random_charge(n, 53)};
    const auto got = gpu::iterate_interactions_gaussian(h, pp, pp, 1.5, xs);
    HierBlockMatrix hr = h;
    for (std::size_t q = 0; q < xs.size(); ++q) {
      update_values(hr, [&](index_t i, index_t j, double) {
        double acc = 0.0;
        for (index_t a = 0; a < d; ++a) {
          const double diff = pp.point(i)[a] - pp.point(j)[a];
          acc += diff * diff;
        }
        return std::exp(-acc / (2.0 * 1.5 * 1.5));
      });
      CHECK(rel(got[q].values, spmv_hier(hr, xs[q]).values) < kTol);
    }
    HierBlockMatrix hg = h;
    CHECK(gpu::update_values_gaussian(hg, pp, pp, 1.5) == static_cast<index_t>(h.nnz));
    CHECK(rel(flatten(hg).values, flatten(hr).values) < kTol);
  }
  {  // resident operator + resident point sets (gpu::Operator / gpu::PointBuffer)
    gpu::Device& dev = gpu::Device::default_device();
    const index_t n = 400, d = 6, k = 9;
    Rng rng(61);
    std::vector<double> c(static_cast<std::size_t>(n) * d), c2(c.size());
    for (double& v : c) v = static_cast<float>(2.0 * rng.normal());
    for (std::size_t q = 0; q < c.size(); ++q) c2[q] = static_cast<float>(c[q] + 0.3 * rng.normal());
    const PointSet pts = make_point_set(n, d, c), tgt = make_point_set(n, d, c2);
    const SparsePattern pat = pattern_from_knn(build_knn(pts, pts, k));
    const SparseMatrix ones{pat, std::vector<double>(pat.entries.size(), 1.0)};
    gpu::Operator op(dev, ones);
    const gpu::PointBuffer pb(dev, pts), tb(dev, tgt);
    // Gaussian recompute: reference gaussian_values + spmv_flat
    const ChargeVector x = random_charge(n, 62);
    CHECK(rel(op.gauss_spmv(tb, pb, 1.3, x).values,
              spmv_flat(gaussian_values(pat, tgt, pts, 1.3), x).values) < kTol);
    // mean shift over the operator's rows: the reference meanshift_step
    MeanShiftState st = meanshift_init(pts, tgt, 1.3, k, 1000);
    const SparsePattern mpat = pattern_from_knn(st.knn);
    gpu::Operator op_ms(dev, SparseMatrix{mpat, std::vector<double>(mpat.entries.size(), 1.0)});
    gpu::PointBuffer tout(dev, n, d);
    op_ms.meanshift(tb, pb, 1.3, tout);
    CHECK(rel(tout.download().coords, meanshift_step(st).targets.coords) < kTol);
    // t-SNE force from the resident P (unchanged) and the fused update
    const SparseMatrix p = random_matrix(64, 700, 63, true);
    gpu::Operator op_p(dev, p);
    std::vector<double> yc(128);
    for (double& v : yc) v = static_cast<float>(rng.normal());
    const PointSet y = make_point_set(64, 2, yc);
    const gpu::PointBuffer yb(dev, y, false);
    gpu::PointBuffer fb(dev, 64, 2, false), yn(dev, 64, 2, false);
    op_p.tsne(yb, fb, 0.5, &yn);
    HierBlockMatrix hr = build_hier_flat(p);
    const PointSet want = tsne_attractive_step(hr, y, 2);
    const PointSet f = fb.download();
    CHECK(rel(f.coords, want.coords) < kTol);
    std::vector<double> p32;
    for (double v : p.values) p32.push_back(static_cast<float>(v));
    CHECK(op_p.values() == p32);
    const PointSet ynew = yn.download();
    std::vector<double> yw(yc.size());
    for (std::size_t q = 0; q < yc.size(); ++q) yw[q] = yc[q] - 0.5 * f.coords[q];
    CHECK(rel(ynew.coords, yw) < 1e-6);  // one fp32 rounding (fused multiply-add)
    expect_errc(errc::dim_mismatch, [&] { op_p.tsne(pb, fb); }, "padded embedding");
  }
  std::printf("test_shim: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
