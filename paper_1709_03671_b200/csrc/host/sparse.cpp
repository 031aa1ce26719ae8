// Host-side sparse formats: canonical CSR from kNN rows, symmetrize, permute
// (the reference's csr_from_coo sort, restated per row), and the cluster-order
// tile format the GPU kernels consume.
#include <algorithm>
#include <numeric>
#include <atomic>
#include <thread>

#include "host.hpp"

namespace knnx {

namespace {

// Runs fn(lo, hi) over [0, n) split across hardware threads (rows are
// independent in every caller, so the result does not depend on the split).
template <typename Fn>
void parallel_rows(index_t n, Fn&& fn) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const index_t workers = static_cast<index_t>(std::min<unsigned>(hw, 32));
  if (workers <= 1 || n < 4096) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const index_t chunk = (n + workers - 1) / workers;
  for (index_t w = 0; w < workers; ++w) {
    const index_t lo = w * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : pool) t.join();
}

}  // namespace

Csr csr_from_knn(const index_t* ids, index_t m, index_t n, index_t k) {
  if (m < 0 || n < 0 || k < 0) throw error(errc::invalid_argument, "negative kNN shape");
  Csr a;
  a.n_rows = m;
  a.n_cols = n;
  a.row_ptr.resize(static_cast<std::size_t>(m) + 1);
  for (index_t i = 0; i <= m; ++i) a.row_ptr[i] = static_cast<std::int64_t>(i) * k;
  a.cols.assign(ids, ids + static_cast<std::size_t>(m) * k);
  std::atomic<bool> bad{false};
  parallel_rows(m, [&](index_t lo, index_t hi) {
    for (index_t i = lo; i < hi; ++i) {
      index_t* row = a.cols.data() + static_cast<std::size_t>(i) * k;
      for (index_t q = 0; q < k; ++q)
        if (row[q] < 0 || row[q] >= n) bad = true;
      std::sort(row, row + k);
      if (std::adjacent_find(row, row + k) != row + k) bad = true;
    }
  });
  if (bad) throw error(errc::out_of_bounds, "kNN ids out of range or repeated within a row");
  return a;
}

Csr symmetrize(const Csr& a) {
  if (a.n_rows != a.n_cols) throw error(errc::not_square, "symmetrize needs a square pattern");
  const index_t n = a.n_rows;
  // transpose pattern
  std::vector<std::int64_t> tptr(static_cast<std::size_t>(n) + 1, 0);
  for (index_t j : a.cols) ++tptr[static_cast<std::size_t>(j) + 1];
  for (index_t i = 0; i < n; ++i) tptr[i + 1] += tptr[i];
  std::vector<index_t> tcols(a.cols.size());
  {
    std::vector<std::int64_t> fill(tptr.begin(), tptr.end() - 1);
    for (index_t i = 0; i < n; ++i)
      for (std::int64_t e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e) tcols[fill[a.cols[e]]++] = i;
  }
  // row-wise sorted union (both inputs are sorted per row; transpose rows are
  // filled in ascending i, hence sorted too)
  std::vector<std::int64_t> len(n);
  parallel_rows(n, [&](index_t lo, index_t hi) {
    for (index_t i = lo; i < hi; ++i) {
      std::int64_t p = a.row_ptr[i], q = tptr[i], c = 0;
      const std::int64_t pe = a.row_ptr[i + 1], qe = tptr[i + 1];
      while (p < pe || q < qe) {
        if (q >= qe || (p < pe && a.cols[p] < tcols[q])) ++p;
        else if (p >= pe || tcols[q] < a.cols[p]) ++q;
        else { ++p; ++q; }
        ++c;
      }
      len[i] = c;
    }
  });
  Csr s;
  s.n_rows = s.n_cols = n;
  s.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  for (index_t i = 0; i < n; ++i) s.row_ptr[i + 1] = s.row_ptr[i] + len[i];
  s.cols.resize(static_cast<std::size_t>(s.row_ptr[n]));
  parallel_rows(n, [&](index_t lo, index_t hi) {
    for (index_t i = lo; i < hi; ++i) {
      std::int64_t p = a.row_ptr[i], q = tptr[i], o = s.row_ptr[i];
      const std::int64_t pe = a.row_ptr[i + 1], qe = tptr[i + 1];
      while (p < pe || q < qe) {
        if (q >= qe || (p < pe && a.cols[p] < tcols[q])) s.cols[o++] = a.cols[p++];
        else if (p >= pe || tcols[q] < a.cols[p]) s.cols[o++] = tcols[q++];
        else { s.cols[o++] = a.cols[p++]; ++q; }
      }
    }
  });
  return s;
}

Csr symmetrize_values(const Csr& a, double scale) {
  if (a.vals.empty()) throw error(errc::invalid_argument, "symmetrize_values needs stored values");
  if (a.n_rows != a.n_cols) throw error(errc::not_square, "symmetrize needs a square pattern");
  Csr s = symmetrize(a);  // union pattern, rows sorted
  const index_t n = a.n_rows;
  // transpose with values (rows filled in ascending source row: sorted)
  std::vector<std::int64_t> tptr(static_cast<std::size_t>(n) + 1, 0);
  for (index_t j : a.cols) ++tptr[static_cast<std::size_t>(j) + 1];
  for (index_t i = 0; i < n; ++i) tptr[i + 1] += tptr[i];
  std::vector<index_t> tcols(a.cols.size());
  std::vector<float> tvals(a.cols.size());
  {
    std::vector<std::int64_t> fill(tptr.begin(), tptr.end() - 1);
    for (index_t i = 0; i < n; ++i)
      for (std::int64_t e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e) {
        const std::int64_t o = fill[a.cols[e]]++;
        tcols[o] = i;
        tvals[o] = a.vals[e];
      }
  }
  s.vals.assign(s.cols.size(), 0.0f);
  // v_ij = scale * (a_ij + a_ji), summed in double, rows independent
  parallel_rows(n, [&](index_t lo, index_t hi) {
    for (index_t i = lo; i < hi; ++i) {
      std::int64_t p = a.row_ptr[i], q = tptr[i];
      for (std::int64_t o = s.row_ptr[i]; o < s.row_ptr[i + 1]; ++o) {
        const index_t c = s.cols[o];
        double v = 0.0;
        if (p < a.row_ptr[i + 1] && a.cols[p] == c) v += a.vals[p++];
        if (q < tptr[i + 1] && tcols[q] == c) v += tvals[q++];
        s.vals[o] = static_cast<float>(scale * v);
      }
    }
  });
  return s;
}

Csr permute(const Csr& a, const std::vector<index_t>& row_fwd, const std::vector<index_t>& col_fwd) {
  if (static_cast<index_t>(row_fwd.size()) != a.n_rows ||
      static_cast<index_t>(col_fwd.size()) != a.n_cols)
    throw error(errc::size_mismatch, "permutation sizes do not match matrix shape");
  std::vector<index_t> row_inv(a.n_rows, -1);
  for (index_t i = 0; i < a.n_rows; ++i) {
    const index_t r = row_fwd[i];
    if (r < 0 || r >= a.n_rows || row_inv[r] != -1)
      throw error(errc::invalid_argument, "row permutation is not a bijection");
    row_inv[r] = i;
  }
  Csr b;
  b.n_rows = a.n_rows;
  b.n_cols = a.n_cols;
  b.row_ptr.assign(static_cast<std::size_t>(a.n_rows) + 1, 0);
  for (index_t r = 0; r < a.n_rows; ++r)
    b.row_ptr[r + 1] = b.row_ptr[r] + (a.row_ptr[row_inv[r] + 1] - a.row_ptr[row_inv[r]]);
  b.cols.resize(a.cols.size());
  const bool has_vals = !a.vals.empty();
  if (has_vals) b.vals.resize(a.vals.size());
  parallel_rows(a.n_rows, [&](index_t lo, index_t hi) {
    std::vector<std::pair<index_t, float>> buf;
    for (index_t r = lo; r < hi; ++r) {
      const index_t i = row_inv[r];
      buf.clear();
      for (std::int64_t e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e)
        buf.emplace_back(col_fwd[a.cols[e]], has_vals ? a.vals[e] : 0.0f);
      std::sort(buf.begin(), buf.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      std::int64_t o = b.row_ptr[r];
      for (const auto& [c, v] : buf) {
        b.cols[o] = c;
        if (has_vals) b.vals[o] = v;
        ++o;
      }
    }
  });
  return b;
}

std::vector<index_t> locality_schedule(const Csr& a, index_t col_base) {
  const index_t m = a.n_rows;
  std::vector<index_t> order;
  order.reserve(m);
  std::vector<char> seen(m, 0);
  for (index_t root = 0; root < m; ++root) {
    if (seen[root]) continue;
    seen[root] = 1;
    std::size_t head = order.size();
    order.push_back(root);
    while (head < order.size()) {
      const index_t r = order[head++];
      for (std::int64_t e = a.row_ptr[r]; e < a.row_ptr[r + 1]; ++e) {
        const std::int64_t c = static_cast<std::int64_t>(a.cols[e]) - col_base;
        if (c < 0 || c >= m || seen[c]) continue;
        seen[c] = 1;
        order.push_back(static_cast<index_t>(c));
      }
    }
  }
  return order;
}

ClusterTiles build_cluster_tiles(const Csr& a, index_t tile_rows, const index_t* schedule,
                                 bool with_halos) {
  if (tile_rows < 32 || tile_rows % 32 != 0 || tile_rows > 1024)
    throw error(errc::invalid_argument, "tile_rows must be a multiple of 32 in [32, 1024]");
  ClusterTiles t;
  t.n_rows = a.n_rows;
  t.n_cols = a.n_cols;
  t.tile_rows = tile_rows;
  t.n_tiles = (a.n_rows + tile_rows - 1) / tile_rows;
  t.nnz = a.nnz();
  const index_t n_slices = (a.n_rows + 31) / 32;
  // SELL-C-sigma with sigma = one tile: when row lengths vary, the rows of
  // each tile are laid out longest first so the 32-row slices pad little;
  // slot_row maps a slot back to its row (empty = identity for uniform rows)
  std::vector<index_t> len(a.n_rows), slot_row(a.n_rows);
  bool uniform = true, scheduled = false;
  for (index_t i = 0; i < a.n_rows; ++i) {
    len[i] = static_cast<index_t>(a.row_ptr[i + 1] - a.row_ptr[i]);
    uniform = uniform && len[i] == len[0];
    slot_row[i] = schedule ? schedule[i] : i;
    scheduled = scheduled || slot_row[i] != i;
  }
  if (schedule) {
    std::vector<char> hit(a.n_rows, 0);
    for (index_t i = 0; i < a.n_rows; ++i) {
      if (slot_row[i] < 0 || slot_row[i] >= a.n_rows || hit[slot_row[i]])
        throw error(errc::invalid_argument, "schedule is not a permutation of the rows");
      hit[slot_row[i]] = 1;
    }
  }
  if (!uniform)
    for (index_t tile = 0; tile < t.n_tiles; ++tile) {
      const index_t r0 = tile * tile_rows, r1 = std::min(a.n_rows, r0 + tile_rows);
      std::stable_sort(slot_row.begin() + r0, slot_row.begin() + r1,
                       [&](index_t x, index_t y) { return len[x] > len[y]; });
    }
  t.row_len.resize(a.n_rows);
  for (index_t p = 0; p < a.n_rows; ++p) t.row_len[p] = len[slot_row[p]];
  t.slice_len.assign(n_slices, 0);
  t.slice_off.assign(static_cast<std::size_t>(n_slices) + 1, 0);
  for (index_t s = 0; s < n_slices; ++s) {
    index_t mx = 0;
    for (index_t r = s * 32; r < std::min(a.n_rows, s * 32 + 32); ++r) mx = std::max(mx, t.row_len[r]);
    t.slice_len[s] = mx;
    t.slice_off[s + 1] = t.slice_off[s] + static_cast<std::int64_t>(mx) * 32;
  }
  t.stored = t.slice_off[n_slices];
  const bool has_vals = !a.vals.empty();
  if (has_vals) t.vals.assign(static_cast<std::size_t>(t.stored), 0.0f);
  if (!with_halos) {
    // original order: the SELL slices and values only -- no halos, so no
    // 16-bit local-index limit (the int32 columns are placed by the caller)
    if (has_vals)
      parallel_rows(a.n_rows, [&](index_t lo, index_t hi) {
        for (index_t p = lo; p < hi; ++p) {
          const index_t r = slot_row[p];
          for (std::int64_t e = a.row_ptr[r]; e < a.row_ptr[r + 1]; ++e)
            t.vals[t.slice_off[p / 32] + (e - a.row_ptr[r]) * 32 + p % 32] = a.vals[e];
        }
      });
    if (!uniform || scheduled) t.slot_row = std::move(slot_row);
    t.halo_off.assign(static_cast<std::size_t>(t.n_tiles) + 1, 0);
    return t;
  }
  t.lidx.assign(static_cast<std::size_t>(t.stored), 0);

  // per-tile halos (sorted unique columns), built in parallel then concatenated
  std::vector<std::vector<index_t>> halos(t.n_tiles);
  std::atomic<bool> overflow{false};
  parallel_rows(t.n_tiles, [&](index_t lo, index_t hi) {
    for (index_t tile = lo; tile < hi; ++tile) {
      const index_t r0 = tile * tile_rows, r1 = std::min(a.n_rows, r0 + tile_rows);
      std::vector<index_t>& h = halos[tile];
      h.clear();
      for (index_t p = r0; p < r1; ++p)
        h.insert(h.end(), a.cols.begin() + a.row_ptr[slot_row[p]], a.cols.begin() + a.row_ptr[slot_row[p] + 1]);
      std::sort(h.begin(), h.end());
      h.erase(std::unique(h.begin(), h.end()), h.end());
      if (h.size() > 65536) {
        overflow = true;
        continue;
      }
      for (index_t p = r0; p < r1; ++p) {
        const index_t r = slot_row[p];
        const index_t s = p / 32, lane = p % 32;
        for (std::int64_t e = a.row_ptr[r]; e < a.row_ptr[r + 1]; ++e) {
          const std::int64_t q = e - a.row_ptr[r];
          const std::int64_t dst = t.slice_off[s] + q * 32 + lane;
          t.lidx[dst] = static_cast<std::uint16_t>(
              std::lower_bound(h.begin(), h.end(), a.cols[e]) - h.begin());
          if (has_vals) t.vals[dst] = a.vals[e];
        }
      }
    }
  });
  if (overflow)
    throw error(errc::local_index_overflow,
                "a tile references more than 65536 distinct columns; use smaller tiles");
  if (!uniform || scheduled) t.slot_row = std::move(slot_row);
  // each tile's halo list is padded to a multiple of 4 ids (16 bytes) so the
  // device can fetch it with one bulk copy; padding repeats the last id
  t.halo_off.assign(static_cast<std::size_t>(t.n_tiles) + 1, 0);
  for (index_t tile = 0; tile < t.n_tiles; ++tile) {
    const std::int64_t padded = (static_cast<std::int64_t>(halos[tile].size()) + 3) / 4 * 4;
    t.halo_off[tile + 1] = t.halo_off[tile] + padded;
    t.max_halo = std::max(t.max_halo, static_cast<index_t>(padded));
  }
  t.halo_ids.assign(static_cast<std::size_t>(t.halo_off[t.n_tiles]), 0);
  for (index_t tile = 0; tile < t.n_tiles; ++tile) {
    std::copy(halos[tile].begin(), halos[tile].end(), t.halo_ids.begin() + t.halo_off[tile]);
    const index_t fill = halos[tile].empty() ? 0 : halos[tile].back();
    for (std::int64_t q = t.halo_off[tile] + static_cast<std::int64_t>(halos[tile].size());
         q < t.halo_off[tile + 1]; ++q)
      t.halo_ids[q] = fill;
  }
  return t;
}

}  // namespace knnx
