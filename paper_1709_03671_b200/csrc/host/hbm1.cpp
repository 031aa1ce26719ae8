// HBM1 reader: the reference's on-disk hierarchical
// block-matrix dump (proj/docs/hbm1-format.md; writer proj/src/hier.cpp:291-323)
// parsed straight into the leaf-block arrays the device loader uploads, so an
// ordering + blocked matrix the reference computed once can be reused without
// rebuilding it.  Little-endian only, like the reference.
#include <bit>
#include <climits>
#include <cstring>
#include <fstream>

#include "host.hpp"

namespace knnx {

static_assert(std::endian::native == std::endian::little, "HBM1 is little-endian");

namespace {

struct Reader {
  std::ifstream in;
  std::string path;
  template <typename T>
  T get() {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof v);
    if (!in) throw error(errc::malformed_record, "truncated HBM1 file " + path);
    return v;
  }
  void skip(std::size_t bytes) {
    in.seekg(static_cast<std::streamoff>(bytes), std::ios::cur);
    if (!in) throw error(errc::malformed_record, "truncated HBM1 file " + path);
  }
};

// one partition tree: node begins (for block offsets) and the leaf order
void read_tree(Reader& r, std::vector<index_t>& begin, std::vector<index_t>& forward) {
  const std::uint32_t dim = r.get<std::uint32_t>();
  r.get<std::uint32_t>();  // leaf_capacity
  r.get<std::uint32_t>();  // max_depth
  const std::uint32_t n_points = r.get<std::uint32_t>();
  const std::uint32_t n_nodes = r.get<std::uint32_t>();
  if (dim < 1 || dim > 3) throw error(errc::malformed_record, "HBM1 tree dim out of range");
  begin.resize(n_nodes);
  for (std::uint32_t q = 0; q < n_nodes; ++q) {
    r.skip(2 * dim * sizeof(double));  // lo, hi
    begin[q] = static_cast<index_t>(r.get<std::uint32_t>());
    r.get<std::uint32_t>();  // end
    r.get<std::uint32_t>();  // depth
    r.get<std::uint32_t>();  // parent + 1
    r.get<std::uint8_t>();   // is_leaf
    const std::uint32_t nc = r.get<std::uint32_t>();
    r.skip(nc * sizeof(std::uint32_t));
  }
  if (n_points > static_cast<std::uint32_t>(INT32_MAX))
    throw error(errc::malformed_record, "HBM1 tree point count out of range");
  forward.resize(n_points);
  // the leaf order must be a permutation, as the reference's load_tree
  // enforces through make_permutation (proj/src/core.cpp:94-109)
  std::vector<char> seen(n_points, 0);
  for (std::uint32_t q = 0; q < n_points; ++q) {
    const std::uint32_t f = r.get<std::uint32_t>();
    if (f >= n_points || seen[f])
      throw error(errc::malformed_record, "HBM1 tree leaf order is not a permutation");
    seen[f] = 1;
    forward[q] = static_cast<index_t>(f);
  }
}

}  // namespace

Hbm1 read_hbm1(const std::string& path) {
  Reader r{std::ifstream(path, std::ios::binary), path};
  if (!r.in) throw error(errc::io_error, "cannot open " + path);
  char magic[4];
  r.in.read(magic, 4);
  if (!r.in || std::memcmp(magic, "HBM1", 4) != 0)
    throw error(errc::malformed_record, "missing HBM1 magic in " + path);
  Hbm1 h;
  h.n_rows = static_cast<index_t>(r.get<std::uint32_t>());
  h.n_cols = static_cast<index_t>(r.get<std::uint32_t>());
  h.nnz = static_cast<std::int64_t>(r.get<std::uint64_t>());
  r.get<std::uint32_t>();  // levels
  h.cut_level = static_cast<index_t>(r.get<std::uint32_t>());
  std::vector<index_t> row_begin, col_begin;
  read_tree(r, row_begin, h.row_forward);
  read_tree(r, col_begin, h.col_forward);
  if (static_cast<std::int64_t>(h.row_forward.size()) != h.n_rows ||
      static_cast<std::int64_t>(h.col_forward.size()) != h.n_cols)
    throw error(errc::malformed_record, "HBM1 tree sizes do not match the matrix shape");
  const std::uint32_t n_blocks = r.get<std::uint32_t>();
  h.block_ptr.push_back(0);
  for (std::uint32_t b = 0; b < n_blocks; ++b) {
    r.get<std::uint32_t>();  // level
    const std::uint32_t rn = r.get<std::uint32_t>(), cn = r.get<std::uint32_t>();
    const bool leaf = r.get<std::uint8_t>() != 0;
    if (!leaf) {
      const std::uint32_t nc = r.get<std::uint32_t>();
      r.skip(nc * sizeof(std::uint32_t));
      continue;
    }
    if (rn >= row_begin.size() || cn >= col_begin.size())
      throw error(errc::malformed_record, "HBM1 block references a missing tree node");
    const std::uint64_t nv = r.get<std::uint64_t>();
    h.row_offset.push_back(row_begin[rn]);
    h.col_offset.push_back(col_begin[cn]);
    const std::size_t o = h.lr.size();
    h.lr.resize(o + nv);
    h.lc.resize(o + nv);
    h.vals.resize(o + nv);
    r.in.read(reinterpret_cast<char*>(h.lr.data() + o), static_cast<std::streamsize>(nv * 2));
    r.in.read(reinterpret_cast<char*>(h.lc.data() + o), static_cast<std::streamsize>(nv * 2));
    for (std::uint64_t e = 0; e < nv; ++e) h.vals[o + e] = static_cast<float>(r.get<double>());
    if (!r.in) throw error(errc::malformed_record, "truncated HBM1 leaf payload in " + path);
    h.block_ptr.push_back(static_cast<std::int64_t>(h.lr.size()));
  }
  if (static_cast<std::int64_t>(h.lr.size()) != h.nnz)
    throw error(errc::malformed_record, "HBM1 leaf payload does not add up to nnz");
  return h;
}

}  // namespace knnx
