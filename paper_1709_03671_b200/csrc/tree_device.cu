// Partition tree on the device (the build_tree half;
// reference: proj/src/tree.cpp:15-112 -- cube root box, centre split into
// orthants, stable buckets, leaf_capacity / max_depth).  The reference (and
// the host build in csrc/host/pca_tree.cpp) recurses over point ranges; here
// the same tree comes out of two sorts:
//   1. every point walks the implicit octree from the root box on its own and
//      records its orthant path (3 bits per level, the reference's centre
//      arithmetic 0.5 * (lo + hi) with separately rounded fp64 add and multiply);
//   2. a stable radix sort by path puts every node's points in one run, so a
//      point's leaf is the shallowest prefix whose run holds at most
//      leaf_capacity points (two binary searches per level);
//   3. a second stable sort, by the path truncated at the leaf, from the
//      original index order gives the leaf order: inside a leaf the points
//      keep ascending original index, exactly what the reference's stable
//      bucket passes leave behind.
// The node array (pre-order ids, boxes, children) is rebuilt on the host from
// the leaf runs.  The result equals the host build field for field
// (tests/test_gpu_parity.py) and, through it, the reference's permutation.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "host/host.hpp"

namespace knnx_dev {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw knnx::error(knnx::errc::cuda_error, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Box {
  double lo[3], hi[3];
};

// orthant path of every point, level 0 in the most significant position
__global__ void path_kernel(const double* __restrict__ emb, int n, int dim, Box root, int max_depth,
                            unsigned long long* __restrict__ code) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double lo[3], hi[3], x[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = root.lo[a];
    hi[a] = root.hi[a];
    x[a] = a < dim ? emb[static_cast<int64_t>(i) * dim + a] : 0.0;
  }
  unsigned long long c = 0;
  for (int l = 0; l < max_depth; ++l) {
    unsigned orth = 0;
    for (int a = 0; a < dim; ++a) {
      const double ctr = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      if (x[a] >= ctr) {
        orth |= 1u << a;
        lo[a] = ctr;
      } else {
        hi[a] = ctr;
      }
    }
    c = (c << 3) | orth;
  }
  code[i] = c;
}

__device__ __forceinline__ int lower_bound(const unsigned long long* a, int lo, int hi, unsigned long long v) {
  while (lo < hi) {
    const int mid = lo + ((hi - lo) >> 1);
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// sorted position i: depth of the leaf holding it and its path truncated there,
// scattered to the point's original index
__global__ void leaf_kernel(const unsigned long long* __restrict__ sorted, const int32_t* __restrict__ idx, int n,
                            int leaf_capacity, int max_depth, unsigned long long* __restrict__ key_by_idx,
                            int32_t* __restrict__ depth_by_idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long c = sorted[i];
  int lo = 0, hi = n, depth = max_depth;
  for (int l = 0; l < max_depth; ++l) {
    const int shift = 3 * (max_depth - l);
    if (l > 0) {  // the run of this point's l-level prefix, inside its parent's run
      const unsigned long long first = (c >> shift) << shift;
      const int nlo = lower_bound(sorted, lo, hi, first);
      const int nhi = lower_bound(sorted, nlo, hi, first + (1ull << shift));
      lo = nlo;
      hi = nhi;
    }
    if (hi - lo <= leaf_capacity) {
      depth = l;
      break;
    }
  }
  const int shift = 3 * (max_depth - depth);
  const int orig = idx[i];
  key_by_idx[orig] = shift >= 64 ? 0ull : (c >> shift) << shift;
  depth_by_idx[orig] = depth;
}

__global__ void iota_kernel(int32_t* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

struct Leaf {
  unsigned long long key;
  int32_t depth, begin, end;
};

// nodes in the reference's creation order: a node, then for every non-empty
// orthant in code order the child and, at once, the child's whole subtree
void grow(knnx::PartitionTree& t, const std::vector<Leaf>& leaves, int32_t node_id, int32_t depth,
          std::size_t l0, std::size_t l1) {
  t.nodes[node_id].begin = leaves[l0].begin;
  t.nodes[node_id].end = leaves[l1 - 1].end;
  t.nodes[node_id].depth = depth;
  if (l1 - l0 == 1 && leaves[l0].depth == depth) {
    t.nodes[node_id].is_leaf = true;
    return;
  }
  const int32_t dim = t.dim;
  std::array<double, 3> ctr{};
  for (int32_t a = 0; a < dim; ++a) ctr[a] = 0.5 * (t.nodes[node_id].lo[a] + t.nodes[node_id].hi[a]);
  const int shift = 3 * (t.max_depth - depth - 1);
  std::size_t p = l0;
  while (p < l1) {
    const unsigned orth = static_cast<unsigned>((leaves[p].key >> shift) & 7u);
    std::size_t q = p;
    while (q < l1 && static_cast<unsigned>((leaves[q].key >> shift) & 7u) == orth) ++q;
    const int32_t child = static_cast<int32_t>(t.nodes.size());
    t.nodes.emplace_back();
    t.nodes[child].parent = node_id;
    for (int32_t a = 0; a < dim; ++a) {
      const bool high = (orth >> a) & 1u;
      t.nodes[child].lo[a] = high ? ctr[a] : t.nodes[node_id].lo[a];
      t.nodes[child].hi[a] = high ? t.nodes[node_id].hi[a] : ctr[a];
    }
    t.nodes[node_id].children.push_back(child);
    grow(t, leaves, child, depth + 1, p, q);
    p = q;
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) { ck(cudaMalloc(&p, sizeof(T) * std::max<std::size_t>(1, n)), "cudaMalloc (tree)"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

knnx::PartitionTree build_tree_device(const double* emb, int n, int dim, int leaf_capacity, int max_depth,
                                      int device) {
  using knnx::errc;
  if (dim < 1 || dim > 3)
    throw knnx::error(errc::dim_too_high, "partition tree supports dim 1..3, got " + std::to_string(dim));
  if (leaf_capacity < 1) throw knnx::error(errc::invalid_argument, "leaf_capacity must be >= 1");
  if (max_depth < 1) throw knnx::error(errc::invalid_argument, "max_depth must be >= 1");
  if (max_depth > 21) throw knnx::error(errc::unsupported, "device tree build packs at most 21 levels");
  knnx::PartitionTree t;
  t.dim = dim;
  t.leaf_capacity = leaf_capacity;
  t.max_depth = max_depth;
  t.n_points = n;
  t.nodes.emplace_back();
  // root cube: the bounding box widened to its longest side around its centre
  // (proj/src/tree.cpp:84-101)
  std::array<double, 3> lo{}, hi{};
  for (int a = 0; a < dim; ++a) lo[a] = hi[a] = n > 0 ? emb[a] : 0.0;
  for (int i = 1; i < n; ++i)
    for (int a = 0; a < dim; ++a) {
      const double v = emb[static_cast<std::size_t>(i) * dim + a];
      lo[a] = std::min(lo[a], v);
      hi[a] = std::max(hi[a], v);
    }
  double side = 0.0;
  for (int a = 0; a < dim; ++a) side = std::max(side, hi[a] - lo[a]);
  Box root{};
  for (int a = 0; a < dim; ++a) {
    const double c = 0.5 * (lo[a] + hi[a]);
    t.nodes[0].lo[a] = root.lo[a] = c - 0.5 * side;
    t.nodes[0].hi[a] = root.hi[a] = c + 0.5 * side;
  }
  t.forward.assign(n, 0);
  if (n == 0) {
    t.nodes[0].is_leaf = true;
    return t;
  }
  int prev = -1;
  cudaGetDevice(&prev);
  ck(cudaSetDevice(device), "cudaSetDevice");
  std::vector<int32_t> order(n), depth_sorted(n);
  std::vector<unsigned long long> key_sorted(n);
  {
    DevBuf<double> d_emb(static_cast<std::size_t>(n) * dim);
    DevBuf<unsigned long long> code(n), code_s(n), key(n), key_s(n);
    DevBuf<int32_t> idx(n), idx_s(n), dep(n), dep_s(n), ord(n);
    ck(cudaMemcpy(d_emb.p, emb, sizeof(double) * static_cast<std::size_t>(n) * dim, cudaMemcpyHostToDevice),
       "upload embedding");
    const int grid = (n + 255) / 256;
    path_kernel<<<grid, 256>>>(d_emb.p, n, dim, root, max_depth, code.p);
    iota_kernel<<<grid, 256>>>(idx.p, n);
    const int bits = 3 * max_depth;
    std::size_t tmp_bytes = 0, tmp2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, code.p, code_s.p, idx.p, idx_s.p, n, 0, bits);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp2, key.p, key_s.p, idx.p, ord.p, n, 0, bits);
    DevBuf<unsigned char> tmp(std::max(tmp_bytes, tmp2));
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, code.p, code_s.p, idx.p, idx_s.p, n, 0, bits), "sort paths");
    leaf_kernel<<<grid, 256>>>(code_s.p, idx_s.p, n, leaf_capacity, max_depth, key.p, dep.p);
    // leaf order: stable sort by truncated path from the original index order
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tmp2, key.p, key_s.p, idx.p, ord.p, n, 0, bits), "sort leaves");
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tmp2, key.p, key_s.p, dep.p, dep_s.p, n, 0, bits), "sort depths");
    ck(cudaGetLastError(), "tree kernels");
    ck(cudaMemcpy(order.data(), ord.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost), "download order");
    ck(cudaMemcpy(key_sorted.data(), key_s.p, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost),
       "download keys");
    ck(cudaMemcpy(depth_sorted.data(), dep_s.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost), "download depths");
  }
  if (prev >= 0 && prev != device) cudaSetDevice(prev);
  for (int pos = 0; pos < n; ++pos) t.forward[order[pos]] = pos;
  std::vector<Leaf> leaves;
  for (int pos = 0; pos < n;) {
    int q = pos;
    while (q < n && key_sorted[q] == key_sorted[pos] && depth_sorted[q] == depth_sorted[pos]) ++q;
    leaves.push_back({key_sorted[pos], depth_sorted[pos], pos, q});
    pos = q;
  }
  grow(t, leaves, 0, 0, 0, leaves.size());
  return t;
}

}  // namespace knnx_dev
