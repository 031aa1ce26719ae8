// Operator construction from a CSR that already lives on the device (SURVEY.md
// §8f next #2; the device counterpart of proj/src/core.cpp:75-92,130-139 +
// hier.cpp:84-155 for the original-order layout): the breadth-first row
// schedule, the SELL-C-sigma sort of each 256-row tile, the slice offsets and
// the entry placement (plain or group-interleaved) all run on the device, so a
// graph produced by knnx_tsne_affinities_dev (C4: 6.0e8 entries) never crosses
// PCIe.  Every array equals what knnx_op_create_csr_ex builds on the host from
// the same CSR (tests/test_gpu_build.py compares results and values).
#include <cuda_runtime.h>

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "knnx_internal.cuh"
#include "knnx_rt.cuh"

using namespace knnx_rt;

namespace {

constexpr int kTile = 256;
constexpr unsigned long long kUnseen = ~0ull;

struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    check(cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), st), "cudaMallocAsync (operator build)");
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// ---- validation: row_ptr monotone from 0 to nnz, columns in range and
// strictly increasing within a row (the canonical CSR of core.cpp:75-92)
__global__ void validate_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                const float* __restrict__ vals, int n_rows, int n_cols, int64_t nnz,
                                int* __restrict__ err) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  // a row block of a larger CSR starts at rp[0] != 0: offsets are relative to it
  const int64_t base = rp[0];
  const int64_t e0 = rp[r], e1 = rp[r + 1];
  if (base < 0 || e1 < e0 || e1 - base > nnz || (r == n_rows - 1 && e1 - base != nnz)) {
    atomicMax(err, 1);
    return;
  }
  int prev = -1;
  for (int64_t e = e0; e < e1; ++e) {
    const int c = cols[e];
    if (c < 0 || c >= n_cols) atomicMax(err, 2);
    else if (c <= prev) atomicMax(err, 3);
    prev = c;
    if (vals && !isfinite(vals[e])) atomicMax(err, 4);
  }
}

// ---- breadth-first schedule, identical to the host's queue order
// (knnx::locality_schedule): a node joins the next level at the position of
// its first discovery, i.e. ordered by (position of the parent in the current
// level, index of the edge in the parent's row)

__global__ void bfs_init_kernel(unsigned long long* key, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = kUnseen;
}

// smallest unseen row in [lo, hi) -> *out (left at its 0x7f7f7f7f fill when none)
__global__ void bfs_next_root_kernel(const unsigned long long* __restrict__ key, int lo, int hi,
                                     int* __restrict__ out) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  const bool hit = i < hi && key[i] == kUnseen;
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicMin(out, i);
}

// warp per frontier node: every unseen neighbour gets the smallest (pos, edge)
__global__ void bfs_expand_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                  const int32_t* __restrict__ order, int lo, int hi, int col_base, int m,
                                  unsigned long long* __restrict__ key) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int pos = lo + w;
  if (pos >= hi) return;
  const int u = order[pos];
  const int64_t e0 = rp[u], e1 = rp[u + 1];
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int64_t c = static_cast<int64_t>(cols[e]) - col_base;
    if (c < 0 || c >= m) continue;
    const unsigned long long k = (static_cast<unsigned long long>(w + 1) << 32) |
                                 static_cast<unsigned long long>(e - e0);
    // key: ~0 = unseen, 0 = placed (sealed after its level), else the best
    // (parent position, edge) found so far in this level
    if (key[c] > k) atomicMin(&key[c], k);
  }
}

// number of edges of frontier node w that won their target
__global__ void bfs_count_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                 const int32_t* __restrict__ order, int lo, int hi, int col_base, int m,
                                 const unsigned long long* __restrict__ key, int* __restrict__ cnt) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int pos = lo + w;
  if (pos >= hi) return;
  const int u = order[pos];
  const int64_t e0 = rp[u], e1 = rp[u + 1];
  int n = 0;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int64_t c = static_cast<int64_t>(cols[e]) - col_base;
    if (c < 0 || c >= m) continue;
    const unsigned long long k = (static_cast<unsigned long long>(w + 1) << 32) |
                                 static_cast<unsigned long long>(e - e0);
    n += key[c] == k ? 1 : 0;
  }
  n = __reduce_add_sync(0xffffffffu, n);
  if (lane == 0) cnt[w] = n;
}

// winners of frontier node w, in edge order, to order[hi + start[w] ...]
__global__ void bfs_emit_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                int32_t* __restrict__ order, int lo, int hi, int col_base, int m,
                                const unsigned long long* __restrict__ key, const int* __restrict__ start) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int pos = lo + w;
  if (pos >= hi) return;
  const int u = order[pos];
  const int64_t e0 = rp[u], e1 = rp[u + 1];
  int out = hi + start[w];
  for (int64_t eb = e0; eb < e1; eb += 32) {
    const int64_t e = eb + lane;
    bool win = false;
    int c32 = 0;
    if (e < e1) {
      const int64_t c = static_cast<int64_t>(cols[e]) - col_base;
      if (c >= 0 && c < m) {
        const unsigned long long k = (static_cast<unsigned long long>(w + 1) << 32) |
                                     static_cast<unsigned long long>(e - e0);
        win = key[c] == k;
        c32 = static_cast<int>(c);
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, win);
    if (win) order[out + __popc(b & ((1u << lane) - 1u))] = c32;
    out += __popc(b);
  }
}

// placed rows must never be rediscovered: their key drops to 0
__global__ void bfs_seal_kernel(const int32_t* __restrict__ order, int lo, int hi,
                                unsigned long long* __restrict__ key) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi) key[order[i]] = 0;
}

// ---- SELL-C-sigma: stable sort of each tile's slots by row length, longest first
__global__ void __launch_bounds__(kTile)
    tile_sort_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ sched, int n_rows,
                     int32_t* __restrict__ slot_row, int32_t* __restrict__ row_len) {
  using Sort = cub::BlockRadixSort<uint32_t, kTile, 1, int32_t>;
  __shared__ typename Sort::TempStorage tmp;
  const int p = blockIdx.x * kTile + threadIdx.x;
  uint32_t key[1] = {0xFFFFFFFFu};
  int32_t val[1] = {-1};
  if (p < n_rows) {
    const int r = sched ? sched[p] : p;
    key[0] = 0xFFFFFFFFu - static_cast<uint32_t>(rp[r + 1] - rp[r]);
    val[0] = r;
  }
  Sort(tmp).Sort(key, val);  // LSD radix sort: stable, so ties keep the schedule order
  if (p < n_rows) {
    slot_row[p] = val[0];
    row_len[p] = static_cast<int32_t>(0xFFFFFFFFu - key[0]);
  }
}

// per 32-slot slice: stored length (the longest row, padded to 8 entries for
// the group-interleaved layout); minmax = {shortest row, longest stored slice,
// longest row}
__global__ void slice_len_kernel(const int32_t* __restrict__ row_len, int n_rows, int interleave,
                                 int32_t* __restrict__ slice_len, int64_t* __restrict__ slice_elems,
                                 int32_t* __restrict__ minmax) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int len = p < n_rows ? row_len[p] : 0;
  const int mx = __reduce_max_sync(0xffffffffu, len);
  const int mn = __reduce_min_sync(0xffffffffu, p < n_rows ? len : 0x7fffffff);
  if ((threadIdx.x & 31) == 0 && p < n_rows) {
    const int stored = interleave ? (mx + 7) / 8 * 8 : mx;
    slice_len[p >> 5] = stored;
    slice_elems[p >> 5] = static_cast<int64_t>(stored) * 32;
    atomicMin(&minmax[0], mn);
    atomicMax(&minmax[1], stored);
    atomicMax(&minmax[2], mx);
  }
}

// warp per slot: entry q of the slot's row to its stored position
__global__ void place_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                             const float* __restrict__ vals, const int32_t* __restrict__ slot_row,
                             const int64_t* __restrict__ slice_off, int n_rows, int interleave,
                             int32_t* __restrict__ out_cols, float* __restrict__ out_vals) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (p >= n_rows) return;
  const int r = slot_row[p];
  const int64_t e0 = rp[r], len = rp[r + 1] - e0;
  const int64_t base = slice_off[p >> 5];
  const int pl = p & 31;
  for (int64_t q = lane; q < len; q += 32) {
    const int64_t dst = interleave ? base + (q >> 3) * 256 + pl * 8 + (q & 7) : base + 32 * q + pl;
    out_cols[dst] = cols[e0 + q];
    if (vals) out_vals[dst] = vals[e0 + q];
  }
}

template <typename T>
std::vector<T> download(const T* d, size_t n, cudaStream_t st) {
  std::vector<T> h(n);
  if (n) check(cudaMemcpyAsync(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, st), "download");
  return h;
}

// Level-synchronous traversal costs a few launches and one host round trip
// per level; a graph of very many tiny components (each a root search plus a
// level or two) would spend minutes there, so past this many host iterations
// the schedule is finished by the host function on a downloaded pattern (the
// result is the same order either way).
constexpr int64_t kMaxDeviceBfsSteps = 20000;

// the host's locality_schedule (csrc/host/sparse.cpp) on the device; returns
// null when the step budget ran out
int32_t* device_schedule(knnx_ctx_t ctx, Scratch& ws, const int64_t* rp, const int32_t* cols, int m,
                         int col_base) {
  cudaStream_t st = ctx->stream;
  int32_t* order = ws.get<int32_t>(m);
  unsigned long long* key = ws.get<unsigned long long>(m);
  int* cnt = ws.get<int>(m + 1);
  int* start = ws.get<int>(m + 1);
  int* d_root = ws.get<int>(1);
  bfs_init_kernel<<<(m + 255) / 256, 256, 0, st>>>(key, m);
  size_t scan_bytes = 0;
  check(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, start, m + 1, st), "scan size");
  void* scan_tmp = ws.get<unsigned char>(scan_bytes);
  int placed = 0, cursor = 0;
  int64_t launches = 1, steps = 0;
  while (placed < m) {
    if (++steps > kMaxDeviceBfsSteps) {
      ctx->launches += launches;
      return nullptr;
    }
    // next root: the smallest unseen row (rows before the cursor are all placed)
    int root = 0x7fffffff;
    for (int lo = cursor; lo < m && root == 0x7fffffff; lo += (1 << 20)) {
      const int hi = std::min(m, lo + (1 << 20));
      check(cudaMemsetAsync(d_root, 0x7f, sizeof(int), st), "memset");
      bfs_next_root_kernel<<<(hi - lo + 255) / 256, 256, 0, st>>>(key, lo, hi, d_root);
      check(cudaMemcpyAsync(&root, d_root, sizeof(int), cudaMemcpyDeviceToHost, st), "root");
      check(cudaStreamSynchronize(st), "sync");
      ++launches;
      if (root >= 0x7f7f7f7f) root = 0x7fffffff;
    }
    require(root != 0x7fffffff, knnx::errc::invalid_argument, "schedule: no unseen row left");
    cursor = root + 1;
    check(cudaMemcpyAsync(order + placed, &root, sizeof(int), cudaMemcpyHostToDevice, st), "root");
    int lo = placed, hi = placed + 1;
    bfs_seal_kernel<<<1, 256, 0, st>>>(order, lo, hi, key);
    while (lo < hi) {
      ++steps;
      const int nf = hi - lo;
      const int grid = static_cast<int>((static_cast<int64_t>(nf) * 32 + 255) / 256);
      bfs_expand_kernel<<<grid, 256, 0, st>>>(rp, cols, order, lo, hi, col_base, m, key);
      bfs_count_kernel<<<grid, 256, 0, st>>>(rp, cols, order, lo, hi, col_base, m, key, cnt);
      check(cudaMemsetAsync(cnt + nf, 0, sizeof(int), st), "memset");
      check(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, start, nf + 1, st), "scan");
      bfs_emit_kernel<<<grid, 256, 0, st>>>(rp, cols, order, lo, hi, col_base, m, key, start);
      int n_new = 0;
      check(cudaMemcpyAsync(&n_new, start + nf, sizeof(int), cudaMemcpyDeviceToHost, st), "level size");
      check(cudaStreamSynchronize(st), "sync");
      launches += 4;
      lo = hi;
      hi += n_new;
      if (n_new > 0) {
        bfs_seal_kernel<<<(n_new + 255) / 256, 256, 0, st>>>(order, lo, hi, key);
        ++launches;
      }
    }
    placed = hi;
  }
  ctx->launches += launches;
  return order;
}

}  // namespace

extern "C" int knnx_op_create_csr_dev(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                                      const int64_t* row_ptr, const int32_t* cols, const float* vals,
                                      int32_t schedule_kind, int32_t col_base, const int32_t* schedule,
                                      int32_t options, knnx_op_t* out) {
  return guard([&] {
    require(ctx != nullptr && out != nullptr, knnx::errc::invalid_argument, "null handle");
    require(n_rows >= 0 && n_cols >= 0 && nnz >= 0, knnx::errc::invalid_argument, "negative shape");
    require(n_rows == 0 || (row_ptr != nullptr && (nnz == 0 || cols != nullptr)),
            knnx::errc::invalid_argument, "null CSR array");
    require(schedule_kind >= KNNX_SCHEDULE_NONE && schedule_kind <= KNNX_SCHEDULE_GIVEN,
            knnx::errc::invalid_argument, "unknown schedule kind");
    require(schedule_kind != KNNX_SCHEDULE_GIVEN || n_rows == 0 || schedule != nullptr,
            knnx::errc::invalid_argument, "null schedule");
    require((options & ~KNNX_OPT_GROUP_INTERLEAVE) == 0, knnx::errc::unsupported,
            "the device build supports KNNX_OPT_GROUP_INTERLEAVE only");
    require(col_base >= 0, knnx::errc::invalid_argument, "negative col_base");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = ctx->stream;
    Scratch ws(st);
    auto op = std::make_unique<knnx_operator>();
    op->ctx = ctx;
    op->n_rows = n_rows;
    op->n_cols = n_cols;
    op->order = KNNX_ORDER_ORIGINAL;
    op->nnz = nnz;
    op->has_vals = vals != nullptr;
    op->interleave = (options & KNNX_OPT_GROUP_INTERLEAVE) ? 8 : 0;
    op->tile_rows = kTile;
    op->n_tiles = (n_rows + kTile - 1) / kTile;
    op->n_slices = (n_rows + 31) / 32;
    if (n_rows == 0) {
      op->h_row_ptr.assign(1, 0);
      op->h_slice_off.assign(1, 0);
      ++ctx->live_ops;
      *out = op.release();
      return KNNX_OK;
    }
    // 1. validate
    int* d_err = ws.get<int>(1);
    check(cudaMemsetAsync(d_err, 0, sizeof(int), st), "memset");
    validate_kernel<<<(n_rows + 255) / 256, 256, 0, st>>>(row_ptr, cols, vals, n_rows, n_cols, nnz, d_err);
    int h_err = 0;
    check(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st), "flag");
    check(cudaStreamSynchronize(st), "sync");
    require(h_err != 1, knnx::errc::invalid_argument, "row_ptr is not monotone from 0 to nnz");
    require(h_err != 2, knnx::errc::out_of_bounds, "column index out of range");
    require(h_err != 3, knnx::errc::duplicate_entry, "columns of a row are not strictly increasing");
    require(h_err != 4, knnx::errc::non_finite_value, "matrix value not finite");
    // 2. schedule
    const int32_t* d_sched = nullptr;
    if (schedule_kind == KNNX_SCHEDULE_GRAPH) {
      d_sched = device_schedule(ctx, ws, row_ptr, cols, n_rows, col_base);
      if (d_sched == nullptr) {  // too many components for the level-synchronous walk
        knnx::Csr a;
        a.n_rows = n_rows;
        a.n_cols = n_cols;
        a.row_ptr = download(row_ptr, static_cast<size_t>(n_rows) + 1, st);
        check(cudaStreamSynchronize(st), "sync");
        const int64_t e0 = a.row_ptr[0];
        a.cols = download(cols + e0, static_cast<size_t>(nnz), st);
        check(cudaStreamSynchronize(st), "sync");
        for (int64_t& v : a.row_ptr) v -= e0;
        const std::vector<int32_t> sched = knnx::locality_schedule(a, col_base);
        int32_t* ds = ws.get<int32_t>(n_rows);
        check(cudaMemcpyAsync(ds, sched.data(), sizeof(int32_t) * n_rows, cudaMemcpyHostToDevice, st), "schedule");
        check(cudaStreamSynchronize(st), "sync");
        d_sched = ds;
      }
    } else if (schedule_kind == KNNX_SCHEDULE_GIVEN) {
      std::vector<char> hit(n_rows, 0);
      for (int32_t i = 0; i < n_rows; ++i) {
        require(schedule[i] >= 0 && schedule[i] < n_rows && !hit[schedule[i]],
                knnx::errc::invalid_argument, "schedule is not a permutation of the rows");
        hit[schedule[i]] = 1;
      }
      int32_t* ds = ws.get<int32_t>(n_rows);
      check(cudaMemcpyAsync(ds, schedule, sizeof(int32_t) * n_rows, cudaMemcpyHostToDevice, st), "schedule");
      d_sched = ds;
    }
    // 3. tile sort, slice lengths and offsets
    int64_t bytes = 0;
    auto dev_alloc = [&](auto** p, size_t n) {
      using T = std::remove_pointer_t<std::remove_pointer_t<decltype(p)>>;
      check(cudaMalloc(p, sizeof(T) * std::max<size_t>(1, n)), "cudaMalloc");
      bytes += sizeof(T) * std::max<size_t>(1, n);
    };
    dev_alloc(&op->d_slot_row, n_rows);
    dev_alloc(&op->d_row_len, n_rows);
    dev_alloc(&op->d_slice_len, op->n_slices);
    dev_alloc(&op->d_slice_off, static_cast<size_t>(op->n_slices) + 1);
    tile_sort_kernel<<<op->n_tiles, kTile, 0, st>>>(row_ptr, d_sched, n_rows, op->d_slot_row, op->d_row_len);
    int64_t* elems = ws.get<int64_t>(static_cast<size_t>(op->n_slices) + 1);
    int32_t* minmax = ws.get<int32_t>(3);
    const int32_t mm0[3] = {0x7fffffff, 0, 0};
    check(cudaMemcpyAsync(minmax, mm0, sizeof mm0, cudaMemcpyHostToDevice, st), "init");
    check(cudaMemsetAsync(elems, 0, sizeof(int64_t) * (static_cast<size_t>(op->n_slices) + 1), st), "memset");
    const int n_pad32 = op->n_slices * 32;
    slice_len_kernel<<<(n_pad32 + 255) / 256, 256, 0, st>>>(op->d_row_len, n_rows, op->interleave,
                                                            op->d_slice_len, elems, minmax);
    size_t scan_bytes = 0;
    check(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, elems, op->d_slice_off, op->n_slices + 1, st),
          "scan size");
    void* scan_tmp = ws.get<unsigned char>(scan_bytes);
    check(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, elems, op->d_slice_off, op->n_slices + 1, st),
          "scan");
    // 4. host mirrors (canonical value order for set/get values; offsets
    // relative to the block's first entry)
    op->h_row_ptr = download(row_ptr, static_cast<size_t>(n_rows) + 1, st);
    op->h_slice_off = download(op->d_slice_off, static_cast<size_t>(op->n_slices) + 1, st);
    std::vector<int32_t> h_slot_row = download(op->d_slot_row, n_rows, st);
    int32_t h_mm[3];
    check(cudaMemcpyAsync(h_mm, minmax, sizeof h_mm, cudaMemcpyDeviceToHost, st), "minmax");
    check(cudaStreamSynchronize(st), "sync");
    {
      const int64_t base = op->h_row_ptr[0];
      if (base != 0)
        for (int64_t& v : op->h_row_ptr) v -= base;
    }
    op->stored = op->h_slice_off[op->n_slices];
    op->max_slice_len = h_mm[1];
    op->uniform_len = h_mm[0] == h_mm[2] ? h_mm[2] : -1;
    bool identity = true;
    for (int32_t p = 0; p < n_rows && identity; ++p) identity = h_slot_row[p] == p;
    if (!identity) {
      op->h_slot_of_row.assign(n_rows, 0);
      for (int32_t p = 0; p < n_rows; ++p) op->h_slot_of_row[h_slot_row[p]] = p;
    }
    // 5. entries
    dev_alloc(&op->d_cols, static_cast<size_t>(op->stored));
    check(cudaMemsetAsync(op->d_cols, 0, sizeof(int32_t) * static_cast<size_t>(op->stored), st), "memset");
    if (op->has_vals) {
      dev_alloc(&op->d_vals, static_cast<size_t>(op->stored));
      check(cudaMemsetAsync(op->d_vals, 0, sizeof(float) * static_cast<size_t>(op->stored), st), "memset");
    }
    place_kernel<<<static_cast<int>((static_cast<int64_t>(n_rows) * 32 + 255) / 256), 256, 0, st>>>(
        row_ptr, cols, vals, op->d_slot_row, op->d_slice_off, n_rows, op->interleave, op->d_cols,
        op->d_vals);
    launched(ctx, "csr_dev build", 8);
    if (identity) {  // like the host build: no slot map when rows run in place
      cudaFree(op->d_slot_row);
      op->d_slot_row = nullptr;
    }
    check(cudaStreamSynchronize(st), "build sync");
    op->device_bytes = bytes;
    ++ctx->live_ops;
    *out = op.release();
    return KNNX_OK;
  });
}
