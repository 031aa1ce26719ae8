// C-ABI runtime of libknnx.so: contexts, operator upload, dispatch.
// See include/knnx.h for the contract of every entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "knnx_internal.cuh"
#include "knnx_rt.cuh"

namespace {

using namespace knnx_rt;

template <typename T>
T* upload(const std::vector<T>& v, cudaStream_t st, int64_t& bytes) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  check(cudaMalloc(&d, sizeof(T) * v.size()), "cudaMalloc");
  check(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st), "upload");
  bytes += static_cast<int64_t>(sizeof(T) * v.size());
  return d;
}

// rows [0, n) split over the host threads (disjoint outputs per row)
template <typename Fn>
void parallel_rows(int32_t n, Fn&& fn) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const int32_t chunk = std::max<int32_t>(1, (n + static_cast<int32_t>(hw) - 1) / static_cast<int32_t>(hw));
  std::vector<std::thread> pool;
  for (int32_t lo = chunk; lo < n; lo += chunk) pool.emplace_back(fn, lo, std::min(n, lo + chunk));
  fn(0, std::min(n, chunk));
  for (auto& t : pool) t.join();
}

// deferred kernel error flag -> status (reads back: synchronising)
int take_flag(knnx_ctx_t ctx) {
  int h[2] = {0, 0};
  check(cudaMemcpyAsync(h, ctx->d_flag, sizeof h, cudaMemcpyDeviceToHost, ctx->stream), "flag");
  check(cudaStreamSynchronize(ctx->stream), "sync");
  if (h[0] == 0) return KNNX_OK;
  const int code = h[0];
  const int zero[2] = {0, 0x7fffffff};
  check(cudaMemcpy(ctx->d_flag, zero, sizeof zero, cudaMemcpyHostToDevice), "flag reset");
  if (code == knnx_dev::kFlagZeroWeight)
    return fail(KNNX_ERR_ZERO_WEIGHT,
                "ZeroWeight: all kernel weights underflowed for target " + std::to_string(h[1]));
  if (code == knnx_dev::kFlagNonFinite)
    return fail(KNNX_ERR_NON_FINITE_VALUE, "NonFiniteValue: update produced a non-finite value in row " +
                                               std::to_string(h[1]));
  return fail(code, "deferred device error in row " + std::to_string(h[1]));
}

void validate_csr(int32_t n_rows, int32_t n_cols, int64_t nnz, const int64_t* row_ptr,
                  const int32_t* cols) {
  require(n_rows >= 0 && n_cols >= 0 && nnz >= 0, knnx::errc::invalid_argument, "negative shape");
  require(row_ptr != nullptr && (nnz == 0 || cols != nullptr), knnx::errc::invalid_argument,
          "null CSR arrays");
  require(row_ptr[0] == 0 && row_ptr[n_rows] == nnz, knnx::errc::size_mismatch,
          "row_ptr does not span nnz entries");
  // messages are built only on failure (this loop sees every entry: 6e8 at C4)
  for (int32_t i = 0; i < n_rows; ++i) {
    if (row_ptr[i + 1] < row_ptr[i])
      throw knnx::error(knnx::errc::invalid_argument, "row_ptr not monotone");
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      if (cols[e] < 0 || cols[e] >= n_cols)
        throw knnx::error(knnx::errc::out_of_bounds,
                          "entry (" + std::to_string(i) + "," + std::to_string(cols[e]) +
                              ") outside " + std::to_string(n_rows) + "x" + std::to_string(n_cols));
      if (e != row_ptr[i] && cols[e - 1] >= cols[e])
        throw knnx::error(knnx::errc::duplicate_entry,
                          "row " + std::to_string(i) +
                              " is not strictly ascending (canonical CSR required)");
    }
  }
}

float gauss_c2(double h) { return static_cast<float>(1.4426950408889634 / (2.0 * h * h)); }

}  // namespace

extern "C" {

int knnx_abi_version(void) { return 1; }
const char* knnx_last_error(void) { return g_last_error.c_str(); }

int knnx_ctx_create(int device, knnx_ctx_t* out) {
  return guard([&] {
    require(out != nullptr, knnx::errc::invalid_argument, "null output handle");
    int n_dev = 0;
    check(cudaGetDeviceCount(&n_dev), "cudaGetDeviceCount");
    require(device >= 0 && device < n_dev, knnx::errc::invalid_argument,
            "device " + std::to_string(device) + " of " + std::to_string(n_dev));
    DeviceGuard dg(device);
    cudaDeviceProp prop{};
    check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
      throw knnx::error(knnx::errc::unsupported,
                        std::string("libknnx is built for sm_100a (B200); device is ") + prop.name);
    auto ctx = std::make_unique<knnx_context>();
    ctx->device = device;
    ctx->n_sms = prop.multiProcessorCount;
    // keep stream-ordered allocations (the _host entry points' staging
    // buffers) cached in the pool instead of returning them at every sync
    cudaMemPool_t pool = nullptr;
    check(cudaDeviceGetDefaultMemPool(&pool, device), "mem pool");
    uint64_t keep = UINT64_MAX;
    check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "mem pool");
    check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
    ctx->stream = ctx->own_stream;
    check(cudaMalloc(&ctx->d_flag, 2 * sizeof(int)), "flag");
    const int zero[2] = {0, 0x7fffffff};
    check(cudaMemcpy(ctx->d_flag, zero, sizeof zero, cudaMemcpyHostToDevice), "flag init");
    *out = ctx.release();
    return KNNX_OK;
  });
}

// Frees a context.  Only the context's own stream is touched: an external
// stream set with knnx_ctx_set_stream may already be gone; cudaFree waits for
// the device anyway.
static void free_context(knnx_context* ctx) {
  cudaSetDevice(ctx->device);
  cudaFree(ctx->d_flag);
  cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int knnx_ctx_destroy(knnx_ctx_t ctx) {
  return guard([&] {
    if (!ctx || ctx->closed) return KNNX_OK;
    if (ctx->live_ops > 0) {  // freed by the last knnx_op_destroy
      ctx->closed = true;
      return KNNX_OK;
    }
    free_context(ctx);
    return KNNX_OK;
  });
}

int knnx_ctx_set_stream(knnx_ctx_t ctx, void* stream) {
  return guard([&] {
    require(ctx != nullptr, knnx::errc::invalid_argument, "null context");
    ctx->stream = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
    return KNNX_OK;
  });
}

int knnx_ctx_use_own_stream(knnx_ctx_t ctx) {
  return guard([&] {
    require(ctx != nullptr, knnx::errc::invalid_argument, "null context");
    ctx->stream = ctx->own_stream;
    return KNNX_OK;
  });
}

void* knnx_ctx_stream(knnx_ctx_t ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int knnx_ctx_sync(knnx_ctx_t ctx) {
  return guard([&] {
    require(ctx != nullptr, knnx::errc::invalid_argument, "null context");
    DeviceGuard dg(ctx->device);
    return take_flag(ctx);
  });
}

int64_t knnx_ctx_launches(knnx_ctx_t ctx) { return ctx ? ctx->launches : -1; }

// ---------------------------------------------------------------------------
// device buffers

int knnx_alloc(knnx_ctx_t ctx, int64_t bytes, void** dev) {
  return guard([&] {
    require(ctx != nullptr && dev != nullptr && bytes >= 0, knnx::errc::invalid_argument,
            "bad argument");
    DeviceGuard dg(ctx->device);
    check(cudaMalloc(dev, static_cast<size_t>(std::max<int64_t>(bytes, 16))), "cudaMalloc");
    return KNNX_OK;
  });
}

int knnx_free(knnx_ctx_t ctx, void* dev) {
  return guard([&] {
    require(ctx != nullptr, knnx::errc::invalid_argument, "null context");
    DeviceGuard dg(ctx->device);
    if (dev) check(cudaFree(dev), "cudaFree");
    return KNNX_OK;
  });
}

int knnx_host_alloc(int64_t bytes, void** host) {
  return guard([&] {
    require(host != nullptr && bytes >= 0, knnx::errc::invalid_argument, "bad argument");
    check(cudaHostAlloc(host, static_cast<size_t>(std::max<int64_t>(bytes, 16)),
                        cudaHostAllocMapped | cudaHostAllocPortable),
          "cudaHostAlloc");
    return KNNX_OK;
  });
}

int knnx_host_free(void* host) {
  return guard([&] {
    if (host) check(cudaFreeHost(host), "cudaFreeHost");
    return KNNX_OK;
  });
}

// rows of `cols` floats at pitch in_ld -> rows at pitch out_ld (columns past
// `cols` zero): the pad / unpad step of the host-buffer entry points
__global__ void repitch_kernel(const float* __restrict__ in, int64_t n, int in_ld, int cols,
                               float* __restrict__ out, int out_ld) {
  const int64_t total = n * out_ld;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / out_ld;
    const int c = static_cast<int>(i - r * out_ld);
    out[i] = c < cols ? in[r * in_ld + c] : 0.0f;
  }
}

static void launch_repitch(const float* in, int64_t n, int in_ld, int cols, float* out, int out_ld,
                           cudaStream_t st) {
  if (n <= 0) return;
  const int64_t total = n * out_ld;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  repitch_kernel<<<grid, 256, 0, st>>>(in, n, in_ld, cols, out, out_ld);
  check(cudaGetLastError(), "repitch");
}

static void check_copy_shape(int32_t n, int32_t dim, int32_t ld, const void* a, const void* b) {
  require(n >= 0 && dim >= 1 && ld >= dim, knnx::errc::invalid_argument, "need n >= 0, 1 <= dim <= ld");
  require(n == 0 || (a != nullptr && b != nullptr), knnx::errc::invalid_argument, "null buffer");
}

int knnx_upload_points(knnx_ctx_t ctx, const float* host, int32_t n, int32_t dim, int32_t ld,
                       float* dev) {
  return guard([&] {
    require(ctx != nullptr, knnx::errc::invalid_argument, "null context");
    check_copy_shape(n, dim, ld, host, dev);
    DeviceGuard dg(ctx->device);
    if (n == 0) return KNNX_OK;
    if (ld == dim) {
      check(cudaMemcpyAsync(dev, host, sizeof(float) * static_cast<size_t>(n) * ld,
                            cudaMemcpyHostToDevice, ctx->stream),
            "h2d");
    } else {
      // one contiguous copy of the packed rows, then the pad on the device
      // (a strided 2-D copy of short rows runs far below the link rate)
      float* packed = nullptr;
      const size_t pbytes = sizeof(float) * static_cast<size_t>(n) * dim;
      check(cudaMallocAsync(&packed, pbytes, ctx->stream), "alloc");
      check(cudaMemcpyAsync(packed, host, pbytes, cudaMemcpyHostToDevice, ctx->stream), "h2d");
      launch_repitch(packed, n, dim, dim, dev, ld, ctx->stream);
      check(cudaFreeAsync(packed, ctx->stream), "free");
    }
    check(cudaStreamSynchronize(ctx->stream), "sync");
    return KNNX_OK;
  });
}

int knnx_download_points(knnx_ctx_t ctx, const float* dev, int32_t n, int32_t dim, int32_t ld,
                         float* host) {
  return guard([&] {
    require(ctx != nullptr, knnx::errc::invalid_argument, "null context");
    check_copy_shape(n, dim, ld, host, dev);
    DeviceGuard dg(ctx->device);
    if (n == 0) return KNNX_OK;
    if (ld == dim) {
      check(cudaMemcpyAsync(host, dev, sizeof(float) * static_cast<size_t>(n) * ld,
                            cudaMemcpyDeviceToHost, ctx->stream),
            "d2h");
    } else {
      float* packed = nullptr;
      const size_t pbytes = sizeof(float) * static_cast<size_t>(n) * dim;
      check(cudaMallocAsync(&packed, pbytes, ctx->stream), "alloc");
      launch_repitch(dev, n, ld, dim, packed, dim, ctx->stream);
      check(cudaMemcpyAsync(host, packed, pbytes, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
      check(cudaFreeAsync(packed, ctx->stream), "free");
    }
    return take_flag(ctx);  // blocking; surfaces deferred kernel errors
  });
}

// ---------------------------------------------------------------------------
// operators

// KNNX_OPT_RELABEL_COLS: renumber columns [col_base, col_base + n_rows) in
// schedule order and re-sort every row by the new number (values follow);
// returns col_order (stored column -> caller column) and h_pos (canonical
// entry -> index within its stored row)
static std::vector<int32_t> relabel_columns(knnx::Csr& a, const int32_t* schedule, int32_t col_base,
                                            std::vector<uint16_t>& h_pos) {
  std::vector<int32_t> rel(a.n_cols), order(a.n_cols);
  for (int32_t c = 0; c < a.n_cols; ++c) rel[c] = c;
  for (int32_t p = 0; p < a.n_rows; ++p) rel[col_base + schedule[p]] = col_base + p;
  for (int32_t c = 0; c < a.n_cols; ++c) order[rel[c]] = c;
  h_pos.assign(static_cast<size_t>(a.nnz()), 0);
  const bool has_vals = !a.vals.empty();
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::atomic<bool> too_long{false};
  for (unsigned w = 0; w < hw; ++w)
    pool.emplace_back([&, w] {
      std::vector<std::pair<int32_t, int64_t>> row;
      std::vector<float> v;
      for (int32_t r = static_cast<int32_t>(w); r < a.n_rows; r += static_cast<int32_t>(hw)) {
        const int64_t e0 = a.row_ptr[r], e1 = a.row_ptr[r + 1];
        if (e1 - e0 > 65536) { too_long = true; return; }
        row.clear();
        for (int64_t e = e0; e < e1; ++e) row.emplace_back(rel[a.cols[e]], e);
        std::sort(row.begin(), row.end());
        if (has_vals) v.assign(a.vals.begin() + e0, a.vals.begin() + e1);
        for (int64_t q = 0; q < e1 - e0; ++q) {
          const int64_t e = row[q].second;
          h_pos[e] = static_cast<uint16_t>(q);
          a.cols[e0 + q] = row[q].first;
          if (has_vals) a.vals[e0 + q] = v[e - e0];
        }
      }
    });
  for (auto& t : pool) t.join();
  require(!too_long, knnx::errc::invalid_argument, "relabelled rows are limited to 65536 entries");
  return order;
}

static int create_from_csr(knnx_ctx_t ctx, knnx::Csr& a, int32_t order, int32_t tile_rows,
                           knnx_op_t* out, bool with_values, const int32_t* schedule = nullptr,
                           int32_t options = 0, int32_t col_base = 0) {
  require(ctx != nullptr && out != nullptr, knnx::errc::invalid_argument, "null handle");
  require(order == KNNX_ORDER_ORIGINAL || order == KNNX_ORDER_CLUSTER,
          knnx::errc::invalid_argument, "unknown order");
  require((options & ~(KNNX_OPT_RELABEL_COLS | KNNX_OPT_GROUP_INTERLEAVE)) == 0,
          knnx::errc::invalid_argument, "unknown option");
  require(!(options & KNNX_OPT_GROUP_INTERLEAVE) || order == KNNX_ORDER_ORIGINAL,
          knnx::errc::invalid_argument, "group interleave needs KNNX_ORDER_ORIGINAL");
  require(!(options & KNNX_OPT_RELABEL_COLS) || (schedule != nullptr || a.n_rows == 0),
          knnx::errc::invalid_argument, "column relabelling needs a schedule");
  require(!(options & KNNX_OPT_RELABEL_COLS) ||
              (col_base >= 0 && static_cast<int64_t>(col_base) + a.n_rows <= a.n_cols),
          knnx::errc::invalid_argument, "relabelled columns out of range");
  std::vector<uint16_t> h_pos;
  std::vector<int32_t> col_order;
  if ((options & KNNX_OPT_RELABEL_COLS) && a.n_rows > 0)
    col_order = relabel_columns(a, schedule, col_base, h_pos);
  if (tile_rows == 0) tile_rows = 256;  // measured best for the stationary SpMV
  require(tile_rows >= 32 && tile_rows <= 1024 && tile_rows % 32 == 0,
          knnx::errc::invalid_argument, "tile_rows must be a multiple of 32 in [32, 1024]");
  DeviceGuard dg(ctx->device);
  auto op = std::make_unique<knnx_operator>();
  op->ctx = ctx;
  op->n_rows = a.n_rows;
  op->n_cols = a.n_cols;
  op->order = order;
  op->nnz = a.nnz();
  op->has_vals = with_values;  // an empty operator can carry (zero) values
  op->h_row_ptr = a.row_ptr;
  op->h_pos = std::move(h_pos);
  op->interleave = (options & KNNX_OPT_GROUP_INTERLEAVE) ? 8 : 0;
  // uniform row length?
  op->uniform_len = -1;
  if (a.n_rows > 0) {
    const int64_t k0 = a.row_ptr[1] - a.row_ptr[0];
    bool uni = true;
    for (int32_t i = 0; i < a.n_rows && uni; ++i) uni = (a.row_ptr[i + 1] - a.row_ptr[i]) == k0;
    if (uni) op->uniform_len = static_cast<int32_t>(k0);
  }
  cudaStream_t st = ctx->stream;
  int64_t bytes = 0;
  // both layouts share the SELL-32 slice structure; cluster tiles add halos
  knnx::ClusterTiles tiles =
      knnx::build_cluster_tiles(a, tile_rows, schedule, order == KNNX_ORDER_CLUSTER);
  op->tile_rows = tile_rows;
  op->n_tiles = tiles.n_tiles;
  op->n_slices = (a.n_rows + 31) / 32;
  op->stored = tiles.stored;
  op->max_halo = tiles.max_halo;
  op->halo_total = static_cast<int64_t>(tiles.halo_ids.size());
  op->h_slice_off = tiles.slice_off;
  for (int32_t s : tiles.slice_len) op->max_slice_len = std::max(op->max_slice_len, s);
  if (!tiles.slot_row.empty()) {
    op->h_slot_of_row.assign(a.n_rows, 0);
    for (int32_t p = 0; p < a.n_rows; ++p) op->h_slot_of_row[tiles.slot_row[p]] = p;
  }
  if (op->interleave) {
    // re-place the entries: slices padded to a multiple of 8 entries per row,
    // entry q of slot p at slice_off + (q/8)*256 + (p%32)*8 + q%8
    std::vector<int64_t> off(static_cast<size_t>(op->n_slices) + 1, 0);
    for (int32_t s = 0; s < op->n_slices; ++s) {
      tiles.slice_len[s] = (tiles.slice_len[s] + 7) / 8 * 8;
      off[s + 1] = off[s] + static_cast<int64_t>(tiles.slice_len[s]) * 32;
    }
    op->h_slice_off = off;
    tiles.slice_off = off;
    op->stored = off[op->n_slices];
    op->max_slice_len = 0;
    for (int32_t sl : tiles.slice_len) op->max_slice_len = std::max(op->max_slice_len, sl);
    if (op->has_vals) {
      tiles.vals.assign(static_cast<size_t>(op->stored), 0.0f);
      parallel_rows(a.n_rows, [&](int32_t lo, int32_t hi) {
        for (int32_t r = lo; r < hi; ++r)
          for (int64_t e = a.row_ptr[r]; e < a.row_ptr[r + 1]; ++e)
            tiles.vals[op->pos_of(op->h_slot_of_row.empty() ? r : op->h_slot_of_row[r],
                                  e - a.row_ptr[r])] = a.vals[e];
      });
    }
  }
  op->d_slice_off = upload(tiles.slice_off, st, bytes);
  op->d_slice_len = upload(tiles.slice_len, st, bytes);
  op->d_row_len = upload(tiles.row_len, st, bytes);
  if (!tiles.slot_row.empty()) op->d_slot_row = upload(tiles.slot_row, st, bytes);
  if (!col_order.empty()) {
    op->d_col_order = upload(col_order, st, bytes);
    op->gather_ws_floats = 3 * static_cast<int64_t>(a.n_cols);  // embedding dim <= 3
    check(cudaMalloc(&op->d_gather_ws, sizeof(float) * op->gather_ws_floats), "cudaMalloc");
    bytes += sizeof(float) * op->gather_ws_floats;
  }
  if (op->has_vals) op->d_vals = upload(tiles.vals, st, bytes);
  if (order == KNNX_ORDER_CLUSTER) {
    require(static_cast<size_t>(tiles.max_halo) * sizeof(float) <= 200 * 1024,
            knnx::errc::local_index_overflow, "tile halo exceeds the shared-memory stage");
    op->d_lidx = upload(tiles.lidx, st, bytes);
    op->d_halo_off = upload(tiles.halo_off, st, bytes);
    op->d_halo_ids = upload(tiles.halo_ids, st, bytes);
    op->halo_total = static_cast<int64_t>(tiles.halo_ids.size());
  } else {
    // global int32 columns in the same slice layout
    std::vector<int32_t> cols(static_cast<size_t>(op->stored), 0);
    op->h_slice_off = tiles.slice_off;
    parallel_rows(a.n_rows, [&](int32_t lo, int32_t hi) {
      for (int32_t r = lo; r < hi; ++r) {
        const int32_t p = op->h_slot_of_row.empty() ? r : op->h_slot_of_row[r];
        for (int64_t e = a.row_ptr[r]; e < a.row_ptr[r + 1]; ++e)
          cols[op->pos_of(p, e - a.row_ptr[r])] = a.cols[e];  // stored (relabelled) order
      }
    });
    op->d_cols = upload(cols, st, bytes);
    op->halo_total = 0;
  }
  check(cudaStreamSynchronize(st), "upload sync");
  op->device_bytes = bytes;
  ++ctx->live_ops;
  *out = op.release();
  return KNNX_OK;
}

int knnx_op_create_csr(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                       const int64_t* row_ptr, const int32_t* cols, const float* vals,
                       int32_t order, int32_t tile_rows, knnx_op_t* out) {
  return guard([&] {
    validate_csr(n_rows, n_cols, nnz, row_ptr, cols);
    knnx::Csr a;
    a.n_rows = n_rows;
    a.n_cols = n_cols;
    a.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
    a.cols.assign(cols, cols + nnz);
    if (vals) {
      a.vals.assign(vals, vals + nnz);
      for (float v : a.vals)
        require(std::isfinite(v), knnx::errc::non_finite_value, "matrix value not finite");
    }
    return create_from_csr(ctx, a, order, tile_rows, out, vals != nullptr);
  });
}

int knnx_op_create_csr_sched(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                             const int64_t* row_ptr, const int32_t* cols, const float* vals,
                             int32_t order, int32_t tile_rows, int32_t schedule_kind,
                             int32_t col_base, const int32_t* schedule, knnx_op_t* out) {
  return knnx_op_create_csr_ex(ctx, n_rows, n_cols, nnz, row_ptr, cols, vals, order, tile_rows,
                               schedule_kind, col_base, schedule, 0, out);
}

int knnx_op_create_csr_ex(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                          const int64_t* row_ptr, const int32_t* cols, const float* vals,
                          int32_t order, int32_t tile_rows, int32_t schedule_kind,
                          int32_t col_base, const int32_t* schedule, int32_t options,
                          knnx_op_t* out) {
  return guard([&] {
    validate_csr(n_rows, n_cols, nnz, row_ptr, cols);
    require(schedule_kind >= KNNX_SCHEDULE_NONE && schedule_kind <= KNNX_SCHEDULE_GIVEN,
            knnx::errc::invalid_argument, "unknown schedule kind");
    require(schedule_kind != KNNX_SCHEDULE_GIVEN || n_rows == 0 || schedule != nullptr,
            knnx::errc::invalid_argument, "null schedule");
    knnx::Csr a;
    a.n_rows = n_rows;
    a.n_cols = n_cols;
    a.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
    a.cols.assign(cols, cols + nnz);
    if (vals) {
      a.vals.assign(vals, vals + nnz);
      for (float v : a.vals)
        require(std::isfinite(v), knnx::errc::non_finite_value, "matrix value not finite");
    }
    std::vector<int32_t> sched;
    if (schedule_kind == KNNX_SCHEDULE_GRAPH) sched = knnx::locality_schedule(a, col_base);
    if (schedule_kind == KNNX_SCHEDULE_GIVEN) sched.assign(schedule, schedule + n_rows);
    return create_from_csr(ctx, a, order, tile_rows, out, vals != nullptr,
                           sched.empty() ? nullptr : sched.data(), options, col_base);
  });
}

int knnx_op_create_hier_leaves(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int32_t n_blocks,
                               const int32_t* row_offset, const int32_t* col_offset,
                               const int64_t* block_ptr, const uint16_t* lr, const uint16_t* lc,
                               const float* vals, int32_t tile_rows, knnx_op_t* out) {
  return guard([&] {
    require(n_blocks >= 0 && block_ptr != nullptr, knnx::errc::invalid_argument, "bad blocks");
    // flatten (proj/src/hier.cpp:182-191) into a canonical CSR
    const int64_t nnz = n_blocks > 0 ? block_ptr[n_blocks] : 0;
    std::vector<int64_t> cnt(static_cast<size_t>(n_rows) + 1, 0);
    for (int32_t b = 0; b < n_blocks; ++b)
      for (int64_t e = block_ptr[b]; e < block_ptr[b + 1]; ++e) {
        const int64_t r = static_cast<int64_t>(row_offset[b]) + lr[e];
        const int64_t c = static_cast<int64_t>(col_offset[b]) + lc[e];
        require(r < n_rows && c < n_cols, knnx::errc::out_of_bounds, "leaf entry out of bounds");
        ++cnt[r + 1];
      }
    for (int32_t i = 0; i < n_rows; ++i) cnt[i + 1] += cnt[i];
    knnx::Csr a;
    a.n_rows = n_rows;
    a.n_cols = n_cols;
    a.row_ptr = cnt;
    a.cols.resize(nnz);
    if (vals) a.vals.resize(nnz);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int32_t b = 0; b < n_blocks; ++b)
      for (int64_t e = block_ptr[b]; e < block_ptr[b + 1]; ++e) {
        const int32_t r = row_offset[b] + lr[e];
        const int64_t o = fill[r]++;
        a.cols[o] = col_offset[b] + lc[e];
        if (vals) a.vals[o] = vals[e];
      }
    for (int32_t i = 0; i < n_rows; ++i) {
      std::vector<std::pair<int32_t, float>> row;
      for (int64_t e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e)
        row.emplace_back(a.cols[e], vals ? a.vals[e] : 0.f);
      std::sort(row.begin(), row.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t q = 0; q < row.size(); ++q) {
        require(q == 0 || row[q - 1].first != row[q].first, knnx::errc::duplicate_entry,
                "repeated entry in leaf payload");
        a.cols[a.row_ptr[i] + q] = row[q].first;
        if (vals) a.vals[a.row_ptr[i] + q] = row[q].second;
      }
    }
    return create_from_csr(ctx, a, KNNX_ORDER_CLUSTER, tile_rows, out, vals != nullptr);
  });
}

int knnx_op_create_knn_dev(knnx_ctx_t ctx, const int32_t* ids, int32_t m, int32_t n_cols,
                           int32_t k, knnx_op_t* out) {
  return guard([&] {
    require(ctx != nullptr && out != nullptr && (m == 0 || ids != nullptr),
            knnx::errc::invalid_argument, "null argument");
    require(m >= 0 && n_cols >= 0 && k >= 1, knnx::errc::invalid_argument, "bad shape");
    require(k <= 32, knnx::errc::unsupported, "device tile build supports k <= 32");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = ctx->stream;
    auto op = std::make_unique<knnx_operator>();
    op->ctx = ctx;
    op->n_rows = m;
    op->n_cols = n_cols;
    op->order = KNNX_ORDER_CLUSTER;
    op->tile_rows = 256;
    op->n_tiles = (m + 255) / 256;
    op->n_slices = (m + 31) / 32;
    op->nnz = static_cast<int64_t>(m) * k;
    op->stored = static_cast<int64_t>(op->n_slices) * 32 * k;
    op->uniform_len = k;
    op->max_slice_len = k;
    op->has_vals = false;
    op->h_row_ptr.resize(static_cast<size_t>(m) + 1);
    for (int32_t i = 0; i <= m; ++i) op->h_row_ptr[i] = static_cast<int64_t>(i) * k;
    op->h_slice_off.resize(static_cast<size_t>(op->n_slices) + 1);
    for (int32_t s = 0; s <= op->n_slices; ++s) op->h_slice_off[s] = static_cast<int64_t>(s) * 32 * k;
    const std::vector<int32_t> slice_len(op->n_slices, k);
    std::vector<int32_t> row_len(m, k);
    int64_t bytes = 0;
    op->d_slice_off = upload(op->h_slice_off, st, bytes);
    op->d_slice_len = upload(slice_len, st, bytes);
    op->d_row_len = upload(row_len, st, bytes);
    knnx_dev::build_tiles_from_knn(ids, m, k, &op->d_halo_off, &op->d_halo_ids, &op->d_lidx,
                                   &op->halo_total, &op->max_halo, st);
    check(cudaGetLastError(), "tile build");
    check(cudaStreamSynchronize(st), "tile build");
    ctx->launches += 2;
    require(op->max_halo <= 65536, knnx::errc::local_index_overflow, "tile halo exceeds 16 bits");
    bytes += static_cast<int64_t>(op->n_tiles + 1) * 8 + op->halo_total * 4 + op->stored * 2;
    op->device_bytes = bytes;
    ++ctx->live_ops;
    *out = op.release();
    return KNNX_OK;
  });
}

int knnx_hbm1_info(const char* path, int32_t* n_rows, int32_t* n_cols, int64_t* nnz,
                   int32_t* cut_level) {
  return guard([&] {
    require(path != nullptr, knnx::errc::invalid_argument, "null path");
    const knnx::Hbm1 h = knnx::read_hbm1(path);
    if (n_rows) *n_rows = h.n_rows;
    if (n_cols) *n_cols = h.n_cols;
    if (nnz) *nnz = h.nnz;
    if (cut_level) *cut_level = h.cut_level;
    return KNNX_OK;
  });
}

int knnx_op_load_hbm1(knnx_ctx_t ctx, const char* path, int32_t tile_rows, int32_t* row_forward,
                      int32_t* col_forward, knnx_op_t* out) {
  return guard([&] {
    require(path != nullptr, knnx::errc::invalid_argument, "null path");
    const knnx::Hbm1 h = knnx::read_hbm1(path);
    if (row_forward) std::copy(h.row_forward.begin(), h.row_forward.end(), row_forward);
    if (col_forward) std::copy(h.col_forward.begin(), h.col_forward.end(), col_forward);
    return knnx_op_create_hier_leaves(ctx, h.n_rows, h.n_cols,
                                      static_cast<int32_t>(h.row_offset.size()), h.row_offset.data(),
                                      h.col_offset.data(), h.block_ptr.data(), h.lr.data(),
                                      h.lc.data(), h.vals.data(), tile_rows, out);
  });
}

int knnx_op_destroy(knnx_op_t op) {
  return guard([&] {
    if (!op) return KNNX_OK;
    knnx_context* ctx = op->ctx;
    delete op;  // ~knnx_operator frees the device arrays
    if (--ctx->live_ops == 0 && ctx->closed) free_context(ctx);
    return KNNX_OK;
  });
}

int knnx_op_slot_rows(knnx_op_t op, int32_t* slot_row_host) {
  return guard([&] {
    require(op != nullptr && (op->n_rows == 0 || slot_row_host != nullptr),
            knnx::errc::invalid_argument, "null argument");
    for (int32_t r = 0; r < op->n_rows; ++r)
      slot_row_host[op->h_slot_of_row.empty() ? r : op->h_slot_of_row[r]] = r;
    return KNNX_OK;
  });
}

int knnx_op_info(knnx_op_t op, knnx_op_info_t* info) {
  return guard([&] {
    require(op != nullptr && info != nullptr, knnx::errc::invalid_argument, "null handle");
    info->n_rows = op->n_rows;
    info->n_cols = op->n_cols;
    info->order = op->order;
    info->tile_rows = op->tile_rows;
    info->nnz = op->nnz;
    info->stored = op->stored;
    info->n_tiles = op->n_tiles;
    info->max_halo = op->max_halo;
    info->halo_total = op->halo_total;
    info->device_bytes = op->device_bytes;
    info->has_values = op->has_vals ? 1 : 0;
    info->uniform_row_len = op->uniform_len;
    return KNNX_OK;
  });
}

int knnx_op_set_row_base(knnx_op_t op, int32_t row_base) {
  return guard([&] {
    require(op != nullptr, knnx::errc::invalid_argument, "null operator");
    require(row_base >= 0 && row_base + op->n_rows <= std::max(op->n_cols, op->n_rows),
            knnx::errc::out_of_bounds, "row block outside the point set");
    op->row_base = row_base;
    op->is_shard = true;
    return KNNX_OK;
  });
}

int knnx_op_set_values(knnx_op_t op, const float* vals_host) {
  return guard([&] {
    require(op != nullptr && vals_host != nullptr, knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(op->ctx->device);
    std::vector<float> stored(static_cast<size_t>(op->stored), 0.0f);
    for (int32_t r = 0; r < op->n_rows; ++r)
      for (int64_t e = op->h_row_ptr[r]; e < op->h_row_ptr[r + 1]; ++e) {
        require(std::isfinite(vals_host[e]), knnx::errc::non_finite_value, "value not finite");
        stored[op->entry_pos(r, e)] = vals_host[e];
      }
    if (!op->d_vals) {
      check(cudaMalloc(&op->d_vals, sizeof(float) * stored.size()), "cudaMalloc");
      op->device_bytes += static_cast<int64_t>(sizeof(float) * stored.size());
    }
    check(cudaMemcpyAsync(op->d_vals, stored.data(), sizeof(float) * stored.size(),
                          cudaMemcpyHostToDevice, op->ctx->stream), "values");
    check(cudaStreamSynchronize(op->ctx->stream), "sync");
    op->has_vals = true;
    return KNNX_OK;
  });
}

int knnx_op_get_values(knnx_op_t op, float* vals_host) {
  return guard([&] {
    require(op != nullptr && vals_host != nullptr, knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(op->ctx->device);
    require(op->has_vals, knnx::errc::invalid_argument, "operator has no stored values");
    std::vector<float> stored(static_cast<size_t>(op->stored));
    check(cudaMemcpyAsync(stored.data(), op->d_vals, sizeof(float) * stored.size(),
                          cudaMemcpyDeviceToHost, op->ctx->stream), "values");
    check(cudaStreamSynchronize(op->ctx->stream), "sync");
    for (int32_t r = 0; r < op->n_rows; ++r)
      for (int64_t e = op->h_row_ptr[r]; e < op->h_row_ptr[r + 1]; ++e)
        vals_host[e] = stored[op->entry_pos(r, e)];
    return KNNX_OK;
  });
}

// ---------------------------------------------------------------------------
// stationary operator

int knnx_spmv_dev(knnx_op_t op, const float* x, float* y) {
  return guard([&] {
    require(op != nullptr && x != nullptr && y != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(op->ctx->device);
    require(op->has_vals, knnx::errc::invalid_argument, "stationary SpMV needs stored values");
    knnx_dev::launch_spmv(*op, x, y, op->ctx->stream);
    launched(op->ctx, "spmv");
    return KNNX_OK;
  });
}

// device address of pinned, mapped host memory (UVA), or null (pageable)
static const void* host_mapped(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

int knnx_spmv_host(knnx_op_t op, const float* x, float* y) {
  return guard([&] {
    require(op != nullptr && x != nullptr && y != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(op->ctx->device);
    require(op->has_vals, knnx::errc::invalid_argument, "stationary SpMV needs stored values");
    cudaStream_t st = op->ctx->stream;
    // pinned (mapped) caller buffers: x read by an SM copy, y stored by the
    // multiply straight into host memory (no copy engines, runtime.cu
    // knnx_spmv_host_batch); pageable buffers: copy engines
    const void* x_dev = host_mapped(x);
    void* y_dev = const_cast<void*>(host_mapped(y));
    float *dx = nullptr, *dy = nullptr;
    check(cudaMallocAsync(&dx, sizeof(float) * std::max(1, op->n_cols), st), "alloc");
    if (!y_dev) check(cudaMallocAsync(&dy, sizeof(float) * std::max(1, op->n_rows), st), "alloc");
    if (x_dev && reinterpret_cast<uintptr_t>(x_dev) % 16 == 0 && op->n_cols % 4 == 0) {
      knnx_dev::launch_copy(dx, x_dev, sizeof(float) * op->n_cols, st);
      launched(op->ctx, "copy");
    } else {
      check(cudaMemcpyAsync(dx, x, sizeof(float) * op->n_cols, cudaMemcpyHostToDevice, st), "h2d");
    }
    knnx_dev::launch_spmv(*op, dx, y_dev ? static_cast<float*>(y_dev) : dy, st);
    launched(op->ctx, "spmv");
    if (!y_dev) {
      check(cudaMemcpyAsync(y, dy, sizeof(float) * op->n_rows, cudaMemcpyDeviceToHost, st), "d2h");
      check(cudaFreeAsync(dy, st), "free");
    }
    check(cudaFreeAsync(dx, st), "free");
    check(cudaStreamSynchronize(st), "sync");
    return KNNX_OK;
  });
}

int knnx_spmv_host_batch(knnx_op_t op, int32_t n_steps, const float* xs, float* ys) {
  return guard([&] {
    require(op != nullptr && xs != nullptr && ys != nullptr && n_steps >= 0,
            knnx::errc::invalid_argument, "bad argument");
    DeviceGuard dg(op->ctx->device);
    require(op->has_vals, knnx::errc::invalid_argument, "stationary SpMV needs stored values");
    if (n_steps == 0) return KNNX_OK;
    knnx_context* ctx = op->ctx;
    // Three-stage pipeline over kSlots device staging slots: a copy-in stream
    // (H2D engine), the context stream (multiply) and a copy-out stream (D2H
    // engine).  Step i's H2D waits only for the multiply that last read its x
    // slot (step i - kSlots) and step i's multiply waits for the D2H that last
    // drained its y slot, so both copy engines stream back to back and the
    // period is max(H2D, multiply, D2H) instead of their sum.
    //
    // When the caller's y buffer is pinned (mapped) host memory the D2H copy
    // engine is bypassed: the multiply stores y straight into the host buffer
    // (posted PCIe writes of whole 128-B lines, overlapping the next step's x
    // copy in the other direction).  Measured at C2: 2.83e11
    // interactions/s vs 2.35e11 with both copy engines; reading x by an SM
    // copy from mapped memory as well was slower (1.9e11) and was removed.
    const void* ys_dev = host_mapped(ys);
    const bool direct_y = ys_dev != nullptr;
    constexpr int kSlots = 3;
    cudaStream_t cin, cout;
    check(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking), "stream");
    check(cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking), "stream");
    cudaStream_t st = ctx->stream;
    cudaEvent_t start, ev_in[kSlots], ev_k[kSlots], ev_out[kSlots];
    for (cudaEvent_t* e : {&start})
      check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    for (int b = 0; b < kSlots; ++b) {
      check(cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming), "event");
      check(cudaEventCreateWithFlags(&ev_k[b], cudaEventDisableTiming), "event");
      check(cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming), "event");
    }
    float *dx = nullptr, *dy = nullptr;
    const int64_t xw = std::max(1, op->n_cols), yw = std::max(1, op->n_rows);
    check(cudaMallocAsync(&dx, sizeof(float) * xw * kSlots, st), "alloc");
    check(cudaMallocAsync(&dy, sizeof(float) * yw * kSlots, st), "alloc");
    check(cudaEventRecord(start, st), "event");  // ordered after prior work + allocs
    check(cudaStreamWaitEvent(cin, start, 0), "wait");
    check(cudaStreamWaitEvent(cout, start, 0), "wait");
    for (int32_t i = 0; i < n_steps; ++i) {
      const int b = i % kSlots;
      float* sx = dx + b * xw;
      float* sy = dy + b * yw;
      if (i >= kSlots) check(cudaStreamWaitEvent(cin, ev_k[b], 0), "wait");
      check(cudaMemcpyAsync(sx, xs + static_cast<int64_t>(i) * op->n_cols,
                            sizeof(float) * op->n_cols, cudaMemcpyHostToDevice, cin), "h2d");
      check(cudaEventRecord(ev_in[b], cin), "event");
      check(cudaStreamWaitEvent(st, ev_in[b], 0), "wait");
      if (!direct_y && i >= kSlots) check(cudaStreamWaitEvent(st, ev_out[b], 0), "wait");
      if (direct_y) {  // the multiply writes y into the caller's pinned buffer
        knnx_dev::launch_spmv(*op, sx,
                              static_cast<float*>(const_cast<void*>(ys_dev)) +
                                  static_cast<int64_t>(i) * op->n_rows,
                              st);
        launched(ctx, "spmv");
        check(cudaEventRecord(ev_k[b], st), "event");
        continue;
      }
      knnx_dev::launch_spmv(*op, sx, sy, st);
      launched(ctx, "spmv");
      check(cudaEventRecord(ev_k[b], st), "event");
      check(cudaStreamWaitEvent(cout, ev_k[b], 0), "wait");
      check(cudaMemcpyAsync(ys + static_cast<int64_t>(i) * op->n_rows, sy,
                            sizeof(float) * op->n_rows, cudaMemcpyDeviceToHost, cout), "d2h");
      check(cudaEventRecord(ev_out[b], cout), "event");
    }
    cudaEvent_t done;
    check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
    check(cudaEventRecord(done, cout), "event");
    check(cudaStreamWaitEvent(st, done, 0), "wait");
    check(cudaFreeAsync(dx, st), "free");
    check(cudaFreeAsync(dy, st), "free");
    check(cudaStreamSynchronize(st), "sync");
    check(cudaStreamDestroy(cin), "stream");
    check(cudaStreamDestroy(cout), "stream");
    check(cudaEventDestroy(start), "event");
    check(cudaEventDestroy(done), "event");
    for (int b = 0; b < kSlots; ++b) {
      check(cudaEventDestroy(ev_in[b]), "event");
      check(cudaEventDestroy(ev_k[b]), "event");
      check(cudaEventDestroy(ev_out[b]), "event");
    }
    return KNNX_OK;
  });
}

int knnx_spmv_batch_strided_dev(knnx_op_t op, int32_t n_steps, const float* xs, int64_t x_stride,
                                float* ys, int64_t y_stride) {
  return guard([&] {
    require(op != nullptr && xs != nullptr && ys != nullptr && n_steps >= 0 && x_stride >= 0 &&
                y_stride >= 0,
            knnx::errc::invalid_argument, "bad argument");
    DeviceGuard dg(op->ctx->device);
    require(op->has_vals, knnx::errc::invalid_argument, "stationary SpMV needs stored values");
    require(op->plain(), knnx::errc::invalid_argument,
            "relabelled / group-interleaved operators serve knnx_tsne_attr_* only");
    cudaStream_t st = op->ctx->stream;
    // stream capture is illegal on the legacy NULL stream
    require(st != nullptr, knnx::errc::invalid_argument,
            "knnx_spmv_batch_dev needs a non-default stream (knnx_ctx_use_own_stream)");
    if (n_steps == 0) return KNNX_OK;
    const knnx_operator::GraphKey key{n_steps, xs, x_stride, ys, y_stride};
    if (!op->graph_exec || !(op->graph_key == key)) {
      if (op->graph_exec) cudaGraphExecDestroy(op->graph_exec);
      op->graph_exec = nullptr;
      cudaGraph_t graph = nullptr;
      check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
      try {
        for (int32_t q = 0; q < n_steps; ++q)
          knnx_dev::launch_spmv(*op, xs + static_cast<int64_t>(q) * x_stride,
                                ys + static_cast<int64_t>(q) * y_stride, st);
      } catch (...) {  // leave the stream usable: end (and drop) the capture
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      check(cudaStreamEndCapture(st, &graph), "end capture");
      const cudaError_t ie = cudaGraphInstantiate(&op->graph_exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) op->graph_exec = nullptr;
      check(ie, "instantiate");
      op->graph_key = key;
    }
    check(cudaGraphLaunch(op->graph_exec, st), "graph launch");
    op->ctx->launches += n_steps;
    return KNNX_OK;
  });
}

int knnx_spmv_batch_dev(knnx_op_t op, int32_t n_steps, const float* xs, float* ys) {
  if (op == nullptr) return knnx_spmv_batch_strided_dev(op, n_steps, xs, 0, ys, 0);
  return knnx_spmv_batch_strided_dev(op, n_steps, xs, op->n_cols, ys, op->n_rows);
}

// ---------------------------------------------------------------------------
// non-stationary operators

static void check_points(const float* p, int32_t ld, int32_t dim) {
  require(p != nullptr, knnx::errc::invalid_argument, "null point array");
  require(dim >= 1, knnx::errc::invalid_argument, "dim must be >= 1");
  require(ld >= dim && ld % 4 == 0, knnx::errc::invalid_argument,
          "leading dimension must be >= dim and a multiple of 4");
  require(reinterpret_cast<uintptr_t>(p) % 16 == 0, knnx::errc::invalid_argument,
          "point arrays must be 16-byte aligned");
  require(dim <= 1024, knnx::errc::dim_too_high, "dim > 1024 is not supported");
}

int knnx_gauss_spmv_dev(knnx_op_t op, const float* t, int32_t ld_t, const float* s, int32_t ld_s,
                        int32_t dim, double h, const float* x, float* y) {
  return guard([&] {
    require(op != nullptr && x != nullptr && y != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(op->ctx->device);
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    check_points(t, ld_t, dim);
    check_points(s, ld_s, dim);
    knnx_dev::launch_gauss_spmv(*op, t, ld_t, s, ld_s, dim, gauss_c2(h), x, y, op->ctx->d_flag,
                                op->ctx->stream);
    launched(op->ctx, "gauss_spmv");
    return KNNX_OK;
  });
}

int knnx_update_gaussian_dev(knnx_op_t op, const float* t, int32_t ld_t, const float* s,
                             int32_t ld_s, int32_t dim, double h) {
  return guard([&] {
    require(op != nullptr, knnx::errc::invalid_argument, "null operator");
    DeviceGuard dg(op->ctx->device);
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    check_points(t, ld_t, dim);
    check_points(s, ld_s, dim);
    if (!op->d_vals) {
      check(cudaMalloc(&op->d_vals, sizeof(float) * std::max<int64_t>(1, op->stored)), "alloc");
      check(cudaMemsetAsync(op->d_vals, 0, sizeof(float) * std::max<int64_t>(1, op->stored),
                            op->ctx->stream), "memset");
      op->device_bytes += sizeof(float) * op->stored;
      op->has_vals = true;
    }
    knnx_dev::launch_update_gaussian(*op, t, ld_t, s, ld_s, dim, gauss_c2(h), op->ctx->d_flag,
                                     op->ctx->stream);
    launched(op->ctx, "update_gaussian");
    return KNNX_OK;
  });
}

int knnx_meanshift_dev(knnx_op_t op, const float* t_in, int32_t ld_t, const float* s,
                       int32_t ld_s, int32_t dim, double h, float* t_out) {
  return guard([&] {
    require(op != nullptr && t_out != nullptr, knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(op->ctx->device);
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    require(t_out != t_in, knnx::errc::invalid_argument, "t_out must not alias t_in");
    check_points(t_in, ld_t, dim);
    check_points(s, ld_s, dim);
    check_points(t_out, ld_t, dim);
    // fp64 exp(-x) == 0 for x > 745.1332191019412 (ln of half the smallest subnormal)
    const double thresh = 745.1332191019412 * 2.0 * h * h;
    const float zt = thresh > 3.0e38 ? INFINITY : static_cast<float>(thresh);
    knnx_dev::launch_meanshift(*op, t_in, ld_t, s, ld_s, dim, gauss_c2(h), zt, t_out,
                               op->ctx->d_flag, op->ctx->stream);
    launched(op->ctx, "meanshift");
    return KNNX_OK;
  });
}

// host n x dim (unpadded) -> device n x ld (zero padded), stream-ordered.
// When dim != ld the packed rows cross PCIe as ONE contiguous copy and are
// re-pitched on the device: a strided cudaMemcpy2D of 196-byte rows (C3)
// runs the copy engine at a few GB/s instead of the link's ~55 GB/s.
static float* stage_points(const float* host, int32_t n, int32_t dim, int32_t ld, cudaStream_t st) {
  float* d = nullptr;
  const size_t bytes = sizeof(float) * static_cast<size_t>(std::max(1, n)) * ld;
  check(cudaMallocAsync(&d, bytes, st), "alloc");
  if (n <= 0) return d;
  if (dim == ld) {
    check(cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, st), "h2d");
    return d;
  }
  float* packed = nullptr;
  const size_t pbytes = sizeof(float) * static_cast<size_t>(n) * dim;
  check(cudaMallocAsync(&packed, pbytes, st), "alloc");
  check(cudaMemcpyAsync(packed, host, pbytes, cudaMemcpyHostToDevice, st), "h2d");
  launch_repitch(packed, n, dim, dim, d, ld, st);
  check(cudaFreeAsync(packed, st), "free");
  return d;
}

// device n x ld -> host n x dim (packed), stream-ordered; the reverse of stage_points
static void unstage_points(float* host, const float* dev, int32_t n, int32_t dim, int32_t ld,
                           cudaStream_t st) {
  if (n <= 0) return;
  if (dim == ld) {
    check(cudaMemcpyAsync(host, dev, sizeof(float) * static_cast<size_t>(n) * ld, cudaMemcpyDeviceToHost, st),
          "d2h");
    return;
  }
  float* packed = nullptr;
  const size_t pbytes = sizeof(float) * static_cast<size_t>(n) * dim;
  check(cudaMallocAsync(&packed, pbytes, st), "alloc");
  launch_repitch(dev, n, ld, dim, packed, dim, st);
  check(cudaMemcpyAsync(host, packed, pbytes, cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaFreeAsync(packed, st), "free");
}

int knnx_gauss_spmv_host(knnx_op_t op, const float* t, const float* s, int32_t dim, double h,
                         const float* x, float* y) {
  return guard([&] {
    require(op != nullptr && t && s && x && y, knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(op->ctx->device);
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    require(dim >= 1 && dim <= 1024, knnx::errc::invalid_argument, "dim out of range");
    const int32_t ld = (dim + 3) / 4 * 4;
    cudaStream_t st = op->ctx->stream;
    // t == s (one point set, the usual kNN-interaction case): staged once
    const bool same = t == s;
    float* ds = stage_points(s, same ? std::max(op->n_cols, op->row_base + op->n_rows) : op->n_cols,
                             dim, ld, st);
    float* dt = same ? ds : stage_points(t, op->row_base + op->n_rows, dim, ld, st);
    float *dx = nullptr, *dy = nullptr;
    check(cudaMallocAsync(&dx, sizeof(float) * std::max(1, op->n_cols), st), "alloc");
    check(cudaMallocAsync(&dy, sizeof(float) * std::max(1, op->n_rows), st), "alloc");
    check(cudaMemcpyAsync(dx, x, sizeof(float) * op->n_cols, cudaMemcpyHostToDevice, st), "h2d");
    knnx_dev::launch_gauss_spmv(*op, dt + static_cast<int64_t>(op->row_base) * ld, ld, ds, ld, dim,
                                gauss_c2(h), dx, dy, op->ctx->d_flag, st);
    launched(op->ctx, "gauss_spmv");
    check(cudaMemcpyAsync(y, dy, sizeof(float) * op->n_rows, cudaMemcpyDeviceToHost, st), "d2h");
    for (void* p : {static_cast<void*>(ds), static_cast<void*>(dx), static_cast<void*>(dy)})
      check(cudaFreeAsync(p, st), "free");
    if (!same) check(cudaFreeAsync(dt, st), "free");
    return take_flag(op->ctx);
  });
}

int knnx_update_gaussian_host(knnx_op_t op, const float* t, const float* s, int32_t dim, double h) {
  return guard([&] {
    require(op != nullptr && t && s, knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(op->ctx->device);
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    require(dim >= 1 && dim <= 1024, knnx::errc::invalid_argument, "dim out of range");
    const int32_t ld = (dim + 3) / 4 * 4;
    cudaStream_t st = op->ctx->stream;
    float* dt = stage_points(t, op->row_base + op->n_rows, dim, ld, st);
    float* ds = stage_points(s, op->n_cols, dim, ld, st);
    const int rc = knnx_update_gaussian_dev(op, dt + static_cast<int64_t>(op->row_base) * ld, ld,
                                            ds, ld, dim, h);
    check(cudaFreeAsync(dt, st), "free");
    check(cudaFreeAsync(ds, st), "free");
    if (rc != KNNX_OK) return rc;
    return take_flag(op->ctx);
  });
}

int knnx_permute_rows_host(knnx_ctx_t ctx, int32_t n, int64_t row_bytes, const void* in,
                           const int32_t* forward, void* out) {
  return guard([&] {
    require(ctx != nullptr && (n == 0 || (in && forward && out)), knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(ctx->device);
    require(row_bytes >= 0 && row_bytes % 4 == 0, knnx::errc::invalid_argument,
            "row_bytes must be a multiple of 4");
    if (n == 0 || row_bytes == 0) return KNNX_OK;
    // validate the bijection like make_permutation (proj/src/core.cpp:94-109)
    std::vector<char> seen(n, 0);
    for (int32_t i = 0; i < n; ++i) {
      require(forward[i] >= 0 && forward[i] < n, knnx::errc::out_of_bounds, "permutation image out of range");
      require(!seen[forward[i]], knnx::errc::duplicate_entry, "permutation image repeated");
      seen[forward[i]] = 1;
    }
    cudaStream_t st = ctx->stream;
    void *din = nullptr, *dout = nullptr, *dfwd = nullptr;
    const size_t bytes = static_cast<size_t>(n) * row_bytes;
    check(cudaMallocAsync(&din, bytes, st), "alloc");
    check(cudaMallocAsync(&dout, bytes, st), "alloc");
    check(cudaMallocAsync(&dfwd, sizeof(int32_t) * n, st), "alloc");
    check(cudaMemcpyAsync(din, in, bytes, cudaMemcpyHostToDevice, st), "h2d");
    check(cudaMemcpyAsync(dfwd, forward, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st), "h2d");
    knnx_dev::launch_permute(n, row_bytes, din, static_cast<const int32_t*>(dfwd), dout, true, st);
    launched(ctx, "permute");
    check(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, st), "d2h");
    for (void* p : {din, dout, dfwd}) check(cudaFreeAsync(p, st), "free");
    check(cudaStreamSynchronize(st), "sync");
    return KNNX_OK;
  });
}

int knnx_meanshift_host(knnx_op_t op, const float* t_in, const float* s, int32_t dim, double h,
                        float* t_out) {
  return guard([&] {
    require(op != nullptr && t_in != nullptr && s != nullptr && t_out != nullptr,
            knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(op->ctx->device);
    require(h > 0.0, knnx::errc::non_positive_bandwidth, "bandwidth must be positive");
    require(dim >= 1 && dim <= 1024, knnx::errc::invalid_argument, "dim out of range");
    const int32_t ld = (dim + 3) / 4 * 4;
    cudaStream_t st = op->ctx->stream;
    float* dout = nullptr;
    const size_t tb = sizeof(float) * static_cast<size_t>(std::max(1, op->n_rows)) * ld;
    // t_in == s (the targets start at the sources): staged once
    const bool same = t_in == s && op->n_rows <= op->n_cols;
    float* ds = stage_points(s, op->n_cols, dim, ld, st);
    float* dt = same ? ds : stage_points(t_in, op->n_rows, dim, ld, st);
    check(cudaMallocAsync(&dout, tb, st), "alloc");
    const double thresh = 745.1332191019412 * 2.0 * h * h;
    const float zt = thresh > 3.0e38 ? INFINITY : static_cast<float>(thresh);
    knnx_dev::launch_meanshift(*op, dt, ld, ds, ld, dim, gauss_c2(h), zt, dout, op->ctx->d_flag, st);
    launched(op->ctx, "meanshift");
    unstage_points(t_out, dout, op->n_rows, dim, ld, st);
    if (!same) check(cudaFreeAsync(dt, st), "free");
    check(cudaFreeAsync(ds, st), "free");
    check(cudaFreeAsync(dout, st), "free");
    return take_flag(op->ctx);
  });
}

int knnx_tsne_attr_dev(knnx_op_t op, const float* y, int32_t dim, float* f,
                       int32_t store_affinities, float step, float* y_out) {
  return guard([&] {
    require(op != nullptr && y != nullptr && f != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(op->ctx->device);
    // a row-block shard holds rows [row_base, row_base + n_rows) of a square problem
    require(op->is_shard ? op->row_base + op->n_rows <= op->n_cols : op->n_rows == op->n_cols,
            knnx::errc::not_square, "affinity matrix is not square");
    require(dim >= 1 && dim <= 3, knnx::errc::dim_mismatch, "embedding dimension must be 1..3");
    require(op->has_vals, knnx::errc::invalid_argument, "t-SNE needs stored affinities");
    require(y_out == nullptr || y_out != y, knnx::errc::invalid_argument, "y_out aliases y");
    knnx_dev::TsneOut out;
    out.local = y_out;
    knnx_dev::launch_tsne(*op, y, dim, f, store_affinities != 0, step, out, op->ctx->stream);
    launched(op->ctx, "tsne");
    return KNNX_OK;
  });
}

int knnx_tsne_attr_host(knnx_op_t op, const float* y, int32_t dim, float* f,
                        int32_t store_affinities) {
  return guard([&] {
    require(op != nullptr && y != nullptr && f != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(op->ctx->device);
    require(op->n_rows == op->n_cols, knnx::errc::not_square, "affinity matrix is not square");
    require(dim >= 1 && dim <= 3, knnx::errc::dim_mismatch, "embedding dimension must be 1..3");
    require(op->has_vals, knnx::errc::invalid_argument, "t-SNE needs stored affinities");
    cudaStream_t st = op->ctx->stream;
    const size_t bytes = sizeof(float) * static_cast<size_t>(std::max(1, op->n_rows)) * dim;
    float *dy = nullptr, *df = nullptr;
    check(cudaMallocAsync(&dy, bytes, st), "alloc");
    check(cudaMallocAsync(&df, bytes, st), "alloc");
    check(cudaMemcpyAsync(dy, y, sizeof(float) * op->n_rows * dim, cudaMemcpyHostToDevice, st), "h2d");
    knnx_dev::launch_tsne(*op, dy, dim, df, store_affinities != 0, 0.0f, knnx_dev::TsneOut{}, st);
    launched(op->ctx, "tsne");
    check(cudaMemcpyAsync(f, df, sizeof(float) * op->n_rows * dim, cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaFreeAsync(dy, st), "free");
    check(cudaFreeAsync(df, st), "free");
    check(cudaStreamSynchronize(st), "sync");
    return KNNX_OK;
  });
}

// ---------------------------------------------------------------------------
// permutations and tools

int knnx_permute_rows_dev(knnx_ctx_t ctx, int32_t n, int64_t row_bytes, const void* in,
                          const int32_t* forward, void* out) {
  return guard([&] {
    require(ctx != nullptr && (n == 0 || (in && forward && out)), knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(ctx->device);
    require(row_bytes >= 0 && row_bytes % 4 == 0, knnx::errc::invalid_argument,
            "row_bytes must be a multiple of 4");
    require(in != out, knnx::errc::invalid_argument, "in-place permutation is not supported");
    knnx_dev::launch_permute(n, row_bytes, in, forward, out, true, ctx->stream);
    launched(ctx, "permute");
    return KNNX_OK;
  });
}

int knnx_gather_rows_dev(knnx_ctx_t ctx, int32_t n, int64_t row_bytes, const void* in,
                         const int32_t* index, void* out) {
  return guard([&] {
    require(ctx != nullptr && (n == 0 || (in && index && out)), knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(ctx->device);
    require(row_bytes >= 0 && row_bytes % 4 == 0, knnx::errc::invalid_argument,
            "row_bytes must be a multiple of 4");
    require(in != out, knnx::errc::invalid_argument, "in-place gather is not supported");
    knnx_dev::launch_permute(n, row_bytes, in, index, out, false, ctx->stream);
    launched(ctx, "gather");
    return KNNX_OK;
  });
}

int knnx_copy_async(knnx_ctx_t ctx, void* dst, const void* src, int64_t bytes) {
  return guard([&] {
    require(ctx != nullptr && (bytes == 0 || (dst && src)), knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(ctx->device);
    require(bytes >= 0 && bytes % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 &&
                reinterpret_cast<uintptr_t>(src) % 16 == 0,
            knnx::errc::invalid_argument, "copy needs 16-byte aligned pointers and sizes");
    knnx_dev::launch_copy(dst, src, bytes, ctx->stream);
    launched(ctx, "copy");
    return KNNX_OK;
  });
}

int knnx_knn_dev(knnx_ctx_t ctx, const float* t, int32_t m, const float* s, int32_t n, int32_t ld,
                 int32_t dim, int32_t k, int32_t self_set, int32_t* ids, float* d2) {
  return guard([&] {
    require(ctx != nullptr && ids != nullptr && d2 != nullptr, knnx::errc::invalid_argument,
            "null argument");
    // wide points go to the tensor-core builder (same output convention)
    if (dim > 64) return knnx_knn_wide_dev(ctx, t, m, s, n, ld, dim, k, 0, self_set, ids, d2, nullptr);
    DeviceGuard dg(ctx->device);
    require(dim >= 1, knnx::errc::invalid_argument, "dim must be >= 1");
    check_points(t, ld, dim);
    check_points(s, ld, dim);
    require(k >= 1, knnx::errc::invalid_argument, "k must be >= 1");
    require(k <= (self_set ? n - 1 : n), knnx::errc::k_too_large,
            "k = " + std::to_string(k) + " with " + std::to_string(n) + " sources");
    require(k <= 256, knnx::errc::too_large, "device kNN supports k <= 256");
    knnx_dev::launch_knn(t, m, s, n, ld, dim, k, self_set != 0, ids, d2, ctx->stream);
    launched(ctx, "knn", 3);
    return KNNX_OK;
  });
}

}  // extern "C"
