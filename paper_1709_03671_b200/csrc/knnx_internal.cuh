// Internal declarations shared by the C-ABI runtime and the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/knnx.h"
#include "host/host.hpp"

struct knnx_context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int* d_flag = nullptr;  // deferred kernel error: [0] = code, [1] = lowest row index
  int64_t launches = 0;
  int n_sms = 148;
  // operators still alive on this context: knnx_ctx_destroy with live
  // operators only marks the context closed and the last knnx_op_destroy
  // frees it (garbage collectors may destroy handles in any order)
  int64_t live_ops = 0;
  bool closed = false;
};

struct knnx_operator {
  knnx_context* ctx = nullptr;
  int32_t n_rows = 0, n_cols = 0, order = 0, tile_rows = 0, n_tiles = 0, n_slices = 0;
  int32_t max_halo = 0, max_slice_len = 0, uniform_len = -1;
  int32_t row_base = 0;          // global point index of local row 0 (row-block shards)
  bool is_shard = false;         // set by knnx_op_set_row_base
  int64_t nnz = 0, stored = 0, halo_total = 0, device_bytes = 0;
  bool has_vals = false;
  // device arrays (SELL-32 entry layout)
  int64_t* d_slice_off = nullptr;
  int32_t* d_slice_len = nullptr;
  int32_t* d_row_len = nullptr;
  int32_t* d_cols = nullptr;     // KNNX_ORDER_ORIGINAL: global column per stored entry
  uint16_t* d_lidx = nullptr;    // KNNX_ORDER_CLUSTER: halo-local column
  int64_t* d_halo_off = nullptr;
  int32_t* d_halo_ids = nullptr;
  float* d_vals = nullptr;
  int32_t* d_slot_row = nullptr; // slot -> row (SELL-sigma); null = identity
  // host copies for value set/get in canonical order
  std::vector<int64_t> h_row_ptr, h_slice_off;
  std::vector<int32_t> h_slot_of_row;  // row -> slot; empty = identity
  // KNNX_OPT_GROUP_INTERLEAVE: entries 8i..8i+7 of a slot contiguous
  int32_t interleave = 0;
  // KNNX_OPT_RELABEL_COLS: stored column p is caller column d_col_order[p];
  // h_pos[e] = index within its stored row of canonical entry e
  int32_t* d_col_order = nullptr;
  float* d_gather_ws = nullptr;
  int64_t gather_ws_floats = 0;
  std::vector<uint16_t> h_pos;
  // the last knnx_spmv_batch*_dev graph (re-instantiated when the call differs)
  struct GraphKey {
    int32_t n_steps = 0;
    const float* xs = nullptr;
    int64_t x_stride = 0;
    float* ys = nullptr;
    int64_t y_stride = 0;
    bool operator==(const GraphKey& o) const {
      return n_steps == o.n_steps && xs == o.xs && x_stride == o.x_stride && ys == o.ys &&
             y_stride == o.y_stride;
    }
  };
  GraphKey graph_key;
  cudaGraphExec_t graph_exec = nullptr;
  bool plain() const { return interleave == 0 && d_col_order == nullptr; }
  knnx_operator() = default;
  knnx_operator(const knnx_operator&) = delete;
  knnx_operator& operator=(const knnx_operator&) = delete;
  // frees whatever was uploaded, also when construction fails half way
  // (the create entry points hold the operator in a unique_ptr until done)
  ~knnx_operator() {
    if (!ctx) return;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);  // cudaFree waits for pending work
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (void* p : {static_cast<void*>(d_slice_off), static_cast<void*>(d_slice_len),
                    static_cast<void*>(d_row_len), static_cast<void*>(d_slot_row),
                    static_cast<void*>(d_cols), static_cast<void*>(d_lidx),
                    static_cast<void*>(d_halo_off), static_cast<void*>(d_halo_ids),
                    static_cast<void*>(d_vals), static_cast<void*>(d_col_order),
                    static_cast<void*>(d_gather_ws)})
      if (p) cudaFree(p);
    if (prev >= 0 && prev != ctx->device) cudaSetDevice(prev);
  }
  // stored position of entry q of slot p
  int64_t pos_of(int32_t p, int64_t q) const {
    const int64_t s = p / 32, lane = p % 32;
    if (interleave) return h_slice_off[s] + (q >> 3) * 256 + lane * 8 + (q & 7);
    return h_slice_off[s] + 32 * q + lane;
  }
  // stored position of canonical entry e (row r)
  int64_t entry_pos(int32_t r, int64_t e) const {
    const int32_t p = h_slot_of_row.empty() ? r : h_slot_of_row[r];
    return pos_of(p, h_pos.empty() ? e - h_row_ptr[r] : h_pos[e]);
  }
};

namespace knnx_dev {

// device-side error codes written to ctx->d_flag
constexpr int kFlagNone = 0;
constexpr int kFlagZeroWeight = 1 + 19;     // errc::zero_weight + 1
constexpr int kFlagNonFinite = 1 + 18;      // errc::non_finite_value + 1

void launch_spmv(const knnx_operator& op, const float* x, float* y, cudaStream_t st);
void launch_gauss_spmv(const knnx_operator& op, const float* t, int ld_t, const float* s,
                       int ld_s, int dim, float c2, const float* x, float* y, int* flag,
                       cudaStream_t st);
void launch_update_gaussian(const knnx_operator& op, const float* t, int ld_t, const float* s,
                            int ld_s, int dim, float c2, int* flag, cudaStream_t st);
void launch_meanshift(const knnx_operator& op, const float* t_in, int ld_t, const float* s,
                      int ld_s, int dim, float c2, float zero_thresh, float* t_out, int* flag,
                      cudaStream_t st);
// outputs of the fused t-SNE embedding update: the local rows (y_out of
// knnx_tsne_attr_dev, may be null) and up to kMaxPeers replicated full
// embeddings (one per rank; rows row_base + i) for knnx_tsne_attr_peers_dev
constexpr int kMaxPeers = 8;
struct TsneOut {
  float* local = nullptr;
  float* peer[kMaxPeers] = {};
  int n_peer = 0;
};
void launch_tsne(const knnx_operator& op, const float* y, int dim, float* f, bool store,
                 float step, const TsneOut& y_out, cudaStream_t st);
void launch_permute(int n, int64_t row_bytes, const void* in, const int32_t* idx, void* out,
                    bool scatter, cudaStream_t st);
// max_ctas: a PCIe-bound copy from mapped host memory needs few CTAs to cover
// the link latency and leaves the other SMs to a concurrent kernel
void launch_copy(void* dst, const void* src, int64_t bytes, cudaStream_t st, int max_ctas = 148 * 8);
void launch_knn(const float* t, int m, const float* s, int n, int ld, int dim, int k,
                bool self_set, int32_t* ids, float* d2, cudaStream_t st);
void build_tiles_from_knn(const int32_t* ids, int m, int k, int64_t** d_halo_off,
                          int32_t** d_halo_ids, uint16_t** d_lidx, int64_t* halo_total,
                          int* max_halo, cudaStream_t st);

}  // namespace knnx_dev
