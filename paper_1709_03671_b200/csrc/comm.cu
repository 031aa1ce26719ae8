// Multi-device communicator of the C ABI (include/knnx.h "multi-device";
// SURVEY.md §8b item 1, §8e).
//
// The reference's only parallelism is spmv_hier_parallel: one call spawns
// worker threads that take block rows (runs of top blocks with the same
// row_node) from an atomic queue (proj/src/kernels.cpp:63-101); results are
// bit-identical for any worker count.  Here the workers are GPUs: the
// cluster-ordered rows are cut into row blocks (one operator shard per rank,
// knnx_op_set_row_base) and every row's sum stays on one device, so sharded
// results are bit-identical to one device.  The iterations that move data
// between steps (power-iteration x, mean-shift targets, the t-SNE embedding)
// exchange it through a knnx_comm:
//
//  * NCCL (one process per GPU, or one process driving distinct GPUs):
//    libnccl.so.2 is opened at run time -- the copy torch already loaded when
//    there is one -- so libknnx.so has no link-time NCCL dependency;
//  * local (one process, ranks may share a device -- the 1-GPU test mode):
//    stream-ordered device / peer copies between the ranks' buffers.
//
// The B200-native exchange for the t-SNE step is fused into the force
// kernel: knnx_tsne_attr_peers_dev stores every updated embedding row straight
// into all ranks' replicated embeddings (NVLink peer stores through P2P or
// CUDA-IPC mappings), so no all-gather runs after the kernel; a stream-ordered
// barrier (knnx_comm_barrier*) then orders the next step.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened with dlopen

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

#include "knnx_internal.cuh"
#include "knnx_rt.cuh"

using namespace knnx_rt;

namespace {

struct Nccl {
  void* h = nullptr;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok() const { return h != nullptr; }
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process's copy first (torch loads libnccl.so.2 from its wheel)
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      const char* e = dlerror();
      n.why = e ? e : "libnccl.so.2 not found";
      return;
    }
    auto sym = [&](auto& fp, const char* s) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(n.h, s));
      if (!fp) n.why = std::string("missing NCCL symbol ") + s;
    };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommInitAll, "ncclCommInitAll");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.AllGather, "ncclAllGather");
    sym(n.AllReduce, "ncclAllReduce");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    sym(n.GetErrorString, "ncclGetErrorString");
    if (!n.why.empty()) n.h = nullptr;
  });
  return n;
}

const Nccl& need_nccl() {
  const Nccl& n = nccl();
  if (!n.ok())
    throw knnx::error(knnx::errc::unsupported, "Unsupported: NCCL unavailable (" + n.why + ")");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw knnx::error(knnx::errc::unsupported,
                      std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

// ranks of one process-local group share this (events for the stream-ordered
// exchanges and barriers)
struct LocalGroup {
  std::vector<knnx_context*> ctxs;
  std::vector<cudaEvent_t> ev;  // one per rank
  ~LocalGroup() {
    for (size_t r = 0; r < ev.size(); ++r) {
      cudaSetDevice(ctxs[r]->device);
      cudaEventDestroy(ev[r]);
    }
  }
};

}  // namespace

struct knnx_comm {
  knnx_context* ctx = nullptr;
  int32_t nranks = 1, rank = 0, transport = KNNX_COMM_LOCAL;
  ncclComm_t nccl = nullptr;
  int* d_scratch = nullptr;  // barrier all-reduce operand
  std::shared_ptr<LocalGroup> group;
};

namespace {

void destroy_comm(knnx_comm* c) {
  if (!c) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(c->ctx->device);
  if (c->nccl) nccl().CommDestroy(c->nccl);
  if (c->d_scratch) cudaFree(c->d_scratch);
  if (prev >= 0) cudaSetDevice(prev);
  delete c;
}

// every rank's stream waits for every other rank's work issued so far
void local_barrier(const knnx_comm_t* comms, int32_t n) {
  LocalGroup& g = *comms[0]->group;
  for (int32_t r = 0; r < n; ++r) {
    DeviceGuard dg(g.ctxs[r]->device);
    check(cudaEventRecord(g.ev[r], g.ctxs[r]->stream), "event");
  }
  for (int32_t q = 0; q < n; ++q) {
    DeviceGuard dg(g.ctxs[q]->device);
    for (int32_t r = 0; r < n; ++r)
      if (r != q) check(cudaStreamWaitEvent(g.ctxs[q]->stream, g.ev[r], 0), "wait");
  }
}

void check_local_set(const knnx_comm_t* comms, int32_t n) {
  require(comms != nullptr && n >= 1 && comms[0] != nullptr && comms[0]->group,
          knnx::errc::invalid_argument, "comms must be the handles of one knnx_comm_init_local group");
  require(n == comms[0]->nranks, knnx::errc::size_mismatch, "pass every rank of the group");
  for (int32_t r = 0; r < n; ++r)
    require(comms[r] && comms[r]->group == comms[0]->group && comms[r]->rank == r,
            knnx::errc::invalid_argument, "comms[r] must be rank r of one local group");
}

}  // namespace

extern "C" {

int knnx_comm_unique_id(void* id) {
  return guard([&] {
    require(id != nullptr, knnx::errc::invalid_argument, "null id buffer");
    ncclUniqueId u;
    nccl_check(need_nccl().GetUniqueId(&u), "GetUniqueId");
    std::memcpy(id, &u, sizeof u);
    return KNNX_OK;
  });
}

int knnx_comm_init_rank(knnx_ctx_t ctx, int32_t nranks, int32_t rank, const void* id,
                        knnx_comm_t* out) {
  return guard([&] {
    require(ctx != nullptr && out != nullptr && id != nullptr, knnx::errc::invalid_argument,
            "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, knnx::errc::invalid_argument,
            "rank outside [0, nranks)");
    DeviceGuard dg(ctx->device);
    auto c = std::unique_ptr<knnx_comm, void (*)(knnx_comm*)>(new knnx_comm, destroy_comm);
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    c->transport = KNNX_COMM_NCCL;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    nccl_check(need_nccl().CommInitRank(&c->nccl, nranks, u, rank), "CommInitRank");
    check(cudaMalloc(&c->d_scratch, sizeof(int)), "cudaMalloc");
    *out = c.release();
    return KNNX_OK;
  });
}

int knnx_comm_init_local(int32_t nranks, const knnx_ctx_t* ctxs, knnx_comm_t* comms) {
  return guard([&] {
    require(nranks >= 1 && nranks <= knnx_dev::kMaxPeers && ctxs != nullptr && comms != nullptr,
            knnx::errc::invalid_argument, "1..8 ranks");
    auto group = std::make_shared<LocalGroup>();
    std::set<int> devs;
    for (int32_t r = 0; r < nranks; ++r) {
      require(ctxs[r] != nullptr, knnx::errc::invalid_argument, "null context");
      group->ctxs.push_back(ctxs[r]);
      devs.insert(ctxs[r]->device);
    }
    for (int32_t r = 0; r < nranks; ++r) {
      DeviceGuard dg(ctxs[r]->device);
      cudaEvent_t e;
      check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      group->ev.push_back(e);
    }
    const bool distinct = static_cast<int32_t>(devs.size()) == nranks;
    // peer access between distinct devices (the fused peer stores and the
    // local copies read / write other GPUs' memory directly)
    for (int d : devs)
      for (int e : devs)
        if (d != e) {
          int can = 0;
          check(cudaDeviceCanAccessPeer(&can, d, e), "peer query");
          if (!can) continue;
          DeviceGuard dg(d);
          const cudaError_t pe = cudaDeviceEnablePeerAccess(e, 0);
          if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) check(pe, "peer access");
          cudaGetLastError();
        }
    std::vector<ncclComm_t> nc(nranks, nullptr);
    const bool use_nccl = distinct && nranks > 1 && nccl().ok();
    if (use_nccl) {
      std::vector<int> devlist;
      for (int32_t r = 0; r < nranks; ++r) devlist.push_back(ctxs[r]->device);
      nccl_check(nccl().CommInitAll(nc.data(), nranks, devlist.data()), "CommInitAll");
    }
    for (int32_t r = 0; r < nranks; ++r) {
      auto* c = new knnx_comm;
      c->ctx = ctxs[r];
      c->nranks = nranks;
      c->rank = r;
      c->transport = use_nccl ? KNNX_COMM_NCCL : KNNX_COMM_LOCAL;
      c->nccl = nc[r];
      c->group = group;
      comms[r] = c;
    }
    return KNNX_OK;
  });
}

int knnx_comm_destroy(knnx_comm_t comm) {
  return guard([&] {
    destroy_comm(comm);
    return KNNX_OK;
  });
}

int knnx_comm_info(knnx_comm_t comm, int32_t* nranks, int32_t* rank, int32_t* transport) {
  return guard([&] {
    require(comm != nullptr, knnx::errc::invalid_argument, "null comm");
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank;
    if (transport) *transport = comm->transport;
    return KNNX_OK;
  });
}

int knnx_allgather_rows_dev(knnx_comm_t comm, void* buf, int64_t rows_per_rank, int64_t row_bytes) {
  return guard([&] {
    require(comm != nullptr && buf != nullptr && rows_per_rank >= 0 && row_bytes >= 0,
            knnx::errc::invalid_argument, "bad argument");
    if (comm->nranks == 1 || rows_per_rank == 0 || row_bytes == 0) return KNNX_OK;
    require(comm->nccl != nullptr && !comm->group, knnx::errc::invalid_argument,
            "a process-local group exchanges with knnx_allgather_rows_local");
    DeviceGuard dg(comm->ctx->device);
    const size_t blk = static_cast<size_t>(rows_per_rank) * row_bytes;
    char* b = static_cast<char*>(buf);
    nccl_check(nccl().AllGather(b + blk * comm->rank, b, blk, ncclUint8, comm->nccl,
                                comm->ctx->stream),
               "AllGather");
    return KNNX_OK;
  });
}

int knnx_allgather_rows_local(const knnx_comm_t* comms, int32_t nranks, void* const* bufs,
                              int64_t rows_per_rank, int64_t row_bytes) {
  return guard([&] {
    check_local_set(comms, nranks);
    require(bufs != nullptr && rows_per_rank >= 0 && row_bytes >= 0, knnx::errc::invalid_argument,
            "bad argument");
    for (int32_t r = 0; r < nranks; ++r)
      require(bufs[r] != nullptr, knnx::errc::invalid_argument, "null buffer");
    if (nranks == 1 || rows_per_rank == 0 || row_bytes == 0) return KNNX_OK;
    const size_t blk = static_cast<size_t>(rows_per_rank) * row_bytes;
    if (comms[0]->transport == KNNX_COMM_NCCL) {
      const Nccl& n = need_nccl();
      nccl_check(n.GroupStart(), "GroupStart");
      for (int32_t r = 0; r < nranks; ++r) {
        DeviceGuard dg(comms[r]->ctx->device);
        char* b = static_cast<char*>(bufs[r]);
        nccl_check(n.AllGather(b + blk * r, b, blk, ncclUint8, comms[r]->nccl, comms[r]->ctx->stream),
                   "AllGather");
      }
      nccl_check(n.GroupEnd(), "GroupEnd");
      return KNNX_OK;
    }
    // local transport: every rank's block copied into every other rank's
    // buffer on the destination's stream, after the source rank's pending
    // work (its block is final) -- then a barrier so no rank overwrites a
    // block before every copy of it has been taken
    LocalGroup& g = *comms[0]->group;
    for (int32_t r = 0; r < nranks; ++r) {
      DeviceGuard dg(g.ctxs[r]->device);
      check(cudaEventRecord(g.ev[r], g.ctxs[r]->stream), "event");
    }
    for (int32_t q = 0; q < nranks; ++q) {
      DeviceGuard dg(g.ctxs[q]->device);
      for (int32_t r = 0; r < nranks; ++r) {
        if (r == q) continue;
        check(cudaStreamWaitEvent(g.ctxs[q]->stream, g.ev[r], 0), "wait");
        check(cudaMemcpyPeerAsync(static_cast<char*>(bufs[q]) + blk * r, g.ctxs[q]->device,
                                  static_cast<const char*>(bufs[r]) + blk * r, g.ctxs[r]->device,
                                  blk, g.ctxs[q]->stream),
              "peer copy");
      }
    }
    local_barrier(comms, nranks);
    return KNNX_OK;
  });
}

int knnx_comm_barrier_local(const knnx_comm_t* comms, int32_t nranks) {
  return guard([&] {
    check_local_set(comms, nranks);
    local_barrier(comms, nranks);
    return KNNX_OK;
  });
}

int knnx_comm_barrier(knnx_comm_t comm) {
  return guard([&] {
    require(comm != nullptr, knnx::errc::invalid_argument, "null comm");
    if (comm->nranks == 1) return KNNX_OK;
    require(comm->nccl != nullptr && !comm->group, knnx::errc::invalid_argument,
            "a process-local group synchronises with knnx_comm_barrier_local");
    DeviceGuard dg(comm->ctx->device);
    // a 1-element all-reduce completes on every rank only after all ranks
    // reached it on their streams: a stream-ordered barrier
    nccl_check(nccl().AllReduce(comm->d_scratch, comm->d_scratch, 1, ncclInt32, ncclSum, comm->nccl,
                                comm->ctx->stream),
               "AllReduce");
    return KNNX_OK;
  });
}

int knnx_tsne_attr_peers_dev(knnx_op_t op, const float* y, int32_t dim, float* f, float step,
                             float* const* y_full_outs, int32_t n_out) {
  return guard([&] {
    require(op != nullptr && y != nullptr && f != nullptr && y_full_outs != nullptr,
            knnx::errc::invalid_argument, "null argument");
    require(n_out >= 1 && n_out <= knnx_dev::kMaxPeers, knnx::errc::invalid_argument,
            "1..8 output embeddings");
    require(op->is_shard ? op->row_base + op->n_rows <= op->n_cols : op->n_rows == op->n_cols,
            knnx::errc::not_square, "affinity matrix is not square");
    require(dim >= 1 && dim <= 3, knnx::errc::dim_mismatch, "embedding dimension must be 1..3");
    require(op->has_vals, knnx::errc::invalid_argument, "t-SNE needs stored affinities");
    DeviceGuard dg(op->ctx->device);
    knnx_dev::TsneOut out;
    for (int32_t q = 0; q < n_out; ++q) {
      require(y_full_outs[q] != nullptr && y_full_outs[q] != y, knnx::errc::invalid_argument,
              "output embeddings must be distinct from the input");
      out.peer[q] = y_full_outs[q];
    }
    out.n_peer = n_out;
    knnx_dev::launch_tsne(*op, y, dim, f, false, step, out, op->ctx->stream);
    launched(op->ctx, "tsne");
    return KNNX_OK;
  });
}

int knnx_ipc_get_handle(knnx_ctx_t ctx, const void* dev_ptr, void* handle) {
  return guard([&] {
    require(ctx != nullptr && dev_ptr != nullptr && handle != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(ctx->device);
    cudaIpcMemHandle_t h;
    check(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof h);
    return KNNX_OK;
  });
}

int knnx_ipc_open(knnx_ctx_t ctx, const void* handle, void** dev_ptr) {
  return guard([&] {
    require(ctx != nullptr && handle != nullptr && dev_ptr != nullptr, knnx::errc::invalid_argument,
            "null argument");
    DeviceGuard dg(ctx->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    check(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return KNNX_OK;
  });
}

int knnx_ipc_close(knnx_ctx_t ctx, void* dev_ptr) {
  return guard([&] {
    require(ctx != nullptr && dev_ptr != nullptr, knnx::errc::invalid_argument, "null argument");
    DeviceGuard dg(ctx->device);
    check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
    return KNNX_OK;
  });
}

}  // extern "C"
