/* include/knnx.h -- C ABI of the B200 kNN-interaction operator library
 * (paper_1709_03671_b200/libknnx.so).
 *
 * This is the drop-in boundary for the hot path of patchord (arXiv
 * 1709.03671's reference): every entry point below replaces one reference
 * interface, cited as proj/<file>:<line> (the reference C++ free-function API,
 * proj/include/patchord/kernels.hpp:23-65 and hier.hpp:58-59).  Plain
 * pointers and sizes only; no exceptions or C++ types cross it.
 *
 * Conventions
 *  - Return 0 on success; otherwise 1 + the ordinal of the reference's
 *    patchord::errc (proj/include/patchord/core.hpp:15-42, so DimMismatch = 4,
 *    NonPositiveBandwidth = 7, OrderingMismatch = 18, NonFiniteValue = 19,
 *    ZeroWeight = 20, InvalidArgument = 26), or KNNX_ERR_CUDA /
 *    KNNX_ERR_UNSUPPORTED.  knnx_last_error() returns the thread's message.
 *  - Arithmetic is fp32 on the device (the reference is fp64; parity is
 *    1e-5 relative).  Indices are int32.
 *  - Bandwidth h uses the reference convention w = exp(-|t - s|^2 / (2 h^2))
 *    (proj/src/knn.cpp:94, kernels.cpp:185).
 *  - "_dev" entry points take device pointers and are asynchronous on the
 *    context's stream; "_host" entry points take host pointers, copy in and
 *    out, and block (the reference's synchronous semantics).
 *  - Point sets on the device are row-major with a leading dimension
 *    (floats per row) that is a multiple of 4, so rows are 16-byte aligned.
 */
#ifndef KNNX_H
#define KNNX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNNX_OK 0
#define KNNX_ERR_DIM_MISMATCH 4
#define KNNX_ERR_NOT_SQUARE 6
#define KNNX_ERR_NON_POSITIVE_BANDWIDTH 7
#define KNNX_ERR_LOCAL_INDEX_OVERFLOW 17
#define KNNX_ERR_ORDERING_MISMATCH 18
#define KNNX_ERR_NON_FINITE_VALUE 19
#define KNNX_ERR_ZERO_WEIGHT 20
#define KNNX_ERR_INVALID_ARGUMENT 26
#define KNNX_ERR_CUDA 65
#define KNNX_ERR_UNSUPPORTED 66

/* operator layouts */
#define KNNX_ORDER_ORIGINAL 0 /* rows/cols as given; int32 columns (spmv_flat path) */
#define KNNX_ORDER_CLUSTER 1  /* tree-ordered rows; cluster tiles with 16-bit halo indices */

typedef struct knnx_context* knnx_ctx_t;
typedef struct knnx_operator* knnx_op_t;

typedef struct {
  int32_t n_rows, n_cols, order, tile_rows;
  int64_t nnz;          /* true nonzeros */
  int64_t stored;       /* stored entries incl. slice padding */
  int32_t n_tiles, max_halo;
  int64_t halo_total;   /* sum of per-tile halo sizes (cluster order) */
  int64_t device_bytes; /* bytes resident on the device for this operator */
  int32_t has_values, uniform_row_len; /* uniform_row_len: k if every row has k entries, else -1 */
} knnx_op_info_t;

int knnx_abi_version(void);
const char* knnx_last_error(void);

/* ---- context: one device, one stream (the reference's implicit CPU
 *      context; threading model proj/include/patchord/kernels.hpp:30-32) ---- */
int knnx_ctx_create(int device, knnx_ctx_t* out);
int knnx_ctx_destroy(knnx_ctx_t ctx);
/* launch on an external cudaStream_t (used as given: NULL is the legacy
 * default stream); knnx_ctx_use_own_stream restores the context's stream */
int knnx_ctx_set_stream(knnx_ctx_t ctx, void* stream);
int knnx_ctx_use_own_stream(knnx_ctx_t ctx);
void* knnx_ctx_stream(knnx_ctx_t ctx);
int knnx_ctx_sync(knnx_ctx_t ctx);
/* number of kernels this library launched on the context (instrumentation) */
int64_t knnx_ctx_launches(knnx_ctx_t ctx);

/* ---- device buffers (coordinate / charge / embedding
 * upload and download).  Point sets live on the device as n x ld floats,
 * ld >= dim (a multiple of 4 for the kernels' 16-byte rows), zero padded;
 * vectors are n x 1 with ld = 1.  The copies are blocking. */
int knnx_alloc(knnx_ctx_t ctx, int64_t bytes, void** dev);
int knnx_free(knnx_ctx_t ctx, void* dev);
/* page-locked, device-mapped host memory for the *_host entry points: with
 * such buffers x is read and y written over PCIe without a staging copy
 * (knnx_spmv_host*); free with knnx_host_free */
int knnx_host_alloc(int64_t bytes, void** host);
int knnx_host_free(void* host);
int knnx_upload_points(knnx_ctx_t ctx, const float* host, int32_t n, int32_t dim, int32_t ld,
                       float* dev);
int knnx_download_points(knnx_ctx_t ctx, const float* dev, int32_t n, int32_t dim, int32_t ld,
                         float* host);

/* ---- operator upload.  Replaces the reference's matrix containers as seen
 * by the kernels: SparseMatrix (proj/include/patchord/core.hpp:71-76) for
 * KNNX_ORDER_ORIGINAL and HierBlockMatrix leaf payload
 * (proj/include/patchord/hier.hpp:15-35, build_hier proj/src/hier.cpp:40-163)
 * for KNNX_ORDER_CLUSTER.  Input is canonical CSR (rows ascending, columns
 * strictly ascending within a row; row_ptr has n_rows+1 entries); vals may be
 * NULL for pattern-only operators (Gaussian / mean-shift recompute their
 * weights).  For the cluster order the rows must already be in the tree's
 * leaf order (proj/src/pipeline.cpp:163-166); tile_rows (multiple of 32,
 * 0 = 256) sets the row-tile height.  The caller keeps its host arrays. */
int knnx_op_create_csr(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                       const int64_t* row_ptr, const int32_t* cols, const float* vals,
                       int32_t order, int32_t tile_rows, knnx_op_t* out);
/* Same, with a row processing schedule (no counterpart in the reference: the
 * reference's rows run in tree order).  y, values and every per-row result
 * are unchanged; only the order in which rows are scheduled on the GPU
 * differs, so rows that share source points run together and their source
 * reads hit L2.  schedule_kind: KNNX_SCHEDULE_NONE (= knnx_op_create_csr),
 * KNNX_SCHEDULE_GRAPH (breadth-first over the operator's own graph; column c
 * is row c - col_base), KNNX_SCHEDULE_GIVEN (schedule[p] = row run p-th, a
 * permutation of n_rows). */
#define KNNX_SCHEDULE_NONE 0
#define KNNX_SCHEDULE_GRAPH 1
#define KNNX_SCHEDULE_GIVEN 2
int knnx_op_create_csr_sched(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                             const int64_t* row_ptr, const int32_t* cols, const float* vals,
                             int32_t order, int32_t tile_rows, int32_t schedule_kind,
                             int32_t col_base, const int32_t* schedule, knnx_op_t* out);
/* Same, with layout options for the high-degree t-SNE operator (C4's
 * symmetrised k = 90 graph).  Only knnx_tsne_attr_* accept such operators
 * (the other entry points return KNNX_ERR_INVALID_ARGUMENT); values, get/set
 * and results stay in the caller's canonical order.
 *  KNNX_OPT_RELABEL_COLS: columns [col_base, col_base + n_rows) are renumbered
 *    in schedule order (column col_base + schedule[p] becomes col_base + p) and
 *    every row's entries are re-sorted by the new number, so a row's
 *    neighbours that the breadth-first schedule placed together share 32-B
 *    sectors of the embedding; each call gathers y into that numbering first
 *    (one pass over n_cols rows).  Needs a schedule; per-row sums then run in
 *    the new column order (within fp32 rounding of the canonical order).
 *  KNNX_OPT_GROUP_INTERLEAVE: KNNX_ORDER_ORIGINAL only.  Inside each 32-row
 *    slice, entries 8i..8i+7 of a row are contiguous (an 8-lane group's loads
 *    of one step are one 32-B sector, a warp's one 128-B line) instead of
 *    SELL-32's row-interleaved columns. */
#define KNNX_OPT_RELABEL_COLS 1
#define KNNX_OPT_GROUP_INTERLEAVE 2
int knnx_op_create_csr_ex(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                          const int64_t* row_ptr, const int32_t* cols, const float* vals,
                          int32_t order, int32_t tile_rows, int32_t schedule_kind,
                          int32_t col_base, const int32_t* schedule, int32_t options,
                          knnx_op_t* out);
/* HierBlockMatrix-shaped input: leaf blocks in traversal order, each with
 * its row/col cluster offsets and a row-major payload of 16-bit local (lr,lc)
 * and values (proj/include/patchord/hier.hpp:15-24).  Flattened on the host
 * (proj/src/hier.cpp:182-191) and uploaded as KNNX_ORDER_CLUSTER. */
int knnx_op_create_hier_leaves(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols,
                               int32_t n_blocks, const int32_t* row_offset,
                               const int32_t* col_offset, const int64_t* block_ptr,
                               const uint16_t* lr, const uint16_t* lc, const float* vals,
                               int32_t tile_rows, knnx_op_t* out);
/* HBM1 dump of a HierBlockMatrix (proj/docs/hbm1-format.md, writer
 * proj/src/hier.cpp:291-323, reader :325-367) loaded straight into a cluster
 * operator; row_forward / col_forward (nullable, n_rows / n_cols entries)
 * receive the trees' leaf orders (forward[original] = position). */
int knnx_hbm1_info(const char* path, int32_t* n_rows, int32_t* n_cols, int64_t* nnz,
                   int32_t* cut_level);
int knnx_op_load_hbm1(knnx_ctx_t ctx, const char* path, int32_t tile_rows, int32_t* row_forward,
                      int32_t* col_forward, knnx_op_t* out);
/* cluster operator built ON THE DEVICE from device-resident kNN rows (ids:
 * m x k cluster positions, uniform k <= 32, rows in tree order): the sort /
 * bucketing of proj/src/core.cpp:75-92,130-139 and proj/src/hier.cpp:84-155
 * done by CUB block sorts per 256-row tile; pattern only (values via
 * knnx_update_gaussian_* or knnx_op_set_values).  Same arrays as
 * knnx_op_create_csr(..., KNNX_ORDER_CLUSTER, 256) on the same rows. */
int knnx_op_create_knn_dev(knnx_ctx_t ctx, const int32_t* ids, int32_t m, int32_t n_cols,
                           int32_t k, knnx_op_t* out);
/* t-SNE joint affinities built ON THE DEVICE from device kNN rows (C4's P;
 * the symmetrize of proj/src/knn.cpp:72-84 with values, whose host form is
 * csr_from_coo's sort of both orientations, proj/src/core.cpp:75-92):
 * ids / d2 are n x k neighbour ids and squared distances (self excluded);
 * p_j|i = exp(-d2_ij / (2 h^2)) / sum over the row, then
 * P = (P_cond + P_cond^T) * scale (scale = 1 / (2n) gives sum P = 1) as a
 * canonical CSR in device buffers allocated by the library (knnx_free):
 * row_ptr (n + 1 int64), cols (nnz int32), vals (nnz fp32). */
int knnx_tsne_affinities_dev(knnx_ctx_t ctx, const int32_t* ids, const float* d2, int32_t n,
                             int32_t k, double h, double scale, int64_t** row_ptr, int32_t** cols,
                             float** vals, int64_t* nnz);
/* Operator from a canonical CSR that already lives on the device (e.g. the
 * output of knnx_tsne_affinities_dev), KNNX_ORDER_ORIGINAL layout, 256-row
 * tiles: validation, the KNNX_SCHEDULE_GRAPH breadth-first schedule, the
 * per-tile length sort, slice offsets and the entry placement (plain or
 * KNNX_OPT_GROUP_INTERLEAVE) run on the device; the result is the operator
 * knnx_op_create_csr_ex builds on the host from the same arrays
 * (proj/src/core.cpp:75-92,130-139, hier.cpp:84-155 on the device).
 * row_ptr / cols / vals: device pointers (vals may be null); schedule: host
 * array for KNNX_SCHEDULE_GIVEN.  The CSR is not consumed.  A row block of a
 * larger device CSR is passed as row_ptr + r0 with the UNSHIFTED cols / vals
 * pointers (row_ptr[0] need not be 0; nnz = row_ptr[n_rows] - row_ptr[0]) and
 * col_base = r0, so a multi-GPU rank builds its shard from the full matrix. */
int knnx_op_create_csr_dev(knnx_ctx_t ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                           const int64_t* row_ptr, const int32_t* cols, const float* vals,
                           int32_t schedule_kind, int32_t col_base, const int32_t* schedule,
                           int32_t options, knnx_op_t* out);
/* slot -> row map of an operator (n_rows int32 on the host): the row the
 * kernels process in slot p (the schedule after the per-tile length sort);
 * identity for unscheduled uniform rows */
int knnx_op_slot_rows(knnx_op_t op, int32_t* slot_row_host);
int knnx_op_destroy(knnx_op_t op);
/* row-block shard (multi-GPU, proj/src/kernels.cpp:74-84 generalised): the
 * operator's local row i is global point row_base + i of a square problem;
 * t-SNE then reads y_i at row_base + i (targets for the other kernels are
 * passed already offset by the caller) */
int knnx_op_set_row_base(knnx_op_t op, int32_t row_base);
int knnx_op_info(knnx_op_t op, knnx_op_info_t* info);
/* replace / read back the stored values, canonical CSR entry order */
int knnx_op_set_values(knnx_op_t op, const float* vals_host);
int knnx_op_get_values(knnx_op_t op, float* vals_host);

/* ---- stationary operator y = A x.
 * replaces spmv_flat (proj/src/kernels.cpp:37-49) for KNNX_ORDER_ORIGINAL and
 * spmv_hier / spmv_hier_parallel (proj/src/kernels.cpp:51-101) for
 * KNNX_ORDER_CLUSTER.  x has n_cols entries, y n_rows. */
int knnx_spmv_dev(knnx_op_t op, const float* x, float* y);
int knnx_spmv_host(knnx_op_t op, const float* x, float* y);
/* n_steps independent host-buffer applications y_s = A x_s (xs: n_steps x
 * n_cols, ys: n_steps x n_rows host arrays, blocking): the H2D of step s+1
 * overlaps the multiply and D2H of step s on two streams.  Page-locked host
 * buffers give full copy bandwidth. */
int knnx_spmv_host_batch(knnx_op_t op, int32_t n_steps, const float* xs, float* ys);
/* n_steps applications y_s = A x_s (xs: n_steps x n_cols, ys: n_steps x
 * n_rows), captured into a CUDA graph; the graph is kept on the operator and
 * replayed while the same arguments come back (the reference's iteration
 * loop, proj/src/pipeline.cpp:296-312).  Needs a non-default stream. */
int knnx_spmv_batch_dev(knnx_op_t op, int32_t n_steps, const float* xs, float* ys);
/* same with explicit element strides between steps (0 = every step reads
 * the same x / writes the same y: the fixed-charge iteration of C2) */
int knnx_spmv_batch_strided_dev(knnx_op_t op, int32_t n_steps, const float* xs, int64_t x_stride,
                                float* ys, int64_t y_stride);

/* ---- non-stationary Gaussian operator: the value model of
 * iterate_interactions with gaussian_values (proj/src/kernels.cpp:217-228,
 * proj/src/hier.cpp:203-222, proj/src/knn.cpp:86-108):
 * y_i = sum_j exp(-|t_i - s_j|^2 / (2 h^2)) x_j, weights recomputed, never
 * stored.  T: n_rows x ld_t, S: n_cols x ld_s device arrays. */
int knnx_gauss_spmv_dev(knnx_op_t op, const float* t, int32_t ld_t, const float* s, int32_t ld_s,
                        int32_t dim, double h, const float* x, float* y);
/* host-pointer form: T (row_base + n_rows) x dim and S n_cols x dim unpadded */
int knnx_gauss_spmv_host(knnx_op_t op, const float* t, const float* s, int32_t dim, double h,
                         const float* x, float* y);
/* update_values(Gaussian) into the stored values (the reference's in-place
 * value refresh, proj/src/hier.cpp:203-222); non-finite -> NonFiniteValue */
int knnx_update_gaussian_dev(knnx_op_t op, const float* t, int32_t ld_t, const float* s,
                             int32_t ld_s, int32_t dim, double h);
int knnx_update_gaussian_host(knnx_op_t op, const float* t, const float* s, int32_t dim, double h);

/* ---- mean shift: one meanshift_step over the operator's fixed neighbor
 * rows (proj/src/kernels.cpp:184-215), targets t_in -> t_out (distinct
 * buffers), sources s fixed.  Weights are evaluated relative to the row's
 * nearest source (same normalised result); ZeroWeight is raised exactly when
 * every fp64 reference weight would underflow. */
int knnx_meanshift_dev(knnx_op_t op, const float* t_in, int32_t ld_t, const float* s,
                       int32_t ld_s, int32_t dim, double h, float* t_out);
int knnx_meanshift_host(knnx_op_t op, const float* t_in, const float* s, int32_t dim, double h,
                        float* t_out);

/* ---- t-SNE attractive force (proj/src/kernels.cpp:103-136):
 * F_i = sum_j p_ij (y_i - y_j) / (1 + |y_i - y_j|^2), dim 1..3, y and F
 * row-major n x dim (no padding).  store_affinities != 0 rewrites the stored
 * values to a_ij = p_ij / (1 + |y_i - y_j|^2) as the reference does in place.
 * step != 0 additionally applies y <- y - step * F (the framework's
 * embedding update), writing y_out (may not alias y). */
int knnx_tsne_attr_dev(knnx_op_t op, const float* y, int32_t dim, float* f,
                       int32_t store_affinities, float step, float* y_out);
int knnx_tsne_attr_host(knnx_op_t op, const float* y, int32_t dim, float* f,
                        int32_t store_affinities);

/* ---- permutation apply / inverse-apply (proj/src/core.cpp:141-148 and the
 * charge / checksum permutes proj/src/pipeline.cpp:67-71,189-191):
 * scatter: out[forward[i]] = in[i]; gather: out[i] = in[index[i]].
 * Rows of row_bytes (multiple of 4), bit-exact copies. */
int knnx_permute_rows_dev(knnx_ctx_t ctx, int32_t n, int64_t row_bytes, const void* in,
                          const int32_t* forward, void* out);
int knnx_gather_rows_dev(knnx_ctx_t ctx, int32_t n, int64_t row_bytes, const void* in,
                         const int32_t* index, void* out);
/* Streaming copy of `bytes` (multiple of 16, 16-B aligned pointers) by SM
 * loads/stores on the context stream.  Either side may be pinned, mapped host
 * memory (a UVA host pointer): the SMs then read or write host memory over
 * PCIe directly, without a copy engine (used by the host-buffer entry points). */
int knnx_copy_async(knnx_ctx_t ctx, void* dst, const void* src, int64_t bytes);
/* host-pointer scatter; validates forward as a bijection (core.cpp:94-109) */
int knnx_permute_rows_host(knnx_ctx_t ctx, int32_t n, int64_t row_bytes, const void* in,
                           const int32_t* forward, void* out);

/* ---- tools: exact brute-force kNN on the device in
 * fp32 (ascending (distance, index); self excluded when self_set) and the
 * bit-exact PCA covariance action used by the host ordering.  dim <= 64: a
 * block-pruned exact SIMT search; dim > 64 forwards to knnx_knn_wide_dev. */
int knnx_knn_dev(knnx_ctx_t ctx, const float* t, int32_t m, const float* s, int32_t n, int32_t ld,
                 int32_t dim, int32_t k, int32_t self_set, int32_t* ids, float* d2);
/* The same tool for wide points (any dim, meant for dim > 64; C5 has dim = 960),
 * where the distance screen |t|^2 + |s|^2 - 2 t.s over all pairs is a real dense
 * contraction: a tcgen05 / TMEM kernel (kind::tf32, TMA-fed, block-pruned by
 * tile bounding balls) keeps the n_cand best TF32 scores per row and an exact
 * fp32 pass re-ranks them (ascending (distance, index)).  Per row a
 * certificate is formed: every dropped source had a screen distance above
 * the row's threshold tau, and its screen error is bounded by the largest
 * signed error (screen - exact) seen on the row's own candidates plus their
 * whole spread; the row is certified when tau minus that bound exceeds its
 * exact k-th distance.  Uncertified rows
 * (clusters tight against their distance from the mean, where TF32 cannot
 * rank) are searched again by the exact SIMT kernel when dim <= 64 and
 * k <= 191, otherwise screened again with 3xTF32 operands (the low parts of
 * both operands multiplied as well, error ~2^-21 |t||s|) and certified anew;
 * what still fails is reported.  n_cand <= 0 picks max(64, 4k), at most 256;
 * k <= n_cand.
 * stats (may be null): 6 doubles -- [0] smallest certificate margin over all
 * rows (+inf for rows recomputed exactly), [1] rows left uncertified,
 * [2] source tiles multiplied, [3] tiles of the dense screen, [4] rows
 * recomputed by the exact search, [5] rows screened again with 3xTF32.
 * The call blocks (it reads the certificate count).
 * With stats == NULL, rows left uncertified make the call fail with
 * DegenerateData instead of returning them unflagged. */
int knnx_knn_wide_dev(knnx_ctx_t ctx, const float* t, int32_t m, const float* s, int32_t n,
                      int32_t ld, int32_t dim, int32_t k, int32_t n_cand, int32_t self_set,
                      int32_t* ids, float* d2, double* stats);

/* ---- multi-device.  The reference's only
 * parallelism is spmv_hier_parallel's worker threads over block rows
 * (proj/src/kernels.cpp:63-101, bit-identical for any worker count); here
 * the workers are GPUs, each holding a row-block shard of the operator
 * (knnx_op_set_row_base), with row sums kept on one device so the results
 * are bit-identical to one GPU.  A communicator carries the exchanges the
 * iterations need.  NCCL is opened at run time (libnccl.so.2, the process's
 * copy when one is loaded); ranks of one process that share a device (the
 * one-GPU test mode) exchange through device copies. */
typedef struct knnx_comm* knnx_comm_t;
#define KNNX_COMM_ID_BYTES 128
#define KNNX_COMM_NCCL 1  /* NCCL communicator (one process per GPU, or distinct GPUs) */
#define KNNX_COMM_LOCAL 2 /* one process, ranks may share a device: stream-ordered copies */
/* an NCCL unique id (KNNX_COMM_ID_BYTES) for knnx_comm_init_rank: made by one
 * rank, distributed by the host (e.g. torch.distributed) */
int knnx_comm_unique_id(void* id);
/* this process's rank of an nranks NCCL communicator on ctx's device */
int knnx_comm_init_rank(knnx_ctx_t ctx, int32_t nranks, int32_t rank, const void* id,
                        knnx_comm_t* out);
/* one process driving nranks contexts (1..8; comms[r] = rank r on ctxs[r]):
 * NCCL (ncclCommInitAll) when the devices are distinct, device copies when
 * they are not; peer access is enabled between distinct devices */
int knnx_comm_init_local(int32_t nranks, const knnx_ctx_t* ctxs, knnx_comm_t* comms);
int knnx_comm_destroy(knnx_comm_t comm);
int knnx_comm_info(knnx_comm_t comm, int32_t* nranks, int32_t* rank, int32_t* transport);
/* in-place all-gather of equal row blocks on the rank's context stream:
 * rank r owns rows [r * rows_per_rank, (r + 1) * rows_per_rank) of buf
 * (nranks * rows_per_rank rows of row_bytes); row blocks are tile-padded by
 * the caller (the x / targets / embedding exchanges of SURVEY.md §8e) */
int knnx_allgather_rows_dev(knnx_comm_t comm, void* buf, int64_t rows_per_rank, int64_t row_bytes);
/* the same exchange for every rank of a knnx_comm_init_local group at once
 * (bufs[r] = rank r's buffer), issued from one host thread */
int knnx_allgather_rows_local(const knnx_comm_t* comms, int32_t nranks, void* const* bufs,
                              int64_t rows_per_rank, int64_t row_bytes);
/* stream-ordered barriers: work issued after it on any rank's stream runs
 * after the work every rank issued before it */
int knnx_comm_barrier(knnx_comm_t comm);
int knnx_comm_barrier_local(const knnx_comm_t* comms, int32_t nranks);
/* t-SNE step with the exchange fused into the kernel: forces of the shard's
 * rows into f (local rows) and y_new = y - step F stored straight into every
 * rank's replicated embedding y_full_outs[q] (rows row_base + i; device
 * pointers valid in this process: own memory, peer memory with peer access,
 * or CUDA-IPC mappings from knnx_ipc_open) -- NVLink peer stores instead of
 * an all-gather after the kernel.  Follow with a barrier before the next
 * step reads the outputs. */
int knnx_tsne_attr_peers_dev(knnx_op_t op, const float* y, int32_t dim, float* f, float step,
                             float* const* y_full_outs, int32_t n_out);
/* CUDA IPC (64-byte handles) so processes of one node can map each other's
 * buffers for knnx_tsne_attr_peers_dev */
int knnx_ipc_get_handle(knnx_ctx_t ctx, const void* dev_ptr, void* handle);
int knnx_ipc_open(knnx_ctx_t ctx, const void* handle, void** dev_ptr);
int knnx_ipc_close(knnx_ctx_t ctx, void* dev_ptr);

/* ---- tensor cores (tcgen05 + TMEM): C = A B^T for row-major fp32 point rows
 * read as TF32 with fp32 accumulation (m x k times n x k, k a multiple of 32,
 * leading dimension ld >= k, ld % 4 == 0; C row-major with ldc).  The Gram
 * block of the kNN distance screen |a - b|^2 = |a|^2 + |b|^2 - 2 a.b (the
 * input builder's dense contraction; the operator itself
 * stays on CUDA cores). */
int knnx_gram_tf32_dev(knnx_ctx_t ctx, const float* a, int32_t m, const float* b, int32_t n,
                       int32_t ld, int32_t k, float* c, int64_t ldc);

#ifdef __cplusplus
}
#endif
#endif /* KNNX_H */
