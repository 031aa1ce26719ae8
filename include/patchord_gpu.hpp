// include/patchord_gpu.hpp -- drop-in GPU versions of patchord's interaction
// kernels, for a patchord maintainer to add beside proj/include/patchord/.
//
// Same types, names, argument meaning and error behaviour as the reference
// (proj/include/patchord/kernels.hpp:23-65, hier.hpp:58-59): inputs are the
// reference's own SparseMatrix / HierBlockMatrix / PointSet / TaggedVector,
// errors are thrown as patchord::error with the reference's errc.  Every
// multiply runs in libknnx.so (sm_100a) through the C ABI of include/knnx.h.
//
// Two levels:
//  * free functions with the reference signatures (upload + compute +
//    download per call; blocking like the reference);
//  * gpu::Operator, which keeps a matrix resident on the device for iterated
//    use (the form a production loop should use).
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "patchord/core.hpp"
#include "patchord/hier.hpp"
#include "patchord/kernels.hpp"

struct knnx_context;
struct knnx_operator;

namespace patchord::gpu {

// one CUDA device + stream (knnx_ctx_create); the free functions use device 0
class Device {
 public:
  explicit Device(int device = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  knnx_context* handle() const { return ctx_; }
  static Device& default_device();

 private:
  knnx_context* ctx_ = nullptr;
};

// A point set resident on the device: n x ld fp32, zero padded.  Coordinates
// use ld = dim rounded up to 4 (16-byte rows for the kernels); t-SNE
// embeddings and forces use ld = dim (padded = false).
class PointBuffer {
 public:
  PointBuffer(Device& dev, const PointSet& p, bool padded = true);  // upload
  PointBuffer(Device& dev, index_t n, index_t dim, bool padded = true);
  ~PointBuffer();
  PointBuffer(const PointBuffer&) = delete;
  PointBuffer& operator=(const PointBuffer&) = delete;
  PointBuffer(PointBuffer&& o) noexcept;
  void upload(const PointSet& p);  // same shape
  PointSet download() const;
  float* data() const { return d_; }
  index_t n_points() const { return n_; }
  index_t dim() const { return dim_; }
  index_t ld() const { return ld_; }

 private:
  Device* dev_ = nullptr;
  float* d_ = nullptr;
  index_t n_ = 0, dim_ = 0, ld_ = 0;
};

// A matrix resident on the device: original order (SparseMatrix, the
// spmv_flat path) or cluster order (HierBlockMatrix leaf payload, the
// spmv_hier path with 16-bit cluster tiles).
class Operator {
 public:
  Operator(Device& dev, const SparseMatrix& m);
  Operator(Device& dev, const HierBlockMatrix& h);
  ~Operator();
  Operator(const Operator&) = delete;
  Operator& operator=(const Operator&) = delete;

  PotentialVector spmv(const ChargeVector& x) const;          // y = A x
  void set_values(const std::vector<double>& canonical_vals);  // canonical entry order
  std::vector<double> values() const;

  // Resident non-stationary forms for iterated loops: the pattern, the
  // affinities and the point sets stay on the device between calls.
  // iterate_interactions with the Gaussian value model, one step
  // (kernels.cpp:217-228): weights exp(-|t_i - s_j|^2 / (2 h^2)) recomputed
  PotentialVector gauss_spmv(const PointBuffer& targets, const PointBuffer& sources,
                             double bandwidth, const ChargeVector& x) const;
  // meanshift_step over the operator's neighbour rows (kernels.cpp:184-208):
  // t_out = sum_j w_ij s_j / sum_j w_ij, sources fixed
  void meanshift(const PointBuffer& t_in, const PointBuffer& sources, double bandwidth,
                 PointBuffer& t_out) const;
  // tsne_attractive_step's force (kernels.cpp:103-136) from the stored P,
  // which stays unchanged; step != 0 also writes y_out = y - step F
  void tsne(const PointBuffer& y, PointBuffer& forces, double step = 0.0,
            PointBuffer* y_out = nullptr) const;
  index_t n_rows() const { return n_rows_; }
  index_t n_cols() const { return n_cols_; }
  knnx_operator* handle() const { return op_; }

 private:
  knnx_operator* op_ = nullptr;
  Device* dev_ = nullptr;
  index_t n_rows_ = 0, n_cols_ = 0;
  std::string row_tag_, col_tag_;
  bool hier_ = false;
  // page-locked fp32 staging for spmv() (one caller at a time per Operator): x is narrowed straight into it and y
  // widened straight out of it (allocated on first use)
  mutable float* x_stage_ = nullptr;
  mutable float* y_stage_ = nullptr;
};

// ---- drop-in replacements (same signatures as proj/include/patchord/kernels.hpp) ----
PotentialVector spmv_flat(const SparseMatrix& m, const ChargeVector& x);
PotentialVector spmv_hier(const HierBlockMatrix& h, const ChargeVector& x);
// `workers` is validated like the reference (>= 1) and otherwise ignored: the
// device result is the same for any worker count (kernels.hpp:33-35 contract)
PotentialVector spmv_hier_parallel(const HierBlockMatrix& h, const ChargeVector& x,
                                   index_t workers);
// rewrites the stored affinities to a_ij in place, like the reference
PointSet tsne_attractive_step(HierBlockMatrix& h, const PointSet& y, index_t dim_out);
// one weighted-mean shift over the state's kNN rows; the kNN refresh every
// refresh_period steps runs on the device too (knnx_knn_dev for dim <= 64,
// the tensor-core knnx_knn_wide_dev beyond), the optional reorder is the reference's
// host ordering + the device permutation
MeanShiftState meanshift_step(MeanShiftState state);
// generic value model: value_fn(kappa) is user code and runs on the host; the
// multiply runs on the device
std::vector<PotentialVector> iterate_interactions(
    HierBlockMatrix& h,
    const std::function<std::function<double(index_t, index_t, double)>(index_t)>& value_fn,
    const std::vector<ChargeVector>& x_seq);
// Gaussian value model entirely on the device: values
// exp(-|t_i - s_j|^2 / (2 h^2)) recomputed every step, never stored
std::vector<PotentialVector> iterate_interactions_gaussian(const HierBlockMatrix& h,
                                                           const PointSet& targets,
                                                           const PointSet& sources,
                                                           double bandwidth,
                                                           const std::vector<ChargeVector>& x_seq);
// update_values with the Gaussian model (hier.hpp:58-59 + knn.cpp:86-108)
index_t update_values_gaussian(HierBlockMatrix& h, const PointSet& targets,
                               const PointSet& sources, double bandwidth);
// permute(PointSet) on the device, bit-exact (core.cpp:141-148)
PointSet permute(const PointSet& pts, const Permutation& p);

}  // namespace patchord::gpu
