/* include/knnx_host.h -- C ABI of the host-side (CPU, C++) half of libknnx.so:
 * the ☆ rows of SURVEY.md §2 that stay on the host and must be bit-exact --
 * ordering (PCA + partition tree), permutation, input formats -- plus the
 * seeded workload generators.  Same return-code convention as knnx.h.
 */
#ifndef KNNX_HOST_H
#define KNNX_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct knnx_csr* knnx_csr_t;
typedef struct knnx_tree* knnx_tree_t;

/* ---- Rng (proj/include/patchord/core.hpp:124-149) ---- */
int knnx_rng_u64(uint64_t seed, int64_t n, uint64_t* out);
int knnx_rng_uniform01(uint64_t seed, int64_t n, double* out);
int knnx_rng_normal(uint64_t seed, int64_t n, double* out);
/* order_scattered (proj/src/orderings.cpp:9-16) */
int knnx_order_scattered(int32_t n, uint64_t seed, int32_t* forward);

/* ---- workload generators (BASELINE.json configs) ----
 * kind 1: C1 mixture (n_clusters components, means U[-10,10]^dim, sigma p0)
 * kind 2: C2/C3 3-level mixture 16x16x16, scales 10/2/0.5, point noise p0
 * kind 3: C5 anisotropic 2-level mixture, n_clusters = n_top * n_sub packed
 *         as n_top = n_clusters >> 16, n_sub = n_clusters & 0xffff
 * kind 4: standard normal times p0 (t-SNE embedding init) */
int knnx_gen_points(int32_t kind, int32_t n, int32_t dim, int32_t n_clusters, double p0,
                    uint64_t seed, float* out);
int knnx_gen_uniform01(int64_t n, uint64_t seed, float* out);
int knnx_median_distance(const float* d2, int64_t count, double* out);

/* ---- canonical CSR handles ---- */
int knnx_csr_from_knn(const int32_t* ids, int32_t m, int32_t n, int32_t k, knnx_csr_t* out);
int knnx_csr_from_arrays(int32_t m, int32_t n, int64_t nnz, const int64_t* row_ptr,
                         const int32_t* cols, const float* vals, knnx_csr_t* out);
/* structural union with the transpose (proj/src/knn.cpp:72-84) */
int knnx_csr_symmetrize(knnx_csr_t a, knnx_csr_t* out);
/* union pattern with values scale * (a_ij + a_ji): the t-SNE joint
 * affinities P = (P_cond + P_cond^T) / 2N from row-conditional values */
int knnx_csr_symmetrize_values(knnx_csr_t a, double scale, knnx_csr_t* out);
/* every row's values divided by the row sum (conditional p_j|i) */
int knnx_csr_row_normalize(knnx_csr_t a);
/* renumber rows and columns by forward (proj/src/core.cpp:130-139) */
int knnx_csr_permute(knnx_csr_t a, const int32_t* forward, knnx_csr_t* out);
/* rows [r0, r1) as a new (r1-r0) x n_cols matrix (row-block shard) */
int knnx_csr_row_block(knnx_csr_t a, int32_t r0, int32_t r1, knnx_csr_t* out);
/* graph-locality row schedule used by KNNX_SCHEDULE_GRAPH (breadth-first,
 * lowest unvisited row first, neighbours in column order; column c is row
 * c - col_base); out receives n_rows row ids */
int knnx_csr_locality_schedule(knnx_csr_t a, int32_t col_base, int32_t* out);
int knnx_csr_set_values(knnx_csr_t a, const float* vals);
int knnx_csr_shape(knnx_csr_t a, int32_t* m, int32_t* n, int64_t* nnz, int32_t* has_values);
int knnx_csr_export(knnx_csr_t a, int64_t* row_ptr, int32_t* cols, float* vals);
void knnx_csr_destroy(knnx_csr_t a);

/* ---- ordering (proj/src/pipeline.cpp:91-129 tree schemes; pca.cpp, tree.cpp) ----
 * d = 2 or 3 (tree2 / tree3).  pca_device >= 0 runs the covariance action of
 * the subspace iteration on that CUDA device with the reference's exact
 * summation order (bit-identical result); -1 keeps it on the host. */
int knnx_order_tree(const double* pts, int32_t n, int32_t dim, int32_t d, int32_t leaf_capacity,
                    int32_t max_depth, int32_t pca_device, knnx_tree_t* out,
                    double* captured_ratio, int32_t* pca_iterations);
/* the same tree built on CUDA device `device` (two radix sorts over the
 * points' orthant paths instead of the recursion, csrc/tree_device.cu);
 * equal to knnx_tree_build field for field.  max_depth <= 21. */
int knnx_tree_build_dev(const double* emb, int32_t n, int32_t dim, int32_t leaf_capacity,
                        int32_t max_depth, int32_t device, knnx_tree_t* out);
int knnx_tree_build(const double* emb, int32_t n, int32_t dim, int32_t leaf_capacity,
                    int32_t max_depth, knnx_tree_t* out);
int knnx_tree_info(knnx_tree_t t, int32_t* n_nodes, int32_t* depth, int32_t* n_points);
int knnx_tree_forward(knnx_tree_t t, int32_t* forward);
int knnx_tree_nodes(knnx_tree_t t, int32_t* begin, int32_t* end, int32_t* depth, int32_t* parent,
                    int32_t* is_leaf);
int knnx_tree_level_blocking(knnx_tree_t t, int32_t level, int32_t* offsets, int32_t* count);
void knnx_tree_destroy(knnx_tree_t t);

/* PCA by blocked subspace iteration (proj/src/pca.cpp:133-264) + project */
int knnx_fit_pca(const double* pts, int32_t n, int32_t dim, int32_t d, int32_t pca_device,
                 double* mean, double* axes, double* singular_values, int32_t* iterations,
                 int32_t* converged, double* projected);

#ifdef __cplusplus
}
#endif
#endif /* KNNX_HOST_H */
