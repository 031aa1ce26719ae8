/* oracle/knn_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 * See knn_oracle.h for scope and pinning.  Compiled with -ffp-contract=off so
 * every multiply and add rounds separately, as the reference's canonical
 * x86-64 build (no -march, hence no FMA) does.
 */
#include "knn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* mt19937_64: the published Matsumoto-Nishimura 64-bit Mersenne twister,
 * as std::mt19937_64 specifies it (used by Rng, core.hpp:124-149). */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

static void mt_twist(orc_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->mti = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->mti >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* core.hpp:131 */
double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* core.hpp:134 */
uint64_t orc_rng_bounded(orc_rng* r, uint64_t n) { return orc_rng_next(r) % n; }

/* Box-Muller with a cached spare (core.cpp:186-199) */
double orc_rng_normal(orc_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double pi = 3.14159265358979323846; /* == std::numbers::pi as a double */
  double u1 = ((double)(orc_rng_next(r) >> 11) + 0.5) * 0x1.0p-53;
  double u2 = ((double)(orc_rng_next(r) >> 11) + 0.5) * 0x1.0p-53;
  double rad = sqrt(-2.0 * log(u1));
  double a = 2.0 * pi * u2;
  r->spare = rad * sin(a);
  r->has_spare = 1;
  return rad * cos(a);
}

void orc_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_next(&r);
}
void orc_rng_uniform01_stream(uint64_t seed, int64_t n, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform01(&r);
}
void orc_rng_normal_stream(uint64_t seed, int64_t n, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_normal(&r);
}

/* order_scattered: Fisher-Yates over the identity (orderings.cpp:9-16, core.hpp:140-143) */
void orc_order_scattered(int32_t n, uint64_t seed, int32_t* forward) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int32_t i = 0; i < n; ++i) forward[i] = i;
  for (int64_t i = n; i > 1; --i) {
    uint64_t j = orc_rng_bounded(&r, (uint64_t)i);
    int32_t tmp = forward[i - 1];
    forward[i - 1] = forward[j];
    forward[j] = tmp;
  }
}

/* ---------------------------------------------------------------------- */
/* operators */

/* kernels.cpp:37-49: y_i += v_e * x_j over the canonical entry list */
int orc_spmv_csr(int32_t m, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                 const double* x, double* y) {
  for (int32_t i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) acc += vals[e] * x[cols[e]];
    y[i] = acc;
  }
  return ORC_OK;
}

static double sq_dist(const double* a, const double* b, int32_t dim) {
  double acc = 0.0;
  for (int32_t d = 0; d < dim; ++d) {
    const double diff = a[d] - b[d];
    acc += diff * diff;
  }
  return acc;
}

/* knn.cpp:86-108 */
int orc_gaussian_values(int32_t m, const int64_t* row_ptr, const int32_t* cols, const double* t,
                        const double* s, int32_t dim, double h, double* vals) {
  if (!(h > 0.0)) return ORC_NON_POSITIVE_BANDWIDTH;
  const double inv = 1.0 / (2.0 * h * h);
  for (int32_t i = 0; i < m; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const double d2 = sq_dist(t + (int64_t)i * dim, s + (int64_t)cols[e] * dim, dim);
      vals[e] = exp(-d2 * inv);
    }
  return ORC_OK;
}

/* iterate_interactions step with the Gaussian value_fn (kernels.cpp:217-228,
 * hier.cpp:203-222 traversal; per-row order == canonical column order) */
int orc_gauss_spmv(int32_t m, const int64_t* row_ptr, const int32_t* cols, const double* t,
                   const double* s, int32_t dim, double h, const double* x, double* y) {
  if (!(h > 0.0)) return ORC_NON_POSITIVE_BANDWIDTH;
  const double inv = 1.0 / (2.0 * h * h);
  for (int32_t i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const double d2 = sq_dist(t + (int64_t)i * dim, s + (int64_t)cols[e] * dim, dim);
      const double v = exp(-d2 * inv);
      if (!isfinite(v)) return ORC_NON_FINITE_VALUE;
      acc += v * x[cols[e]];
    }
    y[i] = acc;
  }
  return ORC_OK;
}

/* kernels.cpp:184-208 */
int orc_meanshift_step(int32_t m, int32_t k, const int32_t* ids, const double* t,
                       const double* s, int32_t dim, double h, double* t_out,
                       int32_t* bad_target) {
  if (!(h > 0.0)) return ORC_NON_POSITIVE_BANDWIDTH;
  const double inv_2h2 = 1.0 / (2.0 * h * h);
  double* mean = (double*)malloc(sizeof(double) * (size_t)(dim > 0 ? dim : 1));
  for (int32_t i = 0; i < m; ++i) {
    const double* yi = t + (int64_t)i * dim;
    double total = 0.0;
    for (int32_t c = 0; c < dim; ++c) mean[c] = 0.0;
    for (int32_t q = 0; q < k; ++q) {
      const double* sj = s + (int64_t)ids[(int64_t)i * k + q] * dim;
      const double w = exp(-sq_dist(yi, sj, dim) * inv_2h2);
      total += w;
      for (int32_t c = 0; c < dim; ++c) mean[c] += w * sj[c];
    }
    if (total == 0.0) {
      if (bad_target) *bad_target = i;
      free(mean);
      return ORC_ZERO_WEIGHT;
    }
    for (int32_t c = 0; c < dim; ++c) t_out[(int64_t)i * dim + c] = mean[c] / total;
  }
  free(mean);
  return ORC_OK;
}

/* kernels.cpp:103-136 */
int orc_tsne_attractive(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* p,
                        const double* y, int32_t dim, double* a_out, double* f) {
  const int64_t nnz = row_ptr[n];
  for (int32_t i = 0; i < n; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
      a_out[e] = p[e] / (1.0 + sq_dist(y + (int64_t)i * dim, y + (int64_t)cols[e] * dim, dim));
  (void)nnz;
  double* r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int32_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) acc += a_out[e] * 1.0;
    r[i] = acc;
  }
  for (int32_t c = 0; c < dim; ++c)
    for (int32_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        acc += a_out[e] * y[(int64_t)cols[e] * dim + c];
      f[(int64_t)i * dim + c] = r[i] * y[(int64_t)i * dim + c] - acc;
    }
  free(r);
  return ORC_OK;
}

/* proj/tests/acceptance.cpp:458-470 (tsne_oracle) */
int orc_tsne_direct(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* p,
                    const double* y, int32_t dim, double* f) {
  for (int64_t q = 0; q < (int64_t)n * dim; ++q) f[q] = 0.0;
  for (int32_t i = 0; i < n; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const double* yi = y + (int64_t)i * dim;
      const double* yj = y + (int64_t)cols[e] * dim;
      const double a = p[e] / (1.0 + sq_dist(yi, yj, dim));
      for (int32_t c = 0; c < dim; ++c) f[(int64_t)i * dim + c] += a * (yi[c] - yj[c]);
    }
  return ORC_OK;
}

/* core.cpp:141-148 */
void orc_permute_rows(int32_t n, int64_t width_bytes, const void* in, const int32_t* forward,
                      void* out) {
  const char* src = (const char*)in;
  char* dst = (char*)out;
  for (int32_t i = 0; i < n; ++i)
    memcpy(dst + (int64_t)forward[i] * width_bytes, src + (int64_t)i * width_bytes,
           (size_t)width_bytes);
}

/* ---------------------------------------------------------------------- */
/* knn.cpp:9-62: exact kNN; candidates ordered by (squared distance, index) */
typedef struct {
  double d;
  int32_t j;
} cand_t;

static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->d < y->d) return -1;
  if (x->d > y->d) return 1;
  return (x->j > y->j) - (x->j < y->j);
}

int orc_build_knn(const double* t, int32_t m, const double* s, int32_t n, int32_t dim, int32_t k,
                  int self_set, int32_t* ids, double* dists) {
  if (k < 1) return ORC_INVALID_ARGUMENT;
  if (k > (self_set ? n - 1 : n)) return ORC_K_TOO_LARGE;
  if (self_set) s = t;
  cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)n);
  for (int32_t i = 0; i < m; ++i) {
    for (int32_t j = 0; j < n; ++j) {
      c[j].d = sq_dist(t + (int64_t)i * dim, s + (int64_t)j * dim, dim);
      c[j].j = j;
    }
    if (self_set) c[i].d = INFINITY;
    qsort(c, (size_t)n, sizeof(cand_t), cand_cmp);
    for (int32_t a = 0; a < k; ++a) {
      ids[(int64_t)i * k + a] = c[a].j;
      dists[(int64_t)i * k + a] = c[a].d;
    }
  }
  free(c);
  return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* tree.cpp:15-112 */
typedef struct {
  double lo[3], hi[3];
} box_t;

typedef struct {
  const double* pts;
  int32_t dim, leaf_capacity, max_depth, max_nodes, n_nodes;
  int32_t *order, *scratch;
  int32_t *begin, *end, *depth, *parent, *is_leaf;
  box_t* box;
  int overflow;
} tree_ctx;

static int32_t orthant(const tree_ctx* tc, int32_t original, const double* center) {
  const double* x = tc->pts + (int64_t)original * tc->dim;
  int32_t code = 0;
  for (int32_t a = 0; a < tc->dim; ++a)
    if (x[a] >= center[a]) code |= 1 << a;
  return code;
}

static void split(tree_ctx* tc, int32_t id, int32_t lo, int32_t hi, int32_t depth) {
  tc->begin[id] = lo;
  tc->end[id] = hi;
  tc->depth[id] = depth;
  tc->is_leaf[id] = 0;
  if (hi - lo <= tc->leaf_capacity || depth >= tc->max_depth) {
    tc->is_leaf[id] = 1;
    return;
  }
  const int32_t n_orth = 1 << tc->dim;
  double center[3];
  for (int32_t a = 0; a < tc->dim; ++a) center[a] = 0.5 * (tc->box[id].lo[a] + tc->box[id].hi[a]);
  int32_t start[9] = {0};
  for (int32_t i = lo; i < hi; ++i) ++start[orthant(tc, tc->order[i], center) + 1];
  for (int32_t c = 0; c < n_orth; ++c) start[c + 1] += start[c];
  int32_t fill[9];
  memcpy(fill, start, sizeof fill);
  for (int32_t i = lo; i < hi; ++i) {
    const int32_t o = tc->order[i];
    tc->scratch[lo + fill[orthant(tc, o, center)]++] = o;
  }
  memcpy(tc->order + lo, tc->scratch + lo, sizeof(int32_t) * (size_t)(hi - lo));
  for (int32_t code = 0; code < n_orth; ++code) {
    const int32_t c_lo = lo + start[code], c_hi = lo + start[code + 1];
    if (c_lo == c_hi) continue;
    if (tc->n_nodes >= tc->max_nodes) {
      tc->overflow = 1;
      return;
    }
    const int32_t child = tc->n_nodes++;
    tc->parent[child] = id;
    for (int32_t a = 0; a < tc->dim; ++a) {
      const int high = (code >> a) & 1;
      tc->box[child].lo[a] = high ? center[a] : tc->box[id].lo[a];
      tc->box[child].hi[a] = high ? tc->box[id].hi[a] : center[a];
    }
    split(tc, child, c_lo, c_hi, depth + 1);
    if (tc->overflow) return;
  }
}

int orc_build_tree(const double* pts, int32_t n, int32_t dim, int32_t leaf_capacity,
                   int32_t max_depth, int32_t* forward, int32_t max_nodes, int32_t* n_nodes,
                   int32_t* begin, int32_t* end, int32_t* depth, int32_t* parent,
                   int32_t* is_leaf) {
  if (dim < 1 || dim > 3) return ORC_DIM_TOO_HIGH;
  if (leaf_capacity < 1 || max_depth < 1 || max_nodes < 1) return ORC_INVALID_ARGUMENT;
  tree_ctx tc;
  memset(&tc, 0, sizeof tc);
  tc.pts = pts;
  tc.dim = dim;
  tc.leaf_capacity = leaf_capacity;
  tc.max_depth = max_depth;
  tc.max_nodes = max_nodes;
  tc.begin = begin;
  tc.end = end;
  tc.depth = depth;
  tc.parent = parent;
  tc.is_leaf = is_leaf;
  tc.box = (box_t*)calloc((size_t)max_nodes, sizeof(box_t));
  tc.order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  tc.scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int32_t a = 0; a < dim; ++a) lo[a] = hi[a] = n > 0 ? pts[a] : 0.0;
  for (int32_t i = 1; i < n; ++i)
    for (int32_t a = 0; a < dim; ++a) {
      const double x = pts[(int64_t)i * dim + a];
      if (x < lo[a]) lo[a] = x; /* std::min(lo, x) keeps lo unless x < lo */
      if (hi[a] < x) hi[a] = x; /* std::max(hi, x) keeps hi unless hi < x */
    }
  double side = 0.0;
  for (int32_t a = 0; a < dim; ++a)
    if (side < hi[a] - lo[a]) side = hi[a] - lo[a];
  for (int32_t a = 0; a < dim; ++a) {
    const double center = 0.5 * (lo[a] + hi[a]);
    tc.box[0].lo[a] = center - 0.5 * side;
    tc.box[0].hi[a] = center + 0.5 * side;
  }
  for (int32_t i = 0; i < n; ++i) tc.order[i] = i;
  tc.n_nodes = 1;
  parent[0] = -1;
  split(&tc, 0, 0, n, 0);
  int rc = ORC_OK;
  if (tc.overflow) {
    rc = ORC_INVALID_ARGUMENT;
  } else {
    for (int32_t pos = 0; pos < n; ++pos) forward[tc.order[pos]] = pos;
    *n_nodes = tc.n_nodes;
  }
  free(tc.box);
  free(tc.order);
  free(tc.scratch);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* BASELINE.json workload generators.  The reference has no
 * generator for these mixtures (its synth.cpp emits one Gaussian mixture per
 * call); these restate the configs' text with the reference Rng so the
 * reference arm of bench.py can build its inputs without the product
 * library.  Pinned bitwise against knnx_gen_points (tests/test_oracle.py). */

/* C1 / C4: n_clusters centres ~ U[-10,10]^dim (-10 + 20 U), point p in
 * component p mod n_clusters, coordinates centre + sigma N(0,1), rounded to
 * fp32 (the emission order of proj/src/synth.cpp:69, round robin) */
int orc_gen_mixture_c1(int32_t n, int32_t dim, int32_t n_clusters, double sigma, uint64_t seed,
                       float* out) {
  if (n <= 0 || dim <= 0 || n_clusters <= 0 || !(sigma > 0.0)) return ORC_INVALID_ARGUMENT;
  orc_rng r;
  orc_rng_seed(&r, seed);
  double* c = (double*)malloc(sizeof(double) * (size_t)n_clusters * dim);
  if (!c) return ORC_INVALID_ARGUMENT;
  for (int64_t i = 0; i < (int64_t)n_clusters * dim; ++i) c[i] = -10.0 + 20.0 * orc_rng_uniform01(&r);
  for (int64_t p = 0; p < n; ++p) {
    const double* cp = c + (size_t)(p % n_clusters) * dim;
    for (int32_t a = 0; a < dim; ++a) out[p * dim + a] = (float)(cp[a] + sigma * orc_rng_normal(&r));
  }
  free(c);
  return ORC_OK;
}

/* C2 / C3: 3-level mixture, 16 x 16 x 16: level-1 centres 10 N(0,1),
 * level-2 = parent + 2 N(0,1), leaves = parent + 0.5 N(0,1); each point picks
 * a leaf with bounded(4096) and adds noise N(0,1) */
int orc_gen_mixture_3level(int32_t n, int32_t dim, double noise, uint64_t seed, float* out) {
  if (n <= 0 || dim <= 0 || !(noise > 0.0)) return ORC_INVALID_ARGUMENT;
  const int fan = 16;
  orc_rng r;
  orc_rng_seed(&r, seed);
  double* l1 = (double*)malloc(sizeof(double) * fan * dim);
  double* l2 = (double*)malloc(sizeof(double) * fan * fan * dim);
  double* l3 = (double*)malloc(sizeof(double) * fan * fan * fan * dim);
  if (!l1 || !l2 || !l3) {
    free(l1); free(l2); free(l3);
    return ORC_INVALID_ARGUMENT;
  }
  for (int i = 0; i < fan * dim; ++i) l1[i] = 10.0 * orc_rng_normal(&r);
  for (int s = 0; s < fan * fan; ++s)
    for (int a = 0; a < dim; ++a) l2[s * dim + a] = l1[(s / fan) * dim + a] + 2.0 * orc_rng_normal(&r);
  for (int s = 0; s < fan * fan * fan; ++s)
    for (int a = 0; a < dim; ++a) l3[s * dim + a] = l2[(s / fan) * dim + a] + 0.5 * orc_rng_normal(&r);
  for (int64_t p = 0; p < n; ++p) {
    const int leaf = (int)orc_rng_bounded(&r, (uint64_t)(fan * fan * fan));
    const double* cp = l3 + (size_t)leaf * dim;
    for (int32_t a = 0; a < dim; ++a) out[p * dim + a] = (float)(cp[a] + noise * orc_rng_normal(&r));
  }
  free(l1); free(l2); free(l3);
  return ORC_OK;
}

/* charges x ~ U[0,1) rounded to fp32 */
void orc_gen_uniform01_f32(int64_t n, uint64_t seed, float* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = (float)orc_rng_uniform01(&r);
}

/* C5: 2-level anisotropic mixture (n_top x n_sub clusters): per top cluster a
 * centre 3 N(0,1), per-axis standard deviations sqrt(10^(-2 + 2U)) and three
 * unit Householder vectors; sub-centres = top + N(0,1); point p of block
 * b = p / 8192 draws from its own stream Rng(seed ^ 0x9E3779B97F4A7C15 (b+1)):
 * sub-cluster bounded(n_top n_sub), z = sd * N(0,1) reflected by the three
 * Householder vectors, x = sub-centre + z */
int orc_gen_mixture_aniso(int32_t n, int32_t dim, int32_t n_top, int32_t n_sub, uint64_t seed,
                          float* out) {
  if (n <= 0 || dim <= 0 || n_top <= 0 || n_sub <= 0) return ORC_INVALID_ARGUMENT;
  enum { kRefl = 3, kBlock = 8192 };
  orc_rng r;
  orc_rng_seed(&r, seed);
  const size_t td = (size_t)n_top * dim;
  double* top = (double*)malloc(sizeof(double) * td);
  double* sd = (double*)malloc(sizeof(double) * td);
  double* house = (double*)malloc(sizeof(double) * td * kRefl);
  double* sub = (double*)malloc(sizeof(double) * td * n_sub);
  double* z = (double*)malloc(sizeof(double) * dim);
  if (!top || !sd || !house || !sub || !z) {
    free(top); free(sd); free(house); free(sub); free(z);
    return ORC_INVALID_ARGUMENT;
  }
  for (size_t i = 0; i < td; ++i) top[i] = 3.0 * orc_rng_normal(&r);
  for (size_t i = 0; i < td; ++i) sd[i] = sqrt(pow(10.0, -2.0 + 2.0 * orc_rng_uniform01(&r)));
  for (int64_t t = 0; t < (int64_t)n_top * kRefl; ++t) {
    double* h = house + (size_t)t * dim;
    double nrm = 0.0;
    for (int32_t a = 0; a < dim; ++a) {
      h[a] = orc_rng_normal(&r);
      nrm += h[a] * h[a];
    }
    nrm = sqrt(nrm);
    for (int32_t a = 0; a < dim; ++a) h[a] /= nrm;
  }
  for (int64_t s = 0; s < (int64_t)n_top * n_sub; ++s)
    for (int32_t a = 0; a < dim; ++a)
      sub[(size_t)s * dim + a] = top[(size_t)(s / n_sub) * dim + a] + 1.0 * orc_rng_normal(&r);
  for (int64_t b = 0; b * kBlock < n; ++b) {
    orc_rng pr;
    orc_rng_seed(&pr, seed ^ (0x9E3779B97F4A7C15ULL * (uint64_t)(b + 1)));
    const int64_t hi = (b + 1) * kBlock < n ? (b + 1) * kBlock : n;
    for (int64_t p = b * kBlock; p < hi; ++p) {
      const int64_t s = (int64_t)orc_rng_bounded(&pr, (uint64_t)n_top * (uint64_t)n_sub);
      const int64_t t = s / n_sub;
      for (int32_t a = 0; a < dim; ++a) z[a] = sd[(size_t)t * dim + a] * orc_rng_normal(&pr);
      for (int q = 0; q < kRefl; ++q) {
        const double* h = house + ((size_t)t * kRefl + q) * dim;
        double dot = 0.0;
        for (int32_t a = 0; a < dim; ++a) dot += h[a] * z[a];
        for (int32_t a = 0; a < dim; ++a) z[a] -= 2.0 * dot * h[a];
      }
      for (int32_t a = 0; a < dim; ++a)
        out[p * dim + a] = (float)(sub[(size_t)s * dim + a] + z[a]);
    }
  }
  free(top); free(sd); free(house); free(sub); free(z);
  return ORC_OK;
}
