/*
 * warmgp_oracle.c -- CPU restatement of the reference algorithm for the
 * warm-started kernel-matvec solve path.  TEST INFRASTRUCTURE ONLY (see
 * warmgp_oracle.h): the parity checker and the CPU baseline, never the product.
 *
 * Every function cites the reference file:line (relative to
 * /root/reference/proj/core) it restates.  Arithmetic is fp64 throughout like
 * the reference; loop orders follow the reference's expressions where they
 * affect results beyond rounding (pivot ties, RNG consumption order,
 * iteration/history semantics).  Dense products do not replicate Eigen's
 * blocked summation order, so agreement with the reference is to rounding
 * (~1e-15 relative), which is what the reference's own tests pin.
 */
#define _GNU_SOURCE
#include "warmgp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* wgo_last_error(void) { return g_err; }

static const double kSqrt3 = 1.7320508075688772935;   /* kernel.cpp:9 */
static const double kTwoPi = 6.283185307179586476925287; /* sampling.cpp:10 */

/* ======================= rng.hpp ======================= */

uint64_t wgo_derive_seed(uint64_t seed, uint64_t stream) { /* rng.hpp:11-16 */
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t wgo_rng_next_u64(wgo_rng* r) { /* rng.hpp:25-30 */
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double wgo_rng_uniform(wgo_rng* r) { /* rng.hpp:33: 53-bit uniform in [0,1) */
  return (double)(wgo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

double wgo_rng_uniform_range(wgo_rng* r, double lo, double hi) { /* rng.hpp:35 */
  return lo + (hi - lo) * wgo_rng_uniform(r);
}

double wgo_rng_normal(wgo_rng* r) { /* rng.hpp:38-43: Box-Muller, cos branch, no cache */
  double u1 = wgo_rng_uniform(r);
  while (u1 <= 0.0) u1 = wgo_rng_uniform(r);
  const double u2 = wgo_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}

double wgo_rng_chi_square3(wgo_rng* r) { /* rng.hpp:46-49 (evaluation order a, b, c) */
  const double a = wgo_rng_normal(r);
  const double b = wgo_rng_normal(r);
  const double c = wgo_rng_normal(r);
  return a * a + b * b + c * c;
}

uint64_t wgo_rng_uniform_index(wgo_rng* r, uint64_t n) { /* rng.hpp:52-54 */
  return (uint64_t)(((unsigned __int128)wgo_rng_next_u64(r) * n) >> 64);
}

void wgo_uniform_inputs(uint64_t seed, int64_t n, int64_t dim, double* X) { /* testutil.hpp:9-16 */
  wgo_rng r = {seed};
  for (int64_t i = 0; i < n; ++i)
    for (int64_t d = 0; d < dim; ++d) X[d * n + i] = wgo_rng_uniform(&r);
}

void wgo_gaussian_vector(uint64_t seed, int64_t n, double* v) { /* testutil.hpp:18-23 */
  wgo_rng r = {seed};
  for (int64_t i = 0; i < n; ++i) v[i] = wgo_rng_normal(&r);
}

/* ======================= kernel.cpp ======================= */

int wgo_hyp_validate(const wgo_hyp* h) { /* kernel.cpp:11-15 */
  if (!(h->lengthscale > 0.0) || !(h->signal_scale > 0.0) || !(h->noise_scale > 0.0))
    return fail(WGO_INVALID_ARGUMENT, "kernel hyperparameters must be strictly positive");
  if (h->kind != WGO_MATERN32 && h->kind != WGO_RBF)
    return fail(WGO_INVALID_ARGUMENT, "unknown kernel kind %d", h->kind);
  return WGO_OK;
}

double wgo_kernel_from_distance(const wgo_hyp* h, double r) {
  if (r < 0.0) r = 0.0;
  const double s2 = h->signal_scale * h->signal_scale;
  if (h->kind == WGO_RBF) { /* extension: s^2 exp(-r^2 / (2 l^2)) */
    const double u = r / h->lengthscale;
    return s2 * exp(-0.5 * u * u);
  }
  const double z = kSqrt3 * r / h->lengthscale; /* kernel.cpp:17-21 */
  return s2 * (1.0 + z) * exp(-z);
}

int wgo_pairwise_distances(const double* A, int64_t m, const double* B, int64_t n, int64_t d,
                           double* D) { /* kernel.cpp:39-46 */
  double* a2 = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  double* b2 = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t k = 0; k < d; ++k) {
    for (int64_t i = 0; i < m; ++i) a2[i] += A[k * m + i] * A[k * m + i];
    for (int64_t j = 0; j < n; ++j) b2[j] += B[k * n + j] * B[k * n + j];
  }
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) {
      double g = 0.0;
      for (int64_t k = 0; k < d; ++k) g += A[k * m + i] * B[k * n + j];
      double d2 = -2.0 * g;
      d2 += a2[i];            /* d2.colwise() += a2 */
      d2 += b2[j];            /* d2.rowwise() += b2^T */
      D[j * m + i] = sqrt(d2 > 0.0 ? d2 : 0.0);
    }
  }
  free(a2);
  free(b2);
  return WGO_OK;
}

/* Squared-norm gram g = X X^T (lower, mirrored) as in kernel.cpp:54-56, then the map of
 * kernel.cpp:58-70.  Shared by the dense gram and the matrix-free operator so both give
 * the same entries. */
static inline double gram_entry(const wgo_hyp* h, double sqi, double sqj, double gij) {
  const double d2 = sqi + sqj - 2.0 * gij;                          /* kernel.cpp:65 */
  return wgo_kernel_from_distance(h, sqrt(d2 > 0.0 ? d2 : 0.0));   /* kernel.cpp:66-67 */
}

int wgo_gram_matrix(const wgo_hyp* h, const double* X, int64_t n, int64_t d, double* H) {
  int st = wgo_hyp_validate(h);
  if (st) return st;
  if (n < 1) return fail(WGO_INVALID_ARGUMENT, "gram_matrix: need at least one row");
  double* sq = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t k = 0; k < d; ++k) s += X[k * n + i] * X[k * n + i];
    sq[i] = s;
  }
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = j; i < n; ++i) {
      double g = 0.0;
      for (int64_t k = 0; k < d; ++k) g += X[k * n + i] * X[k * n + j];
      const double v = gram_entry(h, sq[i], sq[j], g);
      H[j * n + i] = v;
      H[i * n + j] = v; /* exactly symmetric, kernel.cpp:56 */
    }
  }
  const double diag = h->signal_scale * h->signal_scale + h->noise_scale * h->noise_scale;
  for (int64_t i = 0; i < n; ++i) H[i * n + i] = diag; /* kernel.cpp:70 */
  free(sq);
  return WGO_OK;
}

int wgo_cross_kernel(const wgo_hyp* h, const double* Xs, int64_t m, const double* X, int64_t n,
                     int64_t d, double* K) { /* kernel.cpp:74-89 */
  int st = wgo_hyp_validate(h);
  if (st) return st;
  wgo_pairwise_distances(Xs, m, X, n, d, K);
  for (int64_t t = 0; t < m * n; ++t) K[t] = wgo_kernel_from_distance(h, K[t]);
  return WGO_OK;
}

int wgo_extend_assembled(const wgo_hyp* h, const double* H11, const double* X1, int64_t n1,
                         const double* X2, int64_t n2, int64_t d, double* H) {
  /* extend_system kernel.cpp:108-130 followed by BlockedSystem::assembled :91-100 */
  int st = wgo_hyp_validate(h);
  if (st) return st;
  const int64_t n = n1 + n2;
  for (int64_t j = 0; j < n1; ++j) memcpy(H + j * n, H11 + j * n1, sizeof(double) * (size_t)n1);
  if (n2 == 0) return WGO_OK;
  double* H12 = (double*)malloc(sizeof(double) * (size_t)(n1 * n2 + 1));
  double* H22 = (double*)malloc(sizeof(double) * (size_t)(n2 * n2));
  wgo_cross_kernel(h, X1, n1, X2, n2, d, H12);
  wgo_gram_matrix(h, X2, n2, d, H22);
  for (int64_t j = 0; j < n2; ++j)
    for (int64_t i = 0; i < n1; ++i) {
      H[(n1 + j) * n + i] = H12[j * n1 + i];
      H[i * n + (n1 + j)] = H12[j * n1 + i];
    }
  for (int64_t j = 0; j < n2; ++j)
    for (int64_t i = 0; i < n2; ++i) H[(n1 + j) * n + n1 + i] = H22[j * n2 + i];
  free(H12);
  free(H22);
  return WGO_OK;
}

/* Matrix-free K V over a row range.  X is transposed to row-major once and the RHS to
 * row-major so the inner loops are contiguous (OpenMP over row blocks). */
int wgo_kmatvec_rows(const wgo_hyp* h, const double* X, int64_t n, int64_t d, const double* V,
                     int64_t s, int64_t r0, int64_t r1, double* Y, int nthreads) {
  int st = wgo_hyp_validate(h);
  if (st) return st;
  if (r0 < 0 || r1 > n || r0 > r1) return fail(WGO_INVALID_ARGUMENT, "kmatvec_rows: bad range");
  const int64_t nr = r1 - r0;
  double* Xr = (double*)malloc(sizeof(double) * (size_t)(n * d));
  double* Vr = (double*)malloc(sizeof(double) * (size_t)(n * s));
  double* sq = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    double a = 0.0;
    for (int64_t k = 0; k < d; ++k) {
      Xr[i * d + k] = X[k * n + i];
      a += X[k * n + i] * X[k * n + i];
    }
    sq[i] = a;
    for (int64_t c = 0; c < s; ++c) Vr[i * s + c] = V[c * n + i];
  }
  const double diag_noise = h->noise_scale * h->noise_scale;
  const double s2 = h->signal_scale * h->signal_scale;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * (size_t)(s > 0 ? s : 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t i = r0; i < r1; ++i) {
      for (int64_t c = 0; c < s; ++c) acc[c] = 0.0;
      const double* xi = Xr + i * d;
      for (int64_t j = 0; j < n; ++j) {
        double kij;
        if (j == i) {
          kij = s2 + diag_noise; /* diagonal set exactly, kernel.cpp:70 */
        } else {
          const double* xj = Xr + j * d;
          double g = 0.0;
          for (int64_t k = 0; k < d; ++k) g += xi[k] * xj[k];
          kij = gram_entry(h, sq[i], sq[j], g);
        }
        const double* vj = Vr + j * s;
        for (int64_t c = 0; c < s; ++c) acc[c] += kij * vj[c];
      }
      for (int64_t c = 0; c < s; ++c) Y[c * nr + (i - r0)] = acc[c];
    }
    free(acc);
  }
  free(Xr);
  free(Vr);
  free(sq);
  return WGO_OK;
}

int wgo_cross_matvec(const wgo_hyp* h, const double* Xs, int64_t m, const double* X, int64_t n,
                     int64_t d, const double* W, int64_t s, double* Y, int nthreads) {
  int st = wgo_hyp_validate(h);
  if (st) return st;
  double* a2 = (double*)calloc((size_t)(m + 1), sizeof(double));
  double* b2 = (double*)calloc((size_t)(n + 1), sizeof(double));
  for (int64_t k = 0; k < d; ++k) {
    for (int64_t i = 0; i < m; ++i) a2[i] += Xs[k * m + i] * Xs[k * m + i];
    for (int64_t j = 0; j < n; ++j) b2[j] += X[k * n + j] * X[k * n + j];
  }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t c = 0; c < s; ++c) Y[c * m + i] = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double g = 0.0;
      for (int64_t k = 0; k < d; ++k) g += Xs[k * m + i] * X[k * n + j];
      double d2 = -2.0 * g;
      d2 += a2[i];
      d2 += b2[j];
      const double kij = wgo_kernel_from_distance(h, sqrt(d2 > 0.0 ? d2 : 0.0));
      for (int64_t c = 0; c < s; ++c) Y[c * m + i] += kij * W[c * n + j];
    }
  }
  free(a2);
  free(b2);
  return WGO_OK;
}

/* ======================= operators ======================= */

static void dense_matvec(const wgo_op* op, const double* v, double* y) {
  const double* H = (const double*)op->ctx;
  const int64_t n = op->n;
  for (int64_t i = 0; i < n; ++i) y[i] = 0.0;
  for (int64_t j = 0; j < n; ++j) { /* column-major GEMV */
    const double vj = v[j];
    const double* col = H + j * n;
    for (int64_t i = 0; i < n; ++i) y[i] += col[i] * vj;
  }
}

static void dense_block(const wgo_op* op, int64_t r0, int64_t nr, int64_t c0, int64_t nc,
                        double* out) {
  const double* H = (const double*)op->ctx;
  for (int64_t j = 0; j < nc; ++j)
    memcpy(out + j * nr, H + (c0 + j) * op->n + r0, sizeof(double) * (size_t)nr);
}

void wgo_op_dense(wgo_op* op, const double* H, int64_t n) {
  op->n = n;
  op->ctx = H;
  op->matvec = dense_matvec;
  op->block = dense_block;
}

static double mf_entry(const wgo_mf_ctx* c, int64_t i, int64_t j) {
  if (i == j)
    return c->hyp.signal_scale * c->hyp.signal_scale + c->hyp.noise_scale * c->hyp.noise_scale;
  double g = 0.0;
  for (int64_t k = 0; k < c->d; ++k) g += c->X[k * c->n + i] * c->X[k * c->n + j];
  return gram_entry(&c->hyp, c->sq[i], c->sq[j], g);
}

static void mf_matvec(const wgo_op* op, const double* v, double* y) {
  const wgo_mf_ctx* c = (const wgo_mf_ctx*)op->ctx;
  wgo_kmatvec_rows(&c->hyp, c->X, c->n, c->d, v, 1, 0, c->n, y, c->nthreads);
}

static void mf_block(const wgo_op* op, int64_t r0, int64_t nr, int64_t c0, int64_t nc,
                     double* out) {
  const wgo_mf_ctx* c = (const wgo_mf_ctx*)op->ctx;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < nc; ++j)
    for (int64_t i = 0; i < nr; ++i) out[j * nr + i] = mf_entry(c, r0 + i, c0 + j);
}

int wgo_op_matrix_free(wgo_op* op, wgo_mf_ctx* c) {
  int st = wgo_hyp_validate(&c->hyp);
  if (st) return st;
  c->sq = (double*)malloc(sizeof(double) * (size_t)(c->n > 0 ? c->n : 1));
  for (int64_t i = 0; i < c->n; ++i) {
    double a = 0.0;
    for (int64_t k = 0; k < c->d; ++k) a += c->X[k * c->n + i] * c->X[k * c->n + i];
    c->sq[i] = a;
  }
  op->n = c->n;
  op->ctx = c;
  op->matvec = mf_matvec;
  op->block = mf_block;
  return WGO_OK;
}

void wgo_mf_free(wgo_mf_ctx* c) {
  free(c->sq);
  c->sq = NULL;
}

static double op_diag(const wgo_op* op, int64_t i) {
  double v;
  op->block(op, i, 1, i, 1, &v);
  return v;
}

/* ======================= small dense helpers ======================= */

static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

static double nrm2(const double* a, int64_t n) { return sqrt(dot(a, a, n)); }

/* In-place lower Cholesky (Eigen::LLT semantics: fails when a pivot is not > 0). */
static int cholesky_lower(double* A, int64_t n) {
  for (int64_t j = 0; j < n; ++j) {
    double x = A[j * n + j];
    for (int64_t k = 0; k < j; ++k) x -= A[k * n + j] * A[k * n + j];
    if (!(x > 0.0)) return WGO_NOT_SPD;
    const double ljj = sqrt(x);
    A[j * n + j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double y = A[j * n + i];
      for (int64_t k = 0; k < j; ++k) y -= A[k * n + i] * A[k * n + j];
      A[j * n + i] = y / ljj;
    }
  }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < j; ++i) A[j * n + i] = 0.0;
  return WGO_OK;
}

/* x <- (L L^T)^{-1} x */
static void cholesky_solve(const double* L, int64_t n, double* x) {
  for (int64_t i = 0; i < n; ++i) {
    double y = x[i];
    for (int64_t k = 0; k < i; ++k) y -= L[k * n + i] * x[k];
    x[i] = y / L[i * n + i];
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double y = x[i];
    for (int64_t k = i + 1; k < n; ++k) y -= L[i * n + k] * x[k];
    x[i] = y / L[i * n + i];
  }
}

/* ======================= solvers.cpp ======================= */

void wgo_solver_config_default(wgo_solver_config* c) { /* solvers.hpp:27-48 */
  c->method = WGO_CG;
  c->tolerance = 1e-2;
  c->max_iters = 1000;
  c->learning_rate = 0.3;
  c->momentum = 0.9;
  c->batch_size = 100;
  c->sgd_scaling = WGO_SGD_UNBIASED;
  c->block_size = 100;
  c->ap_ordering = WGO_AP_GREEDY;
  c->precond_rank = 100;
  c->precond_shift = 1e-6;
  c->precond_shift_mode = WGO_SHIFT_CALIBRATED;
  c->seed = 0;
}

int wgo_init_weights(int warm, const double* u1, int64_t u1_len, int64_t n1, int64_t n2,
                     double* v) { /* solvers.cpp:27-38 */
  if (n1 < 0 || n2 < 0) return fail(WGO_INVALID_ARGUMENT, "init_weights: negative block size");
  for (int64_t i = 0; i < n1 + n2; ++i) v[i] = 0.0;
  if (warm) {
    if (u1_len != n1)
      return fail(WGO_INVALID_ARGUMENT,
                  "init_weights: warm-start vector length does not match n1");
    memcpy(v, u1, sizeof(double) * (size_t)n1);
  }
  return WGO_OK;
}

/* expand_init, solvers.cpp:43-48 */
static int expand_init(int warm, const double* u1, int64_t n1, int64_t n, double* v) {
  if (!warm) {
    for (int64_t i = 0; i < n; ++i) v[i] = 0.0;
    return WGO_OK;
  }
  if (n1 > n) return fail(WGO_INVALID_ARGUMENT, "initialization longer than the system");
  return wgo_init_weights(1, u1, n1, n1, n - n1, v);
}

/* zero_rhs_result, solvers.cpp:51-58 */
static void zero_rhs_result(int64_t n, wgo_result* res) {
  for (int64_t i = 0; i < n; ++i) res->v[i] = 0.0;
  res->iterations = 0;
  res->history[0] = 0.0;
  res->history_len = 1;
  res->converged = 1;
}

int wgo_relative_residual(const wgo_op* op, const double* v, const double* b, double* out) {
  const int64_t n = op->n; /* solvers.cpp:62-66 */
  const double bnorm = nrm2(b, n);
  if (bnorm == 0.0) return fail(WGO_INVALID_ARGUMENT, "relative_residual: zero right-hand side");
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  op->matvec(op, v, t);
  for (int64_t i = 0; i < n; ++i) t[i] -= b[i];
  *out = nrm2(t, n) / bnorm;
  free(t);
  return WGO_OK;
}

double wgo_quadratic_objective(const wgo_op* op, const double* v, const double* b) {
  const int64_t n = op->n; /* solvers.cpp:68-70 */
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  op->matvec(op, v, t);
  const double q = 0.5 * dot(v, t, n) - dot(v, b, n);
  free(t);
  return q;
}

int wgo_pivoted_cholesky(const wgo_op* op, int64_t rank, double* L, int64_t* achieved_out) {
  const int64_t n = op->n; /* solvers.cpp:72-107 */
  if (rank < 0 || rank > n) return fail(WGO_INVALID_ARGUMENT, "pivoted_cholesky: rank out of range");
  double* d = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  unsigned char* used = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
  double* col = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double dmax = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    d[i] = op_diag(op, i);
    if (d[i] > dmax) dmax = d[i];
  }
  const double floor_ = 1e-12 * (dmax > 0.0 ? dmax : 0.0); /* :77 std::max(maxCoeff, 0) */
  memset(L, 0, sizeof(double) * (size_t)(n * rank));
  int64_t achieved = 0;
  for (int64_t k = 0; k < rank; ++k) {
    int64_t piv = -1;
    double best = floor_;
    for (int64_t i = 0; i < n; ++i) /* strict '>' : first index wins ties, :85-90 */
      if (!used[i] && d[i] > best) {
        best = d[i];
        piv = i;
      }
    if (piv < 0) break; /* :91 */
    const double root = sqrt(d[piv]);
    op->block(op, 0, n, piv, 1, col); /* H.col(piv) */
    if (k > 0) { /* col -= L(:, :k) L(piv, :k)^T, :95 */
      for (int64_t t = 0; t < k; ++t) {
        const double lp = L[t * n + piv];
        const double* Lt = L + t * n;
        for (int64_t i = 0; i < n; ++i) col[i] -= Lt[i] * lp;
      }
    }
    for (int64_t i = 0; i < n; ++i) L[k * n + i] = col[i] / root;
    L[k * n + piv] = root;
    used[piv] = 1;
    for (int64_t i = 0; i < n; ++i)
      if (!used[i]) d[i] -= L[k * n + i] * L[k * n + i];
    d[piv] = 0.0;
    achieved = k + 1;
  }
  *achieved_out = achieved;
  free(d);
  free(used);
  free(col);
  return WGO_OK;
}

int wgo_precond_init(wgo_precond* p, const double* L, int64_t n, int64_t k, double shift) {
  /* CgPreconditioner(L, shift), solvers.cpp:109-121 */
  memset(p, 0, sizeof *p);
  p->n = n;
  p->k = k;
  p->shift = shift;
  if (k == 0) return WGO_OK;
  if (!(shift > 0.0))
    return fail(WGO_INVALID_ARGUMENT, "CgPreconditioner: shift must be positive for rank > 0");
  p->L = (double*)malloc(sizeof(double) * (size_t)(n * k));
  memcpy(p->L, L, sizeof(double) * (size_t)(n * k));
  p->cap = (double*)malloc(sizeof(double) * (size_t)(k * k));
  for (int64_t j = 0; j < k; ++j)
    for (int64_t i = 0; i < k; ++i) p->cap[j * k + i] = dot(p->L + i * n, p->L + j * n, n);
  for (int64_t i = 0; i < k; ++i) p->cap[i * k + i] += shift;
  if (cholesky_lower(p->cap, k) != WGO_OK) {
    wgo_precond_free(p);
    return fail(WGO_NOT_SPD, "CgPreconditioner: capacitance factorization failed");
  }
  return WGO_OK;
}

int wgo_precond_from_op(wgo_precond* p, const wgo_op* op, int64_t rank, double shift, int mode) {
  const int64_t n = op->n; /* from_matrix, solvers.cpp:123-133 */
  memset(p, 0, sizeof *p);
  p->n = n;
  if (rank > n) rank = n;
  if (rank <= 0) return WGO_OK; /* identity */
  double* L = (double*)malloc(sizeof(double) * (size_t)(n * rank));
  int64_t achieved = 0;
  int st = wgo_pivoted_cholesky(op, rank, L, &achieved);
  if (st) {
    free(L);
    return st;
  }
  if (mode == WGO_SHIFT_CALIBRATED) {
    double tr = 0.0, fro = 0.0;
    for (int64_t i = 0; i < n; ++i) tr += op_diag(op, i);
    for (int64_t t = 0; t < n * achieved; ++t) fro += L[t] * L[t];
    const double leftover = (tr - fro) / (double)n;
    shift += leftover > 0.0 ? leftover : 0.0;
  }
  st = wgo_precond_init(p, L, n, achieved, shift);
  free(L);
  return st;
}

void wgo_precond_apply(const wgo_precond* p, const double* r, double* z) {
  const int64_t n = p->n, k = p->k; /* solvers.cpp:135-140 */
  if (k == 0) {
    memcpy(z, r, sizeof(double) * (size_t)n);
    return;
  }
  double* t = (double*)malloc(sizeof(double) * (size_t)k);
  for (int64_t j = 0; j < k; ++j) t[j] = dot(p->L + j * n, r, n);
  cholesky_solve(p->cap, k, t);
  for (int64_t i = 0; i < n; ++i) z[i] = r[i];
  for (int64_t j = 0; j < k; ++j) {
    const double tj = t[j];
    const double* Lj = p->L + j * n;
    for (int64_t i = 0; i < n; ++i) z[i] -= Lj[i] * tj;
  }
  for (int64_t i = 0; i < n; ++i) z[i] /= p->shift;
  free(t);
}

void wgo_precond_free(wgo_precond* p) {
  free(p->L);
  free(p->cap);
  p->L = p->cap = NULL;
}

int wgo_cg_solve_with(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                      const wgo_solver_config* cfg, const wgo_precond* pre, wgo_result* res) {
  const int64_t n = op->n; /* solvers.cpp:142-183 */
  res->iterations = 0;
  res->history_len = 0;
  res->converged = 0;
  res->diverged_at = 0;
  const double bnorm = nrm2(b, n);
  if (bnorm == 0.0) {
    zero_rhs_result(n, res);
    return WGO_OK;
  }
  int st = expand_init(warm, u1, n1, n, res->v);
  if (st) return st;
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* Hp = (double*)malloc(sizeof(double) * (size_t)n);
  op->matvec(op, res->v, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  res->history[res->history_len++] = nrm2(r, n) / bnorm;
  if (res->history[0] <= cfg->tolerance) {
    res->converged = 1;
    goto done;
  }
  wgo_precond_apply(pre, r, z);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = dot(r, z, n);
  for (int k = 1; k <= cfg->max_iters; ++k) {
    op->matvec(op, p, Hp); /* :162 */
    const double pHp = dot(p, Hp, n);
    if (pHp <= 0.0) {
      st = fail(WGO_NOT_SPD, "cg_solve: non-positive curvature encountered");
      goto done;
    }
    const double alpha = rz / pHp;
    for (int64_t i = 0; i < n; ++i) res->v[i] += alpha * p[i];
    op->matvec(op, res->v, r); /* true residual :171 */
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double rel = nrm2(r, n) / bnorm;
    res->history[res->history_len++] = rel;
    res->iterations = k;
    if (rel <= cfg->tolerance) {
      res->converged = 1;
      break;
    }
    wgo_precond_apply(pre, r, z);
    const double rz_next = dot(r, z, n);
    const double beta = rz_next / rz;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_next;
  }
done:
  free(r);
  free(z);
  free(p);
  free(Hp);
  return st;
}

int wgo_cg_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                 const wgo_solver_config* cfg, wgo_result* res) {
  wgo_precond pre; /* solvers.cpp:186-191 */
  int st = wgo_precond_from_op(&pre, op, cfg->precond_rank, cfg->precond_shift,
                               cfg->precond_shift_mode);
  if (st) return st;
  st = wgo_cg_solve_with(op, b, warm, u1, n1, cfg, &pre, res);
  wgo_precond_free(&pre);
  return st;
}

int wgo_sgd_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                  const wgo_solver_config* cfg, wgo_result* res) {
  const int64_t n = op->n; /* solvers.cpp:193-243 */
  res->iterations = 0;
  res->history_len = 0;
  res->converged = 0;
  res->diverged_at = 0;
  const double bnorm = nrm2(b, n);
  if (bnorm == 0.0) {
    zero_rhs_result(n, res);
    return WGO_OK;
  }
  const int64_t batch = cfg->batch_size < n ? cfg->batch_size : n;
  if (batch <= 0) return fail(WGO_INVALID_ARGUMENT, "sgd_solve: batch size must be positive");
  int st = expand_init(warm, u1, n1, n, res->v);
  if (st) return st;
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  double* vel = (double*)calloc((size_t)n, sizeof(double));
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  double* row = (double*)malloc(sizeof(double) * (size_t)n);
  op->matvec(op, res->v, t);
  for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
  res->history[res->history_len++] = nrm2(t, n) / bnorm;
  if (res->history[0] <= cfg->tolerance) {
    res->converged = 1;
    goto done;
  }
  {
    const double scale = cfg->sgd_scaling == WGO_SGD_UNBIASED ? (double)n / (double)batch : 1.0;
    wgo_rng rng = {cfg->seed};
    for (int64_t i = 0; i < n; ++i) idx[i] = i; /* persistent index array :213-214 */
    for (int k = 1; k <= cfg->max_iters; ++k) {
      for (int64_t i = 0; i < batch; ++i) { /* partial Fisher-Yates :219-222 */
        const int64_t j = i + (int64_t)wgo_rng_uniform_index(&rng, (uint64_t)(n - i));
        const int64_t tmp = idx[i];
        idx[i] = idx[j];
        idx[j] = tmp;
      }
      for (int64_t i = 0; i < n; ++i) vel[i] *= cfg->momentum;
      for (int64_t i = 0; i < batch; ++i) { /* :225-228 */
        const int64_t rr = idx[i];
        op->block(op, rr, 1, 0, n, row);
        vel[rr] += scale * (dot(row, res->v, n) - b[rr]);
      }
      for (int64_t i = 0; i < n; ++i) res->v[i] -= cfg->learning_rate * vel[i];
      op->matvec(op, res->v, t);
      for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
      const double rel = nrm2(t, n) / bnorm;
      res->history[res->history_len++] = rel;
      res->iterations = k;
      if (rel > 1e3 || !isfinite(rel)) { /* :234-236 */
        res->diverged_at = k;
        st = fail(WGO_DIVERGED, "sgd_solve: diverged (relative residual above 1e3)");
        goto done;
      }
      if (rel <= cfg->tolerance) {
        res->converged = 1;
        break;
      }
    }
  }
done:
  free(t);
  free(vel);
  free(idx);
  free(row);
  return st;
}

int wgo_ap_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                 const wgo_solver_config* cfg, wgo_result* res) {
  const int64_t n = op->n; /* solvers.cpp:245-309 */
  res->iterations = 0;
  res->history_len = 0;
  res->converged = 0;
  res->diverged_at = 0;
  const double bnorm = nrm2(b, n);
  if (bnorm == 0.0) {
    zero_rhs_result(n, res);
    return WGO_OK;
  }
  const int64_t bs = cfg->block_size < n ? cfg->block_size : n;
  if (bs <= 0) return fail(WGO_INVALID_ARGUMENT, "ap_solve: block size must be positive");
  const int64_t n_blocks = (n + bs - 1) / bs;
  double* fac = (double*)malloc(sizeof(double) * (size_t)(n_blocks * bs * bs));
  for (int64_t blk = 0; blk < n_blocks; ++blk) { /* :255-264 */
    const int64_t start = blk * bs;
    const int64_t len = bs < n - start ? bs : n - start;
    double* F = fac + blk * bs * bs;
    op->block(op, start, len, start, len, F);
    if (cholesky_lower(F, len) != WGO_OK) {
      free(fac);
      return fail(WGO_NOT_SPD, "ap_solve: diagonal block factorization failed");
    }
  }
  int st = expand_init(warm, u1, n1, n, res->v);
  if (st) {
    free(fac);
    return st;
  }
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* delta = (double*)malloc(sizeof(double) * (size_t)bs);
  double* cols = (double*)malloc(sizeof(double) * (size_t)(n * bs));
  op->matvec(op, res->v, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  res->history[res->history_len++] = nrm2(r, n) / bnorm;
  if (res->history[0] <= cfg->tolerance) {
    res->converged = 1;
    goto done;
  }
  for (int k = 1; k <= cfg->max_iters; ++k) {
    int64_t blk = (int64_t)((k - 1) % n_blocks);
    if (cfg->ap_ordering == WGO_AP_GREEDY) { /* :277-286 ties -> lowest index */
      double best = -1.0;
      for (int64_t c = 0; c < n_blocks; ++c) {
        const int64_t len = bs < n - c * bs ? bs : n - c * bs;
        const double norm = nrm2(r + c * bs, len);
        if (norm > best) {
          best = norm;
          blk = c;
        }
      }
    }
    const int64_t start = blk * bs;
    const int64_t len = bs < n - start ? bs : n - start;
    memcpy(delta, r + start, sizeof(double) * (size_t)len);
    cholesky_solve(fac + blk * bs * bs, len, delta); /* :290 */
    for (int64_t i = 0; i < len; ++i) res->v[start + i] += delta[i];
    op->block(op, 0, n, start, len, cols); /* r -= H(:, B) delta, :292 */
    for (int64_t j = 0; j < len; ++j) {
      const double dj = delta[j];
      const double* cj = cols + j * n;
      for (int64_t i = 0; i < n; ++i) r[i] -= cj[i] * dj;
    }
    if (k % (int)n_blocks == 0) { /* refresh against drift :293 */
      op->matvec(op, res->v, r);
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    }
    double rel = nrm2(r, n) / bnorm;
    if (rel <= cfg->tolerance) { /* confirm with the true residual :296-300 */
      op->matvec(op, res->v, r);
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
      rel = nrm2(r, n) / bnorm;
    }
    res->history[res->history_len++] = rel;
    res->iterations = k;
    if (rel <= cfg->tolerance) {
      res->converged = 1;
      break;
    }
  }
done:
  free(fac);
  free(r);
  free(delta);
  free(cols);
  return st;
}

int wgo_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
              const wgo_solver_config* cfg, wgo_result* res) { /* solvers.cpp:311-319 */
  switch (cfg->method) {
    case WGO_CG: return wgo_cg_solve(op, b, warm, u1, n1, cfg, res);
    case WGO_SGD: return wgo_sgd_solve(op, b, warm, u1, n1, cfg, res);
    case WGO_AP: return wgo_ap_solve(op, b, warm, u1, n1, cfg, res);
  }
  return fail(WGO_INVALID_ARGUMENT, "solve: unknown method");
}

int wgo_solve_many(const wgo_op* op, const double* B, int64_t s, int warm, const double* U1,
                   int64_t n1, const wgo_solver_config* cfg, double* V, int* iterations,
                   double* history, int* hist_len, int* converged, int* failed_col,
                   int* diverged_at) { /* solvers.cpp:321-354 */
  const int64_t n = op->n;
  wgo_precond pre;
  memset(&pre, 0, sizeof pre);
  pre.n = n;
  int st = WGO_OK;
  if (failed_col) *failed_col = -1;
  if (cfg->method == WGO_CG) {
    st = wgo_precond_from_op(&pre, op, cfg->precond_rank, cfg->precond_shift,
                             cfg->precond_shift_mode);
    if (st) return st;
  }
  const int64_t hstride = (int64_t)cfg->max_iters + 1;
  for (int64_t i = 0; i < s; ++i) {
    wgo_result res;
    res.v = V + i * n;
    res.history = history + i * hstride;
    const double* b = B + i * n;
    const double* u1 = warm ? U1 + i * n1 : NULL;
    switch (cfg->method) {
      case WGO_CG: st = wgo_cg_solve_with(op, b, warm, u1, n1, cfg, &pre, &res); break;
      case WGO_SGD: {
        wgo_solver_config per = *cfg;
        per.seed = wgo_derive_seed(cfg->seed, (uint64_t)i); /* :344 */
        st = wgo_sgd_solve(op, b, warm, u1, n1, &per, &res);
        break;
      }
      case WGO_AP: st = wgo_ap_solve(op, b, warm, u1, n1, cfg, &res); break;
      default: st = fail(WGO_INVALID_ARGUMENT, "solve_many: unknown method");
    }
    iterations[i] = res.iterations;
    hist_len[i] = res.history_len;
    converged[i] = res.converged;
    if (diverged_at) diverged_at[i] = res.diverged_at;
    if (st) {
      if (failed_col) *failed_col = (int)i;
      break;
    }
  }
  wgo_precond_free(&pre);
  return st;
}

int wgo_exact_solve(const double* H, int64_t n, const double* b, double* x) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(n * n)); /* analysis.cpp:15-26 */
  memcpy(A, H, sizeof(double) * (size_t)(n * n));
  if (cholesky_lower(A, n) != WGO_OK) {
    free(A);
    return fail(WGO_NOT_SPD, "exact_solve: Cholesky factorization failed (matrix not SPD)");
  }
  memcpy(x, b, sizeof(double) * (size_t)n);
  cholesky_solve(A, n, x);
  free(A);
  return WGO_OK;
}

double wgo_rkhs_distance(const wgo_op* op, const double* v_init, const double* v_exact) {
  const int64_t n = op->n; /* analysis.cpp:28-32 */
  double* e = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double* He = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t i = 0; i < n; ++i) e[i] = v_exact[i] - v_init[i];
  op->matvec(op, e, He);
  const double q = dot(e, He, n);
  free(e);
  free(He);
  return sqrt(q > 0.0 ? q : 0.0);
}

/* mll_with_dist, analysis.cpp:99-131.  D: n x n distances (pairwise_distances). */
static int mll_with_dist(const wgo_hyp* h, const double* Dm, int64_t n, const double* y,
                         double* value, double* grad3) {
  const double s2 = h->signal_scale * h->signal_scale;
  const double sn2 = h->noise_scale * h->noise_scale;
  const double l = h->lengthscale;
  const size_t nn = (size_t)(n * n);
  double* K = (double*)malloc(sizeof(double) * nn);
  double* L = (double*)malloc(sizeof(double) * nn);
  for (size_t t = 0; t < nn; ++t) {
    const double r = Dm[t];
    if (h->kind == WGO_RBF) {
      K[t] = s2 * exp(-0.5 * (r / l) * (r / l));
    } else {
      const double z = r * (kSqrt3 / l); /* :103 */
      K[t] = s2 * (1.0 + z) * exp(-z);
    }
    L[t] = K[t];
  }
  for (int64_t i = 0; i < n; ++i) L[i * n + i] += sn2; /* :106 */
  if (cholesky_lower(L, n) != WGO_OK) {
    free(K);
    free(L);
    return fail(WGO_NOT_SPD, "mll: covariance not SPD at these hyperparameters");
  }
  double* alpha = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(alpha, y, sizeof(double) * (size_t)n);
  cholesky_solve(L, n, alpha); /* :112 */
  double logdet = 0.0;
  for (int64_t i = 0; i < n; ++i) logdet += log(L[i * n + i]);
  logdet *= 2.0;
  *value = -0.5 * dot(y, alpha, n) - 0.5 * logdet - 0.5 * (double)n * 1.8378770664093454836;
  /* grad_j = 0.5 tr((alpha alpha^T - H^{-1}) dH_j), H^{-1} column by column (:121-130) */
  double* e = (double*)malloc(sizeof(double) * (size_t)n);
  double g0 = 0.0, g1 = 0.0, tr = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    memset(e, 0, sizeof(double) * (size_t)n);
    e[j] = 1.0;
    cholesky_solve(L, n, e); /* column j of H^{-1} */
    for (int64_t i = 0; i < n; ++i) {
      const double a = alpha[i] * alpha[j] - e[i];
      const double r = Dm[j * n + i];
      const double rho = r / l;
      const double dkl = h->kind == WGO_RBF ? K[j * n + i] * rho * rho
                                            : 3.0 * s2 * rho * rho * exp(-kSqrt3 * rho);
      g0 += a * dkl;
      g1 += a * 2.0 * K[j * n + i];
    }
    tr += alpha[j] * alpha[j] - e[j];
  }
  grad3[0] = 0.5 * g0;
  grad3[1] = 0.5 * g1;
  grad3[2] = 0.5 * tr * 2.0 * sn2;
  free(e);
  free(alpha);
  free(K);
  free(L);
  return WGO_OK;
}

int wgo_mll(const wgo_hyp* h, const double* X, int64_t n, int64_t d, const double* y, double* value,
            double* grad3) { /* analysis.cpp:135-139 */
  int st = wgo_hyp_validate(h);
  if (st) return st;
  if (n < 1) return fail(WGO_INVALID_ARGUMENT, "mll: X rows != y length");
  double* Dm = (double*)malloc(sizeof(double) * (size_t)(n * n));
  wgo_pairwise_distances(X, n, X, n, d, Dm);
  st = mll_with_dist(h, Dm, n, y, value, grad3);
  free(Dm);
  return st;
}

int wgo_optimize_mll(const wgo_hyp* init, const double* X, int64_t n, int64_t d, const double* y,
                     int steps, double step_size, wgo_hyp* out) { /* analysis.cpp:141-182 */
  int st = wgo_hyp_validate(init);
  if (st) return st;
  double* Dm = (double*)malloc(sizeof(double) * (size_t)(n * n));
  wgo_pairwise_distances(X, n, X, n, d, Dm);
  double th[3] = {log(init->lengthscale), log(init->signal_scale), log(init->noise_scale)};
  const double lo[3] = {log(1e-3), log(1e-3), log(1e-4)}, hi[3] = {log(1e3), log(1e3), log(1e2)};
  wgo_hyp cur_h = {init->kind, exp(th[0]), exp(th[1]), exp(th[2])};
  double val, g[3];
  st = mll_with_dist(&cur_h, Dm, n, y, &val, g);
  if (st) {
    free(Dm);
    return st;
  }
  if (!isfinite(val)) {
    free(Dm);
    return fail(WGO_RUNTIME_ERROR, "optimize_mll: non-finite MLL at the initial hyperparameters");
  }
  double best[3] = {th[0], th[1], th[2]}, best_val = val;
  double m[3] = {0, 0, 0}, v[3] = {0, 0, 0};
  for (int t = 1; t <= steps; ++t) {
    const double bc1 = 1.0 - pow(0.9, t), bc2 = 1.0 - pow(0.999, t);
    for (int k = 0; k < 3; ++k) {
      m[k] = 0.9 * m[k] + (1.0 - 0.9) * g[k];
      v[k] = 0.999 * v[k] + (1.0 - 0.999) * (g[k] * g[k]);
      const double step = (m[k] / bc1) / (sqrt(v[k] / bc2) + 1e-8);
      double x = th[k] + step_size * step;
      th[k] = x < lo[k] ? lo[k] : (x > hi[k] ? hi[k] : x);
    }
    cur_h.lengthscale = exp(th[0]);
    cur_h.signal_scale = exp(th[1]);
    cur_h.noise_scale = exp(th[2]);
    st = mll_with_dist(&cur_h, Dm, n, y, &val, g);
    if (st) {
      free(Dm);
      return st;
    }
    if (!isfinite(val)) {
      free(Dm);
      return fail(WGO_RUNTIME_ERROR, "optimize_mll: non-finite MLL at step %d (lengthscale %g)", t,
                  exp(th[0]));
    }
    if (val > best_val) {
      best_val = val;
      best[0] = th[0];
      best[1] = th[1];
      best[2] = th[2];
    }
  }
  free(Dm);
  out->kind = init->kind;
  out->lengthscale = exp(best[0]);
  out->signal_scale = exp(best[1]);
  out->noise_scale = exp(best[2]);
  return WGO_OK;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

double wgo_median_heuristic_lengthscale(const double* X, int64_t n, int64_t d, uint64_t seed) {
  const int64_t cap = n < 256 ? n : 256; /* analysis.cpp:184-203 */
  double* sub = (double*)malloc(sizeof(double) * (size_t)(cap * d + 1));
  wgo_rng rng = {wgo_derive_seed(seed, 0x6d656469ULL)};
  for (int64_t i = 0; i < cap; ++i) {
    const int64_t r = (int64_t)wgo_rng_uniform_index(&rng, (uint64_t)n);
    for (int64_t k = 0; k < d; ++k) sub[k * cap + i] = X[k * n + r];
  }
  double* Dm = (double*)malloc(sizeof(double) * (size_t)(cap * cap + 1));
  wgo_pairwise_distances(sub, cap, sub, cap, d, Dm);
  const int64_t cnt = cap * (cap - 1) / 2;
  double* vals = (double*)malloc(sizeof(double) * (size_t)(cnt + 1));
  int64_t q = 0;
  for (int64_t j = 0; j < cap; ++j)
    for (int64_t i = j + 1; i < cap; ++i) vals[q++] = Dm[j * cap + i];
  double med = 1.0;
  if (cnt > 0) {
    /* nth_element(size/2) == the (size/2)-th order statistic */
    qsort(vals, (size_t)cnt, sizeof(double), cmp_double);
    med = vals[cnt / 2] > 0.0 ? vals[cnt / 2] : 1.0;
  }
  free(vals);
  free(Dm);
  free(sub);
  return med;
}

/* ======================= sampling.cpp ======================= */

int wgo_sample_prior(const wgo_hyp* h, int64_t dim, int64_t F, uint64_t seed, double* Omega,
                     double* phases, double* amps) { /* sampling.cpp:14-35 */
  int st = wgo_hyp_validate(h);
  if (st) return st;
  if (dim < 1 || F < 1)
    return fail(WGO_INVALID_ARGUMENT, "sample_prior: dim and num_features must be positive");
  wgo_rng rng = {seed};
  for (int64_t i = 0; i < F; ++i) {
    double t_scale;
    if (h->kind == WGO_MATERN32) { /* Student-t(3): :26-28 */
      const double u = wgo_rng_chi_square3(&rng);
      t_scale = sqrt(3.0 / u) / h->lengthscale;
    } else { /* RBF spectral density N(0, l^-2 I) (extension) */
      t_scale = 1.0 / h->lengthscale;
    }
    for (int64_t d = 0; d < dim; ++d) Omega[d * F + i] = wgo_rng_normal(&rng) * t_scale;
    phases[i] = wgo_rng_uniform_range(&rng, 0.0, kTwoPi);
    amps[i] = wgo_rng_normal(&rng);
  }
  return WGO_OK;
}

int wgo_eval_prior(const double* Omega, const double* phases, const double* amps, int64_t F,
                   int64_t dim, double signal_scale, const double* Xs, int64_t m, double* out) {
  /* sampling.cpp:37-46: coeff * cos(X Omega^T + phi) w */
  const double coeff = signal_scale * sqrt(2.0 / (double)F);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int64_t f = 0; f < F; ++f) {
      double ph = 0.0;
      for (int64_t d = 0; d < dim; ++d) ph += Xs[d * m + i] * Omega[d * F + f];
      ph += phases[f];
      acc += cos(ph) * amps[f];
    }
    out[i] = coeff * acc;
  }
  return WGO_OK;
}

int wgo_build_sample_rhs(const double* Omega, const double* phases, const double* amps, int64_t F,
                         int64_t dim, double signal_scale, const double* X, int64_t n,
                         double noise_scale, uint64_t seed, double* out) { /* sampling.cpp:56-64 */
  wgo_eval_prior(Omega, phases, amps, F, dim, signal_scale, X, n, out);
  if (noise_scale > 0.0) {
    wgo_rng rng = {seed};
    for (int64_t i = 0; i < n; ++i) out[i] += noise_scale * wgo_rng_normal(&rng);
  }
  return WGO_OK;
}

int wgo_eval_posterior(const wgo_hyp* h, const double* Omega, const double* phases,
                       const double* amps, int64_t F, const double* Xtrain, int64_t n,
                       int64_t dim, const double* weights, const double* Xs, int64_t m,
                       double* out) { /* sampling.cpp:66-75 */
  wgo_eval_prior(Omega, phases, amps, F, dim, h->signal_scale, Xs, m, out);
  if (n > 0) {
    double* corr = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    int st = wgo_cross_matvec(h, Xs, m, Xtrain, n, dim, weights, 1, corr, 0);
    if (st) {
      free(corr);
      return st;
    }
    for (int64_t i = 0; i < m; ++i) out[i] += corr[i];
    free(corr);
  }
  return WGO_OK;
}


/* grad_prior (sampling.cpp:48-54) + the kernel-weighted sum of grad_posterior (:77-87). */
int wgo_grad_posterior(const wgo_hyp* h, const double* Omega, const double* phases,
                       const double* amps, int64_t F, const double* Xtrain, int64_t n,
                       int64_t dim, const double* weights, const double* x, double* g) {
  if (F < 1 || dim < 1) return WGO_INVALID_ARGUMENT;
  const double coeff = h->signal_scale * sqrt(2.0 / (double)F);
  for (int64_t k = 0; k < dim; ++k) g[k] = 0.0;
  /* -coeff * Omega^T (sin(Omega x + phi) .* w) */
  for (int64_t k = 0; k < dim; ++k) {
    double acc = 0.0;
    for (int64_t f = 0; f < F; ++f) {
      double arg = 0.0;
      for (int64_t q = 0; q < dim; ++q) arg += Omega[q * F + f] * x[q];
      arg += phases[f];
      acc += Omega[k * F + f] * (sin(arg) * amps[f]);
    }
    g[k] = -coeff * acc;
  }
  const double l = h->lengthscale, s2 = h->signal_scale * h->signal_scale;
  for (int64_t j = 0; j < n; ++j) {
    double r2 = 0.0;
    for (int64_t k = 0; k < dim; ++k) {
      const double df = Xtrain[k * n + j] - x[k];
      r2 += df * df;
    }
    double f;
    if (h->kind == WGO_RBF) {
      f = weights[j] * (s2 / (l * l)) * exp(-0.5 * r2 / (l * l));
    } else {
      f = weights[j] * (3.0 * s2 / (l * l)) * exp(-sqrt(3.0) * sqrt(r2) / l);
    }
    for (int64_t k = 0; k < dim; ++k) g[k] += f * (Xtrain[k * n + j] - x[k]);
  }
  return WGO_OK;
}

int wgo_ascend_peaks(const wgo_hyp* h, const double* Omega, const double* phases,
                     const double* amps, int64_t F, const double* Xtrain, int64_t n, int64_t dim,
                     const double* weights, const double* peaks, int64_t P, int steps,
                     double rate, double* best_x, double* best_val) {
  if (dim < 1 || dim > 64) return WGO_INVALID_ARGUMENT;
  double x[64], m[64], v[64], g[64], val;
  double bv = -INFINITY;
  for (int64_t k = 0; k < dim; ++k) best_x[k] = 0.0;
  for (int64_t t = 0; t < P; ++t) {
    for (int64_t k = 0; k < dim; ++k) {
      x[k] = peaks[k * P + t];
      m[k] = v[k] = 0.0;
    }
    wgo_eval_posterior(h, Omega, phases, amps, F, Xtrain, n, dim, weights, x, 1, &val);
    if (val > bv) {
      bv = val;
      for (int64_t k = 0; k < dim; ++k) best_x[k] = x[k];
    }
    for (int k = 1; k <= steps; ++k) {
      wgo_grad_posterior(h, Omega, phases, amps, F, Xtrain, n, dim, weights, x, g);
      int finite = 1;
      for (int64_t q = 0; q < dim; ++q) finite &= isfinite(g[q]) ? 1 : 0;
      if (!finite) break;
      const double bc1 = 1.0 - pow(0.9, k), bc2 = 1.0 - pow(0.999, k);
      for (int64_t q = 0; q < dim; ++q) {
        m[q] = 0.9 * m[q] + 0.1 * g[q];
        v[q] = 0.999 * v[q] + 0.001 * (g[q] * g[q]);
        const double step = (m[q] / bc1) / (sqrt(v[q] / bc2) + 1e-8);
        x[q] += rate * step;
        x[q] = x[q] < 0.0 ? 0.0 : (x[q] > 1.0 ? 1.0 : x[q]);
      }
      wgo_eval_posterior(h, Omega, phases, amps, F, Xtrain, n, dim, weights, x, 1, &val);
      if (val > bv) {
        bv = val;
        for (int64_t q = 0; q < dim; ++q) best_x[q] = x[q];
      }
    }
  }
  *best_val = bv;
  return WGO_OK;
}
