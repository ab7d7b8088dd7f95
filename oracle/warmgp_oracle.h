/*
 * warmgp_oracle.h -- CPU restatement of the reference warm-started GP solver
 * path (arXiv 2511.16340, reference at /root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product (paper_2511_16340_b200/libwarmgp_b200.so) never
 * links or calls it, and has no CPU fallback.
 *
 * Conventions follow the reference (Eigen MatrixXd, proj/core/include/warmgp/
 * types.hpp:9-11): every matrix is column-major fp64 with leading dimension =
 * rows; right-hand sides are N x s column-major, one RHS per contiguous column.
 *
 * Parity pins: every function cites the reference file:line it restates.  The
 * restatement is pinned by (i) the reference's own known-answer tests
 * (proj/tests/test_kernel.cpp, test_solvers.cpp, test_sampling.cpp,
 * test_thompson.cpp) re-stated in tests/test_oracle_*.py, and (ii) RNG golden
 * streams produced by compiling the reference's rng.hpp unchanged
 * (oracle/Makefile -> oracle/_ref/rng_golden, fixtures in tests/golden/).
 * Eigen3 is absent, so kernel.cpp / solvers.cpp themselves cannot be built
 * here; their results are pinned through the tests listed above.
 */
#ifndef WARMGP_ORACLE_H
#define WARMGP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same numbering as the product C-ABI (include/warmgp_capi.h) */
enum {
  WGO_OK = 0,
  WGO_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  WGO_NOT_SPD = 2,          /* warmgp::NotSpdError   types.hpp:15-18 */
  WGO_DIVERGED = 3,         /* warmgp::DivergenceError types.hpp:21-26 */
  WGO_RUNTIME_ERROR = 7,    /* std::runtime_error (optimize_mll, analysis.cpp:159,173) */
};
const char* wgo_last_error(void);

/* ---------------- rng.hpp:11-61 ---------------- */
typedef struct { uint64_t state; } wgo_rng;
uint64_t wgo_derive_seed(uint64_t seed, uint64_t stream);
uint64_t wgo_rng_next_u64(wgo_rng* r);
double wgo_rng_uniform(wgo_rng* r);
double wgo_rng_uniform_range(wgo_rng* r, double lo, double hi);
double wgo_rng_normal(wgo_rng* r);
double wgo_rng_chi_square3(wgo_rng* r);
uint64_t wgo_rng_uniform_index(wgo_rng* r, uint64_t n);
/* bulk helpers (fill order = the reference's loops in tests/testutil.hpp:9-23) */
void wgo_uniform_inputs(uint64_t seed, int64_t n, int64_t dim, double* X /* n x dim col-major */);
void wgo_gaussian_vector(uint64_t seed, int64_t n, double* v);

/* ---------------- kernel.hpp / kernel.cpp ---------------- */
enum { WGO_MATERN32 = 0, WGO_RBF = 1 };
typedef struct {
  int kind;              /* WGO_MATERN32 (reference) or WGO_RBF (documented extension) */
  double lengthscale;    /* kernel.hpp:8-14 */
  double signal_scale;
  double noise_scale;    /* sigma_n, NOT the variance: H diag = s^2 + sigma_n^2 */
} wgo_hyp;

int wgo_hyp_validate(const wgo_hyp* h);                          /* kernel.cpp:11-15 */
double wgo_kernel_from_distance(const wgo_hyp* h, double r);     /* kernel.cpp:17-21 (+RBF) */
int wgo_pairwise_distances(const double* A, int64_t m, const double* B, int64_t n, int64_t d,
                           double* D /* m x n */);               /* kernel.cpp:39-46 */
int wgo_gram_matrix(const wgo_hyp* h, const double* X, int64_t n, int64_t d,
                    double* H /* n x n */);                      /* kernel.cpp:48-72 */
int wgo_cross_kernel(const wgo_hyp* h, const double* Xs, int64_t m, const double* X, int64_t n,
                     int64_t d, double* K /* m x n */);          /* kernel.cpp:74-89 */
/* extend_system + BlockedSystem::assembled, kernel.cpp:91-130: H11 (n1 x n1) reused verbatim */
int wgo_extend_assembled(const wgo_hyp* h, const double* H11, const double* X1, int64_t n1,
                         const double* X2, int64_t n2, int64_t d, double* H /* n x n */);

/* Matrix-free (K(X,X)+sigma_n^2 I) V for rows [r0,r1) -- the same per-entry formula as
 * wgo_gram_matrix, evaluated on the fly with OpenMP (CPU baseline for configs 3-4 where
 * dense H cannot exist).  V: n x s col-major; Y: (r1-r0) x s col-major. */
int wgo_kmatvec_rows(const wgo_hyp* h, const double* X, int64_t n, int64_t d, const double* V,
                     int64_t s, int64_t r0, int64_t r1, double* Y, int nthreads);
/* cross mode K(Xs, X) W (no noise), used by eval_posterior (sampling.cpp:66-75) */
int wgo_cross_matvec(const wgo_hyp* h, const double* Xs, int64_t m, const double* X, int64_t n,
                     int64_t d, const double* W, int64_t s, double* Y, int nthreads);

/* ---------------- solvers.hpp / solvers.cpp ---------------- */
enum { WGO_CG = 0, WGO_SGD = 1, WGO_AP = 2 };
enum { WGO_SGD_UNBIASED = 0, WGO_SGD_BLOCK = 1 };
enum { WGO_AP_GREEDY = 0, WGO_AP_CYCLIC = 1 };
enum { WGO_SHIFT_CALIBRATED = 0, WGO_SHIFT_NOISE_ONLY = 1 };

typedef struct {                         /* SolverConfig, solvers.hpp:27-48 */
  int method;
  double tolerance;
  int max_iters;
  double learning_rate;
  double momentum;
  int64_t batch_size;
  int sgd_scaling;
  int64_t block_size;
  int ap_ordering;
  int64_t precond_rank;
  double precond_shift;
  int precond_shift_mode;
  uint64_t seed;
} wgo_solver_config;
void wgo_solver_config_default(wgo_solver_config* c);

/* A symmetric operator the solvers act on: either a dense H (the reference's
 * representation) or the matrix-free kernel operator. */
typedef struct wgo_op {
  int64_t n;
  const void* ctx;
  void (*matvec)(const struct wgo_op* op, const double* v, double* y);   /* y = H v */
  void (*block)(const struct wgo_op* op, int64_t r0, int64_t nr, int64_t c0, int64_t nc,
                double* out /* nr x nc col-major */);
} wgo_op;
void wgo_op_dense(wgo_op* op, const double* H, int64_t n);
typedef struct { wgo_hyp hyp; const double* X; int64_t n; int64_t d; int nthreads; double* sq; } wgo_mf_ctx;
int wgo_op_matrix_free(wgo_op* op, wgo_mf_ctx* ctx); /* ctx->sq allocated; free with wgo_mf_free */
void wgo_mf_free(wgo_mf_ctx* ctx);

/* init_weights, solvers.cpp:27-38.  u1 may be NULL when n1 == 0 and !warm. */
int wgo_init_weights(int warm, const double* u1, int64_t u1_len, int64_t n1, int64_t n2, double* v);
/* relative_residual, solvers.cpp:62-66 (zero b -> WGO_INVALID_ARGUMENT) */
int wgo_relative_residual(const wgo_op* op, const double* v, const double* b, double* out);
double wgo_quadratic_objective(const wgo_op* op, const double* v, const double* b);
/* pivoted_cholesky, solvers.cpp:72-107; L is n x rank (caller-allocated), *achieved <= rank */
int wgo_pivoted_cholesky(const wgo_op* op, int64_t rank, double* L, int64_t* achieved);

typedef struct {                 /* CgPreconditioner, solvers.hpp:82-100 */
  int64_t n, k;
  double shift;
  double* L;    /* n x k */
  double* cap;  /* k x k lower Cholesky factor of shift I + L^T L */
} wgo_precond;
/* CgPreconditioner(L, shift), solvers.cpp:109-121 (copies L) */
int wgo_precond_init(wgo_precond* p, const double* L, int64_t n, int64_t k, double shift);
/* CgPreconditioner::from_matrix, solvers.cpp:123-133 */
int wgo_precond_from_op(wgo_precond* p, const wgo_op* op, int64_t rank, double shift, int mode);
void wgo_precond_apply(const wgo_precond* p, const double* r, double* z); /* solvers.cpp:135-140 */
void wgo_precond_free(wgo_precond* p);

typedef struct {                 /* SolveResult, solvers.hpp:102-109 */
  double* v;            /* n (caller-allocated) */
  int iterations;
  double* history;      /* caller-allocated, capacity max_iters + 1 */
  int history_len;
  int converged;
  int diverged_at;      /* DivergenceError::iterations when status == WGO_DIVERGED */
} wgo_result;

/* init: warm != 0 -> Initialization::warm(u1[0..n1)) else cold */
int wgo_cg_solve_with(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                      const wgo_solver_config* cfg, const wgo_precond* pre,
                      wgo_result* res);                                   /* solvers.cpp:142-183 */
int wgo_cg_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                 const wgo_solver_config* cfg, wgo_result* res);          /* solvers.cpp:186-191 */
int wgo_sgd_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                  const wgo_solver_config* cfg, wgo_result* res);         /* solvers.cpp:193-243 */
int wgo_ap_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
                 const wgo_solver_config* cfg, wgo_result* res);          /* solvers.cpp:245-309 */
int wgo_solve(const wgo_op* op, const double* b, int warm, const double* u1, int64_t n1,
              const wgo_solver_config* cfg, wgo_result* res);             /* solvers.cpp:311-319 */
/* solve_many, solvers.cpp:321-354.  B: n x s col-major; U1: n1 x s col-major (warm != 0);
 * V: n x s; iterations/converged/status: s; history: s x (max_iters+1) row-major, hist_len: s.
 * Columns run sequentially; the first failing column's status is returned (the reference
 * throws there), later columns are not run. */
int wgo_solve_many(const wgo_op* op, const double* B, int64_t s, int warm, const double* U1,
                   int64_t n1, const wgo_solver_config* cfg, double* V, int* iterations,
                   double* history, int* hist_len, int* converged, int* failed_col,
                   int* diverged_at);

/* exact_solve, analysis.cpp:15-26 (dense Cholesky; failure -> WGO_NOT_SPD) */
int wgo_exact_solve(const double* H, int64_t n, const double* b, double* x);
/* rkhs_distance, analysis.cpp:28-32 */
double wgo_rkhs_distance(const wgo_op* op, const double* v_init, const double* v_exact);
/* mll, analysis.cpp:99-139 (mll_with_dist on pairwise_distances(X, X)): value and gradient
 * with respect to (log l, log s_f, log sigma_n).  Matern-3/2 as the reference; kind == WGO_RBF
 * uses the RBF analogue (dK/dlog l = K r^2 / l^2).  X: n x d col-major.  Not SPD ->
 * WGO_NOT_SPD. */
int wgo_mll(const wgo_hyp* h, const double* X, int64_t n, int64_t d, const double* y, double* value,
            double* grad3);
/* optimize_mll, analysis.cpp:141-182: Adam on the log-parameters inside the soft box, best
 * seen returned; a non-finite MLL -> WGO_RUNTIME_ERROR (std::runtime_error). */
int wgo_optimize_mll(const wgo_hyp* init, const double* X, int64_t n, int64_t d, const double* y,
                     int steps, double step_size, wgo_hyp* out);
/* median_heuristic_lengthscale, analysis.cpp:184-203 */
double wgo_median_heuristic_lengthscale(const double* X, int64_t n, int64_t d, uint64_t seed);

/* ---------------- sampling.hpp / sampling.cpp ---------------- */
/* sample_prior, sampling.cpp:14-35.  Omega: F x dim col-major, phases/amps: F.
 * Matern-3/2: Student-t(3) rows (reference).  RBF: Gaussian rows N(0, l^-2 I)
 * drawn in the same per-feature order minus the chi-square draw (extension). */
int wgo_sample_prior(const wgo_hyp* h, int64_t dim, int64_t F, uint64_t seed, double* Omega,
                     double* phases, double* amps);
/* eval_prior, sampling.cpp:37-46.  Xs: m x dim col-major -> out: m */
int wgo_eval_prior(const double* Omega, const double* phases, const double* amps, int64_t F,
                   int64_t dim, double signal_scale, const double* Xs, int64_t m, double* out);
/* build_sample_rhs, sampling.cpp:56-64 */
int wgo_build_sample_rhs(const double* Omega, const double* phases, const double* amps, int64_t F,
                         int64_t dim, double signal_scale, const double* X, int64_t n,
                         double noise_scale, uint64_t seed, double* out);
/* eval_posterior, sampling.cpp:66-75 */
int wgo_eval_posterior(const wgo_hyp* h, const double* Omega, const double* phases,
                       const double* amps, int64_t F, const double* Xtrain, int64_t n,
                       int64_t dim, const double* weights, const double* Xs, int64_t m,
                       double* out);

/* grad_posterior, sampling.cpp:77-87 (with grad_prior :48-54): gradient of eval_posterior at
 * one point x (dim).  Matern-3/2 as in the reference; RBF analogue (s^2/l^2 e^{-r^2/2l^2}) as
 * the documented extension. */
int wgo_grad_posterior(const wgo_hyp* h, const double* Omega, const double* phases,
                       const double* amps, int64_t F, const double* Xtrain, int64_t n,
                       int64_t dim, const double* weights, const double* x, double* g);
/* ascend_peaks for one sample, thompson.cpp:209-258: Adam ascent from each of P start rows
 * (peaks: P x dim col-major), steps/rate as given, clamped to [0,1]^dim; best point and
 * value over all trajectories (strict >, first wins). */
int wgo_ascend_peaks(const wgo_hyp* h, const double* Omega, const double* phases,
                     const double* amps, int64_t F, const double* Xtrain, int64_t n, int64_t dim,
                     const double* weights, const double* peaks, int64_t P, int steps,
                     double rate, double* best_x, double* best_val);

#ifdef __cplusplus
}
#endif
#endif
