/*
 * warmgp_capi.h -- C ABI of the B200-native warm-started GP kernel-matvec path
 * (libwarmgp_b200.so).  Plain pointers and sizes only; no torch, no Eigen.
 *
 * The reference (/root/reference/proj, C++20 + Eigen, fp64 dense H) has no FFI:
 * its boundary is the free-function C++ API of warmgp::{kernel,solvers,
 * sampling}.hpp.  Each entry point below names the reference interface it
 * replaces.  The C++ mirror of that API over this ABI is include/warmgp/gpu.hpp
 * (same type and function names, same exception types); INTEGRATION.md shows
 * how a reference build binds it.
 *
 * Layout conventions at this boundary follow the reference (Eigen MatrixXd,
 * types.hpp:9-11): host matrices are column-major fp64 with an explicit
 * leading dimension; right-hand sides are N x s with one RHS per column.
 * Device-resident buffers (the *_dev entry points) are row-major N x s
 * ("RHS-interleaved") fp64 for every precision; the precision selects the
 * arithmetic inside the kernel-matvec.
 *
 * Threading: calls on one handle are serialised by the caller (one stream per
 * device context); distinct contexts may be used concurrently.  Every call
 * that takes host buffers blocks until results are on the host.
 *
 * Errors: every wgp_status != WGP_OK leaves a thread-local message readable
 * with wgp_last_error().  The C++ wrapper maps WGP_NOT_SPD -> warmgp::NotSpdError,
 * WGP_DIVERGED -> warmgp::DivergenceError(iterations), WGP_INVALID_ARGUMENT ->
 * std::invalid_argument (types.hpp:15-32).  There is no CPU fallback: with no
 * usable CUDA device every call returns WGP_CUDA_ERROR.
 */
#ifndef WARMGP_CAPI_H
#define WARMGP_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WGP_ABI_VERSION 2

typedef enum {
  WGP_OK = 0,
  WGP_INVALID_ARGUMENT = 1, /* std::invalid_argument (solvers.cpp:28-33,46,64,74,113,199,251,326) */
  WGP_NOT_SPD = 2,          /* NotSpdError (solvers.cpp:119,165,262; analysis.cpp:18) */
  WGP_DIVERGED = 3,         /* DivergenceError (solvers.cpp:235) */
  WGP_CUDA_ERROR = 4,
  WGP_NCCL_ERROR = 5,
  WGP_OOM = 6,
  WGP_RUNTIME_ERROR = 7,    /* std::runtime_error (optimize_mll, analysis.cpp:159,173) */
} wgp_status;

typedef enum { WGP_MATERN32 = 0, WGP_RBF = 1 } wgp_kernel;

/* Arithmetic of the kernel-matvec.  F64: fp64 CUDA-core path (<=1e-10 vs the
 * oracle).  F32_3XTF32: fp32 storage, tensor-core contractions with a hi/lo
 * split (<=1e-4).  TF32: single-pass tensor-core contractions (fastest, not
 * parity-grade).  F32_SIMT: fp32 CUDA-core path (validation of the others). */
typedef enum { WGP_F64 = 0, WGP_F32_3XTF32 = 1, WGP_TF32 = 2, WGP_F32_SIMT = 3 } wgp_precision;

/* True residual b - H v of the CG iteration (solvers.cpp:150,171) on fp32 operators.
 * DIRECT: the operator itself (default).  ANCHORED: r_a - H (v - v_a), where v_a is an
 * anchor iterate and r_a = b - H v_a is evaluated by the fp64 kernel; the solver re-anchors
 * when the predicted error of the fp32 part, |v - v_a| times its measured error rate,
 * exceeds 5% of |r|.  ANCHORED removes the attainable-residual floor eps |H||v| / |b| of
 * fp32 operators on ill-conditioned systems for a few fp64 matvecs per solve.  F64
 * operators ignore the mode. */
typedef enum { WGP_RESIDUAL_DIRECT = 0, WGP_RESIDUAL_ANCHORED = 1 } wgp_residual_mode;

typedef enum { WGP_CG = 0, WGP_SGD = 1, WGP_AP = 2 } wgp_method;              /* solvers.hpp:10 */
typedef enum { WGP_SGD_UNBIASED = 0, WGP_SGD_BLOCK = 1 } wgp_sgd_scaling;     /* solvers.hpp:16-19 */
typedef enum { WGP_AP_GREEDY = 0, WGP_AP_CYCLIC = 1 } wgp_ap_ordering;        /* solvers.hpp:25 */
typedef enum { WGP_SHIFT_CALIBRATED = 0, WGP_SHIFT_NOISE_ONLY = 1 } wgp_shift_mode; /* solvers.hpp:43 */

/* warmgp::SolverConfig, solvers.hpp:27-48 (field for field; same defaults via
 * wgp_solver_config_default). */
typedef struct {
  int32_t method;
  double tolerance;
  int32_t max_iters;
  double learning_rate;
  double momentum;
  int64_t batch_size;
  int32_t sgd_scaling;
  int64_t block_size;
  int32_t ap_ordering;
  int64_t precond_rank;
  double precond_shift;
  int32_t precond_shift_mode;
  uint64_t seed;
} wgp_solver_config;

typedef struct wgp_ctx wgp_ctx;
typedef struct wgp_op wgp_op;

int wgp_abi_version(void);
const char* wgp_last_error(void);
void wgp_solver_config_default(wgp_solver_config* cfg);

/* Row partition used by sharded contexts: rows [*row0, *row1) of an n-row
 * operator belong to `rank` of `world`.  Every rank owns an equal slot of
 * ceil(ceil(n / 512) / world) 512-row chunks (the last slots stop at n), so
 * boundaries are multiples of the reduction chunk (per-column sums are
 * bit-identical for every world size) and a full buffer padded to
 * wgp_shard_padded_rows(n, world) rows is exchanged by one in-place all-gather
 * of equal slices. */
void wgp_shard_range(int64_t n, int world, int rank, int64_t* row0, int64_t* row1);
int64_t wgp_shard_padded_rows(int64_t n, int world);

/* ---- device context: one per GPU (one process per GPU) ---- */
wgp_status wgp_ctx_create(int device, wgp_ctx** out);
/* Sharded context: NCCL communicator of `world` ranks built from a unique id
 * produced by rank 0 with wgp_nccl_unique_id (128 bytes), distributed by the
 * caller (e.g. torch.distributed broadcast). */
wgp_status wgp_nccl_unique_id(void* out128);
wgp_status wgp_ctx_create_sharded(int device, int rank, int world, const void* unique_id128,
                                  wgp_ctx** out);
/* Loopback group: `world` ranks emulated by host threads of ONE process on one device
 * (one context per thread, wgp_ctx_create_loopback).  Collectives are host barriers plus
 * device-to-device copies between the ranks' buffers -- no kernel ever waits on another
 * rank -- so the sharded solver code runs unchanged where fewer GPUs than ranks exist
 * (correctness testing; not a performance configuration). */
wgp_status wgp_loopback_group_create(int world, void** group);
void wgp_loopback_group_destroy(void* group);
wgp_status wgp_ctx_create_loopback(int device, int rank, void* group, wgp_ctx** out);
void wgp_ctx_destroy(wgp_ctx* ctx);
/* In-place all-gather of row slices: dV is a full row-major fp64 buffer of
 * wgp_shard_padded_rows(n, world) x s on every rank, rank r holding valid rows
 * wgp_shard_range(n, world, r); afterwards rows [0, n) are valid everywhere (one
 * ncclAllGather of equal slices over NVLink; the exchange step of a sharded matvec). */
wgp_status wgp_allgather_rows_dev(wgp_ctx* ctx, void* dV, int64_t n, int s, void* stream);
/* cudaStream_t the context launches on (for device-pointer callers). */
void* wgp_ctx_stream(wgp_ctx* ctx);

/* ---- kernel operator H = K(X,X) + sigma_n^2 I  (replaces gram_matrix,
 *      kernel.cpp:48-72, and the dense H of CovarianceMatrix kernel.hpp:25-31) ---- */
wgp_status wgp_op_create(wgp_ctx* ctx, int kernel, double lengthscale, double signal_scale,
                         double noise_scale, int precision, int dim, wgp_op** out);
void wgp_op_destroy(wgp_op* op);
/* Append rows to the device-resident X (extend_system, kernel.cpp:108-130;
 * bo_round growth thompson.cpp:403-422).  X_rows: n_new x dim, column-major
 * with leading dimension ld (col_major=1) or row-major with row stride ld. */
wgp_status wgp_op_append_rows(wgp_op* op, const double* X_rows, int64_t n_new, int64_t ld,
                              int col_major);
int64_t wgp_op_size(const wgp_op* op);
/* Select the CG true-residual mode (wgp_residual_mode) of this operator's solves. */
wgp_status wgp_op_set_residual_mode(wgp_op* op, int mode);
int wgp_op_residual_mode(const wgp_op* op);
/* Number of fp64 anchor evaluations made by the last CG solve on this operator (ANCHORED
 * mode; 0 otherwise). */
int wgp_op_last_anchor_count(const wgp_op* op);
int wgp_op_dim(const wgp_op* op);
int wgp_op_precision(const wgp_op* op);

/* Y = H V (the GEMV H*p of solvers.cpp:162 batched over s RHS, without
 * materialising H).  Host column-major fp64 in/out; V: n x s (ldv), Y: n x s (ldy). */
wgp_status wgp_kmatvec(wgp_op* op, const double* V, int64_t ldv, int s, double* Y, int64_t ldy);
/* Device form: dV full n x s row-major, dY this rank's row slice (all n rows
 * unsharded) row-major, both in the op's compute type, on the context stream
 * (stream == NULL) or on `stream`.  Asynchronous. */
wgp_status wgp_kmatvec_dev(wgp_op* op, const void* dV, void* dY, int s, void* stream);
/* Sharded form of wgp_kmatvec_dev (one matvec of solvers.cpp:162 on row-sharded
 * solver vectors): dV is the padded full-row buffer (wgp_shard_padded_rows rows) with this
 * rank's slot up to date; the row slots are all-gathered (NCCL over NVLink, on the context's
 * communication stream) while the local diagonal block K(X_g, X_g) V_g runs, then the other
 * columns.  dY: this rank's rows.  World 1: same as wgp_kmatvec_dev. */
wgp_status wgp_kmatvec_sharded_dev(wgp_op* op, void* dV, void* dY, int s, void* stream);
/* dY = dB - H dV (true residual b - H v, solvers.cpp:150,171,203,231,268,293,298). */
wgp_status wgp_residual_dev(wgp_op* op, const void* dB, const void* dV, void* dY, int s,
                            void* stream);
/* ---- fused solver vector kernels on device [n][s] row-major fp64 arrays (the
 *      per-iteration vector work of cg_solve_with, solvers.cpp:163-180), asynchronous on
 *      `stream` (NULL: the context stream).  dAlpha/dBeta: s fp64; dActive: s int32. ---- */
/* dY[:, c] += alpha_c dX[:, c] for alpha_c != 0   (res.v += alpha * p, solvers.cpp:168) */
wgp_status wgp_axpy_cols_dev(wgp_ctx* ctx, void* dY, const void* dX, const void* dAlpha,
                             int64_t n, int s, void* stream);
/* dP[:, c] = dZ[:, c] + beta_c dP[:, c] where dActive[c] != 0   (p = z + beta p, :180) */
wgp_status wgp_xpby_cols_dev(wgp_ctx* ctx, void* dP, const void* dZ, const void* dBeta,
                             const void* dActive, int64_t n, int s, void* stream);
/* dOut[c] = sum_i dA[i, c] dB[i, c] (p.dot(Hp) :163, r.norm() :172, r.dot(z) :179) in the
 * solvers' fixed order: 512-row chunks, each as 32 sequential 16-row slabs added in slab
 * order, chunks added in index order -- independent of s and of sharding.  dWork: at least
 * ceil(n / 512) * s fp64. */
wgp_status wgp_coldots_dev(wgp_ctx* ctx, const void* dA, const void* dB, int64_t n, int s,
                           void* dOut, void* dWork, void* stream);
/* Cross mode Y = K(X*, X) W, no noise term (cross_kernel kernel.cpp:74-89 times
 * weights, as in eval_posterior sampling.cpp:66-75).  Host column-major fp64. */
wgp_status wgp_cross_matvec(wgp_op* op, const double* Xstar, int64_t m, int64_t ldx,
                            const double* W, int64_t ldw, int s, double* Y, int64_t ldy);

/* ---- solvers (solve_many, solvers.cpp:321-354; cg_solve_with/sgd_solve/ap_solve) ----
 * B: n x s column-major (ldb).  U1: nullable warm starts, n1 x s column-major (ldu)
 * zero-extended to n rows on the device (Initialization::warm, expand_init
 * solvers.cpp:43-48).  Outputs: V n x s (ldv); iterations[s]; converged[s];
 * history: s rows of hist_stride >= max_iters+1 doubles (residual_history,
 * entry 0 = initial residual); history_len[s] = iterations+1 (1 for a zero RHS).
 * col_status (nullable, s): per-column wgp_status; the return value is the
 * status of the lowest failing column (the one the reference would throw
 * from), with diverged_at (nullable, s) holding DivergenceError::iterations. */
wgp_status wgp_solve_many(wgp_op* op, const wgp_solver_config* cfg, const double* B, int64_t ldb,
                          int s, const double* U1, int64_t ldu, int64_t n1, double* V,
                          int64_t ldv, int32_t* iterations, double* history, int64_t hist_stride,
                          int32_t* history_len, int32_t* converged, int32_t* col_status,
                          int32_t* diverged_at);

/* Single right-hand side with the semantics of solve (solvers.cpp:311-319) /
 * cg_solve / sgd_solve / ap_solve: SGD draws from Rng(cfg->seed) itself (solve_many uses
 * derive_seed(cfg->seed, column)).  b: n; u1: nullable warm start of length n1; v: n;
 * history: max_iters+1 doubles.  Errors as wgp_solve_many (diverged_at: nullable). */
wgp_status wgp_solve(wgp_op* op, const wgp_solver_config* cfg, const double* b, const double* u1,
                     int64_t n1, double* v, int32_t* iterations, double* history,
                     int32_t* history_len, int32_t* converged, int32_t* diverged_at);

/* ---- preconditioner (pivoted_cholesky solvers.cpp:72-107, from_matrix :123-133) ----
 * Builds the rank-limited factor on the device and returns it: L (n x rank,
 * column-major, ldl), achieved rank, and the (calibrated) shift. */
wgp_status wgp_pivoted_cholesky(wgp_op* op, int64_t rank, double* L, int64_t ldl,
                                int64_t* achieved);
wgp_status wgp_precond_info(wgp_op* op, int64_t rank, double shift, int mode, int64_t* achieved,
                            double* shift_out);

/* ---- reusable preconditioner (CgPreconditioner, solvers.hpp:82-100) and cg_solve_with
 *      (solvers.hpp:118-119, solvers.cpp:142-183): one factorization shared by many solves,
 *      as bo_round does for its per-column solves (thompson.cpp:359-384).  The handle
 *      lives on the operator's device and is valid while the operator keeps the row count
 *      it was built at (after wgp_op_append_rows, using it returns WGP_INVALID_ARGUMENT). */
typedef struct wgp_precond wgp_precond;
/* CgPreconditioner::from_matrix (solvers.cpp:123-133): pivoted Cholesky of rank
 * min(rank, n) and the Woodbury factors; rank 0 = identity.  mode: wgp_shift_mode. */
wgp_status wgp_precond_create(wgp_op* op, int64_t rank, double shift, int mode, wgp_precond** out);
/* CgPreconditioner(L, shift) (solvers.cpp:109-121): from a host factor L (n x k column-major,
 * ldl), shift used as given (must be > 0 for k > 0; capacitance failure -> WGP_NOT_SPD). */
wgp_status wgp_precond_create_from_factor(wgp_op* op, const double* L, int64_t ldl, int64_t k,
                                          double shift, wgp_precond** out);
void wgp_precond_destroy(wgp_precond* pc);
/* achieved rank and (calibrated) shift of the handle */
wgp_status wgp_precond_get(const wgp_precond* pc, int64_t* rank, double* shift);
/* CgPreconditioner::apply (solvers.cpp:135-140) on host columns: Z = (L L^T + shift I)^{-1} R,
 * R and Z n x s column-major.  Unsharded. */
wgp_status wgp_precond_apply(wgp_precond* pc, const double* R, int64_t ldr, int s, double* Z,
                             int64_t ldz);
/* cg_solve_with: wgp_solve_many's CG (cfg->method is ignored, cfg->precond_* too) with the
 * caller's preconditioner -- no factorization inside.  Same arguments and outputs as
 * wgp_solve_many; a column solved alone gives bitwise the result it gets in a batch. */
wgp_status wgp_cg_solve_with(wgp_op* op, const wgp_precond* pc, const wgp_solver_config* cfg,
                             const double* B, int64_t ldb, int s, const double* U1, int64_t ldu,
                             int64_t n1, double* V, int64_t ldv, int32_t* iterations,
                             double* history, int64_t hist_stride, int32_t* history_len,
                             int32_t* converged);

/* ---- remaining free functions of the reference API ---- */
/* cross_kernel (kernel.cpp:74-89): K (m x n column-major, ldk) = k(X*, X_op), no noise
 * term, fp64 on the device (n <= 65535). */
wgp_status wgp_cross_kernel(wgp_op* op, const double* Xstar, int64_t m, int64_t ldx, double* K,
                            int64_t ldk);
/* relative_residual (solvers.cpp:62-66) per column: out[c] = |H v_c - b_c| / |b_c|; a zero
 * b_c returns WGP_INVALID_ARGUMENT.  V, B n x s column-major; the operator's precision. */
wgp_status wgp_relative_residual(wgp_op* op, const double* V, int64_t ldv, const double* B,
                                 int64_t ldb, int s, double* out);
/* quadratic_objective (solvers.cpp:68-70) per column: 0.5 v.Hv - v.b */
wgp_status wgp_quadratic_objective(wgp_op* op, const double* V, int64_t ldv, const double* B,
                                   int64_t ldb, int s, double* out);
/* init_weights (solvers.cpp:27-38): out (n1 + n2) = u1 == NULL ? 0 : [u1; 0]. */
wgp_status wgp_init_weights(const double* u1, int64_t n1, int64_t n2, double* out);
/* build_sample_rhs (sampling.cpp:56-64): out (n) = prior at the operator's rows (one prior:
 * Omega F x dim column-major, phases F, amps F) + noise_scale Rng(seed).normal() per row. */
wgp_status wgp_build_sample_rhs(wgp_op* op, const double* Omega, const double* phases,
                                const double* amps, int F, double signal_scale,
                                double noise_scale, uint64_t seed, double* out);

/* ---- random Fourier features (eval_prior sampling.cpp:37-46, batched over S
 *      priors; build_sample_rhs :56-64 adds host-drawn noise afterwards) ----
 * Omega: S priors x F x dim (prior-major, each F x dim column-major as RffPrior::
 * frequencies), phases/amps: S x F.  Xstar: m x dim column-major (ldx), or NULL
 * to evaluate at the operator's rows.  out: m x S column-major (ldo). */
wgp_status wgp_rff_eval(wgp_op* op, const double* Omega, const double* phases, const double* amps,
                        int F, int S, double signal_scale, const double* Xstar, int64_t m,
                        int64_t ldx, double* out, int64_t ldo);
/* Same contract in fp32 arithmetic (phases, MUFU cos after a Cody-Waite reduction, fp32
 * sums): ~1e-6 absolute on a unit-variance prior, ~25x faster.  For bulk evaluation at
 * candidate points (posterior sampling for acquisition); right-hand sides use wgp_rff_eval. */
wgp_status wgp_rff_eval_fast(wgp_op* op, const double* Omega, const double* phases,
                             const double* amps, int F, int S, double signal_scale,
                             const double* Xstar, int64_t m, int64_t ldx, double* out, int64_t ldo);

/* ---- host-side randomness (rng.hpp:11-61, bit-identical streams) ----
 * Draws that the reference makes on the host stay on the host: RFF frequencies,
 * observation noise, SGD batch indices.  `state` is warmgp::Rng's 64-bit state. */
uint64_t wgp_derive_seed(uint64_t seed, uint64_t stream);
uint64_t wgp_rng_next_u64(uint64_t* state);
double wgp_rng_uniform(uint64_t* state);
double wgp_rng_normal(uint64_t* state);
double wgp_rng_chi_square3(uint64_t* state);
uint64_t wgp_rng_uniform_index(uint64_t* state, uint64_t n);
/* n consecutive scale * normal() draws from (and advancing) the generator at *state. */
void wgp_rng_normal_fill(uint64_t* state, int64_t n, double scale, double* out);

/* select_peaks' argmax step (thompson.cpp:188-207) on the device: posterior values
 * prior_s(X*) + K(X*, X) W[:, s] (as wgp_rff_eval + wgp_cross_matvec; fast != 0: the fp32
 * RFF kernel and, on tensor-core operators, the tcgen05 cross mode) for S samples at m
 * candidates (X*: m x dim column-major), split into `groups` contiguous candidate groups
 * [m g / groups, m (g+1) / groups); idx[s * groups + g] = the first row of group g with the
 * largest value for sample s.  Only the S x groups indices leave the device. */
wgp_status wgp_posterior_select(wgp_op* op, const double* Omega, const double* phases,
                                const double* amps, int F, int S, double signal_scale,
                                const double* W, int64_t ldw, const double* Xstar, int64_t m,
                                int64_t ldx, int groups, int fast, int64_t* idx);

/* exact_solve (analysis.cpp:15-26): X = H^{-1} B by a dense fp64 Cholesky of the operator's
 * H on the device (materialised once; n <= 60000).  B, X: n x s column-major.  A
 * non-positive pivot returns WGP_NOT_SPD (the reference's LLT failure).  Unsharded only. */
wgp_status wgp_exact_solve(wgp_op* op, const double* B, int64_t ldb, int s, double* X, int64_t ldx);

/* mll (analysis.cpp:99-139): marginal log-likelihood of y (n) under the operator's rows and
 * kernel, at hyperparameters hyp3 = {lengthscale, signal_scale, noise_scale} (nullable: the
 * operator's own), and its gradient with respect to (log l, log s_f, log sigma_n).  Dense
 * fp64 on the device (H factored, [alpha | H^{-1}] by blocked substitution; n <= 30000).
 * Matern-3/2 as the reference; the RBF analogue for RBF operators.  Not SPD -> WGP_NOT_SPD.
 * Unsharded only. */
wgp_status wgp_mll(wgp_op* op, const double* y, const double* hyp3, double* value, double* grad3);
/* optimize_mll (analysis.cpp:141-182): Adam (0.9 / 0.999 / 1e-8) on the log-parameters from
 * init3 (nullable: the operator's), clamped to [1e-3, 1e3] x [1e-3, 1e3] x [1e-4, 1e2],
 * `steps` steps of `step_size`; out3 = the best hyperparameters seen.  A non-finite MLL
 * returns WGP_RUNTIME_ERROR.  The operator itself is not modified. */
wgp_status wgp_optimize_mll(wgp_op* op, const double* y, const double* init3, int steps,
                            double step_size, double* out3);
/* median_heuristic_lengthscale (analysis.cpp:184-203): median pairwise distance of 256 rows
 * drawn with Rng(derive_seed(seed, 0x6d656469)).uniform_index(n); X: n x dim column-major
 * (leading dimension ldx).  Host computation (256 x 256 distances). */
double wgp_median_heuristic_lengthscale(const double* X, int64_t n, int64_t ldx, int dim,
                                        uint64_t seed);

/* grad_posterior (sampling.cpp:77-87): gradients at m points of the posterior samples
 * prior_s + K(., X) W[:, s] (the operator's rows as training inputs; priors as in
 * wgp_rff_eval, W: n x S column-major).  Point i belongs to sample sidx[i]; Xs, G: m x dim
 * column-major.  Matern-3/2 as in the reference; RBF analogue for RBF operators.  fp64. */
wgp_status wgp_grad_posterior(wgp_op* op, const double* Omega, const double* phases,
                              const double* amps, int F, int S, double signal_scale,
                              const double* W, int64_t ldw, const double* Xs, int64_t ldx,
                              const int32_t* sidx, int64_t m, double* G, int64_t ldg);
/* ascend_peaks (thompson.cpp:209-258) for S samples at once: Adam ascent (beta 0.9/0.999,
 * eps 1e-8, clamp to [0,1]^dim, freeze on a non-finite gradient) from P starts per sample
 * (starts: S*P x dim column-major, row s*P + t), best point/value per sample over all its
 * trajectories (strict >, earlier start and step win ties).  best_x: S x dim column-major. */
wgp_status wgp_ascend_peaks(wgp_op* op, const double* Omega, const double* phases,
                            const double* amps, int F, int S, double signal_scale, const double* W,
                            int64_t ldw, const double* starts, int P, int steps, double rate,
                            double* best_x, double* best_val);

/* ---- measurement: CUDA-event timing of the tensor-core kernel-matvec launches only (the
 *      prep kernels around it excluded), for roofline reporting.  enable != 0 starts
 *      recording (and clears); read synchronizes the recorded events and returns the summed
 *      kernel time and launch count since the last enable. ---- */
void wgp_kernel_timer_enable(int enable);
wgp_status wgp_kernel_timer_read(double* total_ms, int64_t* launches);
/* Same for one tagged kernel family: "kmatvec_tc", "kmatvec_f64", "kmatvec_f32", "krows"
 * (SGD minibatch rows), "kcols" (AP block columns), "rff_eval" (fp64), "rff_eval32". */
wgp_status wgp_kernel_timer_read_tag(const char* tag, double* total_ms, int64_t* launches);
/* out[i] = scale * Rng(seed).normal(), i = 0..n-1 (build_sample_rhs noise, sampling.cpp:58-62) */
void wgp_normal_fill(uint64_t seed, int64_t n, double scale, double* out);
/* sample_prior (sampling.cpp:14-35): Omega F x dim column-major, phases F, amps F.
 * Matern-3/2 rows are Student-t(3)/l (reference); RBF rows N(0, l^-2 I) (extension). */
wgp_status wgp_sample_prior(int kernel, double lengthscale, int64_t dim, int64_t F, uint64_t seed,
                            double* Omega, double* phases, double* amps);

#ifdef __cplusplus
}
#endif
#endif
