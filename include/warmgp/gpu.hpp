// warmgp/gpu.hpp -- header-only C++ mirror of the reference warmgp API
// (/root/reference/proj/core/include/warmgp/{kernel,solvers,sampling}.hpp) over the C-ABI
// of libwarmgp_b200.so (include/warmgp_capi.h).
//
// Same type and function names, same argument meaning, same exception types
// (types.hpp:15-32).  The only change a caller sees is that the covariance is a
// device-resident KernelOperator instead of a dense Eigen::MatrixXd (which cannot
// exist at N >= 100k): gram_matrix(X, hyp) -> KernelOperator(X, hyp), extend_system ->
// op.append_rows(X2).  Matrices are column-major doubles like Eigen::MatrixXd; with
// WARMGP_GPU_EIGEN defined, Eigen overloads (to_gpu/to_eigen, gram_matrix, append_rows,
// warm, solve, solve_many, H * V) are provided for drop-in use in the reference build
// (exercised by tests/cpp/test_eigen_overloads.cpp against a shim, since
// Eigen3 is not installed in this image).
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../warmgp_capi.h"

#ifdef WARMGP_GPU_EIGEN
#include <Eigen/Dense>
#endif

namespace warmgp {
namespace gpu {

// ---------------------------------------------------------------- errors (types.hpp:15-26)
class NotSpdError : public std::runtime_error {
 public:
  explicit NotSpdError(const std::string& w) : std::runtime_error(w) {}
};
class DivergenceError : public std::runtime_error {
 public:
  DivergenceError(const std::string& w, int it) : std::runtime_error(w), iterations(it) {}
  int iterations;
};
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(wgp_status st, int iterations = 0) {
  if (st == WGP_OK) return;
  const std::string msg = wgp_last_error();
  switch (st) {
    case WGP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case WGP_NOT_SPD: throw NotSpdError(msg);
    case WGP_DIVERGED: throw DivergenceError(msg, iterations);
    case WGP_OOM: throw std::bad_alloc();
    case WGP_RUNTIME_ERROR: throw std::runtime_error(msg);
    default: throw CudaError(msg);
  }
}

// ---------------------------------------------------------------- value types
struct Matrix {  // column-major, like Eigen::MatrixXd
  int64_t rows = 0, cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(int64_t r, int64_t c) : rows(r), cols(c), data((size_t)(r * c), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return data[(size_t)(j * rows + i)]; }
  double operator()(int64_t i, int64_t j) const { return data[(size_t)(j * rows + i)]; }
  const double* col(int64_t j) const { return data.data() + j * rows; }
};
using Vector = std::vector<double>;

enum class Method { CG = WGP_CG, SGD = WGP_SGD, AP = WGP_AP };            // solvers.hpp:10
enum class SgdScaling { Unbiased = WGP_SGD_UNBIASED, Block = WGP_SGD_BLOCK };
enum class ApOrdering { Greedy = WGP_AP_GREEDY, Cyclic = WGP_AP_CYCLIC };
enum class Kernel { Matern32 = WGP_MATERN32, RBF = WGP_RBF };
enum class Precision { F64 = WGP_F64, F32_3xTF32 = WGP_F32_3XTF32, TF32 = WGP_TF32, F32 = WGP_F32_SIMT };

struct KernelHyperparams {  // kernel.hpp:8-14
  double lengthscale = 1.0;
  double signal_scale = 1.0;
  double noise_scale = 1e-3;
  Kernel kind = Kernel::Matern32;
};

struct SolverConfig {  // solvers.hpp:27-48, same defaults
  enum class PrecondShiftMode { Calibrated = WGP_SHIFT_CALIBRATED, NoiseOnly = WGP_SHIFT_NOISE_ONLY };
  Method method = Method::CG;
  double tolerance = 1e-2;
  int max_iters = 1000;
  double learning_rate = 0.3;
  double momentum = 0.9;
  int64_t batch_size = 100;
  SgdScaling sgd_scaling = SgdScaling::Unbiased;
  int64_t block_size = 100;
  ApOrdering ap_ordering = ApOrdering::Greedy;
  int64_t precond_rank = 100;
  double precond_shift = 1e-6;
  PrecondShiftMode precond_shift_mode = PrecondShiftMode::Calibrated;
  std::uint64_t seed = 0;

  wgp_solver_config c() const {
    wgp_solver_config r;
    r.method = (int32_t)method;
    r.tolerance = tolerance;
    r.max_iters = max_iters;
    r.learning_rate = learning_rate;
    r.momentum = momentum;
    r.batch_size = batch_size;
    r.sgd_scaling = (int32_t)sgd_scaling;
    r.block_size = block_size;
    r.ap_ordering = (int32_t)ap_ordering;
    r.precond_rank = precond_rank;
    r.precond_shift = precond_shift;
    r.precond_shift_mode = (int32_t)precond_shift_mode;
    r.seed = seed;
    return r;
  }
};

struct Initialization {  // solvers.hpp:52-63
  static Initialization cold() { return Initialization{}; }
  static Initialization warm(Vector u1_prev) {
    Initialization i;
    i.warm_start = true;
    i.u1 = std::move(u1_prev);
    return i;
  }
  bool warm_start = false;
  Vector u1;
};

struct SolveResult {  // solvers.hpp:102-109
  Vector v;
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  double final_residual() const { return residual_history.back(); }
};

// ---------------------------------------------------------------- device handles
class Context {
 public:
  explicit Context(int device = 0) { check(wgp_ctx_create(device, &h_)); }
  Context(int device, int rank, int world, const void* nccl_uid128) {
    check(wgp_ctx_create_sharded(device, rank, world, nccl_uid128, &h_));
  }
  // rank of a loopback group (ranks = threads of one process on one device; testing)
  Context(int device, int rank, void* loopback_group) {
    check(wgp_ctx_create_loopback(device, rank, loopback_group, &h_));
  }
  ~Context() { wgp_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  wgp_ctx* get() const { return h_; }

 private:
  wgp_ctx* h_ = nullptr;
};

// H = K(X, X) + sigma_n^2 I, device resident (replaces CovarianceMatrix, kernel.hpp:25-31).
class KernelOperator {
 public:
  KernelOperator(Context& ctx, const Matrix& X, const KernelHyperparams& hyp,
                 Precision precision = Precision::F64) {
    check(wgp_op_create(ctx.get(), (int)hyp.kind, hyp.lengthscale, hyp.signal_scale,
                        hyp.noise_scale, (int)precision, (int)X.cols, &h_));
    if (X.rows > 0) append_rows(X);
  }
  ~KernelOperator() { wgp_op_destroy(h_); }
  KernelOperator(const KernelOperator&) = delete;
  KernelOperator& operator=(const KernelOperator&) = delete;

  // extend_system's growth step (kernel.cpp:108-130): old rows are never re-uploaded
  void append_rows(const Matrix& X2) {
    check(wgp_op_append_rows(h_, X2.data.data(), X2.rows, X2.rows > 0 ? X2.rows : 1, 1));
  }
  int64_t size() const { return wgp_op_size(h_); }
  int64_t rows() const { return size(); }  // Eigen-style, as H.rows() in the reference
  // CG true-residual mode (wgp_residual_mode): ANCHORED removes the fp32 residual floor
  void set_residual_mode(wgp_residual_mode m) { check(wgp_op_set_residual_mode(h_, (int)m)); }
  Matrix operator*(const Matrix& V) const {  // H * V  (solvers.cpp:162)
    Matrix Y(V.rows, V.cols);
    check(wgp_kmatvec(h_, V.data.data(), V.rows, (int)V.cols, Y.data.data(), Y.rows));
    return Y;
  }
  wgp_op* get() const { return h_; }

 private:
  wgp_op* h_ = nullptr;
};

inline KernelOperator gram_matrix(Context& ctx, const Matrix& X, const KernelHyperparams& hyp,
                                  Precision p = Precision::F64) {  // kernel.cpp:48
  if (X.rows < 1) throw std::invalid_argument("gram_matrix: need at least one row");
  return KernelOperator(ctx, X, hyp, p);
}

// ---------------------------------------------------------------- solvers (solvers.hpp:111-141)
inline std::vector<SolveResult> solve_many(const KernelOperator& H, const Matrix& rhs_columns,
                                           const std::vector<Initialization>& inits,
                                           const SolverConfig& cfg) {
  const int64_t n = rhs_columns.rows;
  const int s = (int)rhs_columns.cols;
  if ((int64_t)inits.size() != s)
    throw std::invalid_argument("solve_many: one initialization per right-hand side required");
  if (n != H.size()) throw std::invalid_argument("solve_many: rhs rows != operator size");
  int64_t n1 = 0;
  bool warm = false;
  for (const auto& i : inits)
    if (i.warm_start) {
      warm = true;
      n1 = (int64_t)i.u1.size();
    }
  std::vector<double> U1;
  if (warm) {
    U1.assign((size_t)(n1 * s), 0.0);
    for (int c = 0; c < s; ++c)
      if (inits[c].warm_start) {
        if ((int64_t)inits[c].u1.size() != n1)
          throw std::invalid_argument("solve_many: warm starts must share one length");
        std::copy(inits[c].u1.begin(), inits[c].u1.end(), U1.begin() + c * n1);
      }
  }
  const wgp_solver_config c = cfg.c();
  const int64_t hs = (int64_t)cfg.max_iters + 1;
  std::vector<double> V((size_t)(n * s)), hist((size_t)(hs * s));
  std::vector<int32_t> its(s), hl(s), cv(s), cst(s), dv(s);
  const wgp_status st = wgp_solve_many(H.get(), &c, rhs_columns.data.data(), n, s,
                                       warm ? U1.data() : nullptr, n1 > 0 ? n1 : 1, n1, V.data(), n,
                                       its.data(), hist.data(), hs, hl.data(), cv.data(),
                                       cst.data(), dv.data());
  int fail_iters = 0;
  for (int k = 0; k < s; ++k)
    if (cst[k] != WGP_OK) {
      fail_iters = dv[k];
      break;
    }
  check(st, fail_iters);
  std::vector<SolveResult> out(s);
  for (int k = 0; k < s; ++k) {
    out[k].v.assign(V.begin() + k * n, V.begin() + (k + 1) * n);
    out[k].iterations = its[k];
    out[k].residual_history.assign(hist.begin() + k * hs, hist.begin() + k * hs + hl[k]);
    out[k].converged = cv[k] != 0;
  }
  return out;
}

inline SolveResult solve(const KernelOperator& H, const Vector& b, const Initialization& init,
                         const SolverConfig& cfg) {  // solvers.cpp:311-319
  const int64_t n = (int64_t)b.size();
  if (n != H.size()) throw std::invalid_argument("solve: rhs length != operator size");
  SolveResult r;
  r.v.assign((size_t)n, 0.0);
  std::vector<double> hist((size_t)cfg.max_iters + 1);
  int32_t its = 0, hl = 0, cv = 0, dv = 0;
  const wgp_solver_config c = cfg.c();
  check(wgp_solve(H.get(), &c, b.data(), init.warm_start ? init.u1.data() : nullptr,
                  init.warm_start ? (int64_t)init.u1.size() : 0, r.v.data(), &its, hist.data(), &hl,
                  &cv, &dv),
        dv);
  r.iterations = its;
  r.residual_history.assign(hist.begin(), hist.begin() + hl);
  r.converged = cv != 0;
  return r;
}

inline SolveResult cg_solve(const KernelOperator& H, const Vector& b, const Initialization& i,
                            SolverConfig cfg) {
  cfg.method = Method::CG;
  return solve(H, b, i, cfg);
}
inline SolveResult sgd_solve(const KernelOperator& H, const Vector& b, const Initialization& i,
                             SolverConfig cfg) {
  cfg.method = Method::SGD;
  return solve(H, b, i, cfg);
}
inline SolveResult ap_solve(const KernelOperator& H, const Vector& b, const Initialization& i,
                            SolverConfig cfg) {
  cfg.method = Method::AP;
  return solve(H, b, i, cfg);
}

// init_weights (solvers.cpp:27-38): cold -> 0, warm -> [u1; 0]
inline Vector init_weights(const Initialization& init, int64_t n1, int64_t n2) {
  if (init.warm_start && (int64_t)init.u1.size() != n1)
    throw std::invalid_argument("init_weights: warm-start vector length does not match n1");
  Vector v((size_t)std::max<int64_t>(n1 + n2, 0));
  check(wgp_init_weights(init.warm_start ? init.u1.data() : nullptr, n1, n2, v.data()));
  return v;
}

// relative_residual (solvers.cpp:62-66): |H v - b| / |b|; zero b -> std::invalid_argument
inline double relative_residual(const KernelOperator& H, const Vector& v, const Vector& b) {
  if ((int64_t)v.size() != H.size() || (int64_t)b.size() != H.size())
    throw std::invalid_argument("relative_residual: length mismatch");
  double out = 0.0;
  check(wgp_relative_residual(H.get(), v.data(), (int64_t)v.size(), b.data(), (int64_t)b.size(), 1, &out));
  return out;
}

// quadratic_objective (solvers.cpp:68-70): 0.5 v.Hv - v.b
inline double quadratic_objective(const KernelOperator& H, const Vector& v, const Vector& b) {
  if ((int64_t)v.size() != H.size() || (int64_t)b.size() != H.size())
    throw std::invalid_argument("quadratic_objective: length mismatch");
  double out = 0.0;
  check(wgp_quadratic_objective(H.get(), v.data(), (int64_t)v.size(), b.data(), (int64_t)b.size(), 1, &out));
  return out;
}

// pivoted_cholesky (solvers.cpp:72-107): n x r factor (r <= rank), computed on the device
inline Matrix pivoted_cholesky(const KernelOperator& H, int64_t rank) {
  const int64_t n = H.size();
  Matrix L(n, std::max<int64_t>(rank, 0));
  int64_t achieved = 0;
  check(wgp_pivoted_cholesky(H.get(), rank, rank > 0 ? L.data.data() : nullptr, n > 0 ? n : 1, &achieved));
  L.cols = achieved;
  L.data.resize((size_t)(n * achieved));
  return L;
}

// CgPreconditioner (solvers.hpp:82-100) as a device handle over the operator it was built for.
class CgPreconditioner {
 public:
  CgPreconditioner() = default;  // identity (no handle): cg_solve_with builds a rank-0 one
  static CgPreconditioner from_matrix(const KernelOperator& H, int64_t rank, double shift,
                                      SolverConfig::PrecondShiftMode mode =
                                          SolverConfig::PrecondShiftMode::Calibrated) {
    CgPreconditioner p;
    check(wgp_precond_create(H.get(), rank, shift, (int)mode, &p.h_));
    return p;
  }
  // CgPreconditioner(L, shift) (solvers.cpp:109-121) with L a host factor of the operator's rows
  CgPreconditioner(const KernelOperator& H, const Matrix& L, double shift) {
    check(wgp_precond_create_from_factor(H.get(), L.data.data(), L.rows > 0 ? L.rows : 1, L.cols,
                                         shift, &h_));
  }
  CgPreconditioner(CgPreconditioner&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  CgPreconditioner& operator=(CgPreconditioner&& o) noexcept {
    if (this != &o) {
      wgp_precond_destroy(h_);
      h_ = o.h_;
      o.h_ = nullptr;
    }
    return *this;
  }
  CgPreconditioner(const CgPreconditioner&) = delete;
  CgPreconditioner& operator=(const CgPreconditioner&) = delete;
  ~CgPreconditioner() { wgp_precond_destroy(h_); }

  bool is_identity() const { return rank() == 0; }
  int64_t rank() const {
    if (!h_) return 0;
    int64_t k = 0;
    double sh = 0.0;
    check(wgp_precond_get(h_, &k, &sh));
    return k;
  }
  double shift() const {
    int64_t k = 0;
    double sh = 1.0;
    if (h_) check(wgp_precond_get(h_, &k, &sh));
    return sh;
  }
  Vector apply(const Vector& r) const {  // solvers.cpp:135-140
    if (!h_) return r;
    Vector z(r.size());
    check(wgp_precond_apply(h_, r.data(), (int64_t)r.size(), 1, z.data(), (int64_t)z.size()));
    return z;
  }
  wgp_precond* get() const { return h_; }

 private:
  wgp_precond* h_ = nullptr;
};

// cg_solve_with (solvers.hpp:118-119): CG with an externally built preconditioner (no
// factorization inside); the bo_round pattern calls it per column with one handle.
inline SolveResult cg_solve_with(const KernelOperator& H, const Vector& b, const Initialization& init,
                                 const SolverConfig& cfg, const CgPreconditioner& precond) {
  const int64_t n = (int64_t)b.size();
  if (n != H.size()) throw std::invalid_argument("cg_solve_with: rhs length != operator size");
  CgPreconditioner identity;
  const wgp_precond* pc = precond.get();
  if (!pc) {  // default-constructed identity preconditioner
    identity = CgPreconditioner::from_matrix(H, 0, 1.0);
    pc = identity.get();
  }
  wgp_solver_config c = cfg.c();
  const int64_t hs = (int64_t)cfg.max_iters + 1;
  SolveResult r;
  r.v.assign((size_t)n, 0.0);
  std::vector<double> hist((size_t)hs);
  int32_t its = 0, hl = 0, cv = 0;
  const int64_t n1 = init.warm_start ? (int64_t)init.u1.size() : 0;
  check(wgp_cg_solve_with(H.get(), pc, &c, b.data(), n, 1, init.warm_start ? init.u1.data() : nullptr,
                          n1 > 0 ? n1 : 1, n1, r.v.data(), n, &its, hist.data(), hs, &hl, &cv));
  r.iterations = its;
  r.residual_history.assign(hist.begin(), hist.begin() + hl);
  r.converged = cv != 0;
  return r;
}

// ---------------------------------------------------------------- sampling (sampling.hpp)
struct RffPrior {
  Matrix frequencies;  // F x D
  Vector phases, amplitudes;
  double signal_scale = 1.0;
};

inline RffPrior sample_prior(const KernelHyperparams& hyp, int64_t dim, int64_t F,
                             std::uint64_t seed) {  // sampling.cpp:14-35
  RffPrior p;
  p.frequencies = Matrix(F, dim);
  p.phases.assign((size_t)F, 0.0);
  p.amplitudes.assign((size_t)F, 0.0);
  p.signal_scale = hyp.signal_scale;
  check(wgp_sample_prior((int)hyp.kind, hyp.lengthscale, dim, F, seed, p.frequencies.data.data(),
                         p.phases.data(), p.amplitudes.data()));
  return p;
}

// eval_prior (sampling.cpp:37-46) at the operator's rows for several priors: m x S.
inline Matrix eval_priors(const KernelOperator& H, const std::vector<RffPrior>& priors) {
  const int S = (int)priors.size();
  const int64_t m = H.size();
  Matrix out(m, S);
  if (!S) return out;
  const int64_t F = priors[0].frequencies.rows, D = priors[0].frequencies.cols;
  std::vector<double> Om((size_t)(S * F * D)), ph((size_t)(S * F)), am((size_t)(S * F));
  for (int p = 0; p < S; ++p) {
    std::copy(priors[p].frequencies.data.begin(), priors[p].frequencies.data.end(), Om.begin() + p * F * D);
    std::copy(priors[p].phases.begin(), priors[p].phases.end(), ph.begin() + p * F);
    std::copy(priors[p].amplitudes.begin(), priors[p].amplitudes.end(), am.begin() + p * F);
  }
  check(wgp_rff_eval(H.get(), Om.data(), ph.data(), am.data(), (int)F, S, priors[0].signal_scale,
                     nullptr, m, m, out.data.data(), m));
  return out;
}

// eval_prior (sampling.cpp:37-46) of one prior at the rows of X* (m x D)
inline Vector eval_prior(const KernelOperator& H, const RffPrior& prior, const Matrix& Xstar) {
  const int64_t m = Xstar.rows, F = prior.frequencies.rows;
  Vector out((size_t)m);
  if (!m) return out;
  check(wgp_rff_eval(H.get(), prior.frequencies.data.data(), prior.phases.data(), prior.amplitudes.data(),
                     (int)F, 1, prior.signal_scale, Xstar.data.data(), m, m, out.data(), m));
  return out;
}

// build_sample_rhs (sampling.cpp:56-64) at the operator's rows
inline Vector build_sample_rhs(const KernelOperator& H, const RffPrior& prior, double noise_scale,
                               std::uint64_t seed) {
  Vector out((size_t)H.size());
  check(wgp_build_sample_rhs(H.get(), prior.frequencies.data.data(), prior.phases.data(),
                             prior.amplitudes.data(), (int)prior.frequencies.rows, prior.signal_scale,
                             noise_scale, seed, out.data()));
  return out;
}

// cross_kernel (kernel.cpp:74-89): dense K(X*, X_op), no noise term
inline Matrix cross_kernel(const KernelOperator& H, const Matrix& Xstar) {
  Matrix K(Xstar.rows, H.size());
  check(wgp_cross_kernel(H.get(), Xstar.data.data(), Xstar.rows, Xstar.rows > 0 ? Xstar.rows : 1,
                         K.data.data(), Xstar.rows > 0 ? Xstar.rows : 1));
  return K;
}

// eval_posterior (sampling.cpp:66-75) for S samples at m points at once:
// out(:, s) = prior_s(X*) + K(X*, X) weights(:, s), weights n x S (pathwise samples).
// Reference form: one PosteriorSample per call; here the training rows are the operator's.
inline Matrix eval_posterior(const KernelOperator& H, const std::vector<RffPrior>& priors,
                             const Matrix& weights, const Matrix& Xstar) {
  const int S = (int)priors.size();
  const int64_t m = Xstar.rows;
  if (weights.rows != H.size() || weights.cols != S)
    throw std::invalid_argument("eval_posterior: weights length != training rows");
  Matrix out(m, S);
  if (!S || !m) return out;
  const int64_t F = priors[0].frequencies.rows, D = priors[0].frequencies.cols;
  std::vector<double> Om((size_t)(S * F * D)), ph((size_t)(S * F)), am((size_t)(S * F));
  for (int p = 0; p < S; ++p) {
    std::copy(priors[p].frequencies.data.begin(), priors[p].frequencies.data.end(), Om.begin() + p * F * D);
    std::copy(priors[p].phases.begin(), priors[p].phases.end(), ph.begin() + p * F);
    std::copy(priors[p].amplitudes.begin(), priors[p].amplitudes.end(), am.begin() + p * F);
  }
  check(wgp_rff_eval(H.get(), Om.data(), ph.data(), am.data(), (int)F, S, priors[0].signal_scale,
                     Xstar.data.data(), m, m, out.data.data(), m));
  if (H.size() > 0) {
    Matrix kw(m, S);
    check(wgp_cross_matvec(H.get(), Xstar.data.data(), m, m, weights.data.data(), weights.rows, S,
                           kw.data.data(), m));
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] += kw.data[i];
  }
  return out;
}

// ascend_peaks (thompson.cpp:209-258) for S posterior samples (priors[s], weights column s)
// at once: starts holds S*P rows (sample-major) of dim columns; returns S best points and
// values.  grad_posterior (sampling.cpp:77-87) is wgp_grad_posterior.
struct AscendResult {  // thompson.hpp AscendResult
  Matrix points;
  Vector values;
};
inline AscendResult ascend_peaks(const KernelOperator& H, const std::vector<RffPrior>& priors,
                                 const Matrix& weights, const Matrix& starts, int steps, double rate) {
  const int S = (int)priors.size();
  if (S == 0 || starts.rows % S != 0 || weights.rows != H.size() || weights.cols != S)
    throw std::invalid_argument("ascend_peaks: one peak set per posterior sample required");
  const int64_t F = priors[0].frequencies.rows, D = priors[0].frequencies.cols;
  std::vector<double> Om((size_t)(S * F * D)), ph((size_t)(S * F)), am((size_t)(S * F));
  for (int p = 0; p < S; ++p) {
    std::copy(priors[p].frequencies.data.begin(), priors[p].frequencies.data.end(), Om.begin() + p * F * D);
    std::copy(priors[p].phases.begin(), priors[p].phases.end(), ph.begin() + p * F);
    std::copy(priors[p].amplitudes.begin(), priors[p].amplitudes.end(), am.begin() + p * F);
  }
  AscendResult r;
  r.points = Matrix(S, D);
  r.values.assign((size_t)S, 0.0);
  check(wgp_ascend_peaks(H.get(), Om.data(), ph.data(), am.data(), (int)F, S, priors[0].signal_scale,
                         weights.data.data(), weights.rows, starts.data.data(), (int)(starts.rows / S),
                         steps, rate, r.points.data.data(), r.values.data()));
  return r;
}

// ---------------------------------------------------------------- analysis (analysis.hpp)
// exact_solve (analysis.cpp:15-26): dense fp64 Cholesky of the operator's H on the device.
inline Vector exact_solve(const KernelOperator& H, const Vector& b) {
  if ((int64_t)b.size() != H.size()) throw std::invalid_argument("exact_solve: length mismatch");
  Vector x(b.size());
  check(wgp_exact_solve(H.get(), b.data(), (int64_t)b.size(), 1, x.data(), (int64_t)x.size()));
  return x;
}

struct MllResult {  // analysis.hpp:42-45
  double value = 0.0;
  double grad[3] = {0.0, 0.0, 0.0};  // d/d(log l, log s_f, log sigma_n)
};
// mll (analysis.cpp:99-139) of y under the operator's rows at hyp (the operator's own kind).
inline MllResult mll(const KernelOperator& H, const Vector& y, const KernelHyperparams& hyp) {
  if ((int64_t)y.size() != H.size()) throw std::invalid_argument("mll: X rows != y length");
  const double h3[3] = {hyp.lengthscale, hyp.signal_scale, hyp.noise_scale};
  MllResult r;
  check(wgp_mll(H.get(), y.data(), h3, &r.value, r.grad));
  return r;
}
// optimize_mll (analysis.cpp:141-182): best hyperparameters seen by the Adam ascent.
inline KernelHyperparams optimize_mll(const KernelOperator& H, const Vector& y,
                                      const KernelHyperparams& init, int steps, double step_size) {
  if ((int64_t)y.size() != H.size()) throw std::invalid_argument("mll: X rows != y length");
  const double h3[3] = {init.lengthscale, init.signal_scale, init.noise_scale};
  double out[3];
  check(wgp_optimize_mll(H.get(), y.data(), h3, steps, step_size, out));
  KernelHyperparams r = init;
  r.lengthscale = out[0];
  r.signal_scale = out[1];
  r.noise_scale = out[2];
  return r;
}
// median_heuristic_lengthscale (analysis.cpp:184-203)
inline double median_heuristic_lengthscale(const Matrix& X, uint64_t seed = 0) {
  return wgp_median_heuristic_lengthscale(X.data.data(), X.rows, X.rows > 0 ? X.rows : 1, (int)X.cols,
                                          seed);
}

#ifdef WARMGP_GPU_EIGEN
// ---------------------------------------------------------------- Eigen overloads
// For the reference build (Eigen::MatrixXd is column-major fp64, like Matrix): the call
// sites of INTEGRATION.md keep their Eigen values and gain the device operator.
inline Matrix to_gpu(const Eigen::MatrixXd& A) {
  Matrix M(A.rows(), A.cols());
  std::copy(A.data(), A.data() + A.size(), M.data.begin());
  return M;
}
inline Vector to_gpu(const Eigen::VectorXd& v) { return Vector(v.data(), v.data() + v.size()); }
inline Eigen::MatrixXd to_eigen(const Matrix& M) {
  Eigen::MatrixXd A(M.rows, M.cols);
  std::copy(M.data.begin(), M.data.end(), A.data());
  return A;
}
inline Eigen::VectorXd to_eigen(const Vector& v) {
  Eigen::VectorXd e((Eigen::Index)v.size());
  std::copy(v.begin(), v.end(), e.data());
  return e;
}
inline KernelOperator gram_matrix(Context& ctx, const Eigen::MatrixXd& X, const KernelHyperparams& hyp,
                                  Precision p = Precision::F64) {
  return gram_matrix(ctx, to_gpu(X), hyp, p);
}
inline void append_rows(KernelOperator& H, const Eigen::MatrixXd& X2) { H.append_rows(to_gpu(X2)); }
inline Initialization warm(const Eigen::VectorXd& u1) { return Initialization::warm(to_gpu(u1)); }
inline std::vector<SolveResult> solve_many(const KernelOperator& H, const Eigen::MatrixXd& rhs,
                                           const std::vector<Initialization>& inits,
                                           const SolverConfig& cfg) {
  return solve_many(H, to_gpu(rhs), inits, cfg);
}
inline SolveResult solve(const KernelOperator& H, const Eigen::VectorXd& b, const Initialization& init,
                         const SolverConfig& cfg) {
  return solve(H, to_gpu(b), init, cfg);
}
inline Eigen::MatrixXd operator*(const KernelOperator& H, const Eigen::MatrixXd& V) {
  return to_eigen(H * to_gpu(V));
}
// analysis.hpp signatures: mll(X, y, hyp) / optimize_mll(X, y, init, steps, step) on a
// temporary fp64 device operator over X
inline MllResult mll(Context& ctx, const Eigen::MatrixXd& X, const Eigen::VectorXd& y,
                     const KernelHyperparams& hyp) {
  KernelOperator H(ctx, to_gpu(X), hyp, Precision::F64);
  return mll(H, to_gpu(y), hyp);
}
inline KernelHyperparams optimize_mll(Context& ctx, const Eigen::MatrixXd& X, const Eigen::VectorXd& y,
                                      const KernelHyperparams& init, int steps, double step_size) {
  KernelOperator H(ctx, to_gpu(X), init, Precision::F64);
  return optimize_mll(H, to_gpu(y), init, steps, step_size);
}
inline Eigen::VectorXd exact_solve(const KernelOperator& H, const Eigen::VectorXd& b) {
  return to_eigen(exact_solve(H, to_gpu(b)));
}
inline double median_heuristic_lengthscale(const Eigen::MatrixXd& X, uint64_t seed = 0) {
  return median_heuristic_lengthscale(to_gpu(X), seed);
}
#endif  // WARMGP_GPU_EIGEN

}  // namespace gpu
}  // namespace warmgp
