// C-ABI driver around the reference's OWN kernel.cpp / solvers.cpp / sampling.cpp, compiled
// unchanged from /root/reference (oracle/Makefile `ref`) against the eager Eigen stand-in in
// oracle/eigen_shim.  Test infrastructure only: tests/golden/make_ref_golden.py calls it in
// this container (where the reference tree is mounted) to freeze reference-produced outputs
// into tests/golden/ref_golden.json; nothing in the product, the GPU tests or bench.py loads
// it.  Matrices cross the boundary column-major (Eigen's layout).
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "warmgp/kernel.hpp"
#include "warmgp/sampling.hpp"
#include "warmgp/solvers.hpp"

using warmgp::Index;
using warmgp::Matrix;
using warmgp::Vector;

extern "C" {

struct RefCfg {
  int method;  // 0 CG, 1 SGD, 2 AP
  double tolerance;
  int max_iters;
  double learning_rate;
  double momentum;
  int64_t batch_size;
  int sgd_scaling;  // 0 Unbiased, 1 Block
  int64_t block_size;
  int ap_ordering;  // 0 Greedy, 1 Cyclic
  int64_t precond_rank;
  double precond_shift;
  int precond_shift_mode;  // 0 Calibrated, 1 NoiseOnly
  uint64_t seed;
};

struct RefResult {  // one solve; history written into the caller's buffer
  int status;       // 0 ok, 1 NotSpdError, 2 DivergenceError, 3 invalid_argument, 4 other
  int iterations;   // DivergenceError: the iteration count it carries
  int converged;
  int64_t hist_len;
};
}

namespace {

Matrix mat(const double* p, int64_t r, int64_t c) {
  Matrix m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * r * c);
  return m;
}
Vector vec(const double* p, int64_t n) { return mat(p, n, 1); }
void put(const Matrix& m, double* out) { std::memcpy(out, m.data(), sizeof(double) * m.size()); }

warmgp::KernelHyperparams hyp(double ls, double sf, double sn) {
  warmgp::KernelHyperparams h;
  h.lengthscale = ls;
  h.signal_scale = sf;
  h.noise_scale = sn;
  return h;
}

warmgp::SolverConfig cfg_of(const RefCfg& c) {
  warmgp::SolverConfig s;
  s.method = static_cast<warmgp::Method>(c.method);
  s.tolerance = c.tolerance;
  s.max_iters = c.max_iters;
  s.learning_rate = c.learning_rate;
  s.momentum = c.momentum;
  s.batch_size = c.batch_size;
  s.sgd_scaling = static_cast<warmgp::SgdScaling>(c.sgd_scaling);
  s.block_size = c.block_size;
  s.ap_ordering = static_cast<warmgp::ApOrdering>(c.ap_ordering);
  s.precond_rank = c.precond_rank;
  s.precond_shift = c.precond_shift;
  s.precond_shift_mode = static_cast<warmgp::SolverConfig::PrecondShiftMode>(c.precond_shift_mode);
  s.seed = c.seed;
  return s;
}

warmgp::Initialization init_of(const double* u1, int64_t n1) {
  return u1 ? warmgp::Initialization::warm(vec(u1, n1)) : warmgp::Initialization::cold();
}

void fill(const warmgp::SolveResult& r, double* v_out, double* hist, int64_t hist_cap, RefResult* out) {
  put(r.v, v_out);
  out->status = 0;
  out->iterations = r.iterations;
  out->converged = r.converged ? 1 : 0;
  out->hist_len = static_cast<int64_t>(r.residual_history.size());
  for (int64_t k = 0; k < out->hist_len && k < hist_cap; ++k) hist[k] = r.residual_history[k];
}

template <typename F>
int guarded(RefResult* out, F&& f) {
  try {
    f();
    return 0;
  } catch (const warmgp::NotSpdError&) {
    out->status = 1;
  } catch (const warmgp::DivergenceError& e) {
    out->status = 2;
    out->iterations = e.iterations;
  } catch (const std::invalid_argument&) {
    out->status = 3;
  } catch (const std::exception&) {
    out->status = 4;
  }
  return out->status;
}

}  // namespace

extern "C" {

int ref_gram_matrix(const double* X, int64_t n, int64_t d, double ls, double sf, double sn, double* H) {
  put(warmgp::gram_matrix(mat(X, n, d), hyp(ls, sf, sn)).H, H);
  return 0;
}

int ref_cross_kernel(const double* Xs, int64_t m, const double* X, int64_t n, int64_t d, double ls,
                     double sf, double sn, double* K) {
  put(warmgp::cross_kernel(mat(Xs, m, d), mat(X, n, d), hyp(ls, sf, sn)), K);
  return 0;
}

double ref_matern32_from_distance(double r, double ls, double sf, double sn) {
  return warmgp::matern32_from_distance(r, hyp(ls, sf, sn));
}

int64_t ref_pivoted_cholesky(const double* H, int64_t n, int64_t rank, double* L) {
  const Matrix Lm = warmgp::pivoted_cholesky(mat(H, n, n), rank);
  put(Lm, L);
  return Lm.cols();
}

int ref_precond_apply(const double* H, int64_t n, int64_t rank, double shift, int mode,
                      const double* r, double* z) {
  const auto p = warmgp::CgPreconditioner::from_matrix(
      mat(H, n, n), rank, shift, static_cast<warmgp::SolverConfig::PrecondShiftMode>(mode));
  put(p.apply(vec(r, n)), z);
  return 0;
}

int ref_solve(const double* H, int64_t n, const double* b, const double* u1, int64_t n1, const RefCfg* c,
              double* v_out, double* hist, int64_t hist_cap, RefResult* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded(out, [&] {
    fill(warmgp::solve(mat(H, n, n), vec(b, n), init_of(u1, n1), cfg_of(*c)), v_out, hist, hist_cap, out);
  });
}

// solve_many: s columns of B (n x s), u1 (n1 x s) or null; per-column outputs: V (n x s),
// hist (s x hist_cap), out[s].  The whole call throws as a unit (the reference propagates the
// first exception), reported in out[0].
int ref_solve_many(const double* H, int64_t n, const double* B, int64_t s, const double* U1, int64_t n1,
                   const RefCfg* c, double* V_out, double* hist, int64_t hist_cap, RefResult* out) {
  std::memset(out, 0, sizeof(RefResult) * s);
  return guarded(out, [&] {
    std::vector<warmgp::Initialization> inits;
    for (int64_t i = 0; i < s; ++i) inits.push_back(init_of(U1 ? U1 + i * n1 : nullptr, n1));
    const auto res = warmgp::solve_many(mat(H, n, n), mat(B, n, s), inits, cfg_of(*c));
    for (int64_t i = 0; i < s; ++i) fill(res[i], V_out + i * n, hist + i * hist_cap, hist_cap, out + i);
  });
}

int ref_cg_solve_with(const double* H, int64_t n, const double* b, const double* u1, int64_t n1,
                      const RefCfg* c, int64_t rank, double shift, int mode, double* v_out, double* hist,
                      int64_t hist_cap, RefResult* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded(out, [&] {
    const Matrix Hm = mat(H, n, n);
    const auto p = warmgp::CgPreconditioner::from_matrix(
        Hm, rank, shift, static_cast<warmgp::SolverConfig::PrecondShiftMode>(mode));
    fill(warmgp::cg_solve_with(Hm, vec(b, n), init_of(u1, n1), cfg_of(*c), p), v_out, hist, hist_cap, out);
  });
}

double ref_relative_residual(const double* H, int64_t n, const double* v, const double* b) {
  return warmgp::relative_residual(mat(H, n, n), vec(v, n), vec(b, n));
}

int ref_sample_prior(double ls, double sf, double sn, int64_t dim, int64_t F, uint64_t seed, double* freq,
                     double* phases, double* amps) {
  const auto p = warmgp::sample_prior(hyp(ls, sf, sn), dim, F, seed);
  put(p.frequencies, freq);
  put(p.phases, phases);
  put(p.amplitudes, amps);
  return 0;
}

namespace {
warmgp::RffPrior prior_of(const double* freq, const double* phases, const double* amps, double sf,
                          int64_t F, int64_t d) {
  warmgp::RffPrior p;
  p.frequencies = mat(freq, F, d);
  p.phases = vec(phases, F);
  p.amplitudes = vec(amps, F);
  p.signal_scale = sf;
  return p;
}
}  // namespace

int ref_eval_prior(const double* freq, const double* phases, const double* amps, double sf, int64_t F,
                   int64_t d, const double* Xs, int64_t m, double* out) {
  put(warmgp::eval_prior(prior_of(freq, phases, amps, sf, F, d), mat(Xs, m, d)), out);
  return 0;
}

int ref_build_sample_rhs(const double* freq, const double* phases, const double* amps, double sf,
                         int64_t F, int64_t d, const double* X, int64_t n, double noise, uint64_t seed,
                         double* out) {
  put(warmgp::build_sample_rhs(prior_of(freq, phases, amps, sf, F, d), mat(X, n, d), noise, seed), out);
  return 0;
}

int ref_eval_posterior(const double* freq, const double* phases, const double* amps, double sf, int64_t F,
                       int64_t d, const double* Xtr, int64_t n, const double* w, double ls, double sn,
                       const double* Xs, int64_t m, double* out) {
  warmgp::PosteriorSample s;
  s.prior = prior_of(freq, phases, amps, sf, F, d);
  s.X_train = mat(Xtr, n, d);
  s.weights = vec(w, n);
  s.hyperparams = hyp(ls, sf, sn);
  put(warmgp::eval_posterior(s, mat(Xs, m, d)), out);
  return 0;
}

int ref_grad_posterior(const double* freq, const double* phases, const double* amps, double sf, int64_t F,
                       int64_t d, const double* Xtr, int64_t n, const double* w, double ls, double sn,
                       const double* x, double* out) {
  warmgp::PosteriorSample s;
  s.prior = prior_of(freq, phases, amps, sf, F, d);
  s.X_train = mat(Xtr, n, d);
  s.weights = vec(w, n);
  s.hyperparams = hyp(ls, sf, sn);
  put(warmgp::grad_posterior(s, vec(x, d)), out);
  return 0;
}

int ref_extend_system(const double* X1, int64_t n1, const double* X2, int64_t n2, int64_t d, double ls,
                      double sf, double sn, double* H_out) {
  const auto prev = warmgp::gram_matrix(mat(X1, n1, d), hyp(ls, sf, sn));
  const auto sys = warmgp::extend_system(prev, mat(X2, n2, d), Vector::Zero(n1), Vector::Zero(n2));
  put(sys.assembled(), H_out);
  return 0;
}

}  // extern "C"
