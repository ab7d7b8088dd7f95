// bo_round's solve pattern through include/warmgp/gpu.hpp (thompson.cpp:359-384): ONE
// CgPreconditioner::from_matrix per round, then cg_solve_with per column under per-column
// seeds derive_seed(derive_seed(seed, 0xc0000 + round), col).  The per-column results must
// equal solve_many's bitwise (solve_many factors its own preconditioner with the same rank /
// shift; solvers.hpp:136-141: "results match sequential single-RHS calls exactly").  Also
// exercises the rest of the reference's free functions at the boundary: relative_residual,
// quadratic_objective, init_weights, pivoted_cholesky, cross_kernel, eval_prior,
// build_sample_rhs, CgPreconditioner::apply and its (L, shift) constructor.  Exit 0 = pass.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "warmgp/gpu.hpp"

using namespace warmgp::gpu;

#define REQUIRE(cond, code)                                          \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::printf("FAILED %s (line %d)\n", #cond, __LINE__);         \
      return code;                                                   \
    }                                                                \
  } while (0)

static double kmatern(const Matrix& A, int64_t i, const Matrix& B, int64_t j, double l) {
  double r2 = 0.0;
  for (int64_t k = 0; k < A.cols; ++k) r2 += (A(i, k) - B(j, k)) * (A(i, k) - B(j, k));
  const double z = std::sqrt(3.0) * std::sqrt(r2) / l;
  return (1.0 + z) * std::exp(-z);
}

int main() {
  Context ctx(0);
  const int64_t n1 = 700, n = 764, d = 3, S = 8;
  std::mt19937_64 g(11);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::normal_distribution<double> N01;
  Matrix X(n, d), X1(n1, d), X2(n - n1, d);
  for (auto& x : X.data) x = U(g);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = 0; k < d; ++k) (i < n1 ? X1(i, k) : X2(i - n1, k)) = X(i, k);
  KernelHyperparams hyp{0.3, 1.0, 0.05};
  SolverConfig cfg;
  cfg.tolerance = 1e-8;
  cfg.max_iters = 800;
  cfg.precond_rank = 60;
  cfg.precond_shift = hyp.noise_scale * hyp.noise_scale;

  // previous round: the n1-row system, its solutions are the warm starts
  KernelOperator H(ctx, X1, hyp);
  Matrix rhs1(n1, 1 + S), rhs(n, 1 + S);
  for (auto& x : rhs.data) x = N01(g);
  for (int64_t c = 0; c <= S; ++c)
    for (int64_t i = 0; i < n1; ++i) rhs1(i, c) = rhs(i, c);
  std::vector<Initialization> cold(1 + S, Initialization::cold());
  const std::vector<SolveResult> prev = solve_many(H, rhs1, cold, cfg);

  // this round: append the new rows (extend_system), warm inits [u1; 0]
  H.append_rows(X2);
  REQUIRE(H.size() == n, 10);
  std::vector<Initialization> inits;
  for (const auto& r : prev) inits.push_back(Initialization::warm(r.v));

  const std::uint64_t seed = 5, round = 3;
  const CgPreconditioner precond =
      CgPreconditioner::from_matrix(H, cfg.precond_rank, cfg.precond_shift, cfg.precond_shift_mode);
  int64_t ach = 0;
  double sh = 0.0;
  check(wgp_precond_info(H.get(), cfg.precond_rank, cfg.precond_shift, (int)cfg.precond_shift_mode, &ach, &sh));
  REQUIRE(precond.rank() == ach && precond.shift() == sh, 11);

  std::vector<SolveResult> per;
  for (int64_t col = 0; col <= S; ++col) {
    SolverConfig c = cfg;
    c.seed = wgp_derive_seed(wgp_derive_seed(seed, 0xc0000 + round), (std::uint64_t)col);
    Vector b(rhs.col(col), rhs.col(col) + n);
    per.push_back(cg_solve_with(H, b, inits[col], c, precond));
  }
  const std::vector<SolveResult> batch = solve_many(H, rhs, inits, cfg);
  for (int64_t col = 0; col <= S; ++col) {
    REQUIRE(per[col].iterations == batch[col].iterations, 20);
    REQUIRE(per[col].converged && batch[col].converged, 21);
    REQUIRE(per[col].v == batch[col].v, 22);  // bitwise
    REQUIRE(per[col].residual_history == batch[col].residual_history, 23);
    REQUIRE(per[col].iterations <= prev[0].iterations + 1000, 24);
  }

  // relative_residual of the solution vs its last history entry (same definition)
  Vector b0(rhs.col(0), rhs.col(0) + n);
  const double rr = relative_residual(H, per[0].v, b0);
  REQUIRE(rr <= 1e-8 && std::fabs(rr - per[0].final_residual()) <= 1e-9, 30);
  bool threw = false;
  try {
    relative_residual(H, per[0].v, Vector(n, 0.0));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw, 31);
  // at the solution, 0.5 v.Hv - v.b = -0.5 v.b
  double vb = 0.0;
  for (int64_t i = 0; i < n; ++i) vb += per[0].v[i] * b0[i];
  REQUIRE(std::fabs(quadratic_objective(H, per[0].v, b0) + 0.5 * vb) <= 1e-6 * std::fabs(vb), 32);
  // init_weights
  const Vector w = init_weights(inits[0], n1, n - n1);
  REQUIRE((int64_t)w.size() == n && w[0] == prev[0].v[0] && w[n - 1] == 0.0, 33);
  // pivoted_cholesky: L has the achieved rank; the pivot rows carry sqrt(d) on the diagonal
  const Matrix L = pivoted_cholesky(H, cfg.precond_rank);
  REQUIRE(L.cols == ach && L.rows == n, 34);
  // CgPreconditioner(L, shift) reproduces from_matrix's apply when given its shift
  const CgPreconditioner p2(H, L, precond.shift());
  const Vector z1 = precond.apply(b0), z2 = p2.apply(b0);
  double dz = 0.0, nz = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    dz += (z1[i] - z2[i]) * (z1[i] - z2[i]);
    nz += z1[i] * z1[i];
  }
  REQUIRE(std::sqrt(dz / nz) <= 1e-12, 35);
  // cross_kernel against a direct fp64 evaluation
  const Matrix K = cross_kernel(H, X2);
  double kerr = 0.0;
  for (int64_t i = 0; i < K.rows; ++i)
    for (int64_t j = 0; j < n; j += 7) kerr = std::fmax(kerr, std::fabs(K(i, j) - kmatern(X2, i, X, j, hyp.lengthscale)));
  REQUIRE(kerr <= 1e-12, 36);
  // build_sample_rhs = eval_prior at the operator's rows + Rng(seed) noise
  const RffPrior prior = sample_prior(hyp, d, 256, 77);
  const Vector f = eval_prior(H, prior, X);
  const Vector y = build_sample_rhs(H, prior, 0.1, 99);
  std::uint64_t st = 99;
  double yerr = 0.0;
  for (int64_t i = 0; i < n; ++i) yerr = std::fmax(yerr, std::fabs(y[i] - (f[i] + 0.1 * wgp_rng_normal(&st))));
  REQUIRE(yerr == 0.0, 37);
  // appending rows invalidates the preconditioner handle
  Matrix X3(4, d);
  for (auto& x : X3.data) x = U(g);
  H.append_rows(X3);
  threw = false;
  try {
    cg_solve_with(H, Vector(n + 4, 1.0), Initialization::cold(), cfg, precond);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw, 38);
  std::printf("bo_round pattern ok: %lld columns, rank %lld, shift %.3e, iterations col0 %d\n",
              (long long)(S + 1), (long long)ach, sh, per[0].iterations);
  return 0;
}
