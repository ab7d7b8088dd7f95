// C++ smoke of include/warmgp/gpu.hpp (the reference-API mirror over the C-ABI):
// builds a Matern operator, checks H*v against a direct fp64 evaluation, solves with CG
// cold and warm, and checks the reference exception mapping.  Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <random>

#include "warmgp/gpu.hpp"

using namespace warmgp::gpu;

int main() {
  Context ctx(0);
  const int64_t n = 600, d = 3;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::normal_distribution<double> N01;
  Matrix X(n, d);
  for (auto& x : X.data) x = U(g);
  KernelHyperparams hyp{0.5, 1.0, 0.5};
  KernelOperator H(ctx, X, hyp);
  Matrix v(n, 1);
  for (auto& x : v.data) x = N01(g);
  const Matrix Hv = H * v;
  double err = 0, nrm = 0;
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0;
    for (int64_t j = 0; j < n; ++j) {
      double r2 = 0;
      for (int64_t k = 0; k < d; ++k) r2 += (X(i, k) - X(j, k)) * (X(i, k) - X(j, k));
      const double z = std::sqrt(3.0) * std::sqrt(r2) / hyp.lengthscale;
      acc += ((i == j) ? 1.0 + 0.25 : (1.0 + z) * std::exp(-z)) * v(j, 0);
    }
    err += (acc - Hv(i, 0)) * (acc - Hv(i, 0));
    nrm += acc * acc;
  }
  if (std::sqrt(err / nrm) > 1e-10) { std::printf("matvec mismatch %g\n", std::sqrt(err / nrm)); return 1; }
  Vector b(n);
  for (auto& x : b) x = N01(g);
  SolverConfig cfg;
  cfg.tolerance = 1e-6;
  cfg.precond_rank = 20;
  cfg.precond_shift = 0.25;
  const SolveResult cold = cg_solve(H, b, Initialization::cold(), cfg);
  if (!cold.converged || cold.residual_history.size() != (size_t)cold.iterations + 1) return 2;
  const SolveResult warm = cg_solve(H, b, Initialization::warm(cold.v), cfg);
  if (warm.iterations != 0 || !warm.converged) return 3;
  bool threw = false;
  try {
    cg_solve(H, Vector(n + 1, 1.0), Initialization::cold(), cfg);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!threw) return 4;
  std::printf("gpu.hpp ok: cold %d iters, warm %d iters\n", cold.iterations, warm.iterations);
  return 0;
}
