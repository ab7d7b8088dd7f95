// Exercises include/warmgp/gpu.hpp's WARMGP_GPU_EIGEN overloads (compiled against the
// test shim tests/cpp/eigen_shim, since Eigen3 is absent): Eigen values in, the same
// results as the plain-Matrix API out.
#define WARMGP_GPU_EIGEN 1
#include <warmgp/gpu.hpp>

#include <cmath>
#include <cstdio>

namespace g = warmgp::gpu;

int main() {
  const int n = 200, d = 3;
  Eigen::MatrixXd X(n, d);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) X(i, k) = std::sin(0.37 * i + 1.3 * k);
  g::KernelHyperparams hyp;
  hyp.lengthscale = 0.7;
  hyp.noise_scale = 0.3;
  g::Context ctx(0);
  g::KernelOperator H = g::gram_matrix(ctx, X, hyp);
  Eigen::VectorXd b(n);
  for (int i = 0; i < n; ++i) b(i) = std::cos(0.11 * i);
  g::SolverConfig cfg;
  cfg.tolerance = 1e-8;
  cfg.max_iters = 500;
  const g::SolveResult r = g::solve(H, b, g::Initialization::cold(), cfg);
  const g::SolveResult r2 = g::solve(H, g::to_gpu(b), g::Initialization::cold(), cfg);
  if (!r.converged || r.iterations != r2.iterations) { std::printf("solve mismatch\n"); return 1; }
  Eigen::MatrixXd V(n, 1);
  for (int i = 0; i < n; ++i) V(i, 0) = r.v[(size_t)i];
  const Eigen::MatrixXd HV = H * V;
  double err = 0, nb = 0;
  for (int i = 0; i < n; ++i) {
    err += (HV(i, 0) - b(i)) * (HV(i, 0) - b(i));
    nb += b(i) * b(i);
  }
  if (std::sqrt(err / nb) > 1e-7) { std::printf("residual %g\n", std::sqrt(err / nb)); return 1; }
  Eigen::MatrixXd X2(20, d);
  for (int i = 0; i < 20; ++i)
    for (int k = 0; k < d; ++k) X2(i, k) = std::sin(0.37 * (n + i) + 1.3 * k);
  g::append_rows(H, X2);
  Eigen::MatrixXd B(n + 20, 2);
  for (int i = 0; i < n + 20; ++i) { B(i, 0) = std::cos(0.11 * i); B(i, 1) = std::sin(0.05 * i); }
  std::vector<g::Initialization> inits = {g::warm(g::to_eigen(r.v)), g::Initialization::warm(r.v)};
  const auto rs = g::solve_many(H, B, inits, cfg);
  if (rs.size() != 2 || !rs[0].converged || !rs[1].converged) { std::printf("solve_many failed\n"); return 1; }
  // analysis.hpp overloads: exact_solve, mll / optimize_mll on Eigen values
  g::KernelOperator H0 = g::gram_matrix(ctx, X, hyp);
  const Eigen::VectorXd xs = g::exact_solve(H0, b);
  Eigen::MatrixXd Xs1(n, 1);
  for (int i = 0; i < n; ++i) Xs1(i, 0) = xs(i);
  const Eigen::MatrixXd Hx = H0 * Xs1;
  double e2 = 0;
  for (int i = 0; i < n; ++i) e2 += (Hx(i, 0) - b(i)) * (Hx(i, 0) - b(i));
  if (std::sqrt(e2 / nb) > 1e-10) { std::printf("exact_solve residual %g\n", std::sqrt(e2 / nb)); return 1; }
  const g::MllResult m1 = g::mll(ctx, X, b, hyp);
  const g::MllResult m2 = g::mll(H0, g::to_gpu(b), hyp);
  if (m1.value != m2.value || !std::isfinite(m1.value)) { std::printf("mll mismatch\n"); return 1; }
  const g::KernelHyperparams fit = g::optimize_mll(ctx, X, b, hyp, 5, 0.1);
  if (g::mll(H0, g::to_gpu(b), fit).value < m1.value) { std::printf("optimize_mll worse\n"); return 1; }
  if (!(g::median_heuristic_lengthscale(X) > 0.0)) { std::printf("median heuristic\n"); return 1; }
  std::printf("eigen overloads ok: %d iters, warm %d/%d\n", r.iterations, rs[0].iterations, rs[1].iterations);
  return 0;
}
