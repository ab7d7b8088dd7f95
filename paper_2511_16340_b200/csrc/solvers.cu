// solvers.cu -- batched multi-RHS solvers on the device with the reference's per-column
// semantics (solve_many = k independent solves, solvers.hpp:136-141, solvers.cpp:321-354).
//
// CG restates cg_solve_with (solvers.cpp:142-183) column-wise: each column keeps its own
// alpha, beta, convergence flag, iteration count and residual history; the iteration does
// the reference's TWO operator applications (H p, and the true residual b - H v that
// drives both the stopping test and the next direction).  Columns that converge are
// frozen (alpha = 0, p untouched) so their v is exactly the iterate the reference returns.
//
// Host work per iteration is one small D2H of (rel, active, failure) -- the scalar logic
// (alpha, beta, freeze) runs in single-block "step" kernels on the device.
#include <climits>
#include <cmath>

#include "solvers.h"

namespace wgp {
namespace {

__global__ void init_bnorm_kernel(const double* __restrict__ part, int nch, int s,
                                  double* __restrict__ bnorm, int* __restrict__ active) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < s; c += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < nch; ++q) acc += part[(int64_t)q * s + c];
    bnorm[c] = sqrt(acc);
    active[c] = acc != 0.0;  // zero RHS: zero_rhs_result (solvers.cpp:51-58, :145)
  }
}

// rel = |r| / |b|, freezes converged columns.  nq/qi select the partial slot.
__global__ void resid_step_kernel(const double* __restrict__ part, int nch, int nq, int s,
                                  const double* __restrict__ bnorm, double tol,
                                  double* __restrict__ rel, int* __restrict__ active) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < s; c += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < nch; ++q) acc += part[((int64_t)q * nq) * s + c];
    const double r = bnorm[c] > 0.0 ? sqrt(acc) / bnorm[c] : 0.0;
    rel[c] = r;
    if (active[c] && r <= tol) active[c] = 0;
  }
}

__global__ void cg_alpha_kernel(const double* __restrict__ part, int nch, int s,
                                const double* __restrict__ rz, const int* __restrict__ active,
                                double* __restrict__ alpha, int* __restrict__ fail_col) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < s; c += gridDim.x * blockDim.x) {
    double pHp = 0.0;
    for (int q = 0; q < nch; ++q) pHp += part[(int64_t)q * s + c];
    if (!active[c]) {
      alpha[c] = 0.0;
      continue;
    }
    if (pHp <= 0.0) atomicMin(fail_col, c);  // NotSpdError, solvers.cpp:164-166
    alpha[c] = rz[c] / pHp;
  }
}

// rz_next = r.z ; beta = rz_next / rz (active columns only), solvers.cpp:179-182.
__global__ void cg_beta_kernel(const double* __restrict__ part, int nch, int s,
                               double* __restrict__ rz, const int* __restrict__ active,
                               double* __restrict__ beta, int init) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < s; c += gridDim.x * blockDim.x) {
    double rzn = 0.0;
    for (int q = 0; q < nch; ++q) rzn += part[(int64_t)q * s + c];
    if (init) {
      rz[c] = rzn;
      beta[c] = 0.0;
    } else if (active[c]) {
      beta[c] = rzn / rz[c];
      rz[c] = rzn;
    } else {
      beta[c] = 0.0;
    }
  }
}

inline int sgrid(int s) { return (s + 255) / 256; }

}  // namespace

template <typename T>
void SolverWork<T>::alloc(int64_t n_, int s_) {
  n = n_;
  s = s_;
  nch = ceil_div(n, kChunkRows);
  const size_t ns = (size_t)n * s;
  V.alloc(ns);
  R.alloc(ns);
  Z.alloc(ns);
  P.alloc(ns);
  HP.alloc(ns);
  B.alloc(ns);
  part.alloc((size_t)(nch > 0 ? nch : 1) * 2 * s);
  scal.alloc((size_t)6 * s);
  act.alloc((size_t)s + 1);
}

template <typename T>
void upload_problem(const Op& op, SolverWork<T>& w, const double* B, int64_t ldb, const double* U1,
                    int64_t ldu, int64_t n1, cudaStream_t st) {
  const int64_t n = w.n;
  const int s = w.s;
  // B: host column-major -> device staging (fp64 col-major) -> row-major T
  DBuf<double> stage((size_t)std::max<int64_t>(n, 1) * s);
  WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n, B, sizeof(double) * ldb,
                             sizeof(double) * n, s, cudaMemcpyHostToDevice, st));
  launch_colmajor_to_rows(stage.p, n, n, s, w.B.p, true, st);
  WGP_CUDA(cudaMemsetAsync(w.V.p, 0, sizeof(T) * n * s, st));
  if (U1 && n1 > 0) {  // expand_init: [u1; 0] (solvers.cpp:43-48)
    WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n1, U1, sizeof(double) * ldu,
                               sizeof(double) * n1, s, cudaMemcpyHostToDevice, st));
    launch_colmajor_to_rows(stage.p, n1, n1, s, w.V.p, true, st);
  }
  WGP_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void download_solution(SolverWork<T>& w, double* V, int64_t ldv, cudaStream_t st) {
  const int64_t n = w.n;
  const int s = w.s;
  DBuf<double> stage((size_t)std::max<int64_t>(n, 1) * s);
  launch_rows_to_colmajor(w.V.p, n, s, stage.p, n, true, st);
  WGP_CUDA(cudaMemcpy2DAsync(V, sizeof(double) * ldv, stage.p, sizeof(double) * n,
                             sizeof(double) * n, s, cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void cg_solve_batched(Op& op, const wgp_solver_config& cfg, const PrecondDev& pd,
                      SolverWork<T>& w, SolveOutputs& out, cudaStream_t st) {
  const int64_t n = w.n;
  const int s = w.s;
  double* rz = w.scal.p;
  double* alpha = rz + s;
  double* beta = alpha + s;
  double* bnorm = beta + s;
  double* rel = bnorm + s;
  int* active = w.act.p;
  int* fail = w.act.p + s;
  const int nch = w.nch;
  w.pwork.ensure((size_t)(nch > 0 ? nch : 1) * (pd.k + 1) * s);
  w.tvec.ensure((size_t)(pd.k + 1) * s);

  // |b| per column
  launch_coldots<T>(w.B.p, w.B.p, nullptr, nullptr, n, s, w.part.p, st);
  init_bnorm_kernel<<<sgrid(s), 256, 0, st>>>(w.part.p, nch, s, bnorm, active);
  // r0 = b - H v0 (solvers.cpp:150)
  launch_residual(op, w.B.p, w.V.p, w.R.p, s, st);
  launch_coldots<T>(w.R.p, w.R.p, nullptr, nullptr, n, s, w.part.p, st);
  resid_step_kernel<<<sgrid(s), 256, 0, st>>>(w.part.p, nch, 1, s, bnorm, cfg.tolerance, rel,
                                              active);
  std::vector<double> hrel(s);
  std::vector<int> hact(s + 1), prev_act(s);
  WGP_CUDA(cudaMemcpyAsync(hrel.data(), rel, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaMemcpyAsync(hact.data(), active, sizeof(int) * s, cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaStreamSynchronize(st));
  int n_active = 0;
  for (int c = 0; c < s; ++c) {
    out.history[c].assign(1, hrel[c]);  // zero RHS -> {0} (rel computed as 0)
    out.iterations[c] = 0;
    out.converged[c] = !hact[c];
    n_active += hact[c];
    prev_act[c] = hact[c];
  }
  if (n_active == 0) return;

  // z = P r; p = z; rz = r.z (solvers.cpp:157-159)
  precond_apply<T>(pd, w.R.p, w.Z.p, s, w.tvec.p, w.pwork.p, st);
  WGP_CUDA(cudaMemcpyAsync(w.P.p, w.Z.p, sizeof(T) * n * s, cudaMemcpyDeviceToDevice, st));
  launch_coldots<T>(w.R.p, w.Z.p, nullptr, nullptr, n, s, w.part.p, st);
  cg_beta_kernel<<<sgrid(s), 256, 0, st>>>(w.part.p, nch, s, rz, active, beta, 1);
  const int int_max = INT_MAX;
  WGP_CUDA(cudaMemcpyAsync(fail, &int_max, sizeof(int), cudaMemcpyHostToDevice, st));

  for (int k = 1; k <= cfg.max_iters; ++k) {
    launch_kmatvec_full(op, w.P.p, w.HP.p, s, st);  // Hp = H p (:162)
    launch_coldots<T>(w.P.p, w.HP.p, nullptr, nullptr, n, s, w.part.p, st);
    cg_alpha_kernel<<<sgrid(s), 256, 0, st>>>(w.part.p, nch, s, rz, active, alpha, fail);
    launch_axpy_cols<T>(w.V.p, w.P.p, alpha, n, s, st);  // v += alpha p (:168)
    launch_residual(op, w.B.p, w.V.p, w.R.p, s, st);  // r = b - H v (:171)
    launch_coldots<T>(w.R.p, w.R.p, nullptr, nullptr, n, s, w.part.p, st);
    resid_step_kernel<<<sgrid(s), 256, 0, st>>>(w.part.p, nch, 1, s, bnorm, cfg.tolerance, rel,
                                                active);
    WGP_CUDA(cudaMemcpyAsync(hrel.data(), rel, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaMemcpyAsync(hact.data(), active, sizeof(int) * (s + 1), cudaMemcpyDeviceToHost,
                             st));
    WGP_CUDA(cudaStreamSynchronize(st));
    if (hact[s] != INT_MAX) {
      Error e(WGP_NOT_SPD, "cg_solve: non-positive curvature encountered");
      e.col = hact[s];
      throw e;
    }
    n_active = 0;
    for (int c = 0; c < s; ++c) {
      if (prev_act[c]) {
        out.history[c].push_back(hrel[c]);
        out.iterations[c] = k;
        if (!hact[c]) out.converged[c] = 1;
      }
      prev_act[c] = hact[c];
      n_active += hact[c];
    }
    if (n_active == 0) break;
    precond_apply<T>(pd, w.R.p, w.Z.p, s, w.tvec.p, w.pwork.p, st);  // z = P r (:178)
    launch_coldots<T>(w.R.p, w.Z.p, nullptr, nullptr, n, s, w.part.p, st);
    cg_beta_kernel<<<sgrid(s), 256, 0, st>>>(w.part.p, nch, s, rz, active, beta, 0);
    launch_xpby_cols<T>(w.P.p, w.Z.p, beta, active, n, s, st);  // p = z + beta p (:180)
  }
  WGP_CUDA(cudaGetLastError());
}

template struct SolverWork<double>;
template void upload_problem<double>(const Op&, SolverWork<double>&, const double*, int64_t,
                                     const double*, int64_t, int64_t, cudaStream_t);
template void download_solution<double>(SolverWork<double>&, double*, int64_t, cudaStream_t);
template void cg_solve_batched<double>(Op&, const wgp_solver_config&, const PrecondDev&,
                                       SolverWork<double>&, SolveOutputs&, cudaStream_t);

}  // namespace wgp
