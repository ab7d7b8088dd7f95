// dense.cu -- on-device exact solve H x = b (exact_solve, analysis.cpp:15-26):
// the operator's gram matrix H = K(X, X) + sigma_n^2 I is materialised once in fp64
// (row-major N x N, the reference's dense H), factored in place by a right-looking blocked
// Cholesky (64-wide panels: unblocked factor of the diagonal block in one CTA, a triangular
// solve of the panel below it, a rank-64 update of the trailing lower triangle), and the
// right-hand sides are solved by blocked forward/back substitution.  A non-positive pivot is
// reported as NotSpdError like the reference's LLT failure.  Used for the config-1 warm start
// u1 = exact_solve(H11, y1) (bench_regression.cpp:168) and as a reference solution.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace wgp {
namespace {

constexpr int NBK = 64;  // panel width

__device__ __forceinline__ double kval(double d2, const KParams& p) {
  d2 = d2 > 0.0 ? d2 : 0.0;
  if (p.kind == WGP_RBF) return p.s2 * exp(-p.c1 * d2);
  const double z = p.c1 * sqrt(d2);
  return p.s2 * (1.0 + z) * exp(-z);
}

// H[i][j] for i, j < n (lower and upper), diagonal exactly s^2 + sigma_n^2 (kernel.cpp:70).
__global__ void gram_dense_kernel(const double* __restrict__ X, int dpad, int dim, int64_t n,
                                  KParams p, double* __restrict__ H) {
  __shared__ double sXi[32][33], sXj[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    for (int k = tx; k < dim; k += 32) {
      sXi[r][k] = i0 + r < n ? X[(i0 + r) * dpad + k] : 0.0;
      sXj[r][k] = j0 + r < n ? X[(j0 + r) * dpad + k] : 0.0;
    }
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + tx;
    if (i >= n || j >= n) continue;
    double d2 = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double df = sXi[r][k] - sXj[tx][k];
      d2 = fma(df, df, d2);
    }
    H[i * n + j] = i == j ? p.s2 + p.noise2 : kval(d2, p);
  }
}

// Unblocked Cholesky of the b x b diagonal block at (k0, k0), in place (lower), one CTA.
__global__ void potrf_diag_kernel(double* __restrict__ A, int64_t n, int64_t k0, int b,
                                  int* __restrict__ fail) {
  __shared__ double L[NBK][NBK + 1];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int r = e / b, c = e % b;
    L[r][c] = A[(k0 + r) * n + k0 + c];
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (threadIdx.x == 0) {
      double d = L[j][j];
      for (int t = 0; t < j; ++t) d -= L[j][t] * L[j][t];
      if (!(d > 0.0)) {
        *fail = 1;
        d = 1.0;
      }
      L[j][j] = sqrt(d);
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < b; i += blockDim.x) {
      double a = L[i][j];
      for (int t = 0; t < j; ++t) a -= L[i][t] * L[j][t];
      L[i][j] = a / L[j][j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int r = e / b, c = e % b;
    A[(k0 + r) * n + k0 + c] = c <= r ? L[r][c] : 0.0;
  }
}

// Panel: rows i >= k0 + b, A[i, k0:k0+b] <- A[i, k0:k0+b] L_kk^{-T} (one thread per row).
__global__ void trsm_panel_kernel(double* __restrict__ A, int64_t n, int64_t k0, int b) {
  __shared__ double L[NBK][NBK + 1];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int r = e / b, c = e % b;
    L[r][c] = A[(k0 + r) * n + k0 + c];
  }
  __syncthreads();
  const int64_t i = k0 + b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[NBK];
  for (int c = 0; c < b; ++c) x[c] = A[i * n + k0 + c];
  for (int c = 0; c < b; ++c) {
    double a = x[c];
    for (int t = 0; t < c; ++t) a -= x[t] * L[c][t];
    x[c] = a / L[c][c];
  }
  for (int c = 0; c < b; ++c) A[i * n + k0 + c] = x[c];
}

// Trailing update A[i][j] -= sum_t A[i][k0+t] A[j][k0+t] for k1 <= j <= i < n (64x64 tiles of
// the lower triangle; 256 threads, 4 x 4 outputs each).
__global__ void syrk_update_kernel(double* __restrict__ A, int64_t n, int64_t k0, int b,
                                   int64_t k1) {
  const int64_t ti = (int64_t)blockIdx.y, tj = (int64_t)blockIdx.x;
  if (tj > ti) return;
  const int64_t i0 = k1 + ti * 64, j0 = k1 + tj * 64;
  __shared__ double Pi[64][33], Pj[64][33];  // the panel in 32-wide K slices
  const int tr = (threadIdx.x / 16) * 4, tc = (threadIdx.x % 16) * 4;
  double acc[4][4] = {};
  for (int t0 = 0; t0 < b; t0 += 32) {
    const int kb = min(32, b - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
      const int r = e / 32, c = e % 32;
      Pi[r][c] = (i0 + r < n && c < kb) ? A[(i0 + r) * n + k0 + t0 + c] : 0.0;
      Pj[r][c] = (j0 + r < n && c < kb) ? A[(j0 + r) * n + k0 + t0 + c] : 0.0;
    }
    __syncthreads();
    for (int t = 0; t < kb; ++t) {
      double a[4], c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = Pi[tr + u][t];
        c[u] = Pj[tc + u][t];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], c[v], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t i = i0 + tr + u, j = j0 + tc + v;
      if (i < n && j <= i) A[i * n + j] -= acc[u][v];
    }
}

// Forward substitution block step: Y[k0:k0+b] = L_kk^{-1} (Y[k0:k0+b] - L[k0:k0+b, 0:k0] Y[0:k0]),
// Y row-major [n][s]; one CTA per column.
__global__ void fwd_block_kernel(const double* __restrict__ L, int64_t n, int64_t k0, int b,
                                 double* __restrict__ Y, int s) {
  const int c = blockIdx.x;
  __shared__ double r[NBK];
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double a = Y[(k0 + i) * s + c];
    const double* Li = L + (k0 + i) * n;
    for (int64_t t = 0; t < k0; ++t) a -= Li[t] * Y[t * s + c];
    r[i] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < b; ++i) {
      double a = r[i];
      for (int t = 0; t < i; ++t) a -= L[(k0 + i) * n + k0 + t] * r[t];
      r[i] = a / L[(k0 + i) * n + k0 + i];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < b; i += blockDim.x) Y[(k0 + i) * s + c] = r[i];
}

// Back substitution block step (L^T x = y, last block first): X[k0:k0+b] =
// L_kk^{-T} (Y[k0:k0+b] - L[k0+b:n, k0:k0+b]^T X[k0+b:n]).
__global__ void bwd_block_kernel(const double* __restrict__ L, int64_t n, int64_t k0, int b,
                                 double* __restrict__ Y, int s) {
  const int c = blockIdx.x;
  __shared__ double r[NBK];
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double a = Y[(k0 + i) * s + c];
    for (int64_t t = k0 + b; t < n; ++t) a -= L[t * n + k0 + i] * Y[t * s + c];
    r[i] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = b - 1; i >= 0; --i) {
      double a = r[i];
      for (int t = i + 1; t < b; ++t) a -= L[(k0 + t) * n + k0 + i] * r[t];
      r[i] = a / L[(k0 + i) * n + k0 + i];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < b; i += blockDim.x) Y[(k0 + i) * s + c] = r[i];
}

// Sum of log(L_ii) over the factor's diagonal, one block, fixed order.
__global__ void logdiag_kernel(const double* __restrict__ L, int64_t n, double* __restrict__ out) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += log(L[i * n + i]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// MLL gradient sums over (i, j) 32 x 32 tiles (mll_with_dist, analysis.cpp:121-130):
//   g0 = sum A_ij dK/dlog l (i, j),  g1 = sum A_ij 2 K_ij,  A = alpha alpha^T - H^{-1}.
// Y row-major [n][n + 1]: column 0 = alpha, columns 1.. = H^{-1}.  K and dK/dlog l are
// recomputed from X (direct-difference distances); per-block partials, summed on the host
// in block order.
__global__ void mll_grad_kernel(const double* __restrict__ X, int dpad, int dim, int64_t n,
                                int kind, double l, double s2, const double* __restrict__ Y,
                                double* __restrict__ part) {
  __shared__ double sXi[32][33], sXj[32][33], sa[2][32];
  __shared__ double red[2][256];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int64_t s = n + 1;
  for (int r = ty; r < 32; r += 8) {
    for (int k = tx; k < dim; k += 32) {
      sXi[r][k] = i0 + r < n ? X[(i0 + r) * dpad + k] : 0.0;
      sXj[r][k] = j0 + r < n ? X[(j0 + r) * dpad + k] : 0.0;
    }
  }
  if (ty == 0) sa[0][tx] = i0 + tx < n ? Y[(i0 + tx) * s] : 0.0;
  if (ty == 1) sa[1][tx] = j0 + tx < n ? Y[(j0 + tx) * s] : 0.0;
  __syncthreads();
  double g0 = 0.0, g1 = 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + tx;
    if (i >= n || j >= n) continue;
    double d2 = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double df = sXi[r][k] - sXj[tx][k];
      d2 = fma(df, df, d2);
    }
    const double rho = sqrt(d2) / l;
    double K, dkl;
    if (kind == WGP_RBF) {
      K = s2 * exp(-0.5 * rho * rho);
      dkl = K * rho * rho;
    } else {
      const double z = 1.7320508075688772935 * rho;
      const double e = exp(-z);
      K = s2 * (1.0 + z) * e;
      dkl = 3.0 * s2 * rho * rho * e;
    }
    const double a = sa[0][r] * sa[1][tx] - Y[i * s + 1 + j];
    g0 = fma(a, dkl, g0);
    g1 = fma(a, 2.0 * K, g1);
  }
  const int t = ty * 32 + tx;
  red[0][t] = g0;
  red[1][t] = g1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (t < o) {
      red[0][t] += red[0][t + o];
      red[1][t] += red[1][t + o];
    }
    __syncthreads();
  }
  if (t == 0) {
    const size_t b = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    part[2 * b] = red[0][0];
    part[2 * b + 1] = red[1][0];
  }
}

// sum_i (alpha_i^2 - H^{-1}_ii), one block, fixed order.
__global__ void mll_trace_kernel(const double* __restrict__ Y, int64_t n, double* __restrict__ out) {
  __shared__ double red[256];
  const int64_t s = n + 1;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = Y[i * s];
    acc += a * a - Y[i * s + 1 + i];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

}  // namespace

// H = K(X, X) + sigma_n^2 I for kernel parameters kp, factored in place (lower) by the
// blocked Cholesky.  Returns false if a pivot is not positive.
static bool factor_dense(const Op& op, const KParams& kp, DBuf<double>& H, cudaStream_t st) {
  const int64_t n = op.n;
  H.alloc((size_t)n * n);
  DBuf<int> fail(1);
  WGP_CUDA(cudaMemsetAsync(fail.p, 0, sizeof(int), st));
  dim3 g(ceil_div(n, 32), ceil_div(n, 32));
  gram_dense_kernel<<<g, dim3(32, 8), 0, st>>>(op.X64.p, op.dpad, op.dim, n, kp, H.p);
  WGP_CUDA(cudaGetLastError());
  for (int64_t k0 = 0; k0 < n; k0 += NBK) {
    const int b = (int)std::min<int64_t>(NBK, n - k0);
    potrf_diag_kernel<<<1, 256, 0, st>>>(H.p, n, k0, b, fail.p);
    const int64_t k1 = k0 + b;
    if (k1 < n) {
      trsm_panel_kernel<<<ceil_div(n - k1, 128), 128, 0, st>>>(H.p, n, k0, b);
      const int nt = ceil_div(n - k1, 64);
      syrk_update_kernel<<<dim3(nt, nt), 256, 0, st>>>(H.p, n, k0, b, k1);
    }
    WGP_CUDA(cudaGetLastError());
  }
  int hfail = 0;
  WGP_CUDA(cudaMemcpyAsync(&hfail, fail.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaStreamSynchronize(st));
  return hfail == 0;
}

// Y (n x s row-major) <- (L L^T)^{-1} Y.
static void solve_dense(const double* L, int64_t n, double* Y, int64_t s, cudaStream_t st) {
  for (int64_t k0 = 0; k0 < n; k0 += NBK)
    fwd_block_kernel<<<(unsigned)s, 128, 0, st>>>(L, n, k0, (int)std::min<int64_t>(NBK, n - k0), Y, (int)s);
  for (int64_t k0 = ((n - 1) / NBK) * NBK; k0 >= 0; k0 -= NBK)
    bwd_block_kernel<<<(unsigned)s, 128, 0, st>>>(L, n, k0, (int)std::min<int64_t>(NBK, n - k0), Y, (int)s);
  WGP_CUDA(cudaGetLastError());
}

// Y (n x s row-major, in: B, out: H^{-1} B).  Returns false if H is not numerically SPD.
bool exact_solve_dev(const Op& op, double* Y, int s, cudaStream_t st) {
  const int64_t n = op.n;
  WGP_REQUIRE(n >= 1 && n <= 60000, "exact_solve: n = %lld outside the dense range [1, 60000]",
              (long long)n);
  DBuf<double> H;
  if (!factor_dense(op, op.kp(), H, st)) return false;
  solve_dense(H.p, n, Y, s, st);
  WGP_CUDA(cudaStreamSynchronize(st));
  return true;
}

// mll (analysis.cpp:99-139) at hyperparameters (l, sf, sn) on the operator's rows: dense H
// factored on the device, [alpha | H^{-1}] = H^{-1} [y | I] by blocked substitution, the
// log-determinant from the factor's diagonal and the gradient sums in one fused pass that
// recomputes K and dK/dlog l from X.  y: host, n.  Returns false if H is not SPD.
bool mll_dev(const Op& op, double l, double sf, double sn, const double* y, double* value,
             double* grad3, cudaStream_t st) {
  const int64_t n = op.n;
  WGP_REQUIRE(n >= 1 && n <= 30000, "mll: n = %lld outside the dense range [1, 30000]", (long long)n);
  WGP_REQUIRE(l > 0.0 && sf > 0.0 && sn > 0.0, "KernelHyperparams: all scales must be positive");
  KParams kp;
  kp.kind = op.kind;
  kp.c1 = op.kind == WGP_MATERN32 ? 1.7320508075688772935 / l : 0.5 / (l * l);
  kp.s2 = sf * sf;
  kp.noise2 = sn * sn;
  DBuf<double> H;
  if (!factor_dense(op, kp, H, st)) return false;
  const int64_t s = n + 1;
  std::vector<double> hY((size_t)n * s, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    hY[(size_t)i * s] = y[i];
    hY[(size_t)i * s + 1 + i] = 1.0;
  }
  DBuf<double> Y((size_t)n * s);
  WGP_CUDA(cudaMemcpyAsync(Y.p, hY.data(), sizeof(double) * hY.size(), cudaMemcpyHostToDevice, st));
  solve_dense(H.p, n, Y.p, s, st);
  const dim3 g(ceil_div(n, 32), ceil_div(n, 32));
  const size_t nb = (size_t)g.x * g.y;
  DBuf<double> part(2 * nb), scal(2);
  logdiag_kernel<<<1, 256, 0, st>>>(H.p, n, scal.p);
  mll_trace_kernel<<<1, 256, 0, st>>>(Y.p, n, scal.p + 1);
  mll_grad_kernel<<<g, dim3(32, 8), 0, st>>>(op.X64.p, op.dpad, op.dim, n, op.kind, l, kp.s2, Y.p,
                                             part.p);
  WGP_CUDA(cudaGetLastError());
  std::vector<double> hp(2 * nb), hs(2), alpha((size_t)n);
  WGP_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaMemcpyAsync(hs.data(), scal.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaMemcpy2DAsync(alpha.data(), sizeof(double), Y.p, sizeof(double) * s, sizeof(double), n,
                             cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaStreamSynchronize(st));
  double ya = 0.0, g0 = 0.0, g1 = 0.0;
  for (int64_t i = 0; i < n; ++i) ya += y[i] * alpha[(size_t)i];
  for (size_t b = 0; b < nb; ++b) {
    g0 += hp[2 * b];
    g1 += hp[2 * b + 1];
  }
  const double logdet = 2.0 * hs[0];
  *value = -0.5 * ya - 0.5 * logdet - 0.5 * (double)n * 1.8378770664093454836;
  grad3[0] = 0.5 * g0;
  grad3[1] = 0.5 * g1;
  grad3[2] = 0.5 * hs[1] * 2.0 * kp.noise2;
  return true;
}

}  // namespace wgp
