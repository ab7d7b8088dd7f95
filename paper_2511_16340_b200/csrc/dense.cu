// dense.cu -- on-device exact solve H x = b (exact_solve, analysis.cpp:15-26):
// the operator's gram matrix H = K(X, X) + sigma_n^2 I is materialised once in fp64
// (row-major N x N, the reference's dense H), factored in place by a right-looking blocked
// Cholesky (64-wide panels: unblocked factor of the diagonal block in one CTA, a triangular
// solve of the panel below it, a rank-64 update of the trailing lower triangle), and the
// right-hand sides are solved by blocked forward/back substitution.  A non-positive pivot is
// reported as NotSpdError like the reference's LLT failure.  Used for the config-1 warm start
// u1 = exact_solve(H11, y1) (bench_regression.cpp:168) and as a reference solution.
#include <cmath>

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

}  // namespace

// Y (n x s row-major, in: B, out: H^{-1} B).  Returns false if H is not numerically SPD.
bool exact_solve_dev(const Op& op, double* Y, int s, cudaStream_t st) {
  const int64_t n = op.n;
  WGP_REQUIRE(n >= 1 && n <= 60000, "exact_solve: n = %lld outside the dense range [1, 60000]",
              (long long)n);
  DBuf<double> H((size_t)n * n);
  DBuf<int> fail(1);
  WGP_CUDA(cudaMemsetAsync(fail.p, 0, sizeof(int), st));
  const KParams kp = op.kp();
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
  if (hfail) return false;
  for (int64_t k0 = 0; k0 < n; k0 += NBK)
    fwd_block_kernel<<<s, 128, 0, st>>>(H.p, n, k0, (int)std::min<int64_t>(NBK, n - k0), Y, s);
  for (int64_t k0 = ((n - 1) / NBK) * NBK; k0 >= 0; k0 -= NBK)
    bwd_block_kernel<<<s, 128, 0, st>>>(H.p, n, k0, (int)std::min<int64_t>(NBK, n - k0), Y, s);
  WGP_CUDA(cudaGetLastError());
  WGP_CUDA(cudaStreamSynchronize(st));
  return true;
}

}  // namespace wgp
