// precond.cu -- pivoted-Cholesky preconditioner built and applied on the device.
//
// build_pivoted_cholesky restates pivoted_cholesky (solvers.cpp:72-107) matrix-free:
// the pivot column H(:, piv) is evaluated on the fly from X with the reference's
// norm-form distance (kernel.cpp:65-67, diagonal exactly s^2+sigma_n^2), so the pivot
// sequence (strict '>' over unused rows, first index on ties, floor 1e-12 max diag)
// matches the oracle.  finish_preconditioner computes the Calibrated shift
// (solvers.cpp:128-131), the capacitance shift I + L^T L (:115-117) and factors it on the
// host; the device keeps M = L C^{-T} so that the Woodbury apply (:135-140)
//   z = (r - L cap^{-1} L^T r) / shift  ==  (r - M (M^T r)) / shift
// is two skinny contractions per CG iteration.
#include <cmath>

#include "common.cuh"

namespace wgp {
namespace {

__device__ __forceinline__ double kmap64(double d2, const KParams& p) {
  const double r = sqrt(d2 > 0.0 ? d2 : 0.0);
  if (p.kind == WGP_RBF) return p.s2 * exp(-p.c1 * r * r);
  const double z = p.c1 * r;
  return p.s2 * (1.0 + z) * exp(-z);
}

struct ArgBest {
  double v;
  int64_t i;
};

__device__ __forceinline__ ArgBest better(ArgBest a, ArgBest b) {
  // larger value wins; equal values -> lower index (first index with strict '>' scan)
  if (b.i < 0) return a;
  if (a.i < 0) return b;
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__global__ void argmax_partial_kernel(const double* __restrict__ d, const int* __restrict__ used,
                                      int64_t n, double floor_, double* __restrict__ pv,
                                      int64_t* __restrict__ pi) {
  ArgBest b{0.0, -1};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!used[i] && d[i] > floor_) b = better(b, ArgBest{d[i], i});
  }
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  sv[threadIdx.x] = b.v;
  si[threadIdx.x] = b.i;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ArgBest r = better(ArgBest{sv[threadIdx.x], si[threadIdx.x]},
                         ArgBest{sv[threadIdx.x + o], si[threadIdx.x + o]});
      sv[threadIdx.x] = r.v;
      si[threadIdx.x] = r.i;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = sv[0];
    pi[blockIdx.x] = si[0];
  }
}

// Single block: final argmax; writes the pivot index and root = sqrt(d[piv]).
__global__ void argmax_final_kernel(const double* __restrict__ pv, const int64_t* __restrict__ pi,
                                    int nb, const double* __restrict__ d,
                                    int64_t* __restrict__ piv_out, double* __restrict__ root_out) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  ArgBest b{0.0, -1};
  for (int k = threadIdx.x; k < nb; k += blockDim.x) b = better(b, ArgBest{pv[k], pi[k]});
  sv[threadIdx.x] = b.v;
  si[threadIdx.x] = b.i;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ArgBest r = better(ArgBest{sv[threadIdx.x], si[threadIdx.x]},
                         ArgBest{sv[threadIdx.x + o], si[threadIdx.x + o]});
      sv[threadIdx.x] = r.v;
      si[threadIdx.x] = r.i;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *piv_out = si[0];
    *root_out = si[0] >= 0 ? sqrt(d[si[0]]) : 0.0;
  }
}

// One pivoted-Cholesky step for every row i (solvers.cpp:93-103).
__global__ void pchol_step_kernel(const double* __restrict__ X, const double* __restrict__ sq,
                                  int64_t n, int dpad, int dim, KParams p, int k, int kpad,
                                  const int64_t* __restrict__ piv_p,
                                  const double* __restrict__ root_p, double* __restrict__ L,
                                  double* __restrict__ d, int* __restrict__ used) {
  const int64_t piv = *piv_p;
  if (piv < 0) return;
  const double root = *root_p;
  const double* xp = X + piv * dpad;
  const double* Lp = L + piv * kpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double h;
    if (i == piv) {
      h = p.s2 + p.noise2;
    } else {
      const double* xi = X + i * dpad;
      double g = 0.0;
      for (int t = 0; t < dim; ++t) g += xi[t] * xp[t];
      h = kmap64(sq[i] + sq[piv] - 2.0 * g, p);
    }
    double* Li = L + i * kpad;
    double col = h;
    for (int t = 0; t < k; ++t) col -= Li[t] * Lp[t];
    const double lik = (i == piv) ? root : col / root;
    Li[k] = lik;
    if (i == piv) {
      used[i] = 1;
      d[i] = 0.0;
    } else if (!used[i]) {
      d[i] -= lik * lik;
    }
  }
}

// Per-block partial of G = A^T A over a contiguous slab of rows (fixed assignment).
__global__ void gram_partial_kernel(const double* __restrict__ A, int64_t n, int k, int kpad,
                                    double* __restrict__ part) {
  const int nb = gridDim.x;
  const int64_t per = (n + nb - 1) / nb;
  const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  double* out = part + (int64_t)blockIdx.x * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int a = e / k, b = e % k;
    double acc = 0.0;
    for (int64_t i = r0; i < r1; ++i) acc += A[i * kpad + a] * A[i * kpad + b];
    out[e] = acc;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int np, int count,
                                    double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < np; ++q) acc += part[(int64_t)q * count + e];
    out[e] = acc;
  }
}

// M[i, j] = sum_{t <= j} L[i, t] W[t, j] (W = C^{-T}, upper triangular).
__global__ void apply_upper_kernel(const double* __restrict__ L, const double* __restrict__ W,
                                   int64_t n, int k, int kpad, double* __restrict__ M,
                                   float* __restrict__ M32) {
  extern __shared__ double sW[];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) sW[e] = W[e];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * kpad;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / kpad;
    const int j = (int)(e % kpad);
    double acc = 0.0;
    if (j < k)
      for (int t = 0; t <= j; ++t) acc += L[i * kpad + t] * sW[t * k + j];
    M[e] = acc;
    if (M32) M32[e] = (float)acc;
  }
}

// T[chunk][a][c] = sum_{i in chunk} M[i, a] R[i, c]
template <typename T>
__global__ void __launch_bounds__(256) mtr_partial_kernel(const T* __restrict__ M,
                                                          const T* __restrict__ R, int64_t n,
                                                          int k, int kpad, int s,
                                                          double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RT = 32;
  T* sM = reinterpret_cast<T*>(smem);  // RT x kpad
  T* sR = sM + RT * kpad;               // RT x s
  const int64_t r0 = (int64_t)blockIdx.x * kChunkRows;
  const int64_t r1 = min(n, r0 + (int64_t)kChunkRows);
  const int outs = k * s;
  constexpr int MAXQ = 64;  // supports k*s <= 256*64
  double acc[MAXQ];
  const int nq = (outs + 255) / 256;
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) acc[q] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += RT) {
    __syncthreads();
    for (int e = threadIdx.x; e < RT * kpad; e += 256) {
      const int64_t i = rb + e / kpad;
      sM[e] = i < r1 ? M[i * kpad + e % kpad] : T(0);
    }
    for (int e = threadIdx.x; e < RT * s; e += 256) {
      const int64_t i = rb + e / s;
      sR[e] = i < r1 ? R[i * s + e % s] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      if (q >= nq) break;
      const int o = threadIdx.x + q * 256;
      if (o >= outs) break;
      const int a = o / s, c = o % s;
      double t = acc[q];
      for (int ii = 0; ii < RT; ++ii) t = fma((double)sM[ii * kpad + a], (double)sR[ii * s + c], t);
      acc[q] = t;
    }
  }
  double* out = part + (int64_t)blockIdx.x * outs;
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    if (q >= nq) break;
    const int o = threadIdx.x + q * 256;
    if (o < outs) out[o] = acc[q];
  }
}

// Z[i, c] = (R[i, c] - sum_a M[i, a] t[a, c]) / shift
template <typename T>
__global__ void __launch_bounds__(256) woodbury_out_kernel(const T* __restrict__ M,
                                                           const T* __restrict__ R,
                                                           const double* __restrict__ t, int64_t n,
                                                           int k, int kpad, int s, double inv_shift,
                                                           T* __restrict__ Z) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* st = reinterpret_cast<T*>(smem);  // k x s
  for (int e = threadIdx.x; e < k * s; e += blockDim.x) st[e] = (T)t[e];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * s;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / s;
    const int c = (int)(e % s);
    const T* Mi = M + i * kpad;
    T acc = T(0);
    for (int a = 0; a < k; ++a) acc = fma(Mi[a], st[a * s + c], acc);
    Z[e] = (T)(((double)R[e] - (double)acc) * inv_shift);
  }
}

inline int grid_rows(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void build_pivoted_cholesky(const Op& op, int64_t rank, PrecondDev& pd, cudaStream_t st) {
  const int64_t n = op.n;
  WGP_REQUIRE(rank >= 0 && rank <= n, "pivoted_cholesky: rank out of range");
  pd.n = n;
  pd.k = 0;
  pd.kpad = rank > 0 ? ((rank + 3) / 4) * 4 : 0;
  if (rank == 0) return;
  pd.L.alloc((size_t)n * pd.kpad);
  WGP_CUDA(cudaMemsetAsync(pd.L.p, 0, sizeof(double) * n * pd.kpad, st));
  const KParams p = op.kp();
  const double dval = p.s2 + p.noise2;  // stationary kernels: every diagonal entry is equal
  DBuf<double> d(n);
  DBuf<int> used(n);
  launch_fill<double>(d.p, dval, n, st);
  WGP_CUDA(cudaMemsetAsync(used.p, 0, sizeof(int) * n, st));
  const double floor_ = 1e-12 * (dval > 0.0 ? dval : 0.0);  // solvers.cpp:77
  const int nb = 148 * 2;
  DBuf<double> pv(nb), root(1);
  DBuf<int64_t> pi(nb), piv(1);
  int64_t hpiv = -1;
  for (int64_t k = 0; k < rank; ++k) {
    argmax_partial_kernel<<<nb, 256, 0, st>>>(d.p, used.p, n, floor_, pv.p, pi.p);
    argmax_final_kernel<<<1, 256, 0, st>>>(pv.p, pi.p, nb, d.p, piv.p, root.p);
    WGP_CUDA(cudaMemcpyAsync(&hpiv, piv.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    if (hpiv < 0) break;  // no positive pivot beyond the floor (solvers.cpp:91)
    pchol_step_kernel<<<grid_rows(n), 256, 0, st>>>(op.X64.p, op.sq64.p, n, op.dpad, op.dim, p,
                                                    (int)k, (int)pd.kpad, piv.p, root.p, pd.L.p,
                                                    d.p, used.p);
    WGP_CUDA(cudaGetLastError());
    pd.k = k + 1;
  }
}

void finish_preconditioner(const Op& op, double shift, int mode, PrecondDev& pd, cudaStream_t st) {
  const int64_t n = pd.n;
  const int k = (int)pd.k;
  if (k == 0) return;
  const KParams p = op.kp();
  const int nb = 148;
  DBuf<double> part((size_t)nb * k * k), G((size_t)k * k);
  gram_partial_kernel<<<nb, 256, 0, st>>>(pd.L.p, n, k, (int)pd.kpad, part.p);
  sum_partials_kernel<<<ceil_div((int64_t)k * k, 256), 256, 0, st>>>(part.p, nb, k * k, G.p);
  WGP_CUDA(cudaGetLastError());
  std::vector<double> cap((size_t)k * k);
  WGP_CUDA(cudaMemcpyAsync(cap.data(), G.p, sizeof(double) * k * k, cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaStreamSynchronize(st));
  if (mode == WGP_SHIFT_CALIBRATED) {  // solvers.cpp:128-131
    const double trace = (double)n * (p.s2 + p.noise2);
    double fro = 0.0;
    for (int a = 0; a < k; ++a) fro += cap[(size_t)a * k + a];  // ||L||_F^2 = tr(L^T L)
    const double leftover = (trace - fro) / (double)n;
    shift += leftover > 0.0 ? leftover : 0.0;
  }
  if (!(shift > 0.0))
    throw_error(WGP_INVALID_ARGUMENT, "CgPreconditioner: shift must be positive for rank > 0");
  pd.shift = shift;
  for (int a = 0; a < k; ++a) cap[(size_t)a * k + a] += shift;
  // Cholesky cap = C C^T (lower, row-major here), Eigen::LLT semantics (solvers.cpp:117-120)
  std::vector<double> Cl((size_t)k * k, 0.0);
  for (int j = 0; j < k; ++j) {
    double x = cap[(size_t)j * k + j];
    for (int t = 0; t < j; ++t) x -= Cl[(size_t)j * k + t] * Cl[(size_t)j * k + t];
    if (!(x > 0.0)) throw_error(WGP_NOT_SPD, "CgPreconditioner: capacitance factorization failed");
    const double ljj = std::sqrt(x);
    Cl[(size_t)j * k + j] = ljj;
    for (int i = j + 1; i < k; ++i) {
      double y = cap[(size_t)i * k + j];
      for (int t = 0; t < j; ++t) y -= Cl[(size_t)i * k + t] * Cl[(size_t)j * k + t];
      Cl[(size_t)i * k + j] = y / ljj;
    }
  }
  // W = C^{-T}: upper triangular, W[t][j] (row-major).  Solve C^T W = I column by column.
  std::vector<double> W((size_t)k * k, 0.0);
  for (int j = 0; j < k; ++j) {
    // column j of C^{-T}: back substitution on C^T x = e_j
    std::vector<double> x(k, 0.0);
    for (int i = k - 1; i >= 0; --i) {
      double y = (i == j) ? 1.0 : 0.0;
      for (int t = i + 1; t < k; ++t) y -= Cl[(size_t)t * k + i] * x[t];
      x[i] = y / Cl[(size_t)i * k + i];
    }
    for (int i = 0; i < k; ++i) W[(size_t)i * k + j] = x[i];
  }
  DBuf<double> dW((size_t)k * k);
  WGP_CUDA(cudaMemcpyAsync(dW.p, W.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, st));
  pd.M64.alloc((size_t)n * pd.kpad);
  const size_t smem = sizeof(double) * k * k;
  if (smem > 48 * 1024)
    WGP_CUDA(cudaFuncSetAttribute(apply_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  apply_upper_kernel<<<grid_rows(n * pd.kpad), 256, smem, st>>>(
      pd.L.p, dW.p, n, k, (int)pd.kpad, pd.M64.p, nullptr);
  WGP_CUDA(cudaGetLastError());
  WGP_CUDA(cudaStreamSynchronize(st));  // dW / part / G are freed on return
}

template <typename T>
void precond_apply(const PrecondDev& pd, const T* R, T* Z, int s, double* work_t,
                   double* work_part, cudaStream_t st) {
  const int64_t n = pd.n;
  const int k = (int)pd.k;
  if (k == 0) {
    WGP_CUDA(cudaMemcpyAsync(Z, R, sizeof(T) * n * s, cudaMemcpyDeviceToDevice, st));
    return;
  }
  WGP_REQUIRE((int64_t)k * s <= 256 * 64, "preconditioner: rank*s too large (%d*%d)", k, s);
  const T* M = (const T*)pd.M64.p;  // solver vectors are fp64 for every precision
  const int nch = ceil_div(n, kChunkRows);
  const size_t smem1 = sizeof(T) * 32 * (pd.kpad + s);
  mtr_partial_kernel<T><<<nch, 256, smem1, st>>>(M, R, n, k, (int)pd.kpad, s, work_part);
  sum_partials_kernel<<<ceil_div((int64_t)k * s, 256), 256, 0, st>>>(work_part, nch, k * s, work_t);
  const size_t smem2 = sizeof(T) * k * s;
  if (smem2 > 48 * 1024)
    WGP_CUDA(cudaFuncSetAttribute(woodbury_out_kernel<T>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  woodbury_out_kernel<T><<<grid_rows(n * s), 256, smem2, st>>>(M, R, work_t, n, k, (int)pd.kpad,
                                                               s, 1.0 / pd.shift, Z);
  WGP_CUDA(cudaGetLastError());
}

template void precond_apply<double>(const PrecondDev&, const double*, double*, int, double*,
                                    double*, cudaStream_t);

}  // namespace wgp
