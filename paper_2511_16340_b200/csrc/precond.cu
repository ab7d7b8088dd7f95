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
                                      int64_t n, int64_t r0, double floor_, double* __restrict__ pv,
                                      int64_t* __restrict__ pi) {
  ArgBest b{0.0, -1};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!used[i] && d[i] > floor_) b = better(b, ArgBest{d[i], r0 + i});
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

// Single block: this rank's best (value, global index) as two doubles (index -1: none).
__global__ void argmax_final_kernel(const double* __restrict__ pv, const int64_t* __restrict__ pi,
                                    int nb, double* __restrict__ best2) {
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
    best2[0] = sv[0];
    best2[1] = (double)si[0];
  }
}

// Single GPU: the global argmax, the pivot index (dpiv, -1 when none is left above the
// floor) and the pivot row lpiv in one block, with no host round trip; kcount = steps done.
__global__ void pivot_select_kernel(const double* __restrict__ pv, const int64_t* __restrict__ pi,
                                    int nb, const double* __restrict__ L,
                                    const double* __restrict__ d, int64_t r0, int k, int kpad,
                                    double* __restrict__ lpiv, int64_t* __restrict__ dpiv,
                                    int* __restrict__ kcount) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  ArgBest b{0.0, -1};
  for (int t = threadIdx.x; t < nb; t += blockDim.x) b = better(b, ArgBest{pv[t], pi[t]});
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
  const int64_t piv = si[0];
  if (threadIdx.x == 0) {
    *dpiv = piv;
    if (piv >= 0) *kcount = k + 1;
  }
  if (piv < 0) return;
  const int64_t li = piv - r0;
  for (int t = threadIdx.x; t < k; t += blockDim.x) lpiv[t] = L[li * kpad + t];
  if (threadIdx.x == 0) lpiv[k] = sqrt(d[li]);
}

// Owner of the pivot row: lpiv[0..k) = L[piv, :k], lpiv[k] = sqrt(d[piv]).
__global__ void fill_pivot_kernel(const double* __restrict__ L, const double* __restrict__ d,
                                  int64_t li, int k, int kpad, double* __restrict__ lpiv) {
  for (int t = threadIdx.x; t < k; t += blockDim.x) lpiv[t] = L[li * kpad + t];
  if (threadIdx.x == 0) lpiv[k] = sqrt(d[li]);
}

// One pivoted-Cholesky step for every local row (solvers.cpp:93-103); the pivot row of L
// and root = sqrt(d[piv]) arrive in lpiv (broadcast from the owning rank).
__global__ void pchol_step_kernel(const double* __restrict__ X, const double* __restrict__ sq,
                                  int64_t n_local, int64_t r0, int dpad, int dim, KParams p, int k,
                                  int kpad, const int64_t* __restrict__ dpiv,
                                  const double* __restrict__ lpiv, double* __restrict__ L,
                                  double* __restrict__ d, int* __restrict__ used) {
  const int64_t piv = *dpiv;
  if (piv < 0) return;  // no pivot at this step (the factorisation stopped early)
  const double root = lpiv[k];
  const double* xp = X + piv * dpad;
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n_local;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r0 + li;
    double h;
    if (i == piv) {
      h = p.s2 + p.noise2;
    } else {
      const double* xi = X + i * dpad;
      double g = 0.0;
      for (int t = 0; t < dim; ++t) g += xi[t] * xp[t];
      h = kmap64(sq[i] + sq[piv] - 2.0 * g, p);
    }
    double* Li = L + li * kpad;
    double col = h;
    for (int t = 0; t < k; ++t) col -= Li[t] * lpiv[t];
    const double lik = (i == piv) ? root : col / root;
    Li[k] = lik;
    if (i == piv) {
      used[li] = 1;
      d[li] = 0.0;
    } else if (!used[li]) {
      d[li] -= lik * lik;
    }
  }
}

// Per-chunk partials of A^T B (A: [n][lda], B: [n][ldb] local rows, row-major):
// part[chunk][a][c] = sum over the chunk's rows, in row order, of A[i][a] B[i][c] for a < ka,
// c < kb.  Grid (chunk, a-block of 64, c-block of 64); the chunk's rows are staged 32 at a
// time in shared memory and each thread owns a 4 x 4 output tile (8 shared loads per 16
// FMAs).  Every output is one fma chain over the rows in order, so the partial does not
// depend on the tiling, and chunk q of the local rows is global chunk c0 + q: the fixed-order
// sum over chunks is world-size independent.
__global__ void __launch_bounds__(256) chunk_atb_kernel(const double* __restrict__ A, int lda, int ka,
                                                        const double* __restrict__ B, int ldb, int kb,
                                                        int64_t n, double* __restrict__ part) {
  constexpr int RT = 32;
  __shared__ double sA[RT][64 + 1], sB[RT][64 + 1];
  const int64_t r0 = (int64_t)blockIdx.x * kChunkRows;
  const int64_t r1 = min(n, r0 + (int64_t)kChunkRows);
  const int a0 = blockIdx.y * 64, c0 = blockIdx.z * 64;
  const int ta = (threadIdx.x / 16) * 4, tc = (threadIdx.x % 16) * 4;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += RT) {
    __syncthreads();
    for (int e = threadIdx.x; e < RT * 64; e += 256) {
      const int r = e / 64, q = e % 64;
      const int64_t i = rb + r;
      sA[r][q] = (i < r1 && a0 + q < ka) ? A[i * lda + a0 + q] : 0.0;
      sB[r][q] = (i < r1 && c0 + q < kb) ? B[i * ldb + c0 + q] : 0.0;
    }
    __syncthreads();
    const int rows = (int)(r1 - rb < RT ? r1 - rb : RT);
    for (int ii = 0; ii < rows; ++ii) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = sA[ii][ta + u];
        bv[u] = sB[ii][tc + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
  }
  double* out = part + (int64_t)blockIdx.x * ka * kb;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int a = a0 + ta + u, c = c0 + tc + v;
      if (a < ka && c < kb) out[(int64_t)a * kb + c] = acc[u][v];
    }
}

// Narrow right-hand sides (s <= 8): the same partials as chunk_atb_kernel -- one fma chain per
// output over the chunk's rows in order, so the bits do not depend on which kernel ran -- with
// one thread per (a, column) instead of 4 x 4 register tiles that would leave all but s of
// every 64 output columns idle.  Block = 128 a values (k <= 128 per block), grid.y = s.
__global__ void __launch_bounds__(128) chunk_atb_narrow_kernel(const double* __restrict__ A, int lda,
                                                               int ka, const double* __restrict__ B,
                                                               int ldb, int kb, int64_t n,
                                                               double* __restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * kChunkRows;
  const int64_t r1 = min(n, r0 + (int64_t)kChunkRows);
  const int a = blockIdx.z * 128 + threadIdx.x, c = blockIdx.y;
  if (a >= ka) return;
  double acc = 0.0;
  int64_t i = r0;
  for (; i + 8 <= r1; i += 8) {
    double av[8], bv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      av[u] = A[(i + u) * lda + a];
      bv[u] = B[(i + u) * ldb + c];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fma(av[u], bv[u], acc);
  }
  for (; i < r1; ++i) acc = fma(A[i * lda + a], B[i * ldb + c], acc);
  part[(int64_t)blockIdx.x * ka * kb + (int64_t)a * kb + c] = acc;
}

// Narrow right-hand sides: z = (r - M t) / shift with one thread per row computing all s
// (<= 8) columns -- each output one fma chain over a in order, as woodbury_tile_kernel.
template <int SC>
__global__ void __launch_bounds__(128) woodbury_narrow_kernel(const double* __restrict__ M, int kpad,
                                                              int k, const double* __restrict__ R,
                                                              int64_t ld, const double* __restrict__ t,
                                                              int s, int64_t n, double inv_shift,
                                                              double* __restrict__ Z) {
  constexpr int AT = 32;
  __shared__ double sM[128][AT + 1], sT[AT][SC];
  const int64_t rb = (int64_t)blockIdx.x * 128;
  const int64_t i = rb + threadIdx.x;
  double acc[SC];
#pragma unroll
  for (int v = 0; v < SC; ++v) acc[v] = 0.0;
  for (int a0 = 0; a0 < k; a0 += AT) {
    __syncthreads();
    for (int e = threadIdx.x; e < 128 * AT; e += 128) {
      const int r = e / AT, a = e % AT;
      sM[r][a] = (rb + r < n && a0 + a < k) ? M[(rb + r) * kpad + a0 + a] : 0.0;
    }
    for (int e = threadIdx.x; e < AT * SC; e += 128) {
      const int a = e / SC, c = e % SC;
      sT[a][c] = (a0 + a < k && c < s) ? t[(int64_t)(a0 + a) * s + c] : 0.0;
    }
    __syncthreads();
    const int na = min(AT, k - a0);
    for (int a = 0; a < na; ++a) {
      const double m = sM[threadIdx.x][a];
#pragma unroll
      for (int v = 0; v < SC; ++v) acc[v] = fma(m, sT[a][v], acc[v]);
    }
  }
  if (i >= n) return;
#pragma unroll
  for (int v = 0; v < SC; ++v)
    if (v < s) Z[i * ld + v] = (R[i * ld + v] - acc[v]) * inv_shift;
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int np, int count,
                                    double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
    out[e] = chunk_sum_ordered(part + e, np, count);
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

// Z[i, c] = (R[i, c] - sum_a M[i, a] t[a, c]) / shift  (R, Z: s columns of row-major [n][ld]).
// 64 rows x 64 columns per CTA, 4 x 4 outputs per thread; M and t are staged 32 a at a time
// in shared memory; each output is one fma chain over a in order.
__global__ void __launch_bounds__(256) woodbury_tile_kernel(const double* __restrict__ M, int kpad, int k,
                                                            const double* __restrict__ R, int64_t ld,
                                                            const double* __restrict__ t, int s, int64_t n,
                                                            double inv_shift, double* __restrict__ Z) {
  constexpr int AT = 32;
  __shared__ double sM[64][AT + 1], sT[AT][64 + 1];
  const int64_t rb = (int64_t)blockIdx.x * 64;
  const int cb = blockIdx.y * 64;
  const int tr = (threadIdx.x / 16) * 4, tc = (threadIdx.x % 16) * 4;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int a0 = 0; a0 < k; a0 += AT) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * AT; e += 256) {
      const int r = e / AT, a = e % AT;
      sM[r][a] = (rb + r < n && a0 + a < k) ? M[(rb + r) * kpad + a0 + a] : 0.0;
      const int a2 = e / 64, c = e % 64;
      sT[a2][c] = (a0 + a2 < k && cb + c < s) ? t[(int64_t)(a0 + a2) * s + cb + c] : 0.0;
    }
    __syncthreads();
    const int na = min(AT, k - a0);
    for (int a = 0; a < na; ++a) {
      double mv[4], tv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mv[u] = sM[tr + u][a];
        tv[u] = sT[a][tc + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(mv[u], tv[v], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = rb + tr + u;
    if (i >= n) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = cb + tc + v;
      if (c < s) Z[i * ld + c] = (R[i * ld + c] - acc[u][v]) * inv_shift;
    }
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
  int64_t r0, r1;
  op.local_rows(&r0, &r1);
  const int64_t nl = r1 - r0;
  const Ctx& ctx = *op.ctx;
  pd.n = n;
  pd.r0 = r0;
  pd.n_local = nl;
  pd.k = 0;
  pd.kpad = rank > 0 ? ((rank + 3) / 4) * 4 : 0;
  if (rank == 0) return;
  pd.L.ensure_grow((size_t)std::max<int64_t>(nl, 1) * pd.kpad);
  WGP_CUDA(cudaMemsetAsync(pd.L.p, 0, sizeof(double) * std::max<int64_t>(nl, 1) * pd.kpad, st));
  const KParams p = op.kp();
  const double dval = p.s2 + p.noise2;  // stationary kernels: every diagonal entry is equal
  DBuf<double>& d = pd.w_d;
  DBuf<int>& used = pd.w_used;
  d.ensure_grow(std::max<int64_t>(nl, 1));
  used.ensure_grow(std::max<int64_t>(nl, 1));
  launch_fill<double>(d.p, dval, nl, st);
  WGP_CUDA(cudaMemsetAsync(used.p, 0, sizeof(int) * std::max<int64_t>(nl, 1), st));
  const double floor_ = 1e-12 * (dval > 0.0 ? dval : 0.0);  // solvers.cpp:77
  const int nb = 148 * 2;
  DBuf<double>& pv = pd.w_pv;
  DBuf<double>& best2 = pd.w_best2;
  DBuf<double>& all2 = pd.w_all2;
  DBuf<double>& lpiv = pd.w_lpiv;
  DBuf<int64_t>& pi = pd.w_pi;
  DBuf<int64_t>& dpiv = pd.w_dpiv;
  pv.ensure(nb);
  best2.ensure(2);
  all2.ensure((size_t)2 * ctx.world);
  lpiv.ensure(pd.kpad + 1);
  pi.ensure(nb);
  dpiv.ensure(1);
  if (ctx.world == 1) {
    // no host synchronisation per pivot: selection, pivot row and the early stop all stay
    // on the device; one read of the achieved rank at the end
    DBuf<int>& kcount = pd.w_kcount;
    kcount.ensure(1);
    WGP_CUDA(cudaMemsetAsync(kcount.p, 0, sizeof(int), st));
    for (int64_t k = 0; k < rank; ++k) {
      argmax_partial_kernel<<<nb, 256, 0, st>>>(d.p, used.p, nl, r0, floor_, pv.p, pi.p);
      pivot_select_kernel<<<1, 256, 0, st>>>(pv.p, pi.p, nb, pd.L.p, d.p, r0, (int)k, (int)pd.kpad,
                                             lpiv.p, dpiv.p, kcount.p);
      pchol_step_kernel<<<grid_rows(std::max<int64_t>(nl, 1)), 256, 0, st>>>(
          op.X64.p, op.sq64.p, nl, r0, op.dpad, op.dim, p, (int)k, (int)pd.kpad, dpiv.p, lpiv.p,
          pd.L.p, d.p, used.p);
    }
    WGP_CUDA(cudaGetLastError());
    int kc = 0;
    WGP_CUDA(cudaMemcpyAsync(&kc, kcount.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    pd.k = kc;
    return;
  }
  std::vector<double> h_all((size_t)2 * ctx.world);
  for (int64_t k = 0; k < rank; ++k) {
    argmax_partial_kernel<<<nb, 256, 0, st>>>(d.p, used.p, nl, r0, floor_, pv.p, pi.p);
    argmax_final_kernel<<<1, 256, 0, st>>>(pv.p, pi.p, nb, best2.p);
    dist_allgather(ctx, best2.p, all2.p, 2, st);
    WGP_CUDA(cudaMemcpyAsync(h_all.data(), all2.p, sizeof(double) * h_all.size(),
                             cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    // global argmax: strict '>' scan order == larger value, then lower index
    int64_t piv = -1;
    double bv = 0.0;
    for (int r = 0; r < ctx.world; ++r) {
      const int64_t idx = (int64_t)h_all[2 * r + 1];
      if (idx < 0) continue;
      const double v = h_all[2 * r];
      if (piv < 0 || v > bv || (v == bv && idx < piv)) {
        piv = idx;
        bv = v;
      }
    }
    if (piv < 0) break;  // no positive pivot beyond the floor (solvers.cpp:91)
    const int owner = owner_rank(ctx, n, piv);
    if (owner == ctx.rank) fill_pivot_kernel<<<1, 128, 0, st>>>(pd.L.p, d.p, piv - r0, (int)k, (int)pd.kpad, lpiv.p);
    dist_broadcast(ctx, lpiv.p, sizeof(double) * (pd.kpad + 1), owner, st);
    WGP_CUDA(cudaMemcpyAsync(dpiv.p, &piv, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    pchol_step_kernel<<<grid_rows(std::max<int64_t>(nl, 1)), 256, 0, st>>>(
        op.X64.p, op.sq64.p, nl, r0, op.dpad, op.dim, p, (int)k, (int)pd.kpad, dpiv.p, lpiv.p,
        pd.L.p, d.p, used.p);
    WGP_CUDA(cudaGetLastError());  // (a pageable-source copy has read piv on return)
    pd.k = k + 1;
  }
}

void finish_preconditioner(const Op& op, double shift, int mode, PrecondDev& pd, cudaStream_t st) {
  const int64_t n = pd.n;
  const int k = (int)pd.k;
  if (k == 0) return;
  const KParams p = op.kp();
  const int nch = ceil_div(n, kChunkRows);
  const int c0 = (int)(pd.r0 / kChunkRows);
  DBuf<double>& part = pd.w_part;
  DBuf<double>& G = pd.w_G;
  part.ensure_grow((size_t)padded_chunks(n, op.ctx->world) * k * k);
  G.ensure((size_t)k * k);
  if (pd.n_local > 0)
    chunk_atb_kernel<<<dim3(ceil_div(pd.n_local, kChunkRows), ceil_div(k, 64), ceil_div(k, 64)), 256, 0, st>>>(
        pd.L.p, (int)pd.kpad, k, pd.L.p, (int)pd.kpad, k, pd.n_local, part.p + (int64_t)c0 * k * k);
  dist_allgather_chunks(*op.ctx, part.p, n, (int64_t)k * k, st);
  sum_partials_kernel<<<ceil_div((int64_t)k * k, 256), 256, 0, st>>>(part.p, nch, k * k, G.p);
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
  DBuf<double>& dW = pd.w_W;
  dW.ensure((size_t)k * k);
  WGP_CUDA(cudaMemcpyAsync(dW.p, W.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, st));
  const int64_t nl = std::max<int64_t>(pd.n_local, 1);
  pd.M64.ensure_grow((size_t)nl * pd.kpad);
  const size_t smem = sizeof(double) * k * k;
  if (smem > 48 * 1024)
    WGP_CUDA(cudaFuncSetAttribute(apply_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  apply_upper_kernel<<<grid_rows(nl * pd.kpad), 256, smem, st>>>(
      pd.L.p, dW.p, pd.n_local, k, (int)pd.kpad, pd.M64.p, nullptr);
  WGP_CUDA(cudaGetLastError());
  WGP_CUDA(cudaStreamSynchronize(st));  // (dW is rewritten by the next build's host copy)
}

template <typename T>
void precond_apply(const Op& op, const PrecondDev& pd, const T* R, T* Z, int s, double* work_t,
                   double* work_part, cudaStream_t st) {
  const int64_t nl = pd.n_local;
  const int k = (int)pd.k;
  if (k == 0) {
    if (nl > 0) WGP_CUDA(cudaMemcpyAsync(Z, R, sizeof(T) * nl * s, cudaMemcpyDeviceToDevice, st));
    return;
  }
  static_assert(sizeof(T) == sizeof(double), "solver vectors are fp64 for every precision");
  const double* M = pd.M64.p;
  const int nch = ceil_div(pd.n, kChunkRows);
  const int c0 = (int)(pd.r0 / kChunkRows);
  // t = M^T r: chunk partials (fixed order, world-size independent), then summed
  if (nl > 0 && s <= 8)
    chunk_atb_narrow_kernel<<<dim3(ceil_div(nl, kChunkRows), s, ceil_div(k, 128)), 128, 0, st>>>(
        M, (int)pd.kpad, k, R, s, s, nl, work_part + (int64_t)c0 * k * s);
  else if (nl > 0)
    chunk_atb_kernel<<<dim3(ceil_div(nl, kChunkRows), ceil_div(k, 64), ceil_div(s, 64)), 256, 0, st>>>(
        M, (int)pd.kpad, k, R, s, s, nl, work_part + (int64_t)c0 * k * s);
  WGP_CUDA(cudaGetLastError());
  dist_allgather_chunks(*op.ctx, work_part, pd.n, (int64_t)k * s, st);
  sum_partials_kernel<<<ceil_div((int64_t)k * s, 256), 256, 0, st>>>(work_part, nch, k * s, work_t);
  // z = (r - M t) / shift
  if (nl > 0 && s <= 8) {
    const dim3 g(ceil_div(nl, 128));
    const double is = 1.0 / pd.shift;
    if (s <= 1) woodbury_narrow_kernel<1><<<g, 128, 0, st>>>(M, (int)pd.kpad, k, R, s, work_t, s, nl, is, Z);
    else if (s <= 2) woodbury_narrow_kernel<2><<<g, 128, 0, st>>>(M, (int)pd.kpad, k, R, s, work_t, s, nl, is, Z);
    else if (s <= 4) woodbury_narrow_kernel<4><<<g, 128, 0, st>>>(M, (int)pd.kpad, k, R, s, work_t, s, nl, is, Z);
    else woodbury_narrow_kernel<8><<<g, 128, 0, st>>>(M, (int)pd.kpad, k, R, s, work_t, s, nl, is, Z);
  } else if (nl > 0) {
    woodbury_tile_kernel<<<dim3(ceil_div(nl, 64), ceil_div(s, 64)), 256, 0, st>>>(
        M, (int)pd.kpad, k, R, s, work_t, s, nl, 1.0 / pd.shift, Z);
  }
  WGP_CUDA(cudaGetLastError());
}

template void precond_apply<double>(const Op&, const PrecondDev&, const double*, double*, int,
                                    double*, double*, cudaStream_t);

}  // namespace wgp
