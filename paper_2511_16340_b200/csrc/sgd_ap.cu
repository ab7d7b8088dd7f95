// sgd_ap.cu -- device kernels for the SGD and alternating-projection solvers.
//
//   krows   g[c][i] = H[row_ci, :] . v_c - b_c[row_ci]   (SGD minibatch rows, solvers.cpp:225-228)
//   kcols   r_c -= H[:, B_c] delta_c                      (AP block column update, solvers.cpp:292)
//   block_chol  H_BB = L L^T per contiguous block + L^-1  (AP factorisation, solvers.cpp:255-264)
//   ap_block_solve  delta_c = L^-T L^-1 r_c[B_c]; v_c[B_c] += delta_c   (solvers.cpp:290-291)
//   block_norms / greedy argmax (solvers.cpp:277-286, ties -> lowest block index)
//
// Kernel entries are evaluated on the fly from X with the same per-pair formula as the
// kernel-matvec (explicit differences; H(i,i) = s^2 + sigma_n^2 exactly), in the operator's
// compute type (fp64, or fp32 for the fp32 precisions).  Per-column work of different
// columns is independent, so batching columns never changes a column's result.
#include <algorithm>

#include "solvers.h"

namespace wgp {
namespace {

template <typename T>
__device__ __forceinline__ T kentry(const T* __restrict__ xi, const T* __restrict__ xj, int dim,
                                    const KParams& p) {
  T d2 = T(0);
  for (int k = 0; k < dim; ++k) {
    const T df = xi[k] - xj[k];
    d2 = fma(df, df, d2);
  }
  if (p.kind == WGP_RBF) return T(p.s2) * exp(-T(p.c1) * d2);
  const T z = T(p.c1) * sqrt(d2);
  return T(p.s2) * (T(1) + z) * exp(-z);
}

__device__ __forceinline__ double kexp(double x) { return exp_neg(x); }  // x <= 0
__device__ __forceinline__ float kexp(float x) { return expf(x); }

// One block = 64 gathered rows of one column over one fixed-length j range (grid.z); 4
// threads per row take every 4th j of each 64-column tile.  Partial sums go to
// part[z][c][i] and krows_sum_kernel adds the ranges in order: the j ranges depend on n only,
// so a row's value is the same whichever rank owns it.
// One 64-row tile row of coordinates into registers as 16-byte vector loads: the per-pair
// coordinate reads of krows / kcols were one 4- or 8-byte shared load per dimension (8 per pair
// at d = 8: the kernels were shared-load bound); all lanes read the same row (broadcast).
template <typename T, int DMAX>
__device__ __forceinline__ void load_row(const T (&row)[DMAX], T (&out)[DMAX]) {
  static_assert((DMAX * sizeof(T)) % 16 == 0, "rows of whole 16-byte vectors");
  const uint4* src = reinterpret_cast<const uint4*>(row);
  uint4* dst = reinterpret_cast<uint4*>(out);
#pragma unroll
  for (int q = 0; q < (int)(DMAX * sizeof(T) / 16); ++q) dst[q] = src[q];
}

template <typename T, int DMAX>
__global__ void __launch_bounds__(256) krows_kernel(const T* __restrict__ X, int dpad, int dim,
                                                    int64_t n, int64_t jlen,
                                                    const int* __restrict__ rows, int nb,
                                                    const double* __restrict__ V, int s,
                                                    const int* __restrict__ active, KParams p,
                                                    int64_t r0, int64_t r1,
                                                    double* __restrict__ part) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  // fp32 rows read whole with 16-byte vector loads (broadcast): krows 323 -> 304 us at C2;
  // fp64 rows keep per-element loads (the vector form measured 596 -> 726 us there)
  constexpr int PADX = sizeof(T) == 4 ? 0 : 1;
  __shared__ __align__(16) T sX[64][DMAX + PADX];
  __shared__ double sV[64];
  __shared__ double red[256];
  const int tid = threadIdx.x;
  const int lr = tid >> 2, sub = tid & 3;
  const int bi = blockIdx.x * 64 + lr;
  const int64_t row = bi < nb ? rows[(int64_t)c * nb + bi] : 0;
  // sharded: this rank owns rows [r0, r1) (B holds those rows only); other batch rows get 0
  const bool valid = bi < nb && row >= r0 && row < r1;
  T xr[DMAX];
#pragma unroll
  for (int k = 0; k < DMAX; ++k) xr[k] = (valid && k < dim) ? X[row * dpad + k] : T(0);
  const T s2 = T(p.s2), c1 = T(p.c1), kdiag = T(p.s2 + p.noise2);
  const int64_t j_lo = (int64_t)blockIdx.z * jlen, j_hi = min(n, j_lo + jlen);
  double acc = 0.0;
  for (int64_t j0 = j_lo; j0 < j_hi; j0 += 64) {
    __syncthreads();
    for (int e = tid; e < 64 * DMAX; e += 256) {  // coordinates >= dim are zero
      const int j = e / DMAX, k = e % DMAX;
      sX[j][k] = (j0 + j < j_hi && k < dim) ? X[(j0 + j) * dpad + k] : T(0);
    }
    if (tid < 64) sV[tid] = j0 + tid < j_hi ? V[(j0 + tid) * s + c] : 0.0;
    __syncthreads();
    if (valid) {
      const int jn = (int)(j_hi - j0 < 64 ? j_hi - j0 : 64);
      const int64_t dl = row - j0;  // the diagonal entry's position in this tile, if any
      const int jd = (dl >= 0 && dl < jn) ? (int)dl : -1;
      for (int jj = sub; jj < jn; jj += 4) {
        T d2 = T(0);
        if constexpr (sizeof(T) == 4) {
          T xj[DMAX];
          load_row<T, DMAX>(sX[jj], xj);
#pragma unroll
          for (int k = 0; k < DMAX; ++k) {
            const T df = xr[k] - xj[k];
            d2 = fma(df, df, d2);
          }
        } else {
#pragma unroll
          for (int k = 0; k < DMAX; ++k) {
            const T df = xr[k] - sX[jj][k];
            d2 = fma(df, df, d2);
          }
        }
        T kv;
        if (jj == jd) {
          kv = kdiag;
        } else if (p.kind == WGP_RBF) {
          kv = s2 * kexp(-c1 * d2);
        } else {
          const T z = c1 * sqrt(d2);
          kv = s2 * (T(1) + z) * kexp(-z);
        }
        acc = fma((double)kv, sV[jj], acc);
      }
    }
  }
  red[tid] = acc;
  __syncthreads();
  if (bi < nb && sub == 0)
    part[((int64_t)blockIdx.z * s + c) * nb + bi] = ((red[tid] + red[tid + 1]) + red[tid + 2]) + red[tid + 3];
}

// g[c][i] = sum over the j ranges in order - b_c[row] (owned rows; 0 elsewhere).
__global__ void krows_sum_kernel(const double* __restrict__ part, int nsplit, const int* __restrict__ rows,
                                 int nb, const double* __restrict__ Bm, int s,
                                 const int* __restrict__ active, int64_t r0, int64_t r1,
                                 double* __restrict__ g) {
  const int c = blockIdx.y;
  const int bi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= nb || !active[c]) return;
  const int64_t row = rows[(int64_t)c * nb + bi];
  const bool own = row >= r0 && row < r1;
  double tot = 0.0;
  for (int q = 0; q < nsplit; ++q) tot += part[((int64_t)q * s + c) * nb + bi];
  g[(int64_t)c * nb + bi] = own ? tot - Bm[(row - r0) * s + c] : 0.0;
}

// r[i, c] -= sum_{j in block_c} H[i, j] delta[j - start_c, c]    (thread per row i)
template <typename T, int DMAX>
__global__ void __launch_bounds__(128) kcols_kernel(const T* __restrict__ X, int dpad, int dim,
                                                    int64_t n, const int* __restrict__ blk,
                                                    int bs, const double* __restrict__ delta,
                                                    int s, const int* __restrict__ active,
                                                    KParams p, int64_t r0, int64_t nrows,
                                                    double* __restrict__ R) {
  // rows r0 .. r0 + nrows of the operator (this rank's), R holds those rows
  const int c = blockIdx.y;
  if (!active[c]) return;
  // fp32 rows read whole with 16-byte vector loads (broadcast): krows 323 -> 304 us at C2;
  // fp64 rows keep per-element loads (the vector form measured 596 -> 726 us there)
  constexpr int PADX = sizeof(T) == 4 ? 0 : 1;
  __shared__ __align__(16) T sX[64][DMAX + PADX];
  __shared__ double sD[64];
  const int64_t il = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const bool valid = il < nrows;
  const int64_t i = r0 + il;
  const int64_t start = (int64_t)blk[c] * bs;
  const int len = (int)min((int64_t)bs, n - start);
  T xr[DMAX];
#pragma unroll
  for (int k = 0; k < DMAX; ++k) xr[k] = (valid && k < dim) ? X[i * dpad + k] : T(0);
  const T s2 = T(p.s2), c1 = T(p.c1), kdiag = T(p.s2 + p.noise2);
  double acc = 0.0;
  for (int j0 = 0; j0 < len; j0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * DMAX; e += 128) {  // coordinates >= dim are zero
      const int j = e / DMAX, k = e % DMAX;
      sX[j][k] = (j0 + j < len && k < dim) ? X[(start + j0 + j) * dpad + k] : T(0);
    }
    if (threadIdx.x < 64) sD[threadIdx.x] = j0 + threadIdx.x < len ? delta[(int64_t)(j0 + threadIdx.x) * s + c] : 0.0;
    __syncthreads();
    if (valid) {
      const int m = min(64, len - j0);
      // the diagonal entry of this tile, if row i lies in it (a 32-bit compare per pair
      // instead of a 64-bit index sum and compare)
      const int64_t dl = i - (start + j0);
      const int jd = (dl >= 0 && dl < m) ? (int)dl : -1;
      for (int jj = 0; jj < m; ++jj) {
        T d2 = T(0);
        if constexpr (sizeof(T) == 4) {
          T xj[DMAX];
          load_row<T, DMAX>(sX[jj], xj);
#pragma unroll
          for (int k = 0; k < DMAX; ++k) {
            const T df = xr[k] - xj[k];
            d2 = fma(df, df, d2);
          }
        } else {
#pragma unroll
          for (int k = 0; k < DMAX; ++k) {
            const T df = xr[k] - sX[jj][k];
            d2 = fma(df, df, d2);
          }
        }
        T kv;
        if (jj == jd) {
          kv = kdiag;
        } else if (p.kind == WGP_RBF) {
          kv = s2 * kexp(-c1 * d2);
        } else {
          const T z = c1 * sqrt(d2);
          kv = s2 * (T(1) + z) * kexp(-z);
        }
        acc = fma((double)kv, sD[jj], acc);
      }
    }
  }
  if (valid) R[il * s + c] -= acc;
}

// One CTA per block: A = H_BB (fp64, from X64), in-place lower Cholesky, then L^-1.
// fac: [n_blocks][bs][bs] row-major (lower L); inv: same shape (lower L^-1).
__global__ void __launch_bounds__(512) block_chol_kernel(const double* __restrict__ X, int dpad,
                                                         int dim, int64_t n, int bs, KParams p,
                                                         double* __restrict__ fac,
                                                         double* __restrict__ inv,
                                                         int* __restrict__ fail) {
  const int blkid = blockIdx.x;
  const int64_t start = (int64_t)blkid * bs;
  const int len = (int)min((int64_t)bs, n - start);
  double* A = fac + (int64_t)blkid * bs * bs;
  double* Li = inv + (int64_t)blkid * bs * bs;
  // H_BB with the reference's exactly-set diagonal (kernel.cpp:70)
  for (int e = threadIdx.x; e < len * len; e += blockDim.x) {
    const int a = e / len, b = e % len;
    double v;
    if (a == b) {
      v = p.s2 + p.noise2;
    } else {
      v = kentry<double>(X + (start + a) * dpad, X + (start + b) * dpad, dim, p);
    }
    A[a * bs + b] = v;
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  // right-looking Cholesky (Eigen::LLT semantics: pivot must be > 0)
  for (int j = 0; j < len; ++j) {
    __shared__ double ljj;
    if (threadIdx.x == 0) {
      const double x = A[j * bs + j];
      if (!(x > 0.0)) bad = 1;
      ljj = sqrt(x > 0.0 ? x : 1.0);
      A[j * bs + j] = ljj;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < len; i += blockDim.x) A[i * bs + j] /= ljj;
    __syncthreads();
    const int m = len - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int a = j + 1 + e / m, b = j + 1 + e % m;
      if (b <= a) A[a * bs + b] -= A[a * bs + j] * A[b * bs + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && bad) atomicExch(fail, 1);
  // L^-1 column by column (thread per column): Li[i][col] = (delta_i,col - sum_k L_ik Li_k,col)/L_ii
  for (int col = threadIdx.x; col < len; col += blockDim.x) {
    for (int i = 0; i < len; ++i) {
      double v = (i == col) ? 1.0 : 0.0;
      if (i < col) {
        Li[i * bs + col] = 0.0;
        continue;
      }
      for (int k = col; k < i; ++k) v -= A[i * bs + k] * Li[k * bs + col];
      Li[i * bs + col] = v / A[i * bs + i];
    }
  }
}

// delta_c = L^-T (L^-1 r_c[B]) for the column's chosen block; v_c[B] += delta_c.  The block's
// residual rows come from the full residual R (rows [start, start + len)) or, when Rblk is
// given, from the gathered block rows Rblk[i][c] (sharded solves).
// delta = (L L^T)^{-1} r_B for each active column's chosen block, with Li = L^{-1} (lower,
// block_chol): y = Li r in ap_block_y_kernel, delta = Li^T y (and v_B += delta) in
// ap_block_delta_kernel.  Grids of (column, row slice) CTAs -- one CTA per column left 131 of
// 148 SMs idle (138 us per iteration at C2) -- and y's rows by warps with lanes along k, so
// the reads of Li are coalesced (one thread per row of Li read it 4 KB apart).  Fixed orders:
// y[i] = 32-lane partial sums over k combined by xor-shuffle; delta[j] = 8 warp partials (rows
// i = w mod 8, ascending) added in warp order.
constexpr int kApRowsPerCta = 32;
__global__ void __launch_bounds__(256) ap_block_y_kernel(
    const double* __restrict__ inv, int bs, int64_t n, const int* __restrict__ blk,
    const int* __restrict__ active, const double* __restrict__ R, const double* __restrict__ Rblk,
    int s, double* __restrict__ ybuf) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  extern __shared__ double rb[];  // bs
  const int64_t start = (int64_t)blk[c] * bs;
  const int len = (int)min((int64_t)bs, n - start);
  const double* Li = inv + (int64_t)blk[c] * bs * bs;
  for (int i = threadIdx.x; i < len; i += blockDim.x)
    rb[i] = Rblk ? Rblk[(int64_t)i * s + c] : R[(start + i) * s + c];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * kApRowsPerCta;
  for (int i = i0 + warp; i < min(len, i0 + kApRowsPerCta); i += blockDim.x / 32) {
    double a = 0.0;
    for (int k = lane; k <= i; k += 32) a = fma(Li[(int64_t)i * bs + k], rb[k], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) ybuf[(int64_t)i * s + c] = a;
  }
}

__global__ void __launch_bounds__(256) ap_block_delta_kernel(
    const double* __restrict__ inv, int bs, int64_t n, const int* __restrict__ blk,
    const int* __restrict__ active, const double* __restrict__ ybuf, int s, double* __restrict__ V,
    double* __restrict__ delta) {
  // CTA = (32 consecutive j, column c); warp w adds rows i = j0 + w, j0 + w + 8, ... (lanes
  // along j: coalesced rows of Li), the 8 warp partials are then added in warp order
  const int c = blockIdx.y;
  if (!active[c]) return;
  __shared__ double part[8][32];
  extern __shared__ double ys[];  // y[j0 .. len)
  const int64_t start = (int64_t)blk[c] * bs;
  const int len = (int)min((int64_t)bs, n - start);
  const double* Li = inv + (int64_t)blk[c] * bs * bs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * 32, j = j0 + lane;
  for (int i = j0 + threadIdx.x; i < len; i += blockDim.x) ys[i - j0] = ybuf[(int64_t)i * s + c];
  __syncthreads();
  double a = 0.0;
  if (j < len)
    for (int i = j0 + warp; i < len; i += 8)
      if (i >= j) a = fma(Li[(int64_t)i * bs + j], ys[i - j0], a);
  part[warp][lane] = a;
  __syncthreads();
  if (warp == 0 && j < len) {
    double d = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) d += part[w][lane];
    delta[(int64_t)j * s + c] = d;
    V[(start + j) * s + c] += d;
  }
}

// Greedy block choice (solvers.cpp:277-286), in two steps so that a row-sharded residual
// gives bitwise the one-GPU choice: the rows are cut into segments at every block boundary
// and every kChunkRows boundary (a segment lies in one block and one chunk, so one rank owns
// it); seg_norms writes the squared norm of each segment this rank owns (32-lane
// interleaved sums + xor-shuffle, a fixed order) and 0 for the others -- summed over ranks
// exactly, since one rank contributes each value -- and greedy_from_segments adds a block's
// segments in order, takes the square root and the argmax (strict >, first wins).
__global__ void seg_norms_kernel(const double* __restrict__ Rloc, int64_t r0, int64_t nloc,
                                 const int64_t* __restrict__ seg_start, int nseg, int s,
                                 const int* __restrict__ active, double* __restrict__ segn) {
  const int c = blockIdx.x;
  for (int g = threadIdx.y; g < nseg; g += blockDim.y) {
    const int64_t a0 = seg_start[g], a1 = seg_start[g + 1];
    double a = 0.0;
    if (active[c] && a0 >= r0 && a0 < r0 + nloc) {
      for (int64_t i = a0 + threadIdx.x; i < a1; i += 32) {
        const double r = Rloc[(i - r0) * s + c];
        a = fma(r, r, a);
      }
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    }
    if (threadIdx.x == 0) segn[(int64_t)g * s + c] = a;
  }
}

__global__ void __launch_bounds__(128) greedy_from_segments_kernel(
    const double* __restrict__ segn, const int* __restrict__ seg_block, int nseg, int nblk, int s,
    const int* __restrict__ active, int* __restrict__ blk) {
  // one block per column: the segment norms load in parallel (the single-thread scan of
  // round 1 was a chain of dependent L2 loads, 48 us at C2), then one thread adds each
  // block's segments in order and takes the argmax
  extern __shared__ double sn[];  // nseg
  const int c = blockIdx.x;
  if (!active[c]) return;
  for (int g = threadIdx.x; g < nseg; g += blockDim.x) sn[g] = segn[(int64_t)g * s + c];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double best = -1.0, cur = 0.0;
  int arg = 0;
  for (int g = 0; g < nseg; ++g) {
    cur += sn[g];
    if (g + 1 == nseg || seg_block[g + 1] != seg_block[g]) {
      const double nrm = sqrt(cur);
      if (nrm > best) {
        best = nrm;
        arg = seg_block[g];
      }
      cur = 0.0;
    }
  }
  blk[c] = arg;
}

// Rows of each active column's chosen block that this rank owns -> Rblk[i][c] (0 for rows of
// other ranks): the exact all-reduce of these gives every rank the block's residual.
__global__ void gather_block_rows_kernel(const double* __restrict__ Rloc, int64_t r0, int64_t nloc,
                                         int64_t n, int bs, const int* __restrict__ blk,
                                         const int* __restrict__ active, int s,
                                         double* __restrict__ Rblk) {
  const int c = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= bs) return;
  double v = 0.0;
  if (active[c]) {
    const int64_t row = (int64_t)blk[c] * bs + i;
    if (row < n && row >= r0 && row < r0 + nloc) v = Rloc[(row - r0) * s + c];
  }
  Rblk[(int64_t)i * s + c] = v;
}

__global__ void set_cyclic_kernel(int* blk, int s, int value) {
  for (int c = threadIdx.x; c < s; c += blockDim.x) blk[c] = value;
}

// velocity *= momentum; velocity[rows] += scale * g; v -= lr * velocity   (active columns)
__global__ void sgd_momentum_kernel(double* __restrict__ vel, int64_t n, int s,
                                    const int* __restrict__ active, double momentum) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * s;
       e += (int64_t)gridDim.x * blockDim.x)
    if (active[e % s]) vel[e] *= momentum;
}
__global__ void sgd_scatter_kernel(double* __restrict__ vel, const int* __restrict__ rows,
                                   const double* __restrict__ g, int nb, int s,
                                   const int* __restrict__ active, double scale, int64_t r0,
                                   int64_t r1) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const int64_t row = rows[(int64_t)c * nb + i];
    if (row >= r0 && row < r1) vel[(row - r0) * s + c] += scale * g[(int64_t)c * nb + i];
  }
}
__global__ void sgd_step_kernel(double* __restrict__ V, const double* __restrict__ vel, int64_t n,
                                int s, const int* __restrict__ active, double lr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * s;
       e += (int64_t)gridDim.x * blockDim.x)
    if (active[e % s]) V[e] -= lr * vel[e];
}

// Copy columns flagged in mask from src to dst (AP convergence confirmation).
__global__ void copy_masked_cols_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                        int64_t n, int s, const int* __restrict__ mask) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * s;
       e += (int64_t)gridDim.x * blockDim.x)
    if (mask[e % s]) dst[e] = src[e];
}

inline int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

template <typename T, int DM>
static void krows_launch(const Op& op, const T* X, dim3 grid, int64_t jlen, const int* rows, int nb,
                         const double* V, int s, const int* active, int64_t r0, int64_t r1,
                         cudaStream_t st) {
  krows_kernel<T, DM><<<grid, 256, 0, st>>>(X, op.dpad, op.dim, op.n, jlen, rows, nb, V, s, active, op.kp(),
                                            r0, r1, op.krows_part.p);
}

void launch_krows(const Op& op, const int* rows, int nb, const double* V, const double* B, int s,
                  const int* active, double* g, int64_t r0, int64_t r1, cudaStream_t st) {
  TimedScope ts_("krows", st);
  // fixed j ranges of >= 1024 columns (at most 64), a function of n only
  const int64_t n = op.n;
  const int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(64, n / 1024));
  const int64_t jlen = (((n + nsplit - 1) / nsplit + 63) / 64) * 64;
  op.krows_part.ensure((size_t)nsplit * s * nb);
  const dim3 grid(ceil_div(nb, 64), s, nsplit);
  const int d = op.dim;
  if (op.f64()) {
    if (d <= 8) krows_launch<double, 8>(op, op.X64.p, grid, jlen, rows, nb, V, s, active, r0, r1, st);
    else if (d <= 16) krows_launch<double, 16>(op, op.X64.p, grid, jlen, rows, nb, V, s, active, r0, r1, st);
    else krows_launch<double, 32>(op, op.X64.p, grid, jlen, rows, nb, V, s, active, r0, r1, st);
  } else {
    if (d <= 8) krows_launch<float, 8>(op, op.X32.p, grid, jlen, rows, nb, V, s, active, r0, r1, st);
    else if (d <= 16) krows_launch<float, 16>(op, op.X32.p, grid, jlen, rows, nb, V, s, active, r0, r1, st);
    else krows_launch<float, 32>(op, op.X32.p, grid, jlen, rows, nb, V, s, active, r0, r1, st);
  }
  WGP_CUDA(cudaGetLastError());
  krows_sum_kernel<<<dim3(ceil_div(nb, 128), s), 128, 0, st>>>(op.krows_part.p, nsplit, rows, nb, B, s,
                                                               active, r0, r1, g);
  WGP_CUDA(cudaGetLastError());
}

template <typename T, int DM>
static void kcols_launch(const Op& op, const T* X, dim3 grid, const int* blk, int bs, const double* delta,
                         int s, const int* active, int64_t r0, int64_t nrows, double* R, cudaStream_t st) {
  kcols_kernel<T, DM><<<grid, 128, 0, st>>>(X, op.dpad, op.dim, op.n, blk, bs, delta, s, active, op.kp(),
                                            r0, nrows, R);
}

void launch_kcols(const Op& op, const int* blk, int bs, const double* delta, int s,
                  const int* active, double* R, int64_t r0, int64_t nrows, cudaStream_t st) {
  if (nrows <= 0) return;
  TimedScope ts_("kcols", st);
  const dim3 grid(ceil_div(nrows, 128), s);
  const int d = op.dim;
  if (op.f64()) {
    if (d <= 8) kcols_launch<double, 8>(op, op.X64.p, grid, blk, bs, delta, s, active, r0, nrows, R, st);
    else if (d <= 16) kcols_launch<double, 16>(op, op.X64.p, grid, blk, bs, delta, s, active, r0, nrows, R, st);
    else kcols_launch<double, 32>(op, op.X64.p, grid, blk, bs, delta, s, active, r0, nrows, R, st);
  } else {
    if (d <= 8) kcols_launch<float, 8>(op, op.X32.p, grid, blk, bs, delta, s, active, r0, nrows, R, st);
    else if (d <= 16) kcols_launch<float, 16>(op, op.X32.p, grid, blk, bs, delta, s, active, r0, nrows, R, st);
    else kcols_launch<float, 32>(op, op.X32.p, grid, blk, bs, delta, s, active, r0, nrows, R, st);
  }
  WGP_CUDA(cudaGetLastError());
}

void launch_block_chol(const Op& op, int bs, int nblk, double* fac, double* inv, int* fail,
                       cudaStream_t st) {
  block_chol_kernel<<<nblk, 512, 0, st>>>(op.X64.p, op.dpad, op.dim, op.n, bs, op.kp(), fac, inv,
                                          fail);
  WGP_CUDA(cudaGetLastError());
}

void launch_ap_block_solve(const double* inv, int bs, int64_t n, const int* blk, const int* active,
                           const double* R, const double* Rblk, int s, double* V, double* delta,
                           double* ybuf, cudaStream_t st) {
  const size_t smem = sizeof(double) * bs;  // <= 8 KB (bs <= 1024)
  ap_block_y_kernel<<<dim3((unsigned)ceil_div(bs, kApRowsPerCta), (unsigned)s), 256, smem, st>>>(
      inv, bs, n, blk, active, R, Rblk, s, ybuf);
  ap_block_delta_kernel<<<dim3((unsigned)ceil_div(bs, 32), (unsigned)s), 256, smem, st>>>(
      inv, bs, n, blk, active, ybuf, s, V, delta);
  WGP_CUDA(cudaGetLastError());
}

void launch_seg_norms(const double* Rloc, int64_t r0, int64_t nloc, const int64_t* seg_start, int nseg,
                      int s, const int* active, double* segn, cudaStream_t st) {
  seg_norms_kernel<<<s, dim3(32, 16), 0, st>>>(Rloc, r0, nloc, seg_start, nseg, s, active, segn);
  WGP_CUDA(cudaGetLastError());
}

void launch_greedy_from_segments(const double* segn, const int* seg_block, int nseg, int nblk, int s,
                                 const int* active, int* blk, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)std::max(nseg, 1);
  if (smem > 48 * 1024)
    WGP_CUDA(cudaFuncSetAttribute(greedy_from_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::min<size_t>(smem, 227 * 1024)));
  WGP_REQUIRE(smem <= 227 * 1024, "ap_solve: too many row segments for the greedy choice");
  greedy_from_segments_kernel<<<s, 128, smem, st>>>(segn, seg_block, nseg, nblk, s, active, blk);
  WGP_CUDA(cudaGetLastError());
}

void launch_gather_block_rows(const double* Rloc, int64_t r0, int64_t nloc, int64_t n, int bs,
                              const int* blk, const int* active, int s, double* Rblk, cudaStream_t st) {
  gather_block_rows_kernel<<<dim3((bs + 127) / 128, s), 128, 0, st>>>(Rloc, r0, nloc, n, bs, blk, active, s,
                                                                     Rblk);
  WGP_CUDA(cudaGetLastError());
}

void launch_set_cyclic(int* blk, int s, int value, cudaStream_t st) {
  set_cyclic_kernel<<<1, 256, 0, st>>>(blk, s, value);
  WGP_CUDA(cudaGetLastError());
}

void launch_sgd_update(double* V, double* vel, const int* rows, const double* g, int nb, int64_t n,
                       int s, const int* active, double momentum, double scale, double lr,
                       int64_t r0, cudaStream_t st) {
  // V, vel: this rank's rows [r0, r0 + n)
  sgd_momentum_kernel<<<grid_for(n * s), 256, 0, st>>>(vel, n, s, active, momentum);
  sgd_scatter_kernel<<<dim3(ceil_div(nb, 256), s), 256, 0, st>>>(vel, rows, g, nb, s, active, scale,
                                                                 r0, r0 + n);
  sgd_step_kernel<<<grid_for(n * s), 256, 0, st>>>(V, vel, n, s, active, lr);
  WGP_CUDA(cudaGetLastError());
}

void launch_copy_masked_cols(double* dst, const double* src, int64_t n, int s, const int* mask,
                             cudaStream_t st) {
  copy_masked_cols_kernel<<<grid_for(n * s), 256, 0, st>>>(dst, src, n, s, mask);
  WGP_CUDA(cudaGetLastError());
}

}  // namespace wgp
