// vecops.cu -- fused solver vector kernels over RHS-interleaved [n][s] arrays
// (solvers.cpp:163-182: p^T H p, v += alpha p, |r|, r^T z, p = z + beta p), layout
// conversion at the host boundary, and fixed-order column reductions.
//
// Reductions are deterministic and world-size independent: each block reduces one
// kChunkRows-row chunk in a fixed order to fp64 partials part[chunk][q][c]; the
// scalar-step kernels (solver_kernels.cu) then add the chunks in index order.
#include <type_traits>

#include "solvers.h"

namespace wgp {
namespace {

template <typename T>
__global__ void colmajor_to_rows_kernel(const double* __restrict__ src, int64_t ld, int64_t n,
                                        int s, T* __restrict__ dst) {
  // 32x32 tile transpose through shared memory: coalesced on both sides.
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int c = c0 + k;
    const int64_t i = i0 + threadIdx.x;
    tile[k][threadIdx.x] = (c < s && i < n) ? src[(int64_t)c * ld + i] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t i = i0 + k;
    const int c = c0 + threadIdx.x;
    if (i < n && c < s) dst[i * s + c] = (T)tile[threadIdx.x][k];
  }
}

template <typename T>
__global__ void rows_to_colmajor_kernel(const T* __restrict__ src, int64_t n, int s,
                                        double* __restrict__ dst, int64_t ld) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t i = i0 + k;
    const int c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (i < n && c < s) ? (double)src[i * s + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int c = c0 + k;
    const int64_t i = i0 + threadIdx.x;
    if (c < s && i < n) dst[(int64_t)c * ld + i] = tile[threadIdx.x][k];
  }
}

// Per column the chunk is 32 fixed 16-row slabs, each summed sequentially, slab sums added
// in slab order: the order of every column's sum depends only on the row index, never on s
// or on the other columns (solve_many must equal single-RHS solves bitwise,
// test_solvers.cpp:397-413).  Work item = (chunk, group of up to 32 columns), one thread per
// (column, slab): a warp reads 32 consecutive columns of a row (256 contiguous bytes per fp64
// load); blocks of CB columns x 32 slabs walk the items, 1024 / (32 CB) of them per SM.  Each
// slab is loaded in 8-row halves (4-row quarters for two dot products), all loads of a part
// issued before its FMA chain: 16 loads in flight per thread, 128 KB per SM.  Two 512-thread
// blocks per SM (CB = 16) measured 20.2 us per launch at [101000][64] (ncu, cold L2; 79% of
// the measured HBM copy bandwidth) against 21.8 us for one 1024-thread block (its reduction
// and item change leave the SM without loads in flight; the other block covers them); a
// rolling load ring across slab rows and items (no drain at all) measured slower (21.3 /
// 22.8 us: per-load index arithmetic and predication).
constexpr int kSlabRows = kChunkRows / 32;
template <typename T, int NQ, int CB>
__global__ void __launch_bounds__(CB * 32, 32 / CB)
    coldots_kernel(const T* __restrict__ A0, const T* __restrict__ B0, const T* __restrict__ A1,
                   const T* __restrict__ B1, int64_t n, int s, int cb, int ngroups, int64_t items,
                   double* __restrict__ part) {
  __shared__ double red[NQ][32][CB];
  const int cl = threadIdx.x % cb;
  const int q = threadIdx.x / cb;  // slab
  constexpr int NH = NQ == 1 ? 2 : 4;  // loads in flight per thread: 16 (64 registers at 1024 threads)
  constexpr int H = kSlabRows / NH;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t chunk = item / ngroups;
    const int grp = (int)(item - chunk * ngroups);
    const int c = grp * cb + cl;
    if (q < 32 && c < s) {
      const int64_t i0 = chunk * kChunkRows + (int64_t)q * kSlabRows;
      const int64_t i1 = min(n, i0 + kSlabRows);
      double a0 = 0.0, a1 = 0.0;
      const T* pa0 = A0 + i0 * s + c;
      const T* pb0 = B0 + i0 * s + c;
      const T* pa1 = A1 + i0 * s + c;
      const T* pb1 = B1 + i0 * s + c;
      if (i1 - i0 == kSlabRows) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          T xa[H], xb[H], ya[NQ > 1 ? H : 1], yb[NQ > 1 ? H : 1];
#pragma unroll
          for (int k = 0; k < H; ++k) {
            const int64_t o = (int64_t)(h * H + k) * s;
            xa[k] = pa0[o];
            xb[k] = pb0[o];
            if (NQ > 1) {
              ya[k] = pa1[o];
              yb[k] = pb1[o];
            }
          }
#pragma unroll
          for (int k = 0; k < H; ++k) {
            a0 = fma((double)xa[k], (double)xb[k], a0);
            if (NQ > 1) a1 = fma((double)ya[k], (double)yb[k], a1);
          }
        }
      } else {
        for (int64_t k = 0; k < i1 - i0; ++k) {
          a0 = fma((double)pa0[k * s], (double)pb0[k * s], a0);
          if (NQ > 1) a1 = fma((double)pa1[k * s], (double)pb1[k * s], a1);
        }
      }
      red[0][q][cl] = a0;
      if (NQ > 1) red[NQ - 1][q][cl] = a1;
    }
    __syncthreads();
    if (threadIdx.x < cb * NQ) {
      const int col = threadIdx.x % cb, qq = threadIdx.x / cb;
      const int cc = grp * cb + col;
      if (cc < s) {
        double t = 0.0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) t += red[qq][k][col];
        part[chunk * NQ * s + (int64_t)qq * s + cc] = t;
      }
    }
    __syncthreads();
  }
}

// Column sums of chunk partials part[chunk][s] in chunk order (the scalar-step kernels'
// order), for the standalone device dot product of the C-ABI.
// One block per column: the block stages the column's nch partials in shared memory with
// parallel loads, then one thread adds them in chunk order (the same order as
// chunk_sum_ordered) -- a chain of dependent fp64 adds instead of dependent L2 round trips.
__global__ void __launch_bounds__(256) chunk_sum_kernel(const double* __restrict__ part, int nch,
                                                        int s, double* __restrict__ out) {
  __shared__ double buf[2048];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int base = 0; base < nch; base += 2048) {
    const int m = min(2048, nch - base);
    for (int q = threadIdx.x; q < m; q += blockDim.x) buf[q] = part[(int64_t)(base + q) * s + c];
    __syncthreads();
    if (threadIdx.x == 0) {
      int q = 0;
      for (; q + 8 <= m; q += 8) {  // shared loads 8 ahead of the ordered adds
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = buf[q + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; q < m; ++q) acc += buf[q];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = acc;
}

// Element-wise column updates of [n][s] arrays.  The grid covers `rows_step` whole rows per
// step (rows_step * s threads), so every thread keeps one column -- its coefficient and
// activity flag stay in registers, with no index division in the loop -- and a warp still
// touches consecutive addresses.
template <typename T>
__global__ void __launch_bounds__(256) axpy_cols_kernel(T* __restrict__ Y, const T* __restrict__ X,
                                                        const double* __restrict__ alpha,
                                                        int64_t total, int s, int64_t stride) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= stride) return;
  const double a = alpha[t % s];
  if (a == 0.0) return;
#pragma unroll 4
  for (int64_t e = t; e < total; e += stride) Y[e] = (T)((double)Y[e] + a * (double)X[e]);
}

template <typename T>
__global__ void __launch_bounds__(256) xpby_cols_kernel(T* __restrict__ P, const T* __restrict__ Z,
                                                        const double* __restrict__ beta,
                                                        const int* __restrict__ active,
                                                        int64_t total, int s, int64_t stride) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= stride) return;
  const int c = (int)(t % s);
  if (!active[c]) return;
  const double b = beta[c];
#pragma unroll 4
  for (int64_t e = t; e < total; e += stride) P[e] = (T)((double)Z[e] + b * (double)P[e]);
}

// fp64 pairs (s even): 16-byte accesses, one column pair per thread
__global__ void __launch_bounds__(256) axpy_cols2_kernel(double2* __restrict__ Y,
                                                         const double2* __restrict__ X,
                                                         const double* __restrict__ alpha,
                                                         int64_t total2, int s2, int64_t stride2) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= stride2) return;
  const int c = 2 * (int)(t % s2);
  const double a0 = alpha[c], a1 = alpha[c + 1];
  if (a0 == 0.0 && a1 == 0.0) return;
#pragma unroll 4
  for (int64_t e = t; e < total2; e += stride2) {
    double2 y = Y[e];
    const double2 x = X[e];
    if (a0 != 0.0) y.x = y.x + a0 * x.x;
    if (a1 != 0.0) y.y = y.y + a1 * x.y;
    Y[e] = y;
  }
}

__global__ void __launch_bounds__(256) xpby_cols2_kernel(double2* __restrict__ P,
                                                         const double2* __restrict__ Z,
                                                         const double* __restrict__ beta,
                                                         const int* __restrict__ active,
                                                         int64_t total2, int s2, int64_t stride2) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= stride2) return;
  const int c = 2 * (int)(t % s2);
  const bool on0 = active[c] != 0, on1 = active[c + 1] != 0;
  if (!on0 && !on1) return;
  const double b0 = beta[c], b1 = beta[c + 1];
#pragma unroll 4
  for (int64_t e = t; e < total2; e += stride2) {
    double2 pv = P[e];
    const double2 z = Z[e];
    if (on0) pv.x = z.x + b0 * pv.x;
    if (on1) pv.y = z.y + b1 * pv.y;
    P[e] = pv;
  }
}

template <typename T>
__global__ void fill_kernel(T* p, T v, size_t count) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
       e += (size_t)gridDim.x * blockDim.x)
    p[e] = v;
}

inline int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_colmajor_to_rows(const double* src, int64_t ld, int64_t n, int s, void* dst, bool f64,
                             cudaStream_t st) {
  if (n <= 0 || s <= 0) return;
  dim3 grid(ceil_div(n, 32), ceil_div(s, 32)), block(32, 8);
  if (f64)
    colmajor_to_rows_kernel<double><<<grid, block, 0, st>>>(src, ld, n, s, (double*)dst);
  else
    colmajor_to_rows_kernel<float><<<grid, block, 0, st>>>(src, ld, n, s, (float*)dst);
  WGP_CUDA(cudaGetLastError());
}

void launch_rows_to_colmajor(const void* src, int64_t n, int s, double* dst, int64_t ld, bool f64,
                             cudaStream_t st) {
  if (n <= 0 || s <= 0) return;
  dim3 grid(ceil_div(n, 32), ceil_div(s, 32)), block(32, 8);
  if (f64)
    rows_to_colmajor_kernel<double><<<grid, block, 0, st>>>((const double*)src, n, s, dst, ld);
  else
    rows_to_colmajor_kernel<float><<<grid, block, 0, st>>>((const float*)src, n, s, dst, ld);
  WGP_CUDA(cudaGetLastError());
}

template <typename T>
void launch_coldots(const T* A0, const T* B0, const T* A1, const T* B1, int64_t n, int s,
                    double* part, cudaStream_t st) {
  if (s <= 0) return;
  const int nch = ceil_div(n, kChunkRows);
  if (nch <= 0) return;
  static const int forced_cb = getenv("WGP_COLDOTS_CB") ? atoi(getenv("WGP_COLDOTS_CB")) : 0;
  const int CBmax = forced_cb == 8 || forced_cb == 16 || forced_cb == 32 ? forced_cb : 16;
  const int cb = s < CBmax ? s : CBmax;
  const int ngroups = ceil_div(s, cb);
  const int64_t items = (int64_t)nch * ngroups;
  const int grid = (int)std::min<int64_t>(items, (int64_t)148 * (32 / CBmax));
  TimedScope ts_("coldots", st);
  auto go = [&](auto kern2, auto kern1) {
    if (A1)
      kern2<<<grid, cb * 32, 0, st>>>(A0, B0, A1, B1, n, s, cb, ngroups, items, part);
    else
      kern1<<<grid, cb * 32, 0, st>>>(A0, B0, A0, B0, n, s, cb, ngroups, items, part);
  };
  if (CBmax == 8)
    go(coldots_kernel<T, 2, 8>, coldots_kernel<T, 1, 8>);
  else if (CBmax == 16)
    go(coldots_kernel<T, 2, 16>, coldots_kernel<T, 1, 16>);
  else
    go(coldots_kernel<T, 2, 32>, coldots_kernel<T, 1, 32>);
  WGP_CUDA(cudaGetLastError());
}

void launch_chunk_sum(const double* part, int nch, int s, double* out, cudaStream_t st) {
  if (s <= 0) return;
  chunk_sum_kernel<<<s, 256, 0, st>>>(part, nch, s, out);
  WGP_CUDA(cudaGetLastError());
}

// rows per grid step: about 2048 resident threads per SM, whole rows
static int64_t col_stride(int64_t n, int s) {
  const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)148 * 2048 / s));
  return rows * s;
}

template <typename T>
void launch_axpy_cols(T* Y, const T* X, const double* alpha, int64_t n, int s, cudaStream_t st) {
  const int64_t total = n * s;
  if (total <= 0) return;
  if (std::is_same<T, double>::value && s % 2 == 0 && ((uintptr_t)Y % 16 == 0) &&
      ((uintptr_t)X % 16 == 0)) {
    const int64_t stride2 = col_stride(n, s / 2);
    axpy_cols2_kernel<<<(unsigned)((stride2 + 255) / 256), 256, 0, st>>>(
        (double2*)Y, (const double2*)X, alpha, total / 2, s / 2, stride2);
    WGP_CUDA(cudaGetLastError());
    return;
  }
  const int64_t stride = col_stride(n, s);
  axpy_cols_kernel<T><<<(unsigned)((stride + 255) / 256), 256, 0, st>>>(Y, X, alpha, total, s, stride);
  WGP_CUDA(cudaGetLastError());
}

template <typename T>
void launch_xpby_cols(T* P, const T* Z, const double* beta, const int* active, int64_t n, int s,
                      cudaStream_t st) {
  const int64_t total = n * s;
  if (total <= 0) return;
  if (std::is_same<T, double>::value && s % 2 == 0 && ((uintptr_t)P % 16 == 0) &&
      ((uintptr_t)Z % 16 == 0)) {
    const int64_t stride2 = col_stride(n, s / 2);
    xpby_cols2_kernel<<<(unsigned)((stride2 + 255) / 256), 256, 0, st>>>(
        (double2*)P, (const double2*)Z, beta, active, total / 2, s / 2, stride2);
    WGP_CUDA(cudaGetLastError());
    return;
  }
  const int64_t stride = col_stride(n, s);
  xpby_cols_kernel<T><<<(unsigned)((stride + 255) / 256), 256, 0, st>>>(P, Z, beta, active, total,
                                                                         s, stride);
  WGP_CUDA(cudaGetLastError());
}

template <typename T>
void launch_fill(T* p, T v, size_t count, cudaStream_t st) {
  if (!count) return;
  fill_kernel<T><<<grid_for((int64_t)count), 256, 0, st>>>(p, v, count);
  WGP_CUDA(cudaGetLastError());
}

#define WGP_INST(T)                                                                          \
  template void launch_coldots<T>(const T*, const T*, const T*, const T*, int64_t, int,      \
                                  double*, cudaStream_t);                                    \
  template void launch_axpy_cols<T>(T*, const T*, const double*, int64_t, int, cudaStream_t); \
  template void launch_xpby_cols<T>(T*, const T*, const double*, const int*, int64_t, int,   \
                                    cudaStream_t);                                           \
  template void launch_fill<T>(T*, T, size_t, cudaStream_t);
WGP_INST(double)
WGP_INST(float)
template void launch_fill<int>(int*, int, size_t, cudaStream_t);

}  // namespace wgp
