// vecops.cu -- fused solver vector kernels over RHS-interleaved [n][s] arrays
// (solvers.cpp:163-182: p^T H p, v += alpha p, |r|, r^T z, p = z + beta p), layout
// conversion at the host boundary, and fixed-order column reductions.
//
// Reductions are deterministic and world-size independent: each block reduces one
// kChunkRows-row chunk in a fixed order to fp64 partials part[chunk][q][c]; the
// scalar-step kernels (solver_kernels.cu) then add the chunks in index order.
#include "common.cuh"

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

// One block per chunk.  Lanes map to (row-sub, column) with SP = pow2 >= min(s,32)
// columns per warp step; the 8 warps stride rows; fixed-order combine at the end.
template <typename T, int NQ>
__global__ void __launch_bounds__(256) coldots_kernel(const T* __restrict__ A0,
                                                      const T* __restrict__ B0,
                                                      const T* __restrict__ A1,
                                                      const T* __restrict__ B1, int64_t n, int s,
                                                      int SP, double* __restrict__ part) {
  __shared__ double red[8][NQ][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kChunkRows;
  const int64_t r1 = min(n, r0 + (int64_t)kChunkRows);
  const int RS = 32 / SP;  // rows per warp step
  const int rsub = lane / SP, cl = lane % SP;
  for (int cb = 0; cb < s; cb += SP) {
    const int c = cb + cl;
    double a0 = 0.0, a1 = 0.0;
    if (c < s) {
      for (int64_t i = r0 + warp * RS + rsub; i < r1; i += 8 * RS) {
        const int64_t e = i * s + c;
        a0 = fma((double)A0[e], (double)B0[e], a0);
        if (NQ > 1) a1 = fma((double)A1[e], (double)B1[e], a1);
      }
    }
    // combine row-subs inside the warp (lanes with equal cl), fixed butterfly order
    for (int off = SP; off < 32; off <<= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, off);
      if (NQ > 1) a1 += __shfl_xor_sync(0xffffffffu, a1, off);
    }
    if (rsub == 0) {
      red[warp][0][cl] = a0;
      if (NQ > 1) red[warp][NQ - 1][cl] = a1;
    }
    __syncthreads();
    if (threadIdx.x < SP && cb + (int)threadIdx.x < s) {
      const int cc = threadIdx.x;
      double t0 = 0.0, t1 = 0.0;
      for (int w = 0; w < 8; ++w) {
        t0 += red[w][0][cc];
        if (NQ > 1) t1 += red[w][NQ - 1][cc];
      }
      double* out = part + (int64_t)blockIdx.x * NQ * s;
      out[cb + cc] = t0;
      if (NQ > 1) out[s + cb + cc] = t1;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void axpy_cols_kernel(T* __restrict__ Y, const T* __restrict__ X,
                                 const double* __restrict__ alpha, int64_t total, int s) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double a = alpha[e % s];
    if (a != 0.0) Y[e] = (T)((double)Y[e] + a * (double)X[e]);
  }
}

template <typename T>
__global__ void xpby_cols_kernel(T* __restrict__ P, const T* __restrict__ Z,
                                 const double* __restrict__ beta, const int* __restrict__ active,
                                 int64_t total, int s) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % s);
    if (active[c]) P[e] = (T)((double)Z[e] + beta[c] * (double)P[e]);
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
  int SP = 1;
  while (SP < s && SP < 32) SP <<= 1;
  if (A1)
    coldots_kernel<T, 2><<<nch, 256, 0, st>>>(A0, B0, A1, B1, n, s, SP, part);
  else
    coldots_kernel<T, 1><<<nch, 256, 0, st>>>(A0, B0, A0, B0, n, s, SP, part);
  WGP_CUDA(cudaGetLastError());
}

template <typename T>
void launch_axpy_cols(T* Y, const T* X, const double* alpha, int64_t n, int s, cudaStream_t st) {
  const int64_t total = n * s;
  if (total <= 0) return;
  axpy_cols_kernel<T><<<grid_for(total), 256, 0, st>>>(Y, X, alpha, total, s);
  WGP_CUDA(cudaGetLastError());
}

template <typename T>
void launch_xpby_cols(T* P, const T* Z, const double* beta, const int* active, int64_t n, int s,
                      cudaStream_t st) {
  const int64_t total = n * s;
  if (total <= 0) return;
  xpby_cols_kernel<T><<<grid_for(total), 256, 0, st>>>(P, Z, beta, active, total, s);
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
