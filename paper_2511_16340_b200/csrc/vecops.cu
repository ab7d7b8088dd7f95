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

// One block per chunk.  Per column the chunk is cut into 32 fixed 16-row slabs summed
// sequentially, then the 32 slab sums are added in slab order: the order of every column's
// sum depends only on the row index, never on s or on the other columns (solve_many must
// equal single-RHS solves bitwise, test_solvers.cpp:397-413).
constexpr int kSlabRows = kChunkRows / 32;

template <typename T, int NQ>
__global__ void __launch_bounds__(256) coldots_kernel(const T* __restrict__ A0,
                                                      const T* __restrict__ B0,
                                                      const T* __restrict__ A1,
                                                      const T* __restrict__ B1, int64_t n, int s,
                                                      double* __restrict__ part) {
  extern __shared__ double red[];  // [NQ][32][s]
  const int64_t r0 = (int64_t)blockIdx.x * kChunkRows;
  for (int f = threadIdx.x; f < 32 * s; f += blockDim.x) {
    const int q = f / s, c = f % s;
    const int64_t i0 = r0 + (int64_t)q * kSlabRows;
    const int64_t i1 = min(n, i0 + kSlabRows);
    double a0 = 0.0, a1 = 0.0;
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t e = i * s + c;
      a0 = fma((double)A0[e], (double)B0[e], a0);
      if (NQ > 1) a1 = fma((double)A1[e], (double)B1[e], a1);
    }
    red[q * s + c] = a0;
    if (NQ > 1) red[(32 + q) * s + c] = a1;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < s; c += blockDim.x) {
    double t0 = 0.0, t1 = 0.0;
    for (int q = 0; q < 32; ++q) {
      t0 += red[q * s + c];
      if (NQ > 1) t1 += red[(32 + q) * s + c];
    }
    double* out = part + (int64_t)blockIdx.x * NQ * s;
    out[c] = t0;
    if (NQ > 1) out[s + c] = t1;
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
  const size_t smem = sizeof(double) * 32 * s * (A1 ? 2 : 1);
  if (A1) {
    if (smem > 48 * 1024)
      WGP_CUDA(cudaFuncSetAttribute(coldots_kernel<T, 2>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    coldots_kernel<T, 2><<<nch, 256, smem, st>>>(A0, B0, A1, B1, n, s, part);
  } else {
    if (smem > 48 * 1024)
      WGP_CUDA(cudaFuncSetAttribute(coldots_kernel<T, 1>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    coldots_kernel<T, 1><<<nch, 256, smem, st>>>(A0, B0, A0, B0, n, s, part);
  }
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
