// fp64 throughput on B200: DFMA (CUDA cores) vs DMMA (mma.sync.m8n8k4.f64, tensor cores).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_bench(double* out, int iters, long long* clk) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

__global__ void dmma_bench(double* out, int iters, long long* clk) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&clk, 8);
  const int iters = 4096;
  for (int warps : {8, 16, 32}) {
    dfma_bench<<<148, warps * 32>>>(out, iters, clk);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("DFMA warps %2d: %.1f FMA/clk/SM\n", warps, (double)warps * 32 * iters * 8 / c);
    dmma_bench<<<148, warps * 32>>>(out, iters, clk);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("DMMA warps %2d: %.1f FMA/clk/SM\n", warps, (double)warps * iters * 4 * 256 / c);
  }
  return 0;
}
