// TMEM load/store throughput per SM (tcgen05.ld 32x32b.x32 / tcgen05.st 32x32b.x16) with W
// warps (4*k, each warp reads its lane quadrant).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2511_16340_b200/csrc/ptx.cuh"

template <int MODE>
__global__ void bench(int iters, long long* clk, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) wgp::ptx::tmem_alloc(&slot, 512);
  wgp::ptx::tc_fence_before();
  __syncthreads();
  wgp::ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 32 % 512;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t addr = tmem + lane_off + ((col0 + it * 32) & 511);
    if (MODE == 0) {
      uint32_t v[32];
      wgp::ptx::tmem_ld32(addr, v);
      wgp::ptx::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[i];
    } else {
      uint32_t v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = it + i;
      wgp::ptx::tmem_st16(addr, v);
      wgp::ptx::tmem_wait_st();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  wgp::ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    wgp::ptx::tc_fence_after();
    wgp::ptx::tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* clk;
  float* sink;
  cudaMalloc(&clk, 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 2000;
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      if (mode == 0) bench<0><<<148, warps * 32>>>(iters, clk, sink);
      else bench<1><<<148, warps * 32>>>(iters, clk, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * iters * 32 * (mode == 0 ? 32 : 16) * 4;
      printf("%s warps %2d: %.1f B/clk/SM  (%s)\n", mode == 0 ? "LDTM.x32" : "STTM.x16", warps,
             bytes / c, cudaGetErrorString(e));
    }
  return 0;
}
