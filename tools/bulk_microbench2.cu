// Bulk-copy concurrency: P producer warps (each its own ring of R slots of S bytes), copies
// optionally split into k pieces.  One CTA per SM, all 148 SMs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2511_16340_b200/csrc/ptx.cuh"

__global__ void bench(const char* src, size_t src_bytes, int S, int R, int P, int K, int iters,
                      long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)P * R * S);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * P * R; ++i) wgp::ptx::mbar_init(&bars[i], 1);
    wgp::ptx::fence_mbar_init();
  }
  __syncthreads();
  const size_t nchunks = src_bytes / S;
  long long t0 = clock64();
  if (w < P && lane < (K < 0 ? -K : 1)) {  // producer p (K < 0: -K lanes each issue one piece)
    uint64_t* full = bars + (size_t)w * 2 * R;
    uint64_t* empty = full + R;
    size_t pos = ((size_t)blockIdx.x * 977 + w * 131) % nchunks;
    unsigned char* ring = sm + (size_t)w * R * S;
    for (int it = 0; it < iters; ++it) {
      const int st = it % R;
      if (it >= R) wgp::ptx::mbar_wait(&empty[st], ((it / R) - 1) & 1);
      if (K > 0) {
        wgp::ptx::mbar_arrive_expect_tx(&full[st], S);
        for (int k = 0; k < K; ++k)
          wgp::ptx::bulk_g2s(ring + (size_t)st * S + k * (S / K), src + pos * S + k * (S / K), S / K, &full[st]);
      } else {
        const int L = -K;
        if (lane == 0) wgp::ptx::mbar_arrive_expect_tx(&full[st], S);
        __syncwarp((1u << L) - 1);
        wgp::ptx::bulk_g2s(ring + (size_t)st * S + lane * (S / L), src + pos * S + lane * (S / L), S / L, &full[st]);
      }
      pos = (pos + 1) % nchunks;
    }
  } else if (w >= P && w < 2 * P && lane == 0) {  // consumer of producer w - P
    uint64_t* full = bars + (size_t)(w - P) * 2 * R;
    uint64_t* empty = full + R;
    for (int it = 0; it < iters; ++it) {
      const int st = it % R;
      wgp::ptx::mbar_wait(&full[st], (it / R) & 1);
      wgp::ptx::mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  const size_t bytes = 24u << 20;
  char* src;
  long long* out;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaMalloc(&out, 16);
  struct C { int S, R, P, K; } cs[] = {{16384, 4, 1, 1}, {16384, 4, 1, -2}, {16384, 4, 1, -4}, {16384, 4, 1, -8},
                                       {16384, 4, 1, -16}, {16384, 4, 2, 1}, {16384, 4, 2, -4}, {16384, 8, 1, -4},
                                       {32768, 4, 1, -8}, {8192, 8, 1, -4}};
  for (auto c : cs) {
    const size_t smem = (size_t)c.P * c.R * c.S + 2048;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = 1000;
    bench<<<148, 64 * c.P, smem>>>(src, bytes, c.S, c.R, c.P, c.K, iters, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("S=%6d R=%d P=%d K=%2d: %7.1f B/clk/SM (%.0f clk per copy per producer) %s\n", c.S, c.R, c.P, c.K,
           (double)c.S * iters * c.P / cyc, (double)cyc / iters, cudaGetErrorString(e));
  }
  return 0;
}
