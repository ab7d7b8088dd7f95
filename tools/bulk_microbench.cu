// Bulk-copy (cp.async.bulk, UBLKCP) streaming throughput/latency per SM: one CTA per SM, a
// producer lane keeps a ring of R copies of S bytes in flight over a shared L2-resident
// buffer; a consumer lane waits each full barrier and frees the slot.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2511_16340_b200/csrc/ptx.cuh"

__global__ void bench(const char* src, size_t src_bytes, int S, int R, int iters, long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)R * S);
  uint64_t* empty = full + R;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) { wgp::ptx::mbar_init(&full[i], 1); wgp::ptx::mbar_init(&empty[i], 1); }
    wgp::ptx::fence_mbar_init();
  }
  __syncthreads();
  const size_t nchunks = src_bytes / S;
  size_t pos = ((size_t)blockIdx.x * 977) % nchunks;
  long long t0 = clock64(), lat = 0;
  if (threadIdx.x == 0) {  // producer
    for (int it = 0; it < iters; ++it) {
      const int st = it % R;
      if (it >= R) wgp::ptx::mbar_wait(&empty[st], ((it / R) - 1) & 1);
      wgp::ptx::mbar_arrive_expect_tx(&full[st], S);
      wgp::ptx::bulk_g2s(sm + (size_t)st * S, src + pos * S, S, &full[st]);
      pos = (pos + 1) % nchunks;
    }
  } else if (threadIdx.x == 32) {  // consumer
    for (int it = 0; it < iters; ++it) {
      const int st = it % R;
      wgp::ptx::mbar_wait(&full[st], (it / R) & 1);
      wgp::ptx::mbar_arrive(&empty[st]);
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
  }
}

int main() {
  const size_t bytes = 24u << 20;
  char* src;
  long long* out;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaMalloc(&out, 16);
  for (int S : {4096, 8192, 16384, 32768})
    for (int R : {2, 4, 8}) {
      const size_t smem = (size_t)R * S + 1024;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 2000;
      for (int grid : {1, 148}) {
        bench<<<grid, 64, smem>>>(src, bytes, S, R, iters, out);
        cudaError_t e = cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        const double bpc = (double)S * iters / c;
        printf("S=%6d R=%d grid=%3d: %7.1f B/clk/SM  (%.0f clk per copy, ~latency %.0f clk) %s\n", S, R,
               grid, bpc, (double)c / iters, (double)c / iters * R, cudaGetErrorString(e));
      }
    }
  return 0;
}
