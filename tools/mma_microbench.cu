// mma_microbench.cu -- measures tcgen05.mma issue/execution cost on this GPU (not product
// code): per-instruction cycles for the shapes the kmatvec kernel uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I.. -o mma_microbench mma_microbench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2511_16340_b200/csrc/ptx.cuh"

using namespace wgp;

template <int MODE>  // 0: tf32 SS N=64, 1: f16 TS N=64, 2: f16 TS N=128, 3: tf32 TS N=64, 4: f16 SS N=64
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&tslot, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint64_t d0 = ptx::umma_desc(ptx::smem_u32(smem), 128, 1024);
    const uint32_t i_tf = ptx::idesc_tf32(128, MODE == 2 ? 128 : 64);
    const uint32_t i_f16 = ptx::idesc_f16(128, MODE == 2 ? 128 : 64);
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int i = 0; i < iters; ++i) {
        if (MODE == 0) ptx::mma_tf32_ss(tmem, d0, d0 + 16, i_tf, 1);
        if (MODE == 1 || MODE == 2) ptx::mma_f16_ts(tmem + 256, tmem + (i & 3) * 8, d0, i_f16, 1);
        if (MODE == 3) ptx::mma_tf32_ts(tmem + 256, tmem + (i & 3) * 8, d0, i_tf, 1);
        if (MODE == 4) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(d0), "l"(d0 + 16), "r"(i_f16), "r"(1));
        }
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    unsigned long long t1 = clock64();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(const char* name, int iters) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 2 * 148);
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  bench<MODE><<<148, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%-28s iters %6d  issue %8.1f cyc/inst  complete %8.1f cyc/inst  (%s)\n", name, iters,
         (double)h[0] / iters, (double)h[1] / iters, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int it : {64, 1024}) {
    run<0>("tf32 SS M128 N64 K8", it);
    run<3>("tf32 TS M128 N64 K8", it);
    run<1>("f16  TS M128 N64 K16", it);
    run<2>("f16  TS M128 N128 K16", it);
    run<4>("f16  SS M128 N64 K16", it);
  }
  return 0;
}
