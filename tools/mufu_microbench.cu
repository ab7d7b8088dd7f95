// Throughput of the SFU (MUFU) ops used by the kernel-map epilogue, per SM per clock, and of
// a software exp2 on the FMA pipe.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__device__ __forceinline__ float op(float x) {
  float y;
  if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 1) asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 2) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  if (OP == 3) {  // software 2^x, x in [-126, 0]: Cody-Waite split + degree-5 minimax on [0,1)
    const float xf = floorf(x);
    const float f = x - xf;
    float p = 1.8775767e-3f;
    p = fmaf(p, f, 8.9893397e-3f);
    p = fmaf(p, f, 5.5826318e-2f);
    p = fmaf(p, f, 2.4015361e-1f);
    p = fmaf(p, f, 6.9315308e-1f);
    p = fmaf(p, f, 9.9999994e-1f);
    y = __int_as_float(__float_as_int(p) + ((int)xf << 23));
  }
  if (OP == 4) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int OP>
__global__ void bench(float* out, int iters, long long* clk) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = op<OP>(a[i]) * -1.0f - 0.5f;  // keep in range
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4 * 4);
  cudaMalloc(&clk, 8);
  const char* names[] = {"ex2.approx", "sqrt.approx", "rsqrt.approx", "sw exp2 (FMA)", "tanh.approx"};
  const int iters = 4096;
  for (int o = 0; o < 5; ++o) {
    for (int threads : {256, 512, 1024}) {
      auto k = o == 0 ? bench<0> : o == 1 ? bench<1> : o == 2 ? bench<2> : o == 3 ? bench<3> : bench<4>;
      k<<<148, threads>>>(out, iters, clk);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      // per SM: threads * iters * 8 ops in c cycles (one CTA per SM)
      printf("%-16s threads/SM %4d: %.2f ops/clk/SM (+fmul,fadd per op)\n", names[o], threads,
             (double)threads * iters * 8 / c);
    }
  }
  return 0;
}
