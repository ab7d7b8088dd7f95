// Throughput of the kernel-map instruction mix alone (no TMEM, no sync): per element
// sqrt.approx(|d2|) -> FFMA2 -> ex2.approx -> FMUL2/FFMA2 -> fp16 hi/lo split (LOP3, FADD2,
// F2FP), 16-element chunks per iteration like the tcgen05 epilogue.  Reports pairs/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float sqa(float x) { float y; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pk(float a, float b) { __half2 h = __floats2half2_rn(a, b); return *reinterpret_cast<uint32_t*>(&h); }

template <int MODE>
__global__ void bench(const float* in, uint32_t* out, int iters, long long* clk) {
  float v[16];
  for (int c = 0; c < 16; ++c) v[c] = in[(threadIdx.x + c) & 255] * 0.01f;
  uint32_t sink = 0;
  const float2 NC = make_float2(-1.5f, -1.5f), OFF = make_float2(10.f, 10.f), C1 = make_float2(1.7f, 1.7f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float kv[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float2 r;
      if (MODE == 2) {
        r = make_float2(fabsf(v[2 * q]), fabsf(v[2 * q + 1]));
      } else {
        r.x = sqa(fabsf(v[2 * q]));
        r.y = sqa(fabsf(v[2 * q + 1]));
      }
      const float2 a = __ffma2_rn(r, NC, OFF);
      float2 e;
      e.x = ex2a(a.x);
      e.y = ex2a(a.y);
      const float2 z = __fmul2_rn(r, C1);
      const float2 k = __ffma2_rn(z, e, e);
      kv[2 * q] = k.x;
      kv[2 * q + 1] = k.y;
    }
    if (MODE >= 1) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float2 hf = make_float2(__uint_as_float(__float_as_uint(kv[2 * c]) & 0xFFFFE000u),
                                      __uint_as_float(__float_as_uint(kv[2 * c + 1]) & 0xFFFFE000u));
        const float2 rem = __fadd2_rn(make_float2(kv[2 * c], kv[2 * c + 1]), make_float2(-hf.x, -hf.y));
        sink ^= pk(hf.x, hf.y) + pk(rem.x, rem.y);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 16; ++c) sink ^= __float_as_uint(kv[c]);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = v[c] + 1e-7f;  // new inputs each iteration
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* in; uint32_t* out; long long* clk;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4);
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  const char* names[] = {"map (2 MUFU) no pack", "map + fp16 split", "ex2 only + split"};
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {8, 16, 24, 32}) {
      const int iters = 2000;
      if (mode == 0) bench<0><<<148, warps * 32>>>(in, out, iters, clk);
      if (mode == 1) bench<1><<<148, warps * 32>>>(in, out, iters, clk);
      if (mode == 2) bench<2><<<148, warps * 32>>>(in, out, iters, clk);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      printf("%-22s warps %2d: %.2f elements/clk/SM\n", names[mode], warps, (double)warps * 32 * iters * 16 / c);
    }
  return 0;
}
