// rff.cu -- random-Fourier-feature prior evaluation for S priors at once (K7):
//   out[i, p] = s_f sqrt(2/F) sum_f w_pf cos(x_i . omega_pf + phi_pf)
// restating eval_prior (sampling.cpp:37-46), which the reference runs once per prior as a
// dense X Omega^T GEMM followed by cos and a GEMV.  Here the phase contraction (K = d),
// the cos and the amplitude reduction are fused per (row tile, prior): the m x F phase
// matrix never exists.  fp64 throughout (RHS generation is not precision-relaxed).
#include "solvers.h"

namespace wgp {
namespace {

constexpr int RT = 128, FT = 64;

__global__ void __launch_bounds__(RT) rff_eval_kernel(const double* __restrict__ X, int ldx_row,
                                                      int dim, int64_t m,
                                                      const double* __restrict__ Om,
                                                      const double* __restrict__ ph,
                                                      const double* __restrict__ amp, int F,
                                                      double coeff, double* __restrict__ out,
                                                      int64_t ldo) {
  extern __shared__ double sm[];
  double* sOm = sm;                 // FT x dim  (row-major within the tile)
  double* sPh = sOm + FT * dim;     // FT
  double* sAm = sPh + FT;           // FT
  const int p = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x;
  const double* Omp = Om + (int64_t)p * F * dim;  // F x dim column-major
  const double* php = ph + (int64_t)p * F;
  const double* amp_p = amp + (int64_t)p * F;
  double x[32];
  const bool valid = i < m;
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = (valid && k < dim) ? X[i * ldx_row + k] : 0.0;
  double acc = 0.0;
  for (int f0 = 0; f0 < F; f0 += FT) {
    const int nf = min(FT, F - f0);
    __syncthreads();
    for (int e = threadIdx.x; e < nf * dim; e += RT) {
      const int f = e % nf, k = e / nf;
      sOm[f * dim + k] = Omp[(int64_t)k * F + f0 + f];
    }
    for (int e = threadIdx.x; e < nf; e += RT) {
      sPh[e] = php[f0 + e];
      sAm[e] = amp_p[f0 + e];
    }
    __syncthreads();
    for (int f = 0; f < nf; ++f) {
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k < dim) a = fma(x[k], sOm[f * dim + k], a);
      a += sPh[f];
      acc = fma(cos(a), sAm[f], acc);
    }
  }
  if (valid) out[(int64_t)p * ldo + i] = coeff * acc;
}

// fp32 variant for bulk evaluation at candidate points (posterior sampling for acquisition,
// SURVEY 8f.1): phases in fp32, Cody-Waite reduction to [-pi, pi] and MUFU cos.approx,
// fp32 accumulation.  Absolute error ~1e-6 of a unit-variance prior; not used for RHS
// construction (the solves' right-hand sides stay on the fp64 kernel above).
__global__ void __launch_bounds__(RT) rff_eval32_kernel(const double* __restrict__ X, int ldx_row,
                                                        int dim, int64_t m,
                                                        const double* __restrict__ Om,
                                                        const double* __restrict__ ph,
                                                        const double* __restrict__ amp, int F,
                                                        double coeff, double* __restrict__ out,
                                                        int64_t ldo) {
  extern __shared__ float smf[];
  float* sOm = smf;                 // FT x dim
  float* sPh = sOm + FT * dim;      // FT
  float* sAm = sPh + FT;            // FT
  const int p = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x;
  const double* Omp = Om + (int64_t)p * F * dim;
  const double* php = ph + (int64_t)p * F;
  const double* amp_p = amp + (int64_t)p * F;
  float x[32];
  const bool valid = i < m;
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = (valid && k < dim) ? (float)X[i * ldx_row + k] : 0.0f;
  float acc = 0.0f;
  const float inv2pi = 0.15915494309189535f, twopi_hi = 6.28318548202514648f,
              twopi_lo = -1.74845553e-7f;
  for (int f0 = 0; f0 < F; f0 += FT) {
    const int nf = min(FT, F - f0);
    __syncthreads();
    for (int e = threadIdx.x; e < nf * dim; e += RT) {
      const int f = e % nf, k = e / nf;
      sOm[f * dim + k] = (float)Omp[(int64_t)k * F + f0 + f];
    }
    for (int e = threadIdx.x; e < nf; e += RT) {
      sPh[e] = (float)php[f0 + e];
      sAm[e] = (float)amp_p[f0 + e];
    }
    __syncthreads();
    for (int f = 0; f < nf; ++f) {
      float a = sPh[f];
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k < dim) a = fmaf(x[k], sOm[f * dim + k], a);
      const float nrev = (a * inv2pi + 12582912.0f) - 12582912.0f;  // rn(a / 2pi)
      a = fmaf(-nrev, twopi_hi, a);
      a = fmaf(-nrev, twopi_lo, a);
      float c;
      asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(a));
      acc = fmaf(c, sAm[f], acc);
    }
  }
  if (valid) out[(int64_t)p * ldo + i] = coeff * (double)acc;
}

}  // namespace

void launch_rff_eval32(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st) {
  TimedScope ts_("rff_eval32", st);
  WGP_REQUIRE(dim <= 32, "rff_eval: dim <= 32 supported, got %d", dim);
  if (m <= 0 || S <= 0) return;
  const size_t smem = sizeof(float) * (FT * dim + 2 * FT);
  dim3 grid(ceil_div(m, RT), S);
  rff_eval32_kernel<<<grid, RT, smem, st>>>(X, ldx_row, dim, m, Om, ph, amp, F, coeff, out, ldo);
  WGP_CUDA(cudaGetLastError());
}

void launch_rff_eval64(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st) {
  TimedScope ts_("rff_eval", st);
  WGP_REQUIRE(dim <= 32, "rff_eval: dim <= 32 supported, got %d", dim);
  if (m <= 0 || S <= 0) return;
  const size_t smem = sizeof(double) * (FT * dim + 2 * FT);
  dim3 grid(ceil_div(m, RT), S);
  rff_eval_kernel<<<grid, RT, smem, st>>>(X, ldx_row, dim, m, Om, ph, amp, F, coeff, out, ldo);
  WGP_CUDA(cudaGetLastError());
}

}  // namespace wgp
