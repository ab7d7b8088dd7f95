// rff.cu -- random-Fourier-feature prior evaluation for S priors at once (K7):
//   out[i, p] = s_f sqrt(2/F) sum_f w_pf cos(x_i . omega_pf + phi_pf)
// restating eval_prior (sampling.cpp:37-46), which the reference runs once per prior as a
// dense X Omega^T GEMM followed by cos and a GEMV.  Here the phase contraction (K = d),
// the cos and the amplitude reduction are fused per (row tile, prior): the m x F phase
// matrix never exists.  fp64 for right-hand sides (not precision-relaxed); an fp32 variant
// (MUFU cos) for bulk candidate evaluation.
#include "solvers.h"

namespace wgp {
namespace {

constexpr int RT = 128, FT = 64;

// Phase, cos and amplitude FMA of one (point, feature); the operation order of the reference's
// dense form per entry (sampling.cpp:43-45): x.omega accumulated over k, + phi, cos, * w summed
// over features in order.
template <typename T>
__device__ __forceinline__ T rff_cos(T a);
template <>
__device__ __forceinline__ double rff_cos<double>(double a) { return cos(a); }
// fp32: Cody-Waite reduction to [-pi, pi] then MUFU cos.approx
template <>
__device__ __forceinline__ float rff_cos<float>(float a) {
  const float inv2pi = 0.15915494309189535f, twopi_hi = 6.28318548202514648f,
              twopi_lo = -1.74845553e-7f;
  const float nrev = (a * inv2pi + 12582912.0f) - 12582912.0f;  // rn(a / 2pi)
  a = fmaf(-nrev, twopi_hi, a);
  a = fmaf(-nrev, twopi_lo, a);
  float c;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(a));
  return c;
}

// One block per (tile of RT * PT points, prior): every thread keeps PT points' coordinates in
// registers (D a compile-time dimension: no predicated k loop), the block stages FT features
// of the prior in shared memory, and each staged feature row is read once per PT points.
// T = double: the RHS path (fp64, libdevice cos); T = float: candidate evaluation (fp32
// phases, MUFU cos, ~1e-6 absolute on a unit-variance prior).
template <typename T, int D, int PT>
__global__ void __launch_bounds__(RT) rff_kernel(const double* __restrict__ X, int ldx_row,
                                                 int64_t m, const double* __restrict__ Om,
                                                 const double* __restrict__ ph,
                                                 const double* __restrict__ amp, int F,
                                                 double coeff, double* __restrict__ out,
                                                 int64_t ldo) {
  __shared__ T sOm[FT * D];  // [f][k]
  __shared__ T sPh[FT], sAm[FT];
  const int p = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * RT * PT + threadIdx.x;
  const double* Omp = Om + (int64_t)p * F * D;  // F x D column-major
  const double* php = ph + (int64_t)p * F;
  const double* amp_p = amp + (int64_t)p * F;
  T x[PT][D];
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    const int64_t i = i0 + (int64_t)q * RT;
#pragma unroll
    for (int k = 0; k < D; ++k) x[q][k] = i < m ? (T)X[i * ldx_row + k] : T(0);
  }
  T acc[PT];
#pragma unroll
  for (int q = 0; q < PT; ++q) acc[q] = T(0);
  for (int f0 = 0; f0 < F; f0 += FT) {
    const int nf = min(FT, F - f0);
    __syncthreads();
    for (int e = threadIdx.x; e < nf * D; e += RT) {
      const int f = e % nf, k = e / nf;
      sOm[f * D + k] = (T)Omp[(int64_t)k * F + f0 + f];
    }
    for (int e = threadIdx.x; e < nf; e += RT) {
      sPh[e] = (T)php[f0 + e];
      sAm[e] = (T)amp_p[f0 + e];
    }
    __syncthreads();
    for (int f = 0; f < nf; ++f) {
      T om[D];
#pragma unroll
      for (int k = 0; k < D; ++k) om[k] = sOm[f * D + k];
      const T phf = sPh[f], amf = sAm[f];
#pragma unroll
      for (int q = 0; q < PT; ++q) {
        T a;
        if constexpr (sizeof(T) == 8) {  // fp64: sum_k x_k omega_k, then + phi (sampling.cpp:43)
          a = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) a = fma(x[q][k], om[k], a);
          a += phf;
        } else {  // fp32: phi folded in as the accumulator's start
          a = phf;
#pragma unroll
          for (int k = 0; k < D; ++k) a = fmaf(x[q][k], om[k], a);
        }
        acc[q] = fma(rff_cos<T>(a), amf, acc[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    const int64_t i = i0 + (int64_t)q * RT;
    if (i < m) out[(int64_t)p * ldo + i] = coeff * (double)acc[q];
  }
}

template <typename T, int PT>
void rff_dispatch(int dim, dim3 grid, cudaStream_t st, const double* X, int ldx_row, int64_t m,
                  const double* Om, const double* ph, const double* amp, int F, double coeff,
                  double* out, int64_t ldo) {
  switch (dim) {
#define WGP_RFF_CASE(D)                                                                      \
  case D:                                                                                    \
    rff_kernel<T, D, PT><<<grid, RT, 0, st>>>(X, ldx_row, m, Om, ph, amp, F, coeff, out, ldo); \
    break;
    WGP_RFF_CASE(1) WGP_RFF_CASE(2) WGP_RFF_CASE(3) WGP_RFF_CASE(4) WGP_RFF_CASE(5)
    WGP_RFF_CASE(6) WGP_RFF_CASE(7) WGP_RFF_CASE(8) WGP_RFF_CASE(9) WGP_RFF_CASE(10)
    WGP_RFF_CASE(11) WGP_RFF_CASE(12) WGP_RFF_CASE(13) WGP_RFF_CASE(14) WGP_RFF_CASE(15)
    WGP_RFF_CASE(16) WGP_RFF_CASE(17) WGP_RFF_CASE(18) WGP_RFF_CASE(19) WGP_RFF_CASE(20)
    WGP_RFF_CASE(21) WGP_RFF_CASE(22) WGP_RFF_CASE(23) WGP_RFF_CASE(24) WGP_RFF_CASE(25)
    WGP_RFF_CASE(26) WGP_RFF_CASE(27) WGP_RFF_CASE(28) WGP_RFF_CASE(29) WGP_RFF_CASE(30)
    WGP_RFF_CASE(31) WGP_RFF_CASE(32)
#undef WGP_RFF_CASE
    default:
      throw_error(WGP_INVALID_ARGUMENT, "rff_eval: dim <= 32 supported, got %d", dim);
  }
}

}  // namespace

void launch_rff_eval32(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st) {
  TimedScope ts_("rff_eval32", st);
  WGP_REQUIRE(dim >= 1 && dim <= 32, "rff_eval: dim <= 32 supported, got %d", dim);
  if (m <= 0 || S <= 0) return;
  constexpr int PT = 4;
  dim3 grid(ceil_div(m, RT * PT), S);
  rff_dispatch<float, PT>(dim, grid, st, X, ldx_row, m, Om, ph, amp, F, coeff, out, ldo);
  WGP_CUDA(cudaGetLastError());
}

void launch_rff_eval64(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st) {
  TimedScope ts_("rff_eval", st);
  WGP_REQUIRE(dim >= 1 && dim <= 32, "rff_eval: dim <= 32 supported, got %d", dim);
  if (m <= 0 || S <= 0) return;
  constexpr int PT = 2;
  dim3 grid(ceil_div(m, RT * PT), S);
  rff_dispatch<double, PT>(dim, grid, st, X, ldx_row, m, Om, ph, amp, F, coeff, out, ldo);
  WGP_CUDA(cudaGetLastError());
}

}  // namespace wgp
