// ascent.cu -- posterior-sample gradients and batched Adam peak ascent on the device
// (SURVEY 8f.2): grad_posterior (sampling.cpp:77-87, with grad_prior :48-54) and
// ascend_peaks (thompson.cpp:209-258) for all samples and all start points at once.  The
// reference runs one trajectory at a time on the host, re-evaluating the posterior sample at
// every step; here one CTA owns one trajectory (sample s, start t) and evaluates value and
// gradient together per step: the n representer terms and the F random features are split
// over the threads and reduced in a fixed order (deterministic), fp64 throughout.
#include <cmath>

#include "common.cuh"

namespace wgp {
namespace {

constexpr int AT = 256;  // threads per trajectory
constexpr int MAXD = 32;

struct PostArgs {
  const double* X;   // training rows, row-major [n][dpad]
  int dpad, dim;
  int64_t n;
  const double* Om;  // S priors x (F x dim column-major)
  const double* ph;  // S x F
  const double* am;  // S x F
  int F;
  double coeff;      // s_f sqrt(2 / F)
  const double* W;   // representer weights [S][n]
  int kind;
  double l, s2;
};

// value and gradient of posterior sample s at x (shared, dim entries); result in out[0..dim]
// (value first), valid in every thread after the call.
__device__ void eval_grad(const PostArgs& a, int s, const double* x, double* red, double* out) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int dim = a.dim;
  double acc[MAXD + 1];
#pragma unroll
  for (int k = 0; k <= MAXD; ++k) acc[k] = 0.0;
  // representer part: sum_j w_j k(x, x_j) and its gradient
  const double* w = a.W + (int64_t)s * a.n;
  const double il2 = 1.0 / (a.l * a.l);
  for (int64_t j = tid; j < a.n; j += AT) {
    double r2 = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double df = a.X[j * a.dpad + k] - x[k];
      r2 = fma(df, df, r2);
    }
    double kv, f;
    if (a.kind == WGP_RBF) {
      const double e = exp(-0.5 * r2 * il2);
      kv = a.s2 * e;
      f = w[j] * a.s2 * il2 * e;
    } else {
      const double z = 1.7320508075688772935 * sqrt(r2) / a.l;
      const double e = exp(-z);
      kv = a.s2 * (1.0 + z) * e;
      f = w[j] * 3.0 * a.s2 * il2 * e;
    }
    acc[0] = fma(w[j], kv, acc[0]);
    for (int k = 0; k < dim; ++k) acc[1 + k] = fma(f, a.X[j * a.dpad + k] - x[k], acc[1 + k]);
  }
  // prior part: coeff sum_f a_f cos(w_f.x + phi_f) and -coeff sum_f a_f sin(.) w_f
  const double* Om = a.Om + (int64_t)s * a.F * dim;
  const double* ph = a.ph + (int64_t)s * a.F;
  const double* am = a.am + (int64_t)s * a.F;
  for (int f = tid; f < a.F; f += AT) {
    double arg = ph[f];
    for (int k = 0; k < dim; ++k) arg = fma(Om[(int64_t)k * a.F + f], x[k], arg);
    double sn, cs;
    sincos(arg, &sn, &cs);
    acc[0] = fma(a.coeff * am[f], cs, acc[0]);
    const double gs = -a.coeff * am[f] * sn;
    for (int k = 0; k < dim; ++k) acc[1 + k] = fma(gs, Om[(int64_t)k * a.F + f], acc[1 + k]);
  }
  // fixed-order block reduction: warp shuffles, then warp partials summed in warp order
  for (int k = 0; k <= dim; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid * (MAXD + 1) + k] = v;
  }
  __syncthreads();
  if (tid <= dim) {
    double v = 0.0;
    for (int q = 0; q < AT / 32; ++q) v += red[q * (MAXD + 1) + tid];
    out[tid] = v;
  }
  __syncthreads();
}

// grad_posterior at m points; point i belongs to sample sidx[i].  Xs, G: [m][dim].
__global__ void __launch_bounds__(AT) grad_kernel(PostArgs a, const double* __restrict__ Xs,
                                                  const int* __restrict__ sidx,
                                                  double* __restrict__ G) {
  __shared__ double x[MAXD], red[(AT / 32) * (MAXD + 1)], out[MAXD + 1];
  const int64_t i = blockIdx.x;
  if (threadIdx.x < a.dim) x[threadIdx.x] = Xs[i * a.dim + threadIdx.x];
  __syncthreads();
  eval_grad(a, sidx[i], x, red, out);
  if (threadIdx.x < a.dim) G[i * a.dim + threadIdx.x] = out[1 + threadIdx.x];
}

// One Adam trajectory per CTA: start starts[(s * P + t)][dim]; best value / point written
// per trajectory (the host combines them per sample in start order, strict >).
__global__ void __launch_bounds__(AT) ascend_kernel(PostArgs a, const double* __restrict__ starts,
                                                    int P, int steps, double rate,
                                                    double* __restrict__ best_val,
                                                    double* __restrict__ best_x) {
  __shared__ double x[MAXD], mo[MAXD], ve[MAXD], red[(AT / 32) * (MAXD + 1)], out[MAXD + 1];
  __shared__ double bx[MAXD];
  __shared__ double bv;
  __shared__ int stop;
  const int t = blockIdx.x, s = blockIdx.y;
  const int dim = a.dim;
  const int64_t traj = (int64_t)s * P + t;
  if (threadIdx.x < dim) {
    x[threadIdx.x] = starts[traj * dim + threadIdx.x];
    mo[threadIdx.x] = 0.0;
    ve[threadIdx.x] = 0.0;
  }
  __syncthreads();
  eval_grad(a, s, x, red, out);
  if (threadIdx.x == 0) {
    bv = out[0];  // > -inf always for a finite value
    for (int k = 0; k < dim; ++k) bx[k] = x[k];
    stop = 0;
  }
  __syncthreads();
  for (int k = 1; k <= steps; ++k) {
    if (threadIdx.x == 0) {
      bool finite = true;
      for (int q = 0; q < dim; ++q) finite = finite && isfinite(out[1 + q]);
      if (!finite) {
        stop = 1;  // freeze this trajectory, keep best-seen
      } else {
        const double bc1 = 1.0 - pow(0.9, (double)k), bc2 = 1.0 - pow(0.999, (double)k);
        for (int q = 0; q < dim; ++q) {
          const double g = out[1 + q];
          mo[q] = 0.9 * mo[q] + 0.1 * g;
          ve[q] = 0.999 * ve[q] + 0.001 * (g * g);
          const double step = (mo[q] / bc1) / (sqrt(ve[q] / bc2) + 1e-8);
          double xn = x[q] + rate * step;
          x[q] = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
        }
      }
    }
    __syncthreads();
    if (stop) break;
    eval_grad(a, s, x, red, out);
    if (threadIdx.x == 0 && out[0] > bv) {
      bv = out[0];
      for (int q = 0; q < dim; ++q) bx[q] = x[q];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) best_val[traj] = bv;
  if (threadIdx.x < dim) best_x[traj * dim + threadIdx.x] = bx[threadIdx.x];
}

}  // namespace

static PostArgs post_args(const Op& op, const double* Om, const double* ph, const double* am, int F,
                          double coeff, const double* W) {
  PostArgs a;
  a.X = op.X64.p;
  a.dpad = op.dpad;
  a.dim = op.dim;
  a.n = op.n;
  a.Om = Om;
  a.ph = ph;
  a.am = am;
  a.F = F;
  a.coeff = coeff;
  a.W = W;
  a.kind = op.kind;
  a.l = op.lengthscale;
  a.s2 = op.signal_scale * op.signal_scale;
  return a;
}

void launch_grad_posterior(const Op& op, const double* Om, const double* ph, const double* am,
                           int F, double coeff, const double* W, const double* Xs,
                           const int* sidx, int64_t m, double* G, cudaStream_t st) {
  WGP_REQUIRE(op.dim <= MAXD, "grad_posterior: dim <= %d supported", MAXD);
  if (m <= 0) return;
  grad_kernel<<<(unsigned)m, AT, 0, st>>>(post_args(op, Om, ph, am, F, coeff, W), Xs, sidx, G);
  WGP_CUDA(cudaGetLastError());
}

void launch_ascend(const Op& op, const double* Om, const double* ph, const double* am, int F,
                   double coeff, const double* W, int S, const double* starts, int P, int steps,
                   double rate, double* best_val, double* best_x, cudaStream_t st) {
  WGP_REQUIRE(op.dim <= MAXD, "ascend_peaks: dim <= %d supported", MAXD);
  if (S <= 0 || P <= 0) return;
  ascend_kernel<<<dim3(P, S), AT, 0, st>>>(post_args(op, Om, ph, am, F, coeff, W), starts, P, steps,
                                           rate, best_val, best_x);
  WGP_CUDA(cudaGetLastError());
}

}  // namespace wgp
