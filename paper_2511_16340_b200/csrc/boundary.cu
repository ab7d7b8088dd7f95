// boundary.cu -- the remaining free functions of the reference API at the C-ABI:
//   cross_kernel       (kernel.cpp:74-89)       dense K(X*, X) block, fp64
//   relative_residual  (solvers.cpp:62-66)      |H v - b| / |b|, zero b -> invalid_argument
//   quadratic_objective(solvers.cpp:68-70)      0.5 v.Hv - v.b
//   init_weights       (solvers.cpp:27-48)      cold -> 0, warm -> [u1; 0]
//   build_sample_rhs   (sampling.cpp:56-64)     prior at the operator's rows + Rng(seed) noise
// The operator matvecs run on the device with the operator's precision; the final norms and
// dot products over n values are host fp64 sums in index order.
#include <cmath>
#include <cstring>
#include <vector>

#include "rng.h"
#include "solvers.h"

namespace wgp {
namespace {

// K[i + j*ldk] = k(x*_i, x_j): the reference's norm-form distance sqrt(max(|a|^2 + |b|^2 -
// 2 a.b, 0)) (kernel.cpp:39-46), Matern-3/2 s^2 (1+z) e^{-z} / RBF s^2 e^{-d^2/2l^2}, fp64.
__global__ void cross_kernel_kernel(const double* __restrict__ Xs, const double* __restrict__ sqs,
                                    int64_t m, const double* __restrict__ X,
                                    const double* __restrict__ sq, int64_t n, int dpad, int dim,
                                    KParams p, double* __restrict__ K, int64_t ldk) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i >= m || j >= n) return;
  double g = 0.0;
  for (int k = 0; k < dim; ++k) g = fma(Xs[i * dpad + k], X[j * dpad + k], g);
  double d2 = sqs[i] + sq[j] - 2.0 * g;
  d2 = d2 > 0.0 ? d2 : 0.0;
  double kv;
  if (p.kind == WGP_RBF) {
    kv = p.s2 * exp(-p.c1 * d2);
  } else {
    const double z = p.c1 * sqrt(d2);
    kv = p.s2 * (1.0 + z) * exp(-z);
  }
  K[i + j * ldk] = kv;
}

// select_peaks' per-sample argmax (thompson.cpp:199-203) over candidate groups: block
// (sample s, group g) scans rows [g0, g1) of value(i, s) = prior(i, s) + cross(i, s) and keeps
// the largest value, the lowest index on ties (Eigen maxCoeff / numpy argmax: first max).
__global__ void __launch_bounds__(256) group_argmax_kernel(const double* __restrict__ prior,
                                                           const double* __restrict__ cross, int64_t m,
                                                           int S, int groups,
                                                           int64_t* __restrict__ idx) {
  const int sidx = blockIdx.x, g = blockIdx.y;
  const int64_t g0 = m * g / groups, g1 = m * (g + 1) / groups;
  double best = -INFINITY;
  int64_t bi = g1;
  for (int64_t i = g0 + threadIdx.x; i < g1; i += blockDim.x) {
    const double v = prior[i + (int64_t)sidx * m] + cross[i * S + sidx];
    if (v > best) {  // strided scan in increasing i: strict > keeps the first max per thread
      best = v;
      bi = i;
    }
  }
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const double ov = sv[threadIdx.x + off];
      const int64_t oi = si[threadIdx.x + off];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) idx[(int64_t)sidx * groups + g] = si[0] < g1 ? si[0] : g0;
}

}  // namespace

void op_append_rows(Op& op, const double* host_rows, int64_t n_new, int64_t ld, int col_major);
void launch_rff_eval32(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st);
void launch_rff_eval64(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st);

}  // namespace wgp

using namespace wgp;

struct wgp_op : Op {};

template <typename F>
static wgp_status guard2(F&& f) {
  try {
    f();
    return WGP_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return WGP_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return WGP_CUDA_ERROR;
  }
}

// H V for host column-major V (n x s), into host Y (n x s), unsharded.
static void host_matvec(Op& op, const double* V, int64_t ldv, int s, std::vector<double>& Y) {
  WGP_REQUIRE(op.ctx->world == 1, "host-buffer operator applications need an unsharded context");
  const int64_t n = op.n;
  cudaStream_t st = op.ctx->stream;
  DBuf<double> stage((size_t)n * s), dV((size_t)n * s), dY((size_t)n * s);
  WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n, V, sizeof(double) * ldv,
                             sizeof(double) * n, s, cudaMemcpyHostToDevice, st));
  launch_colmajor_to_rows(stage.p, n, n, s, dV.p, true, st);
  launch_kmatvec_full(op, dV.p, dY.p, s, st);
  launch_rows_to_colmajor(dY.p, n, s, stage.p, n, true, st);
  Y.resize((size_t)n * s);
  WGP_CUDA(cudaMemcpyAsync(Y.data(), stage.p, sizeof(double) * n * s, cudaMemcpyDeviceToHost, st));
  WGP_CUDA(cudaStreamSynchronize(st));
}

extern "C" {

wgp_status wgp_cross_kernel(wgp_op* op, const double* Xstar, int64_t m, int64_t ldx, double* K,
                            int64_t ldk) {
  return guard2([&] {
    WGP_REQUIRE(op && (m == 0 || (Xstar && K)), "wgp_cross_kernel: null argument");
    WGP_REQUIRE(m >= 0 && ldx >= m && ldk >= m, "cross_kernel: bad shape");
    const int64_t n = op->n;
    if (m == 0 || n == 0) return;
    WGP_REQUIRE(n <= 65535, "wgp_cross_kernel: dense block limited to 65535 columns");
    WGP_CUDA(cudaSetDevice(op->ctx->device));
    cudaStream_t st = op->ctx->stream;
    Op tmp;  // X* rows staged row-major with their squared norms
    tmp.ctx = op->ctx;
    tmp.precision = WGP_F64;
    tmp.dim = op->dim;
    tmp.dpad = op->dpad;
    op_append_rows(tmp, Xstar, m, ldx, 1);
    DBuf<double> dK((size_t)m * n);
    dim3 grid((unsigned)((m + 127) / 128), (unsigned)n);
    cross_kernel_kernel<<<grid, 128, 0, st>>>(tmp.X64.p, tmp.sq64.p, m, op->X64.p, op->sq64.p, n,
                                              op->dpad, op->dim, op->kp(), dK.p, m);
    WGP_CUDA(cudaGetLastError());
    WGP_CUDA(cudaMemcpy2DAsync(K, sizeof(double) * ldk, dK.p, sizeof(double) * m,
                               sizeof(double) * m, n, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}

wgp_status wgp_relative_residual(wgp_op* op, const double* V, int64_t ldv, const double* B,
                                 int64_t ldb, int s, double* out) {
  return guard2([&] {
    WGP_REQUIRE(op && V && B && out && s >= 1, "wgp_relative_residual: bad argument");
    const int64_t n = op->n;
    WGP_REQUIRE(n >= 1 && ldv >= n && ldb >= n, "relative_residual: length mismatch");
    for (int c = 0; c < s; ++c) {  // solvers.cpp:63-64: zero b throws before any work
      double bb = 0.0;
      for (int64_t i = 0; i < n; ++i) bb += B[c * ldb + i] * B[c * ldb + i];
      WGP_REQUIRE(bb != 0.0, "relative_residual: zero right-hand side");
    }
    WGP_CUDA(cudaSetDevice(op->ctx->device));
    std::vector<double> Y;
    host_matvec(*op, V, ldv, s, Y);
    for (int c = 0; c < s; ++c) {
      double rr = 0.0, bb = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        const double r = Y[(size_t)c * n + i] - B[c * ldb + i];
        rr += r * r;
        bb += B[c * ldb + i] * B[c * ldb + i];
      }
      out[c] = std::sqrt(rr) / std::sqrt(bb);
    }
  });
}

wgp_status wgp_quadratic_objective(wgp_op* op, const double* V, int64_t ldv, const double* B,
                                   int64_t ldb, int s, double* out) {
  return guard2([&] {
    WGP_REQUIRE(op && V && B && out && s >= 1, "wgp_quadratic_objective: bad argument");
    const int64_t n = op->n;
    WGP_REQUIRE(n >= 1 && ldv >= n && ldb >= n, "quadratic_objective: length mismatch");
    WGP_CUDA(cudaSetDevice(op->ctx->device));
    std::vector<double> Y;
    host_matvec(*op, V, ldv, s, Y);
    for (int c = 0; c < s; ++c) {
      double vhv = 0.0, vb = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        vhv += V[c * ldv + i] * Y[(size_t)c * n + i];
        vb += V[c * ldv + i] * B[c * ldb + i];
      }
      out[c] = 0.5 * vhv - vb;
    }
  });
}

wgp_status wgp_init_weights(const double* u1, int64_t n1, int64_t n2, double* out) {
  return guard2([&] {
    WGP_REQUIRE(n1 >= 0 && n2 >= 0, "init_weights: negative block size");
    WGP_REQUIRE(out || n1 + n2 == 0, "wgp_init_weights: null output");
    for (int64_t i = 0; i < n1 + n2; ++i) out[i] = 0.0;
    if (u1)  // warm: [u1; 0] (length checked by the caller's u1 size = n1)
      for (int64_t i = 0; i < n1; ++i) out[i] = u1[i];
  });
}

wgp_status wgp_build_sample_rhs(wgp_op* op, const double* Omega, const double* phases,
                                const double* amps, int F, double signal_scale,
                                double noise_scale, uint64_t seed, double* out) {
  const wgp_status st = wgp_rff_eval(op, Omega, phases, amps, F, 1, signal_scale, nullptr, 0, 0, out,
                                     op ? (op->n > 0 ? op->n : 1) : 1);
  if (st != WGP_OK) return st;
  if (noise_scale > 0.0) {  // Rng(seed), one normal per row in index order
    Rng rng{seed};
    for (int64_t i = 0; i < op->n; ++i) out[i] += noise_scale * rng.normal();
  }
  return WGP_OK;
}

}  // extern "C"

extern "C" wgp_status wgp_posterior_select(wgp_op* op, const double* Omega, const double* phases,
                                           const double* amps, int F, int S, double signal_scale,
                                           const double* W, int64_t ldw, const double* Xstar,
                                           int64_t m, int64_t ldx, int groups, int fast,
                                           int64_t* idx) {
  return guard2([&] {
    WGP_REQUIRE(op && Omega && phases && amps && W && Xstar && idx, "wgp_posterior_select: null argument");
    WGP_REQUIRE(F >= 1 && S >= 1 && m >= 1 && groups >= 1 && groups <= m && ldx >= m && ldw >= op->n,
                "wgp_posterior_select: bad shape");
    WGP_REQUIRE(op->ctx->world == 1, "posterior_select: unsharded operators only");
    WGP_REQUIRE(op->n >= 1, "posterior_select: empty operator");
    WGP_CUDA(cudaSetDevice(op->ctx->device));
    cudaStream_t st = op->ctx->stream;
    const int64_t n = op->n;
    const int dim = op->dim;
    Op tmp;  // candidates, row-major with norms
    tmp.ctx = op->ctx;
    tmp.precision = WGP_F64;
    tmp.dim = dim;
    tmp.dpad = op->dpad;
    op_append_rows(tmp, Xstar, m, ldx, 1);
    const size_t nom = (size_t)S * F * dim, nf = (size_t)S * F;
    DBuf<double> dOm(nom), dPh(nf), dAm(nf), dPrior((size_t)m * S), dCross((size_t)m * S);
    DBuf<double> stage((size_t)n * S), dW((size_t)n * S);
    DBuf<int64_t> dIdx((size_t)S * groups);
    WGP_CUDA(cudaMemcpyAsync(dOm.p, Omega, sizeof(double) * nom, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(dPh.p, phases, sizeof(double) * nf, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(dAm.p, amps, sizeof(double) * nf, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n, W, sizeof(double) * ldw, sizeof(double) * n, S,
                               cudaMemcpyHostToDevice, st));
    launch_colmajor_to_rows(stage.p, n, n, S, dW.p, true, st);
    const double coeff = signal_scale * std::sqrt(2.0 / (double)F);  // sampling.cpp:40-41
    if (fast)
      launch_rff_eval32(tmp.X64.p, tmp.dpad, dim, m, dOm.p, dPh.p, dAm.p, F, S, coeff, dPrior.p, m, st);
    else
      launch_rff_eval64(tmp.X64.p, tmp.dpad, dim, m, dOm.p, dPh.p, dAm.p, F, S, coeff, dPrior.p, m, st);
    // K(X*, X) W: the tcgen05 cross mode on tensor-core operators when asked (and the
    // candidates fit its operand range), else the fp64 kernel
    if (!(fast && op_cross_tc(*op, tmp.X64.p, m, tmp.dpad, dW.p, S, dCross.p, st)))
      launch_kmatvec_simt<double>(*op, tmp.X64.p, m, 0, op->X64.p, n, dW.p, S, nullptr, dCross.p, false, st);
    group_argmax_kernel<<<dim3((unsigned)S, (unsigned)groups), 256, 0, st>>>(dPrior.p, dCross.p, m, S, groups,
                                                                            dIdx.p);
    WGP_CUDA(cudaGetLastError());
    WGP_CUDA(cudaMemcpyAsync(idx, dIdx.p, sizeof(int64_t) * S * groups, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}
