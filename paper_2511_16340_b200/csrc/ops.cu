// ops.cu -- device-resident operator state: row append (K8) and kernel-matvec dispatch.
//
// append_rows restates the growth half of extend_system (kernel.cpp:108-130) and
// bo_round (thompson.cpp:403-422) for a matrix-free operator: new rows of X are
// appended to the device copy (capacity doubling, old rows never re-uploaded) with their
// squared norms, so the next system is ready without recomputing or storing H11.
#include <cstdlib>
#include <vector>
#include "solvers.h"

namespace wgp {
namespace {

__global__ void append_rows_kernel(const double* __restrict__ src, int64_t ld, int col_major,
                                   int64_t n_new, int dim, int dpad, int64_t row_off,
                                   double* __restrict__ X64, double* __restrict__ sq64,
                                   float* __restrict__ X32, float* __restrict__ sq32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_new;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    float acc32 = 0.0f;
    const int64_t g = row_off + i;
    for (int k = 0; k < dpad; ++k) {
      double x = 0.0;
      if (k < dim) x = col_major ? src[(int64_t)k * ld + i] : src[i * ld + k];
      X64[g * dpad + k] = x;
      acc += x * x;  // sum in k order, as Eigen's rowwise().squaredNorm() / rankUpdate diagonal
      if (X32) {
        const float xf = (float)x;
        X32[g * dpad + k] = xf;
        acc32 = fmaf(xf, xf, acc32);
      }
    }
    sq64[g] = acc;
    if (sq32) sq32[g] = acc32;
  }
}

}  // namespace

// out[e] = sum over q of slots[q][e], in rank order (loopback all-reduce).
__global__ void sum_slots_kernel(const double* __restrict__ slots, int world, size_t count,
                                 double* __restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
       e += (size_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int q = 0; q < world; ++q) a += slots[(size_t)q * count + e];
    out[e] = a;
  }
}

void launch_sum_slots(const double* slots, int world, size_t count, double* out, cudaStream_t st) {
  if (!count) return;
  const unsigned g = (unsigned)std::min<size_t>((count + 255) / 256, 148 * 8);
  sum_slots_kernel<<<g, 256, 0, st>>>(slots, world, count, out);
  WGP_CUDA(cudaGetLastError());
}

void op_append_rows(Op& op, const double* host_rows, int64_t n_new, int64_t ld, int col_major) {
  if (n_new <= 0) return;
  cudaStream_t st = op.ctx->stream;
  const int64_t need = op.n + n_new;
  if (need > op.cap) {
    int64_t cap = op.cap > 0 ? op.cap : 1024;
    while (cap < need) cap *= 2;
    DBuf<double> X64((size_t)cap * op.dpad), sq64(cap);
    DBuf<float> X32, sq32;
    if (!op.f64()) {
      X32.alloc((size_t)cap * op.dpad);
      sq32.alloc(cap);
    }
    if (op.n > 0) {
      WGP_CUDA(cudaMemcpyAsync(X64.p, op.X64.p, sizeof(double) * op.n * op.dpad,
                               cudaMemcpyDeviceToDevice, st));
      WGP_CUDA(cudaMemcpyAsync(sq64.p, op.sq64.p, sizeof(double) * op.n, cudaMemcpyDeviceToDevice,
                               st));
      if (!op.f64()) {
        WGP_CUDA(cudaMemcpyAsync(X32.p, op.X32.p, sizeof(float) * op.n * op.dpad,
                                 cudaMemcpyDeviceToDevice, st));
        WGP_CUDA(cudaMemcpyAsync(sq32.p, op.sq32.p, sizeof(float) * op.n,
                                 cudaMemcpyDeviceToDevice, st));
      }
    }
    WGP_CUDA(cudaStreamSynchronize(st));
    op.X64 = std::move(X64);
    op.sq64 = std::move(sq64);
    op.X32 = std::move(X32);
    op.sq32 = std::move(sq32);
    op.cap = cap;
  }
  // stage the host rows (column-major n_new x dim with ld, or row-major with stride ld)
  const size_t elems = col_major ? (size_t)ld * (op.dim - 1) + n_new : (size_t)ld * (n_new - 1) + op.dim;
  DBuf<double> stage(elems);
  WGP_CUDA(cudaMemcpyAsync(stage.p, host_rows, sizeof(double) * elems, cudaMemcpyHostToDevice, st));
  int grid = ceil_div(n_new, 256);
  if (grid > 148 * 8) grid = 148 * 8;
  append_rows_kernel<<<grid, 256, 0, st>>>(stage.p, ld, col_major, n_new, op.dim, op.dpad, op.n,
                                           op.X64.p, op.sq64.p, op.f64() ? nullptr : op.X32.p,
                                           op.f64() ? nullptr : op.sq32.p);
  WGP_CUDA(cudaGetLastError());
  if (op.h_center.empty()) {
    // Translation for the tensor-core operands: the mean of the first batch.  Distances
    // are translation invariant; centering shrinks |x|^2 and with it the cancellation in
    // |x|^2 + |y|^2 - 2 x.y.  Fixed afterwards so appended rows reuse it.
    op.h_center.assign(op.dim, 0.0);
    for (int64_t i = 0; i < n_new; ++i)
      for (int k = 0; k < op.dim; ++k)
        op.h_center[k] += col_major ? host_rows[(int64_t)k * ld + i] : host_rows[i * ld + k];
    for (int k = 0; k < op.dim; ++k) op.h_center[k] /= (double)n_new;
    op.center.alloc(op.dim);
    WGP_CUDA(cudaMemcpyAsync(op.center.p, op.h_center.data(), sizeof(double) * op.dim,
                             cudaMemcpyHostToDevice, st));
  }
  WGP_CUDA(cudaStreamSynchronize(st));
  op.n = need;
  op.tc_dirty = true;
}

static void ensure_tc_operands(Op& op, cudaStream_t st) {
  if (!op.tc_dirty) return;
  tc_build_operands(op, op.XA, op.XB, op.center.p, st);
  op.tc_dirty = false;
}

// Cross mode on the tensor cores: Y (m x s) = K(X*, X) W for device rows X* (row-major,
// stride dpad).  Returns false if this operator / these points need the fp64 path.
bool op_cross_tc(Op& op, const double* Xs, int64_t m, int dpad, const double* W, int s, double* Y,
                 cudaStream_t st) {
  if (!op.tensor() || !tc_supported(op.dim, op.precision)) return false;
  ensure_tc_operands(op, st);
  DBuf<float> XAc;
  if (!tc_build_cross_rows(op, Xs, m, dpad, XAc, st)) return false;
  launch_kmatvec_tc(op, XAc.p, op.XB.p, m, 0, op.n, W, s, nullptr, Y, false, op.vt, op.vchunk,
                    op.ychunk, op.ysplit, st);
  return true;
}

static void dispatch(Op& op, const double* B, const double* V, double* Y, int s, cudaStream_t st) {
  int64_t r0, r1;
  op.local_rows(&r0, &r1);
  if (op.tensor() && tc_supported(op.dim, op.precision)) {
    ensure_tc_operands(op, st);
    launch_kmatvec_tc(op, op.XA.p, op.XB.p, r1 - r0, r0, op.n, V, s, B, Y, true, op.vt,
                      op.vchunk, op.ychunk, op.ysplit, st);
  } else if (op.f64()) {
    launch_kmatvec_simt<double>(op, op.X64.p + r0 * op.dpad, r1 - r0, r0, op.X64.p, op.n, V, s, B,
                                Y, true, st);
  } else {
    launch_kmatvec_simt<float>(op, op.X32.p + r0 * op.dpad, r1 - r0, r0, op.X32.p, op.n, V, s, B,
                               Y, true, st);
  }
}

int launch_kmatvec_parts(Op& op, const double* V, double* Y, int s, cudaStream_t st, int parts,
                         cudaEvent_t* part_done) {
  if (op.ctx->world == 1 && op.tensor() && tc_supported(op.dim, op.precision) && s <= 64 &&
      op.n >= 2 * 128 * parts) {
    ensure_tc_operands(op, st);
    launch_kmatvec_tc(op, op.XA.p, op.XB.p, op.n, 0, op.n, V, s, nullptr, Y, true, op.vt, op.vchunk,
                      op.ychunk, op.ysplit, st, parts, part_done);
    return parts;
  }
  dispatch(op, nullptr, V, Y, s, st);
  return 1;
}

namespace {
// comma-separated cumulative sixteenths from the environment (probe overrides), else def
std::vector<int> sixteenths(const char* env, std::vector<int> def) {
  const char* e = getenv(env);
  if (!e || !*e) return def;
  std::vector<int> v;
  for (const char* p = e; *p;) {
    char* end = nullptr;
    const long x = strtol(p, &end, 10);
    if (end == p) break;
    if (x > 0 && x < 16 && (v.empty() || x > v.back())) v.push_back((int)x);
    p = *end == ',' ? end + 1 : end;
  }
  return v;
}
}  // namespace

int64_t row_part_begin(int64_t nrows, int part, int parts) {
  const int64_t tiles = (nrows + 127) / 128;
  int64_t t = tiles * part / parts;
  if (parts == Ctx::kHostParts && part > 0 && part < parts) {
    static const std::vector<int> cuts = sixteenths("WGP_HOST_ROWCUTS", {8, 12, 15});
    if ((int)cuts.size() == parts - 1) t = tiles * cuts[part - 1] / 16;
  }
  return std::min(nrows, t * 128);
}

int host_col_parts(int64_t n, int64_t* cb) {
  static const std::vector<int> cuts = sixteenths("WGP_HOST_COLCUTS", {2, 8});
  int ncp = 0;
  cb[0] = 0;
  for (int c : cuts) {
    if (ncp + 1 >= Ctx::kColParts) break;
    const int64_t b = n * c / 16 / 128 * 128;
    if (b > cb[ncp]) cb[++ncp] = b;
  }
  cb[++ncp] = n;
  return ncp;
}

bool kmatvec_colphased_ok(const Op& op, int s, int parts) {
  return op.ctx->world == 1 && op.tensor() && tc_supported(op.dim, op.precision) && s <= 64 &&
         op.n >= 2 * 128 * parts && op.n >= 16384;
}

int launch_kmatvec_colphased(Op& op, const double* V, double* Y, int s, cudaStream_t st,
                             const int64_t* cb, int ncp, const cudaEvent_t* vready, int parts,
                             cudaEvent_t* part_done) {
  if (!kmatvec_colphased_ok(op, s, parts)) return 0;
  ensure_tc_operands(op, st);
  const size_t rb = (size_t)tc_k1(op.dim, op.precision, op.tc_f16) * (op.tc_f16 ? 2 : 4);
  const char* XB = reinterpret_cast<const char*>(op.XB.p);
  for (int k = 0; k < ncp; ++k) {
    const int64_t a = cb[k], b = cb[k + 1];
    WGP_REQUIRE(a % 128 == 0 && b > a && b <= op.n, "kmatvec_colphased: bad column parts");
    WGP_CUDA(cudaStreamWaitEvent(st, vready[k], 0));
    const bool last = k == ncp - 1;
    // gram for every part (the exact diagonal wherever it falls); the noise term once, in the
    // last part, from the complete V
    launch_kmatvec_tc(op, op.XA.p, reinterpret_cast<const float*>(XB + a * rb), op.n, 0, b - a,
                      V + a * s, s, nullptr, Y, true, op.vt, op.vchunk, op.ychunk, op.ysplit, st,
                      last ? parts : 1, last ? part_done : nullptr, a, k > 0 ? Y : nullptr, 1.0,
                      last ? 1 : 0, V);
  }
  return parts;
}

void launch_kmatvec_overlap(Op& op, const double* B, const double* V, double* Y, int s,
                            cudaEvent_t gathered, cudaStream_t st) {
  if (!gathered) return dispatch(op, B, V, Y, s, st);
  int64_t r0, r1;
  op.local_rows(&r0, &r1);
  if (op.tensor() && tc_supported(op.dim, op.precision)) {
    // local diagonal block (gram: sigma^2 V and the exact diagonal), then, once V is
    // complete, the columns before and after the slot accumulated into Y
    ensure_tc_operands(op, st);
    const size_t rb = (size_t)tc_k1(op.dim, op.precision, op.tc_f16) * (op.tc_f16 ? 2 : 4);
    const char* XB = reinterpret_cast<const char*>(op.XB.p);
    launch_kmatvec_tc(op, op.XA.p, reinterpret_cast<const float*>(XB + r0 * rb), r1 - r0, r0, r1 - r0,
                      V + r0 * s, s, B, Y, true, op.vt, op.vchunk, op.ychunk, op.ysplit, st, 1, nullptr, r0);
    WGP_CUDA(cudaStreamWaitEvent(st, gathered, 0));
    const double sg = B ? -1.0 : 1.0;
    launch_kmatvec_tc(op, op.XA.p, op.XB.p, r1 - r0, r0, r0, V, s, nullptr, Y, false, op.vt, op.vchunk,
                      op.ychunk, op.ysplit, st, 1, nullptr, 0, Y, sg);
    launch_kmatvec_tc(op, op.XA.p, reinterpret_cast<const float*>(XB + r1 * rb), r1 - r0, r0, op.n - r1,
                      V + r1 * s, s, nullptr, Y, false, op.vt, op.vchunk, op.ychunk, op.ysplit, st, 1,
                      nullptr, r1, Y, sg);
  } else if (op.f64()) {
    ColPhase ph;
    ph.c0 = r0;
    ph.c1 = r1;
    ph.ready = gathered;
    launch_kmatvec_simt<double>(op, op.X64.p + r0 * op.dpad, r1 - r0, r0, op.X64.p, op.n, V, s, B, Y,
                                true, st, &ph);
  } else {
    WGP_CUDA(cudaStreamWaitEvent(st, gathered, 0));
    dispatch(op, B, V, Y, s, st);
  }
}

// Y (this rank's rows) = H V, V full n x s (fp64 row-major).
void launch_kmatvec_full(Op& op, const double* V, double* Y, int s, cudaStream_t st) {
  dispatch(op, nullptr, V, Y, s, st);
}

void launch_residual_f64(Op& op, const double* B, const double* V, double* Y, int s,
                         cudaStream_t st) {
  int64_t r0, r1;
  op.local_rows(&r0, &r1);
  launch_kmatvec_simt<double>(op, op.X64.p + r0 * op.dpad, r1 - r0, r0, op.X64.p, op.n, V, s, B, Y,
                              true, st);
}

// Y = B - H V  (B and Y: this rank's rows; V full)
void launch_residual(Op& op, const double* B, const double* V, double* Y, int s, cudaStream_t st) {
  dispatch(op, B, V, Y, s, st);
}

}  // namespace wgp
