// common.cuh -- shared internals of libwarmgp_b200.so (not part of the ABI).
//
// Device data layout:
//   X    : row-major [cap][dpad]   fp64 (always) and fp32 (fp32 precisions), dpad = dim
//          rounded up to 8 (one tf32 K-atom = 32 bytes), zero padded.
//   sq   : [cap] squared row norms (fp64 and fp32), used by the norm-form distance
//          |x|^2 + |y|^2 - 2 x.y of kernel.cpp:39-46/48-72.
//   RHS  : row-major [n][s] in the compute type ("RHS-interleaved"): one row of X
//          meets all s right-hand sides in one contiguous 4*s / 8*s byte span.
//   L/M  : preconditioner factors row-major [n][kpad] fp64 (+ fp32 copy of M).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/warmgp_capi.h"

namespace wgp {

constexpr int kChunkRows = 512;  // fixed reduction chunk: sums are world-size independent

struct Error : std::runtime_error {
  wgp_status code;
  int col = -1;
  int iterations = 0;
  Error(wgp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_error(wgp_status code, const char* fmt, ...);
void set_last_error(const char* msg);  // the thread-local message of wgp_last_error()

#define WGP_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::wgp::throw_error(e_ == cudaErrorMemoryAllocation ? WGP_OOM : WGP_CUDA_ERROR,     \
                         "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
  } while (0)

#define WGP_REQUIRE(cond, ...)                                  \
  do {                                                          \
    if (!(cond)) ::wgp::throw_error(WGP_INVALID_ARGUMENT, __VA_ARGS__); \
  } while (0)

// Device block cache (mem.cpp): freed blocks are kept per (device, size bucket) and handed
// out again instead of a new cudaMalloc; a free synchronises the device first, as cudaFree
// did, so a cached block is never still in use by queued work.  Per-call cudaMalloc /
// cudaFree pairs showed as sporadic 0.1-0.25 s stalls of the solves.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);

// Owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
    n = count;
  }
  void ensure(size_t count) { if (count > n) alloc(count); }
  // for buffers sized by a growing system (append_rows sweeps): 25% headroom per reallocation
  void ensure_grow(size_t count) { if (count > n) alloc(count + count / 4); }
  void release() { if (p) dev_free(p, n * sizeof(T)); p = nullptr; n = 0; }
};

// Owning pinned host buffer (async device-to-host copies of per-iteration records).
struct PinnedBuf {
  unsigned char* p = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() { if (p) cudaFreeHost(p); }
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    WGP_CUDA(cudaMallocHost(&p, bytes));
    n = bytes;
  }
};

// Kernel-map parameters (kernel.cpp:17-21 Matern-3/2; RBF extension).
struct KParams {
  int kind;        // WGP_MATERN32 / WGP_RBF
  double c1;       // Matern: sqrt(3)/l   RBF: 1/(2 l^2)
  double s2;       // signal^2
  double noise2;   // sigma_n^2 (diagonal of H only)
};

#ifdef __CUDACC__
// e^x for x <= 0 in fp64 DFMA/integer ops: n = rn(x log2 e) via the 1.5*2^52 shifter,
// r = x - n ln2 (Cody-Waite hi/lo, |r| <= ln2/2), e^r by its degree-11 Taylor polynomial
// (max relative error 9e-15 over [-708, 0], measured against libm), 2^n inserted into the
// exponent field.  x is clamped at -708 (e^-708 ~ 3e-308: below that a kernel entry
// contributes nothing at fp64 resolution).  ~16 DP ops against ~25+ for the libdevice exp
// with its special-case handling, on the pipe that bounds this kernel.
__device__ __forceinline__ double exp_neg(double x) {
  x = fmax(x, -708.0);
  const double shifter = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, 1.4426950408889634, shifter);
  const double n = t - shifter;
  double r = fma(-n, 6.93147180369123816490e-01, x);
  r = fma(-n, 1.90821492927058770002e-10, r);
  double q = 2.505210838544171877505e-08;  // 1/11!
  q = fma(q, r, 2.755731922398589065256e-07);
  q = fma(q, r, 2.755731922398589065256e-06);
  q = fma(q, r, 2.480158730158730158730e-05);
  q = fma(q, r, 1.984126984126984126984e-04);
  q = fma(q, r, 1.388888888888888888889e-03);
  q = fma(q, r, 8.333333333333333333333e-03);
  q = fma(q, r, 4.166666666666666666667e-02);
  q = fma(q, r, 1.666666666666666666667e-01);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const long long ni = __double_as_longlong(t) - __double_as_longlong(shifter);
  return __longlong_as_double(__double_as_longlong(q) + (ni << 52));
}
#endif

struct Comm;  // NCCL / loopback plumbing (dist.cpp)

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host-API result copies overlapping compute
  static constexpr int kHostParts = 4;  // row parts of the host-buffer matvec (copy overlap)
  cudaEvent_t part_ev[kHostParts] = {};
  static constexpr int kColParts = 4;  // max column parts of its input copy (copy overlap)
  cudaEvent_t col_ev[kColParts] = {};
  // sharded operators: the row all-gather runs on comm_stream while the compute stream works
  // on the local diagonal block (comm_ev[0]: slot ready, comm_ev[1]: gather complete)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comm_ev[2] = {nullptr, nullptr};
  int rank = 0, world = 1;
  Comm* comm = nullptr;
};

struct Op {
  Ctx* ctx = nullptr;
  int kind = WGP_MATERN32;
  double lengthscale = 1, signal_scale = 1, noise_scale = 1e-3;
  int precision = WGP_F64;
  int dim = 0, dpad = 0;
  int64_t n = 0, cap = 0;
  DBuf<double> X64, sq64;
  DBuf<float> X32, sq32;
  DBuf<unsigned char> scratch[3];  // host-boundary staging, reused across calls
  // tensor-core path: tiled 3xTF32 operand rows (rebuilt lazily after appends), the
  // translation applied before forming them, and per-call V staging.
  DBuf<float> XA, XB, vt;
  DBuf<double> center, vchunk, ychunk, ysplit;
  mutable DBuf<double> f64split;  // fp64 kernel-matvec column-split partials
  mutable DBuf<double> krows_part;  // SGD minibatch-row partials per j range
  std::vector<double> h_center;
  // solver work buffers (SolverWork<double>) and preconditioner factors (PrecondDev), kept
  // across solve calls on this operator: reallocated only when they must grow, so a solve
  // pays no cudaMalloc / synchronous cudaFree for its [n][s] vectors (calls on one handle
  // are never concurrent)
  std::shared_ptr<void> solve_cache, precond_cache;
  // true-residual mode of the CG solver on fp32 operators (wgp_op_set_residual_mode):
  // WGP_RESIDUAL_DIRECT recomputes b - H v with the operator itself; WGP_RESIDUAL_ANCHORED
  // evaluates it as r_a - H (v - v_a) with r_a = b - H v_a from the fp64 kernel at anchor
  // iterates v_a, re-anchoring when the predicted error of the fast part reaches a fraction
  // of the residual (solvers.cu).
  int resid_mode = WGP_RESIDUAL_DIRECT;
  int last_anchors = 0;  // fp64 anchor evaluations of the last CG solve
  bool tc_dirty = true;
  // GEMM1 operand format chosen at operand build: fp16 splits of x / l (kind::f16, half the
  // bytes and MMA time of tf32) when the scaled coordinates fit fp16, else tf32 splits of x.
  bool tc_f16 = false;
  KParams kp() const {
    KParams p;
    p.kind = kind;
    p.c1 = kind == WGP_MATERN32 ? 1.7320508075688772935 / lengthscale
                                : 0.5 / (lengthscale * lengthscale);
    p.s2 = signal_scale * signal_scale;
    p.noise2 = noise_scale * noise_scale;
    return p;
  }
  bool f64() const { return precision == WGP_F64; }
  bool tensor() const { return precision == WGP_F32_3XTF32 || precision == WGP_TF32; }
  void local_rows(int64_t* r0, int64_t* r1) const {
    wgp_shard_range(n, ctx->world, ctx->rank, r0, r1);
  }
};

// Sum of chunk partials part[q * stride] for q = 0..nch-1 in index order (the fixed order
// that keeps sums independent of s and of the world size).  The loads are independent of the
// running sum, so they are issued 8 ahead instead of one dependent L2 round trip per chunk.
__device__ __forceinline__ double chunk_sum_ordered(const double* __restrict__ part, int nch,
                                                    int64_t stride) {
  double acc = 0.0;
  int q = 0;
  for (; q + 8 <= nch; q += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = part[(int64_t)(q + k) * stride];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  for (; q < nch; ++q) acc += part[(int64_t)q * stride];
  return acc;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Row partition (wgp_shard_range): every rank owns an equal, chunk-aligned slot of
// shard_chunks(n, world) chunks (the last ranks' rows stop at n), so a full buffer padded
// to padded_chunks(n, world) chunks is exchanged by ONE in-place all-gather of equal
// slices.  Full [rows][s] buffers and [chunk][...] partial arrays that are all-gathered
// are allocated with padded_chunks(...) chunks.
inline int64_t shard_chunks(int64_t n, int world) {
  const int64_t nch = (n + kChunkRows - 1) / kChunkRows;
  if (world < 1) world = 1;
  const int64_t c = (nch + world - 1) / world;
  return c > 0 ? c : 1;
}
inline int64_t padded_chunks(int64_t n, int world) {
  return shard_chunks(n, world) * (world < 1 ? 1 : world);
}
inline int64_t padded_rows(int64_t n, int world) { return padded_chunks(n, world) * kChunkRows; }

// ------------------------------------------------------------------ collectives (dist.cpp)
// All are no-ops (or local copies) when ctx.world == 1.
void dist_allgather_rows(const Ctx& ctx, void* full, int64_t n, int64_t row_elems, size_t esize,
                         cudaStream_t st);
// Start the all-gather of the row slots of `full` (this rank's slot final on `st`); work
// queued on `st` afterwards overlaps it.  Returns the event that completes the gather
// (world 1: nullptr, nothing to wait for; loopback: the exchange is done before returning
// and the event is already recorded).
cudaEvent_t dist_allgather_rows_begin(const Ctx& ctx, void* full, int64_t n, int64_t row_elems,
                                      size_t esize, cudaStream_t st);
void dist_allgather_chunks(const Ctx& ctx, double* part, int64_t n, int64_t per_chunk,
                           cudaStream_t st);
void dist_broadcast(const Ctx& ctx, void* buf, size_t bytes, int root, cudaStream_t st);
// In-place sum over ranks of `count` doubles (NCCL all-reduce; loopback: rank order).  Used
// where every entry has a single non-zero contributor, so the sum is exact and the result
// bitwise the one-GPU value.
void dist_allreduce_sum(const Ctx& ctx, double* buf, size_t count, cudaStream_t st);
void launch_sum_slots(const double* slots, int world, size_t count, double* out, cudaStream_t st);
void dist_allgather(const Ctx& ctx, const double* in, double* out, size_t count, cudaStream_t st);
int owner_rank(const Ctx& ctx, int64_t n, int64_t row);

// ------------------------------------------------------------------ launchers
// vecops.cu
void launch_colmajor_to_rows(const double* src, int64_t ld, int64_t n, int s, void* dst,
                             bool f64, cudaStream_t st);
void launch_rows_to_colmajor(const void* src, int64_t n, int s, double* dst, int64_t ld, bool f64,
                             cudaStream_t st);
template <typename T>
void launch_coldots(const T* A0, const T* B0, const T* A1, const T* B1, int64_t n, int s,
                    double* part, cudaStream_t st);  // part: [nchunks][nq][s]
void launch_chunk_sum(const double* part, int nch, int s, double* out, cudaStream_t st);
template <typename T>
void launch_axpy_cols(T* Y, const T* X, const double* alpha, int64_t n, int s, cudaStream_t st);
template <typename T>
void launch_xpby_cols(T* P, const T* Z, const double* beta, const int* active, int64_t n, int s,
                      cudaStream_t st);
template <typename T>
void launch_fill(T* p, T v, size_t count, cudaStream_t st);

// precond.cu
struct PrecondDev {
  int64_t n = 0, k = 0, kpad = 0;
  int64_t r0 = 0, n_local = 0;  // this rank's rows of L / M
  double shift = 1.0;
  DBuf<double> L;    // [n][kpad] row-major (pivoted Cholesky factor)
  DBuf<double> M64;  // [n][kpad]  M = L C^{-T}, C = chol(shift I + L^T L): M M^T = L cap^{-1} L^T
  // factorisation workspaces, kept (grown only) across builds: per-call cudaMalloc /
  // synchronous cudaFree of them showed as sporadic 0.1-0.25 s stalls of a C3 solve
  DBuf<double> w_d, w_pv, w_best2, w_all2, w_lpiv, w_part, w_G, w_W;
  DBuf<int> w_used, w_kcount;
  DBuf<int64_t> w_pi, w_dpiv;
};
void build_pivoted_cholesky(const Op& op, int64_t rank, PrecondDev& pd, cudaStream_t st);
void finish_preconditioner(const Op& op, double shift, int mode, PrecondDev& pd, cudaStream_t st);
template <typename T>
void precond_apply(const Op& op, const PrecondDev& pd, const T* R, T* Z, int s, double* work_t,
                   double* work_part, cudaStream_t st);


}  // namespace wgp
