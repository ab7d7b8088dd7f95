// capi.cpp -- extern "C" boundary of libwarmgp_b200.so (include/warmgp_capi.h).
//
// Every entry point converts C++ exceptions into a wgp_status plus a thread-local
// message; no exception crosses the ABI.  Host buffers use the reference's Eigen layout
// (column-major fp64); they are converted to the device layout on the GPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "rng.h"
#include "solvers.h"

namespace wgp {

static thread_local std::string g_last_error;

void set_last_error(const char* msg) { g_last_error = msg; }

void throw_error(wgp_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Error(code, buf);
}

void op_append_rows(Op& op, const double* host_rows, int64_t n_new, int64_t ld, int col_major);
bool exact_solve_dev(const Op& op, double* Y, int s, cudaStream_t st);
bool mll_dev(const Op& op, double l, double sf, double sn, const double* y, double* value,
             double* grad3, cudaStream_t st);
void launch_grad_posterior(const Op& op, const double* Om, const double* ph, const double* am,
                           int F, double coeff, const double* W, const double* Xs,
                           const int* sidx, int64_t m, double* G, cudaStream_t st);
void launch_ascend(const Op& op, const double* Om, const double* ph, const double* am, int F,
                   double coeff, const double* W, int S, const double* starts, int P, int steps,
                   double rate, double* best_val, double* best_x, cudaStream_t st);
void launch_rff_eval32(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st);
void launch_rff_eval64(const double* X, int ldx_row, int dim, int64_t m, const double* Om,
                       const double* ph, const double* amp, int F, int S, double coeff,
                       double* out, int64_t ldo, cudaStream_t st);
void dist_init(Ctx& ctx, const void* uid);
struct LoopGroup;
void dist_init_loopback(Ctx& ctx, LoopGroup* g);
void dist_destroy(Ctx& ctx);
int loop_group_world(const LoopGroup* g);

template <typename F>
static wgp_status guard(F&& f) {
  try {
    f();
    return WGP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return WGP_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return WGP_CUDA_ERROR;
  }
}

static void set_device(const Ctx& ctx) { WGP_CUDA(cudaSetDevice(ctx.device)); }

// Opt-in phase timing of a solve (WGP_PHASE_TIMING=1): synchronises the stream at each
// phase boundary and prints wall times to stderr.  Off by default (no extra syncs).
struct PhaseTimer {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(cudaStream_t s) : st(s) {
    const char* e = getenv("WGP_PHASE_TIMING");
    on = e && atoi(e) != 0;
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    WGP_CUDA(cudaStreamSynchronize(st));
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[wgp phase] %-14s %9.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

static void run_solve(Op& op, const wgp_solver_config& cfg, const double* B, int64_t ldb, int s,
                      const double* U1, int64_t ldu, int64_t n1, double* V, int64_t ldv,
                      SolveOutputs& out, bool derive_seeds, const PrecondDev* given = nullptr) {
  cudaStream_t st = op.ctx->stream;
  PhaseTimer pt(st);
  if (!op.solve_cache) op.solve_cache = std::make_shared<SolverWork<double>>();
  SolverWork<double>& w = *static_cast<SolverWork<double>*>(op.solve_cache.get());
  w.alloc(op, s);
  pt.mark("alloc");
  upload_problem<double>(op, w, B, ldb, U1, ldu, n1, st);
  pt.mark("upload");
  switch (cfg.method) {
    case WGP_CG: {
      if (given) {  // cg_solve_with (solvers.cpp:142): the caller's preconditioner, no rebuild
        cg_solve_batched<double>(op, cfg, *given, w, out, st);
        pt.mark("cg_loop");
        break;
      }
      if (!op.precond_cache) op.precond_cache = std::make_shared<PrecondDev>();
      PrecondDev& pd = *static_cast<PrecondDev*>(op.precond_cache.get());
      const int64_t rank = std::min<int64_t>(cfg.precond_rank, op.n);  // from_matrix :125-126
      if (rank > 0) {
        build_pivoted_cholesky(op, rank, pd, st);
        pt.mark("pivchol");
        finish_preconditioner(op, cfg.precond_shift, cfg.precond_shift_mode, pd, st);
        pt.mark("precond");
      } else {
        int64_t a, b;
        op.local_rows(&a, &b);
        pd.n = op.n;
        pd.r0 = a;
        pd.n_local = b - a;
        pd.k = 0;  // identity (the cached factors of an earlier solve are not used)
        pd.kpad = 0;
      }
      cg_solve_batched<double>(op, cfg, pd, w, out, st);
      pt.mark("cg_loop");
      break;
    }
    case WGP_SGD: {
      // solve_many derives one stream per RHS (solvers.cpp:343-345); sgd_solve uses cfg.seed
      std::vector<uint64_t> seeds(s);
      for (int c = 0; c < s; ++c) seeds[c] = derive_seeds ? derive_seed(cfg.seed, (uint64_t)c) : cfg.seed;
      WGP_REQUIRE(op.dim <= 32, "sgd_solve: dim > 32 not supported on the device path");
      sgd_solve_batched(op, cfg, seeds, w, out, st);
      break;
    }
    case WGP_AP:
      ap_solve_batched(op, cfg, w, out, st);
      break;
    default:
      throw_error(WGP_INVALID_ARGUMENT, "solve: unknown method");
  }
  download_solution<double>(w, V, ldv, st);
  pt.mark("download");
}

}  // namespace wgp

using namespace wgp;

struct wgp_ctx : Ctx {};
struct wgp_op : Op {};

extern "C" {

int wgp_abi_version(void) { return WGP_ABI_VERSION; }

void wgp_kernel_timer_enable(int enable) {
  wgp::KernelTimer& kt = wgp::kernel_timer();
  kt.clear();
  kt.on = enable != 0;
}

wgp_status wgp_kernel_timer_read_tag(const char* tag, double* total_ms, int64_t* launches) {
  return guard([&] {
    WGP_REQUIRE(tag && total_ms && launches, "wgp_kernel_timer_read: null argument");
    wgp::KernelTimer& kt = wgp::kernel_timer();
    double tot = 0.0;
    int64_t cnt = 0;
    for (auto& e : kt.ev) {
      if (std::strcmp(e.tag, tag) != 0) continue;
      WGP_CUDA(cudaEventSynchronize(e.b));
      float ms = 0.f;
      WGP_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
      tot += ms;
      ++cnt;
    }
    *total_ms = tot;
    *launches = cnt;
  });
}

wgp_status wgp_kernel_timer_read(double* total_ms, int64_t* launches) {
  return wgp_kernel_timer_read_tag("kmatvec_tc", total_ms, launches);
}

const char* wgp_last_error(void) { return g_last_error.c_str(); }

void wgp_solver_config_default(wgp_solver_config* c) {  // solvers.hpp:27-48
  c->method = WGP_CG;
  c->tolerance = 1e-2;
  c->max_iters = 1000;
  c->learning_rate = 0.3;
  c->momentum = 0.9;
  c->batch_size = 100;
  c->sgd_scaling = WGP_SGD_UNBIASED;
  c->block_size = 100;
  c->ap_ordering = WGP_AP_GREEDY;
  c->precond_rank = 100;
  c->precond_shift = 1e-6;
  c->precond_shift_mode = WGP_SHIFT_CALIBRATED;
  c->seed = 0;
}

void wgp_shard_range(int64_t n, int world, int rank, int64_t* row0, int64_t* row1) {
  // equal chunk-aligned slots of shard_chunks(n, world) chunks (common.cuh); the rows of
  // the last slot(s) stop at n
  if (world < 1) world = 1;
  const int64_t c = shard_chunks(n, world);
  int64_t a = (int64_t)rank * c * kChunkRows, b = (int64_t)(rank + 1) * c * kChunkRows;
  if (a > n) a = n;
  if (b > n) b = n;
  *row0 = a;
  *row1 = b;
}

int64_t wgp_shard_padded_rows(int64_t n, int world) { return padded_rows(n, world); }

wgp_status wgp_ctx_create(int device, wgp_ctx** out) {
  return guard([&] {
    WGP_REQUIRE(out, "wgp_ctx_create: null output");
    int count = 0;
    WGP_CUDA(cudaGetDeviceCount(&count));
    WGP_REQUIRE(device >= 0 && device < count, "wgp_ctx_create: device %d of %d", device, count);
    std::unique_ptr<wgp_ctx> c(new wgp_ctx());
    c->device = device;
    WGP_CUDA(cudaSetDevice(device));
    WGP_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    WGP_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (auto& e : c->part_ev) WGP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->col_ev) WGP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    WGP_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    for (auto& e : c->comm_ev) WGP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *out = c.release();
  });
}

wgp_status wgp_ctx_create_sharded(int device, int rank, int world, const void* uid,
                                  wgp_ctx** out) {
  return guard([&] {
    WGP_REQUIRE(world >= 1 && rank >= 0 && rank < world, "wgp_ctx_create_sharded: bad rank/world");
    wgp_ctx* c = nullptr;
    wgp_status stc = wgp_ctx_create(device, &c);
    if (stc != WGP_OK) throw Error(stc, g_last_error);
    c->rank = rank;
    c->world = world;
    try {
      if (world > 1) dist_init(*c, uid);
    } catch (...) {
      wgp_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

wgp_status wgp_ctx_create_loopback(int device, int rank, void* group, wgp_ctx** out) {
  return guard([&] {
    WGP_REQUIRE(group && out, "wgp_ctx_create_loopback: null argument");
    LoopGroup* g = static_cast<LoopGroup*>(group);
    const int world = loop_group_world(g);
    WGP_REQUIRE(rank >= 0 && rank < world, "wgp_ctx_create_loopback: bad rank");
    wgp_ctx* c = nullptr;
    wgp_status stc = wgp_ctx_create(device, &c);
    if (stc != WGP_OK) throw Error(stc, g_last_error);
    c->rank = rank;
    c->world = world;
    if (world > 1) dist_init_loopback(*c, g);
    *out = c;
  });
}

void wgp_ctx_destroy(wgp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->comm) dist_destroy(*c);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (auto& e : c->part_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->col_ev)
    if (e) cudaEventDestroy(e);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  for (auto& e : c->comm_ev)
    if (e) cudaEventDestroy(e);
  delete c;
}

void* wgp_ctx_stream(wgp_ctx* c) { return c ? (void*)c->stream : nullptr; }

wgp_status wgp_op_create(wgp_ctx* ctx, int kernel, double lengthscale, double signal_scale,
                         double noise_scale, int precision, int dim, wgp_op** out) {
  return guard([&] {
    WGP_REQUIRE(ctx && out, "wgp_op_create: null argument");
    // KernelHyperparams::validate (kernel.cpp:11-15)
    WGP_REQUIRE(lengthscale > 0.0 && signal_scale > 0.0 && noise_scale > 0.0,
                "kernel hyperparameters must be strictly positive");
    WGP_REQUIRE(kernel == WGP_MATERN32 || kernel == WGP_RBF, "unknown kernel %d", kernel);
    WGP_REQUIRE(precision >= WGP_F64 && precision <= WGP_F32_SIMT, "unknown precision %d",
                precision);
    WGP_REQUIRE(dim >= 1 && dim <= 256, "dim must be in [1, 256], got %d", dim);
    set_device(*ctx);
    std::unique_ptr<wgp_op> op(new wgp_op());
    op->ctx = ctx;
    op->kind = kernel;
    op->lengthscale = lengthscale;
    op->signal_scale = signal_scale;
    op->noise_scale = noise_scale;
    op->precision = precision;
    op->dim = dim;
    op->dpad = ((dim + 7) / 8) * 8;
    *out = op.release();
  });
}

void wgp_op_destroy(wgp_op* op) {
  if (!op) return;
  cudaSetDevice(op->ctx->device);
  delete op;
}

wgp_status wgp_op_append_rows(wgp_op* op, const double* X, int64_t n_new, int64_t ld,
                              int col_major) {
  return guard([&] {
    WGP_REQUIRE(op, "wgp_op_append_rows: null op");
    WGP_REQUIRE(n_new >= 0, "extend_system: negative row count");
    if (n_new == 0) return;
    WGP_REQUIRE(X, "wgp_op_append_rows: null rows");
    WGP_REQUIRE(col_major ? ld >= n_new : ld >= op->dim, "wgp_op_append_rows: bad leading dim");
    set_device(*op->ctx);
    op_append_rows(*op, X, n_new, ld, col_major);
  });
}

int64_t wgp_op_size(const wgp_op* op) { return op ? op->n : 0; }

wgp_status wgp_op_set_residual_mode(wgp_op* op, int mode) {
  return guard([&] {
    WGP_REQUIRE(op, "wgp_op_set_residual_mode: null op");
    WGP_REQUIRE(mode == WGP_RESIDUAL_DIRECT || mode == WGP_RESIDUAL_ANCHORED,
                "unknown residual mode %d", mode);
    op->resid_mode = mode;
  });
}

int wgp_op_residual_mode(const wgp_op* op) { return op ? op->resid_mode : -1; }
int wgp_op_last_anchor_count(const wgp_op* op) { return op ? op->last_anchors : 0; }
int wgp_op_dim(const wgp_op* op) { return op ? op->dim : 0; }
int wgp_op_precision(const wgp_op* op) { return op ? op->precision : -1; }

wgp_status wgp_kmatvec_dev(wgp_op* op, const void* dV, void* dY, int s, void* stream) {
  return guard([&] {
    WGP_REQUIRE(op && dV && dY && s >= 1, "wgp_kmatvec_dev: bad argument");
    WGP_REQUIRE(op->n >= 1, "wgp_kmatvec_dev: empty operator");
    cudaStream_t st = stream ? (cudaStream_t)stream : op->ctx->stream;
    launch_kmatvec_full(*op, (const double*)dV, (double*)dY, s, st);
  });
}

wgp_status wgp_kmatvec_sharded_dev(wgp_op* op, void* dV, void* dY, int s, void* stream) {
  return guard([&] {
    WGP_REQUIRE(op && dV && dY && s >= 1, "wgp_kmatvec_sharded_dev: bad argument");
    WGP_REQUIRE(op->n >= 1, "wgp_kmatvec_sharded_dev: empty operator");
    cudaStream_t st = stream ? (cudaStream_t)stream : op->ctx->stream;
    cudaEvent_t ev = dist_allgather_rows_begin(*op->ctx, dV, op->n, s, sizeof(double), st);
    launch_kmatvec_overlap(*op, nullptr, (const double*)dV, (double*)dY, s, ev, st);
  });
}

wgp_status wgp_residual_dev(wgp_op* op, const void* dB, const void* dV, void* dY, int s,
                            void* stream) {
  return guard([&] {
    WGP_REQUIRE(op && dB && dV && dY && s >= 1, "wgp_residual_dev: bad argument");
    WGP_REQUIRE(op->n >= 1, "wgp_residual_dev: empty operator");
    cudaStream_t st = stream ? (cudaStream_t)stream : op->ctx->stream;
    launch_residual(*op, (const double*)dB, (const double*)dV, (double*)dY, s, st);
  });
}

wgp_status wgp_axpy_cols_dev(wgp_ctx* ctx, void* dY, const void* dX, const void* dAlpha,
                             int64_t n, int s, void* stream) {
  return guard([&] {
    WGP_REQUIRE(ctx && dY && dX && dAlpha && n >= 0 && s >= 1, "wgp_axpy_cols_dev: bad argument");
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    launch_axpy_cols<double>((double*)dY, (const double*)dX, (const double*)dAlpha, n, s, st);
  });
}

wgp_status wgp_xpby_cols_dev(wgp_ctx* ctx, void* dP, const void* dZ, const void* dBeta,
                             const void* dActive, int64_t n, int s, void* stream) {
  return guard([&] {
    WGP_REQUIRE(ctx && dP && dZ && dBeta && dActive && n >= 0 && s >= 1,
                "wgp_xpby_cols_dev: bad argument");
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    launch_xpby_cols<double>((double*)dP, (const double*)dZ, (const double*)dBeta,
                             (const int*)dActive, n, s, st);
  });
}

wgp_status wgp_coldots_dev(wgp_ctx* ctx, const void* dA, const void* dB, int64_t n, int s,
                           void* dOut, void* dWork, void* stream) {
  return guard([&] {
    WGP_REQUIRE(ctx && dA && dB && dOut && dWork && n >= 1 && s >= 1,
                "wgp_coldots_dev: bad argument");
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    const int nch = (int)((n + kChunkRows - 1) / kChunkRows);
    launch_coldots<double>((const double*)dA, (const double*)dB, nullptr, nullptr, n, s,
                           (double*)dWork, st);
    launch_chunk_sum((const double*)dWork, nch, s, (double*)dOut, st);
  });
}

wgp_status wgp_kmatvec(wgp_op* op, const double* V, int64_t ldv, int s, double* Y, int64_t ldy) {
  return guard([&] {
    WGP_REQUIRE(op && V && Y && s >= 1, "wgp_kmatvec: bad argument");
    const int64_t n = op->n;
    WGP_REQUIRE(n >= 1, "wgp_kmatvec: empty operator");
    WGP_REQUIRE(ldv >= n && ldy >= n, "wgp_kmatvec: leading dimension < n");
    WGP_REQUIRE(op->ctx->world == 1, "wgp_kmatvec: host form needs an unsharded context");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    const size_t bytes = (size_t)n * s * sizeof(double);
    op->scratch[0].ensure(bytes);
    op->scratch[1].ensure(bytes);
    op->scratch[2].ensure(bytes);
    double* stage = (double*)op->scratch[0].p;
    double* dV = (double*)op->scratch[1].p;
    double* dY = (double*)op->scratch[2].p;
    Ctx& c = *op->ctx;
    // Tensor-core operators: V crosses in column parts (rows of V; host_col_parts: 1/8,
    // 3/8, 1/2) on the copy stream and the columns of each part are computed as soon as it
    // lands, so only the first part of the upload is exposed.  The rows of the result are
    // computed in Ctx::kHostParts parts (row_part_begin: 1/2, 1/4, 3/16, 1/16); each
    // finished part's rows are transposed and copied back on the copy stream while the next
    // parts compute, so only the last part's copy is exposed.
    int parts = 0;
    if (kmatvec_colphased_ok(*op, s, Ctx::kHostParts)) {
      int64_t cb[Ctx::kColParts + 1];
      const int ncp = host_col_parts(n, cb);
      WGP_CUDA(cudaEventRecord(c.col_ev[0], st));  // the stage / dV buffers are free
      WGP_CUDA(cudaStreamWaitEvent(c.copy_stream, c.col_ev[0], 0));
      for (int k = 0; k < ncp; ++k) {
        const int64_t a = cb[k], rows = cb[k + 1] - a;
        WGP_CUDA(cudaMemcpy2DAsync(stage + a, sizeof(double) * n, V + a, sizeof(double) * ldv,
                                   sizeof(double) * rows, s, cudaMemcpyHostToDevice, c.copy_stream));
        launch_colmajor_to_rows(stage + a, n, rows, s, dV + a * s, true, c.copy_stream);
        WGP_CUDA(cudaEventRecord(c.col_ev[k], c.copy_stream));
      }
      parts = launch_kmatvec_colphased(*op, dV, dY, s, st, cb, ncp, c.col_ev, Ctx::kHostParts,
                                       c.part_ev);
    } else {
      WGP_CUDA(cudaMemcpy2DAsync(stage, sizeof(double) * n, V, sizeof(double) * ldv,
                                 sizeof(double) * n, s, cudaMemcpyHostToDevice, st));
      launch_colmajor_to_rows(stage, n, n, s, dV, true, st);
      parts = launch_kmatvec_parts(*op, dV, dY, s, st, Ctx::kHostParts, c.part_ev);
    }
    if (parts == 1) {
      launch_rows_to_colmajor(dY, n, s, stage, n, true, st);
      WGP_CUDA(cudaMemcpy2DAsync(Y, sizeof(double) * ldy, stage, sizeof(double) * n,
                                 sizeof(double) * n, s, cudaMemcpyDeviceToHost, st));
      WGP_CUDA(cudaStreamSynchronize(st));
      return;
    }
    for (int part = 0; part < parts; ++part) {  // same split as launch_kmatvec_tc's row parts
      const int64_t a = row_part_begin(n, part, parts);
      const int64_t b = row_part_begin(n, part + 1, parts);
      WGP_CUDA(cudaStreamWaitEvent(c.copy_stream, c.part_ev[part], 0));
      if (b <= a) continue;
      launch_rows_to_colmajor(dY + a * s, b - a, s, stage + a, n, true, c.copy_stream);
      WGP_CUDA(cudaMemcpy2DAsync(Y + a, sizeof(double) * ldy, stage + a, sizeof(double) * n,
                                 sizeof(double) * (b - a), s, cudaMemcpyDeviceToHost, c.copy_stream));
    }
    WGP_CUDA(cudaStreamSynchronize(c.copy_stream));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}

wgp_status wgp_cross_matvec(wgp_op* op, const double* Xs, int64_t m, int64_t ldx, const double* W,
                            int64_t ldw, int s, double* Y, int64_t ldy) {
  return guard([&] {
    WGP_REQUIRE(op && Xs && W && Y && s >= 1 && m >= 0, "wgp_cross_matvec: bad argument");
    WGP_REQUIRE(ldx >= m && ldy >= m && ldw >= op->n, "wgp_cross_matvec: bad leading dimension");
    if (m == 0) return;
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    const int64_t n = op->n;
    // stage X* into a scratch operator sharing the hyperparameters (row-major, padded)
    Op tmp;
    tmp.ctx = op->ctx;
    tmp.kind = op->kind;
    tmp.lengthscale = op->lengthscale;
    tmp.signal_scale = op->signal_scale;
    tmp.noise_scale = op->noise_scale;
    tmp.precision = op->precision == WGP_F64 ? WGP_F64 : WGP_F32_SIMT;
    tmp.dim = op->dim;
    tmp.dpad = op->dpad;
    op_append_rows(tmp, Xs, m, ldx, 1);
    DBuf<double> stage((size_t)std::max(n, m) * s);
    DBuf<double> dW((size_t)n * s), dY((size_t)m * s);
    WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n, W, sizeof(double) * ldw,
                               sizeof(double) * n, s, cudaMemcpyHostToDevice, st));
    launch_colmajor_to_rows(stage.p, n, n, s, dW.p, true, st);
    if (op->f64()) {
      launch_kmatvec_simt<double>(*op, tmp.X64.p, m, 0, op->X64.p, n, dW.p, s, nullptr, dY.p,
                                  false, st);
    } else if (op->tensor()) {
      // tensor-core cross mode (no sigma^2 term); points outside the fp16 operand range of
      // this operator fall back to the fp64 CUDA-core kernel
      if (!op_cross_tc(*op, tmp.X64.p, m, tmp.dpad, dW.p, s, dY.p, st))
        launch_kmatvec_simt<double>(*op, tmp.X64.p, m, 0, op->X64.p, n, dW.p, s, nullptr, dY.p,
                                    false, st);
    } else {
      launch_kmatvec_simt<float>(*op, tmp.X32.p, m, 0, op->X32.p, n, dW.p, s, nullptr, dY.p,
                                 false, st);
    }
    launch_rows_to_colmajor(dY.p, m, s, stage.p, m, true, st);
    WGP_CUDA(cudaMemcpy2DAsync(Y, sizeof(double) * ldy, stage.p, sizeof(double) * m,
                               sizeof(double) * m, s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

static wgp_status solve_impl(wgp_op* op, const wgp_solver_config* cfg, const double* B, int64_t ldb,
                             int s, const double* U1, int64_t ldu, int64_t n1, double* V, int64_t ldv,
                             int32_t* iterations, double* history, int64_t hist_stride,
                             int32_t* history_len, int32_t* converged, int32_t* col_status,
                             int32_t* diverged_at, bool derive_seeds,
                             const PrecondDev* given = nullptr) {
  int fail_col = -1;
  int fail_iters = 0;
  wgp_status st = guard([&] {
    WGP_REQUIRE(op && cfg && B && V && iterations && history && history_len && converged,
                "wgp_solve_many: null argument");
    WGP_REQUIRE(s >= 0, "solve_many: negative RHS count");
    const int64_t n = op->n;
    WGP_REQUIRE(n >= 1, "solve_many: empty operator");
    WGP_REQUIRE(ldb >= n && ldv >= n, "solve_many: leading dimension < n");
    WGP_REQUIRE(cfg->max_iters >= 0, "solve_many: negative max_iters");
    WGP_REQUIRE(hist_stride >= (int64_t)cfg->max_iters + 1, "solve_many: history stride too small");
    if (U1) {
      WGP_REQUIRE(n1 <= n, "initialization longer than the system");  // solvers.cpp:46
      WGP_REQUIRE(n1 >= 0 && (n1 == 0 || ldu >= n1), "solve_many: bad warm-start shape");
    }
    if (s == 0) return;
    set_device(*op->ctx);
    SolveOutputs out(s);
    try {
      run_solve(*op, *cfg, B, ldb, s, U1, ldu, n1, V, ldv, out, derive_seeds, given);
    } catch (Error& e) {
      fail_col = e.col;
      fail_iters = e.iterations;
      throw;
    }
    for (int c = 0; c < s; ++c) {
      iterations[c] = out.iterations[c];
      converged[c] = out.converged[c];
      history_len[c] = (int32_t)out.history[c].size();
      std::memcpy(history + (int64_t)c * hist_stride, out.history[c].data(),
                  sizeof(double) * out.history[c].size());
      if (col_status) col_status[c] = out.status[c];
      if (diverged_at) diverged_at[c] = out.diverged_at[c];
      // zero right-hand side: v = 0 exactly (zero_rhs_result, solvers.cpp:51-58)
      bool zero = true;
      for (int64_t i = 0; i < n && zero; ++i) zero = B[(int64_t)c * ldb + i] == 0.0;
      if (zero)
        for (int64_t i = 0; i < n; ++i) V[(int64_t)c * ldv + i] = 0.0;
    }
    // the reference throws from the lowest failing column (DivergenceError, solvers.cpp:235)
    for (int c = 0; c < s; ++c)
      if (out.status[c] != WGP_OK) {
        fail_col = c;
        fail_iters = out.diverged_at[c];
        Error e((wgp_status)out.status[c], "sgd_solve: diverged (relative residual above 1e3)");
        e.col = c;
        e.iterations = out.diverged_at[c];
        throw e;
      }
  });
  if (st != WGP_OK && col_status && fail_col >= 0 && fail_col < s) col_status[fail_col] = st;
  if (st != WGP_OK && diverged_at && fail_col >= 0 && fail_col < s) diverged_at[fail_col] = fail_iters;
  return st;
}

extern "C" {

wgp_status wgp_solve_many(wgp_op* op, const wgp_solver_config* cfg, const double* B, int64_t ldb,
                          int s, const double* U1, int64_t ldu, int64_t n1, double* V, int64_t ldv,
                          int32_t* iterations, double* history, int64_t hist_stride,
                          int32_t* history_len, int32_t* converged, int32_t* col_status,
                          int32_t* diverged_at) {
  return solve_impl(op, cfg, B, ldb, s, U1, ldu, n1, V, ldv, iterations, history, hist_stride,
                    history_len, converged, col_status, diverged_at, true);
}

wgp_status wgp_solve(wgp_op* op, const wgp_solver_config* cfg, const double* b, const double* u1,
                     int64_t n1, double* v, int32_t* iterations, double* history,
                     int32_t* history_len, int32_t* converged, int32_t* diverged_at) {
  const int64_t n = op ? op->n : 0;
  return solve_impl(op, cfg, b, n, 1, u1, n1 > 0 ? n1 : 1, n1, v, n, iterations, history,
                    cfg ? (int64_t)cfg->max_iters + 1 : 1, history_len, converged, nullptr,
                    diverged_at, false);
}

wgp_status wgp_pivoted_cholesky(wgp_op* op, int64_t rank, double* L, int64_t ldl, int64_t* achieved) {
  return guard([&] {
    WGP_REQUIRE(op && achieved, "wgp_pivoted_cholesky: null argument");
    WGP_REQUIRE(rank >= 0 && rank <= op->n, "pivoted_cholesky: rank out of range");
    WGP_REQUIRE(!L || ldl >= op->n, "wgp_pivoted_cholesky: ldl < n");
    WGP_REQUIRE(!L || op->ctx->world == 1, "pivoted_cholesky: L download needs an unsharded context");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    PrecondDev pd;
    build_pivoted_cholesky(*op, rank, pd, st);
    *achieved = pd.k;
    if (L && pd.k > 0) {
      const int64_t n = op->n;
      std::vector<double> h((size_t)n * pd.kpad);
      WGP_CUDA(cudaMemcpyAsync(h.data(), pd.L.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
      WGP_CUDA(cudaStreamSynchronize(st));
      for (int64_t t = 0; t < pd.k; ++t)
        for (int64_t i = 0; i < n; ++i) L[t * ldl + i] = h[(size_t)i * pd.kpad + t];
    }
  });
}

wgp_status wgp_precond_info(wgp_op* op, int64_t rank, double shift, int mode, int64_t* achieved,
                            double* shift_out) {
  return guard([&] {
    WGP_REQUIRE(op && achieved && shift_out, "wgp_precond_info: null argument");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    PrecondDev pd;
    rank = std::min<int64_t>(rank, op->n);
    *achieved = 0;
    *shift_out = shift;
    if (rank <= 0) return;
    build_pivoted_cholesky(*op, rank, pd, st);
    finish_preconditioner(*op, shift, mode, pd, st);
    *achieved = pd.k;
    *shift_out = pd.shift;
  });
}

static wgp_status rff_eval_impl(wgp_op* op, const double* Omega, const double* phases,
                                const double* amps, int F, int S, double signal_scale,
                                const double* Xs, int64_t m, int64_t ldx, double* out, int64_t ldo,
                                bool fast) {
  return guard([&] {
    WGP_REQUIRE(op && Omega && phases && amps && out, "wgp_rff_eval: null argument");
    WGP_REQUIRE(F >= 1 && S >= 0, "sample_prior: dim and num_features must be positive");
    if (S == 0) return;
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    const int dim = op->dim;
    Op tmp;
    const double* Xd = op->X64.p;
    if (Xs) {  // evaluation points given on the host (candidates); else the operator's rows
      WGP_REQUIRE(m >= 0 && ldx >= m, "wgp_rff_eval: bad X* shape");
      tmp.ctx = op->ctx;
      tmp.precision = WGP_F64;
      tmp.dim = dim;
      tmp.dpad = op->dpad;
      op_append_rows(tmp, Xs, m, ldx, 1);
      Xd = tmp.X64.p;
    } else {
      m = op->n;
    }
    WGP_REQUIRE(ldo >= m, "wgp_rff_eval: ldo < m");
    if (m == 0) return;
    const size_t nom = (size_t)S * F * dim, nf = (size_t)S * F;
    DBuf<double> dOm(nom), dPh(nf), dAm(nf), dOut((size_t)m * S);
    WGP_CUDA(cudaMemcpyAsync(dOm.p, Omega, sizeof(double) * nom, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(dPh.p, phases, sizeof(double) * nf, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(dAm.p, amps, sizeof(double) * nf, cudaMemcpyHostToDevice, st));
    const double coeff = signal_scale * std::sqrt(2.0 / (double)F);  // sampling.cpp:40-41
    if (fast)
      launch_rff_eval32(Xd, op->dpad, dim, m, dOm.p, dPh.p, dAm.p, F, S, coeff, dOut.p, m, st);
    else
      launch_rff_eval64(Xd, op->dpad, dim, m, dOm.p, dPh.p, dAm.p, F, S, coeff, dOut.p, m, st);
    WGP_CUDA(cudaMemcpy2DAsync(out, sizeof(double) * ldo, dOut.p, sizeof(double) * m,
                               sizeof(double) * m, S, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}

wgp_status wgp_rff_eval(wgp_op* op, const double* Omega, const double* phases, const double* amps,
                        int F, int S, double signal_scale, const double* Xs, int64_t m, int64_t ldx,
                        double* out, int64_t ldo) {
  return rff_eval_impl(op, Omega, phases, amps, F, S, signal_scale, Xs, m, ldx, out, ldo, false);
}

wgp_status wgp_rff_eval_fast(wgp_op* op, const double* Omega, const double* phases,
                             const double* amps, int F, int S, double signal_scale, const double* Xs,
                             int64_t m, int64_t ldx, double* out, int64_t ldo) {
  return rff_eval_impl(op, Omega, phases, amps, F, S, signal_scale, Xs, m, ldx, out, ldo, true);
}

wgp_status wgp_exact_solve(wgp_op* op, const double* B, int64_t ldb, int s, double* X, int64_t ldx) {
  return guard([&] {
    WGP_REQUIRE(op && B && X && s >= 1, "wgp_exact_solve: bad argument");
    WGP_REQUIRE(op->ctx->world == 1, "exact_solve: unsharded operators only");
    const int64_t n = op->n;
    WGP_REQUIRE(n >= 1 && ldb >= n && ldx >= n, "exact_solve: bad shape");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    DBuf<double> stage((size_t)n * s), Y((size_t)n * s);
    WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n, B, sizeof(double) * ldb, sizeof(double) * n,
                               s, cudaMemcpyHostToDevice, st));
    launch_colmajor_to_rows(stage.p, n, n, s, Y.p, true, st);
    if (!exact_solve_dev(*op, Y.p, s, st)) throw_error(WGP_NOT_SPD, "exact_solve: Cholesky failed");
    launch_rows_to_colmajor(Y.p, n, s, stage.p, n, true, st);
    WGP_CUDA(cudaMemcpy2DAsync(X, sizeof(double) * ldx, stage.p, sizeof(double) * n, sizeof(double) * n,
                               s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}

wgp_status wgp_mll(wgp_op* op, const double* y, const double* hyp3, double* value, double* grad3) {
  return guard([&] {
    WGP_REQUIRE(op && y && value && grad3, "wgp_mll: null argument");
    WGP_REQUIRE(op->ctx->world == 1, "mll: unsharded operators only");
    WGP_REQUIRE(op->n >= 1, "mll: X rows != y length");
    set_device(*op->ctx);
    const double l = hyp3 ? hyp3[0] : op->lengthscale, sf = hyp3 ? hyp3[1] : op->signal_scale,
                 sn = hyp3 ? hyp3[2] : op->noise_scale;
    if (!mll_dev(*op, l, sf, sn, y, value, grad3, op->ctx->stream))
      throw_error(WGP_NOT_SPD, "mll: covariance not SPD at these hyperparameters");
  });
}

wgp_status wgp_optimize_mll(wgp_op* op, const double* y, const double* init3, int steps,
                            double step_size, double* out3) {
  return guard([&] {
    WGP_REQUIRE(op && y && out3, "wgp_optimize_mll: null argument");
    WGP_REQUIRE(op->ctx->world == 1, "optimize_mll: unsharded operators only");
    WGP_REQUIRE(steps >= 0, "optimize_mll: negative step count");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    const double h0[3] = {init3 ? init3[0] : op->lengthscale, init3 ? init3[1] : op->signal_scale,
                          init3 ? init3[2] : op->noise_scale};
    WGP_REQUIRE(h0[0] > 0.0 && h0[1] > 0.0 && h0[2] > 0.0,
                "KernelHyperparams: all scales must be positive");
    // analysis.cpp:141-182: Adam on theta = log(l, s_f, sigma_n) inside the soft box
    double th[3] = {std::log(h0[0]), std::log(h0[1]), std::log(h0[2])};
    const double lo[3] = {std::log(1e-3), std::log(1e-3), std::log(1e-4)};
    const double hi[3] = {std::log(1e3), std::log(1e3), std::log(1e2)};
    double val = 0.0, g[3];
    auto eval = [&](const double* t) {
      if (!mll_dev(*op, std::exp(t[0]), std::exp(t[1]), std::exp(t[2]), y, &val, g, st))
        throw_error(WGP_NOT_SPD, "mll: covariance not SPD at these hyperparameters");
    };
    eval(th);
    if (!std::isfinite(val))
      throw_error(WGP_RUNTIME_ERROR, "optimize_mll: non-finite MLL at the initial hyperparameters");
    double best[3] = {th[0], th[1], th[2]}, best_val = val;
    double m[3] = {0.0, 0.0, 0.0}, v[3] = {0.0, 0.0, 0.0};
    for (int t = 1; t <= steps; ++t) {
      const double bc1 = 1.0 - std::pow(0.9, t), bc2 = 1.0 - std::pow(0.999, t);
      for (int k = 0; k < 3; ++k) {
        m[k] = 0.9 * m[k] + (1.0 - 0.9) * g[k];
        v[k] = 0.999 * v[k] + (1.0 - 0.999) * (g[k] * g[k]);
        const double step = (m[k] / bc1) / (std::sqrt(v[k] / bc2) + 1e-8);
        th[k] = std::min(std::max(th[k] + step_size * step, lo[k]), hi[k]);
      }
      eval(th);
      if (!std::isfinite(val))
        throw_error(WGP_RUNTIME_ERROR, "optimize_mll: non-finite MLL at step %d (lengthscale %g)", t,
                    std::exp(th[0]));
      if (val > best_val) {
        best_val = val;
        for (int k = 0; k < 3; ++k) best[k] = th[k];
      }
    }
    for (int k = 0; k < 3; ++k) out3[k] = std::exp(best[k]);
  });
}

double wgp_median_heuristic_lengthscale(const double* X, int64_t n, int64_t ldx, int dim,
                                        uint64_t seed) {
  if (!X || n < 1 || dim < 1 || ldx < n) return 1.0;
  const int64_t cap = std::min<int64_t>(n, 256);  // analysis.cpp:184-203
  std::vector<double> sub((size_t)(cap * dim));
  Rng rng{derive_seed(seed, 0x6d656469ULL)};
  for (int64_t i = 0; i < cap; ++i) {
    const int64_t r = (int64_t)rng.uniform_index((uint64_t)n);
    for (int k = 0; k < dim; ++k) sub[(size_t)(k * cap + i)] = X[k * ldx + r];
  }
  // pairwise_distances (kernel.cpp:39-46): sqrt(max(|a|^2 + |b|^2 - 2 a.b, 0))
  std::vector<double> sq((size_t)cap, 0.0);
  for (int k = 0; k < dim; ++k)
    for (int64_t i = 0; i < cap; ++i) sq[(size_t)i] += sub[(size_t)(k * cap + i)] * sub[(size_t)(k * cap + i)];
  std::vector<double> vals;
  vals.reserve((size_t)(cap * (cap - 1) / 2));
  for (int64_t j = 0; j < cap; ++j)
    for (int64_t i = j + 1; i < cap; ++i) {
      double gsum = 0.0;
      for (int k = 0; k < dim; ++k) gsum += sub[(size_t)(k * cap + i)] * sub[(size_t)(k * cap + j)];
      double d2 = -2.0 * gsum;
      d2 += sq[(size_t)i];
      d2 += sq[(size_t)j];
      vals.push_back(std::sqrt(d2 > 0.0 ? d2 : 0.0));
    }
  if (vals.empty()) return 1.0;
  std::nth_element(vals.begin(), vals.begin() + vals.size() / 2, vals.end());
  const double med = vals[vals.size() / 2];
  return med > 0.0 ? med : 1.0;
}

// upload S priors (prior-major, each F x dim column-major) and W (n x S column-major)
static void upload_posterior(const Op& op, const double* Omega, const double* phases,
                             const double* amps, int F, int S, const double* W, int64_t ldw,
                             DBuf<double>& dOm, DBuf<double>& dPh, DBuf<double>& dAm,
                             DBuf<double>& dW, cudaStream_t st) {
  const size_t nom = (size_t)S * F * op.dim, nf = (size_t)S * F;
  dOm.alloc(nom);
  dPh.alloc(nf);
  dAm.alloc(nf);
  dW.alloc((size_t)std::max<int64_t>(op.n, 1) * S);
  WGP_CUDA(cudaMemcpyAsync(dOm.p, Omega, sizeof(double) * nom, cudaMemcpyHostToDevice, st));
  WGP_CUDA(cudaMemcpyAsync(dPh.p, phases, sizeof(double) * nf, cudaMemcpyHostToDevice, st));
  WGP_CUDA(cudaMemcpyAsync(dAm.p, amps, sizeof(double) * nf, cudaMemcpyHostToDevice, st));
  if (op.n > 0)
    WGP_CUDA(cudaMemcpy2DAsync(dW.p, sizeof(double) * op.n, W, sizeof(double) * ldw,
                               sizeof(double) * op.n, S, cudaMemcpyHostToDevice, st));
}

wgp_status wgp_grad_posterior(wgp_op* op, const double* Omega, const double* phases,
                              const double* amps, int F, int S, double signal_scale,
                              const double* W, int64_t ldw, const double* Xs, int64_t ldx,
                              const int32_t* sidx, int64_t m, double* G, int64_t ldg) {
  return guard([&] {
    WGP_REQUIRE(op && Omega && phases && amps && W && Xs && sidx && G, "wgp_grad_posterior: null argument");
    WGP_REQUIRE(F >= 1 && S >= 1 && m >= 0 && ldw >= op->n && ldx >= m && ldg >= m,
                "grad_posterior: bad shape");
    WGP_REQUIRE(op->ctx->world == 1, "grad_posterior: unsharded operators only");
    for (int64_t i = 0; i < m; ++i)
      WGP_REQUIRE(sidx[i] >= 0 && sidx[i] < S, "grad_posterior: sample index out of range");
    if (m == 0) return;
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    const int dim = op->dim;
    DBuf<double> dOm, dPh, dAm, dW, dX((size_t)m * dim), dG((size_t)m * dim);
    DBuf<int> dS((size_t)m);
    upload_posterior(*op, Omega, phases, amps, F, S, W, ldw, dOm, dPh, dAm, dW, st);
    std::vector<double> hx((size_t)m * dim);
    for (int64_t i = 0; i < m; ++i)
      for (int k = 0; k < dim; ++k) hx[(size_t)i * dim + k] = Xs[(int64_t)k * ldx + i];
    WGP_CUDA(cudaMemcpyAsync(dX.p, hx.data(), sizeof(double) * hx.size(), cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(dS.p, sidx, sizeof(int) * m, cudaMemcpyHostToDevice, st));
    const double coeff = signal_scale * std::sqrt(2.0 / (double)F);
    launch_grad_posterior(*op, dOm.p, dPh.p, dAm.p, F, coeff, dW.p, dX.p, dS.p, m, dG.p, st);
    WGP_CUDA(cudaMemcpyAsync(hx.data(), dG.p, sizeof(double) * hx.size(), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < m; ++i)
      for (int k = 0; k < dim; ++k) G[(int64_t)k * ldg + i] = hx[(size_t)i * dim + k];
  });
}

wgp_status wgp_ascend_peaks(wgp_op* op, const double* Omega, const double* phases,
                            const double* amps, int F, int S, double signal_scale, const double* W,
                            int64_t ldw, const double* starts, int P, int steps, double rate,
                            double* best_x, double* best_val) {
  return guard([&] {
    WGP_REQUIRE(op && Omega && phases && amps && W && starts && best_x && best_val,
                "wgp_ascend_peaks: null argument");
    WGP_REQUIRE(F >= 1 && S >= 1 && P >= 1 && steps >= 0 && ldw >= op->n, "ascend_peaks: bad shape");
    WGP_REQUIRE(op->ctx->world == 1, "ascend_peaks: unsharded operators only");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    const int dim = op->dim;
    const int64_t m = (int64_t)S * P;
    DBuf<double> dOm, dPh, dAm, dW, dX((size_t)m * dim), dBX((size_t)m * dim), dBV((size_t)m);
    upload_posterior(*op, Omega, phases, amps, F, S, W, ldw, dOm, dPh, dAm, dW, st);
    std::vector<double> hx((size_t)m * dim), hv((size_t)m);
    for (int64_t i = 0; i < m; ++i)
      for (int k = 0; k < dim; ++k) hx[(size_t)i * dim + k] = starts[(int64_t)k * m + i];
    WGP_CUDA(cudaMemcpyAsync(dX.p, hx.data(), sizeof(double) * hx.size(), cudaMemcpyHostToDevice, st));
    const double coeff = signal_scale * std::sqrt(2.0 / (double)F);
    launch_ascend(*op, dOm.p, dPh.p, dAm.p, F, coeff, dW.p, S, dX.p, P, steps, rate, dBV.p, dBX.p, st);
    WGP_CUDA(cudaMemcpyAsync(hx.data(), dBX.p, sizeof(double) * hx.size(), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaMemcpyAsync(hv.data(), dBV.p, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    for (int s = 0; s < S; ++s) {  // start order, strict > (thompson.cpp:227-252)
      int64_t best = (int64_t)s * P;
      for (int t = 1; t < P; ++t)
        if (hv[(size_t)s * P + t] > hv[(size_t)best]) best = (int64_t)s * P + t;
      best_val[s] = hv[(size_t)best];
      for (int k = 0; k < dim; ++k) best_x[(int64_t)k * S + s] = hx[(size_t)best * dim + k];
    }
  });
}

}  // extern "C"

// ------------------------------------------------------------------------------------------
// Reusable preconditioner (CgPreconditioner, solvers.hpp:82-100) and cg_solve_with
// (solvers.hpp:118-119): bo_round builds ONE preconditioner per round and reuses it for every
// per-column solve (thompson.cpp:359-384).
struct wgp_precond {
  wgp_op* op = nullptr;
  int64_t n_at_build = 0;
  PrecondDev pd;
};

static void check_precond(const wgp_precond* pc, const wgp_op* op) {
  WGP_REQUIRE(pc, "null preconditioner");
  WGP_REQUIRE(!op || pc->op == op, "preconditioner built for another operator");
  WGP_REQUIRE(pc->op->n == pc->n_at_build,
              "preconditioner built for %lld rows, operator now has %lld (rows appended)",
              (long long)pc->n_at_build, (long long)pc->op->n);
}

extern "C" {

wgp_status wgp_precond_create(wgp_op* op, int64_t rank, double shift, int mode, wgp_precond** out) {
  return guard([&] {
    WGP_REQUIRE(op && out, "wgp_precond_create: null argument");
    WGP_REQUIRE(rank >= 0, "CgPreconditioner: negative rank");
    WGP_REQUIRE(mode == WGP_SHIFT_CALIBRATED || mode == WGP_SHIFT_NOISE_ONLY, "unknown shift mode");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    std::unique_ptr<wgp_precond> pc(new wgp_precond());
    pc->op = op;
    pc->n_at_build = op->n;
    rank = std::min<int64_t>(rank, op->n);  // from_matrix (solvers.cpp:123-133)
    if (rank > 0) {
      build_pivoted_cholesky(*op, rank, pc->pd, st);
      finish_preconditioner(*op, shift, mode, pc->pd, st);
    } else {
      int64_t a, b;
      op->local_rows(&a, &b);
      pc->pd.n = op->n;
      pc->pd.r0 = a;
      pc->pd.n_local = b - a;
      pc->pd.shift = shift;
    }
    *out = pc.release();
  });
}

wgp_status wgp_precond_create_from_factor(wgp_op* op, const double* L, int64_t ldl, int64_t k,
                                          double shift, wgp_precond** out) {
  return guard([&] {
    WGP_REQUIRE(op && out && (k == 0 || L), "wgp_precond_create_from_factor: null argument");
    WGP_REQUIRE(k >= 0 && (k == 0 || ldl >= op->n), "CgPreconditioner: bad factor shape");
    set_device(*op->ctx);
    cudaStream_t st = op->ctx->stream;
    std::unique_ptr<wgp_precond> pc(new wgp_precond());
    pc->op = op;
    pc->n_at_build = op->n;
    int64_t a, b;
    op->local_rows(&a, &b);
    PrecondDev& pd = pc->pd;
    pd.n = op->n;
    pd.r0 = a;
    pd.n_local = b - a;
    pd.k = k;
    pd.shift = shift;
    pd.kpad = k > 0 ? ((k + 3) / 4) * 4 : 0;
    if (k > 0) {
      // CgPreconditioner(L, shift) (solvers.cpp:109-121): this rank's rows of L, row-major
      const int64_t nl = std::max<int64_t>(pd.n_local, 1);
      std::vector<double> h((size_t)nl * pd.kpad, 0.0);
      for (int64_t i = 0; i < pd.n_local; ++i)
        for (int64_t t = 0; t < k; ++t) h[(size_t)i * pd.kpad + t] = L[t * ldl + a + i];
      pd.L.ensure(h.size());
      WGP_CUDA(cudaMemcpyAsync(pd.L.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st));
      finish_preconditioner(*op, shift, WGP_SHIFT_NOISE_ONLY, pd, st);  // shift used as given
    }
    *out = pc.release();
  });
}

void wgp_precond_destroy(wgp_precond* pc) {
  if (!pc) return;
  cudaSetDevice(pc->op->ctx->device);
  delete pc;
}

wgp_status wgp_precond_get(const wgp_precond* pc, int64_t* rank, double* shift) {
  return guard([&] {
    WGP_REQUIRE(pc && rank && shift, "wgp_precond_get: null argument");
    *rank = pc->pd.k;
    *shift = pc->pd.shift;
  });
}

wgp_status wgp_precond_apply(wgp_precond* pc, const double* R, int64_t ldr, int s, double* Z,
                             int64_t ldz) {
  return guard([&] {
    check_precond(pc, nullptr);
    Op& op = *pc->op;
    WGP_REQUIRE(R && Z && s >= 1, "wgp_precond_apply: bad argument");
    WGP_REQUIRE(op.ctx->world == 1, "wgp_precond_apply: host form needs an unsharded context");
    const int64_t n = op.n;
    WGP_REQUIRE(ldr >= n && ldz >= n, "CgPreconditioner::apply: length mismatch");
    set_device(*op.ctx);
    cudaStream_t st = op.ctx->stream;
    DBuf<double> stage((size_t)n * s), dR((size_t)n * s), dZ((size_t)n * s);
    const int64_t k = pc->pd.k;
    DBuf<double> wt((size_t)(k + 1) * s), wp((size_t)padded_chunks(n, 1) * (k + 1) * s);
    WGP_CUDA(cudaMemcpy2DAsync(stage.p, sizeof(double) * n, R, sizeof(double) * ldr,
                               sizeof(double) * n, s, cudaMemcpyHostToDevice, st));
    launch_colmajor_to_rows(stage.p, n, n, s, dR.p, true, st);
    precond_apply<double>(op, pc->pd, dR.p, dZ.p, s, wt.p, wp.p, st);
    launch_rows_to_colmajor(dZ.p, n, s, stage.p, n, true, st);
    WGP_CUDA(cudaMemcpy2DAsync(Z, sizeof(double) * ldz, stage.p, sizeof(double) * n,
                               sizeof(double) * n, s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  });
}

wgp_status wgp_cg_solve_with(wgp_op* op, const wgp_precond* pc, const wgp_solver_config* cfg,
                             const double* B, int64_t ldb, int s, const double* U1, int64_t ldu,
                             int64_t n1, double* V, int64_t ldv, int32_t* iterations,
                             double* history, int64_t hist_stride, int32_t* history_len,
                             int32_t* converged) {
  try {
    check_precond(pc, op);
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  }
  if (!cfg) return WGP_INVALID_ARGUMENT;
  wgp_solver_config c = *cfg;
  c.method = WGP_CG;
  return solve_impl(op, &c, B, ldb, s, U1, ldu, n1, V, ldv, iterations, history, hist_stride,
                    history_len, converged, nullptr, nullptr, true, &pc->pd);
}

}  // extern "C"
