// solvers.h -- internal solver interfaces (device work buffers, operator applications).
#pragma once

#include "common.cuh"

namespace wgp {

// Per-solve device buffers, row-major [rows][s] fp64.  Sharded (world > 1): this rank owns
// rows [r0, r0 + n) of N; V and P are full N-row buffers (the matvec reads every row,
// all-gathered after each update), R, Z, HP, B hold the local rows only.  Chunk partials
// `part` are indexed by global chunk (c0 = r0 / kChunkRows).
template <typename T>
struct SolverWork {
  int64_t n = 0;        // local rows
  int64_t N = 0, r0 = 0;
  int s = 0;
  int nch = 0;          // global chunk count
  int c0 = 0;
  DBuf<T> V, R, Z, P, HP, B;
  // anchored true residual (Op::resid_mode): V then holds d = v - v_a, VA the anchor v_a
  // (full rows), RA = b - H v_a (local rows, fp64 kernel); warm = nonzero initial v
  DBuf<T> VA, RA;
  DBuf<double> anc;  // [4][s]: ones, minus ones, |d| per column, spare
  bool warm = false;
  // per-iteration records of a CG block between host synchronisations (solvers.cu)
  DBuf<double> blk_rel;
  DBuf<int> blk_act;
  PinnedBuf h_blk;
  T* Vl() const { return V.p + r0 * s; }
  T* Pl() const { return P.p + r0 * s; }
  DBuf<double> part;   // [nch][2][s] chunk partials
  DBuf<double> scal;   // rz, alpha, beta, bnorm, rel, spare (6 x s)
  DBuf<int> act;       // active[s] + failure column
  DBuf<double> pwork;  // preconditioner chunk partials
  DBuf<double> tvec;   // M^T r  (k x s)
  DBuf<double> stage;  // host-boundary staging (column-major) for upload / download
  PinnedBuf h_stage;   // pinned host staging of large uploads / downloads (upload_problem)
  // SGD / AP workspaces (grown only: no per-solve cudaMalloc / synchronous cudaFree)
  DBuf<int> sgd_rows, ap_fail, ap_seg_block, ap_blk, ap_conf;
  DBuf<double> sgd_g, sgd_vel, ap_fac, ap_inv, ap_segn, ap_rblk, ap_delta, ap_y;
  DBuf<int64_t> ap_seg_start;
  void alloc(const Op& op, int s);
};

struct SolveOutputs {
  std::vector<std::vector<double>> history;
  std::vector<int> iterations, converged, status, diverged_at;
  explicit SolveOutputs(int s) : history(s), iterations(s, 0), converged(s, 0), status(s, 0),
                                 diverged_at(s, 0) {}
};

// Operator applications on this rank's rows (all rows when world = 1).  Solver vectors are
// fp64 for every precision; the precision selects the kernel (SIMT fp64 / SIMT fp32 /
// tcgen05 3xTF32), which converts on the fly.
void launch_kmatvec_full(Op& op, const double* V, double* Y, int s, cudaStream_t st);
void launch_residual(Op& op, const double* B, const double* V, double* Y, int s, cudaStream_t st);
// Y = B - H V on this rank's rows with the fp64 kernel whatever the operator's precision
// (the anchor residuals of WGP_RESIDUAL_ANCHORED)
void launch_residual_f64(Op& op, const double* B, const double* V, double* Y, int s,
                         cudaStream_t st);
// Sharded matvec overlapped with the row all-gather of V: columns [c0, c1) (this rank's
// slot) are valid on the stream at launch, the others only once `ready` has fired.
struct ColPhase {
  int64_t c0 = 0, c1 = 0;
  cudaEvent_t ready = nullptr;
};
// Y (this rank's rows) = H V, or B - H V, with V's rows outside this rank's slot arriving
// through `gathered` (dist_allgather_rows_begin; nullptr = V already complete): the local
// diagonal block runs first, the rest after the event.
void launch_kmatvec_overlap(Op& op, const double* B, const double* V, double* Y, int s,
                            cudaEvent_t gathered, cudaStream_t st);
template <typename T>
void launch_kmatvec_simt(const Op& op, const T* Xr, int64_t nrows, int64_t row0, const T* Xc,
                         int64_t ncols, const double* V, int s, const double* B, double* Y,
                         bool gram, cudaStream_t st, const ColPhase* ph = nullptr);
// C: Y = C + sgn (K V [+ sigma^2 V_i when gram]) on rows [row0, row0 + nrows) and columns
// [col0, col0 + ncols) (XB, V64 already offset to col0); B64 given: C = B64, sgn = -1.
// gram: the exact diagonal k(x, x) where global row == global column, and the noise term,
// taken from V64's row i - col0 (noise_mode -1), from noiseV's row i (1: the full V, for a
// column-range launch), or left out (0: another launch of the same product adds it).
void launch_kmatvec_tc(const Op& op, const float* XA_all, const float* XB, int64_t nrows,
                       int64_t row0, int64_t ncols, const double* V64, int s, const double* B64,
                       double* Y64, bool gram, DBuf<float>& vt_scratch, DBuf<double>& vchunk,
                       DBuf<double>& ychunk, DBuf<double>& ysplit, cudaStream_t st,
                       int row_parts = 1, cudaEvent_t* part_done = nullptr, int64_t col0 = 0,
                       const double* C64 = nullptr, double sgn = 1.0, int noise_mode = -1,
                       const double* noiseV = nullptr);
// Host-API form of the gram matvec: on tensor-core operators the rows are computed in
// `parts` parts, part_done[p] recorded as each part's rows are final (else one part).
// Returns the number of parts used.
int launch_kmatvec_parts(Op& op, const double* V, double* Y, int s, cudaStream_t st, int parts,
                         cudaEvent_t* part_done);
// First row of row part `part` of `parts` (CTA-tile aligned; part == parts gives nrows).
// Equal parts, except the host API's four: 1/2, 1/4, 3/16, 1/16 of the rows, so each part's
// copy-back hides under the next part's compute and the exposed last one is small
// (WGP_HOST_ROWCUTS="a,b,c" overrides the cumulative sixteenths 8,12,15 -- probes).
int64_t row_part_begin(int64_t nrows, int part, int parts);
// Column parts of the host API's upload: boundaries cb[0..ncp] (multiples of 128) of the
// cumulative shares 1/8, 1/2 (WGP_HOST_COLCUTS="a,b,..." overrides the sixteenths 2,8);
// returns ncp (<= Ctx::kColParts).
int host_col_parts(int64_t n, int64_t* cb);
// The same with V arriving in column parts (host API: the host-to-device copy of part p + 1
// overlaps the columns of part p): V rows [cb[k], cb[k + 1]) are valid after vready[k]
// (ncp parts).  Column part k < ncp - 1 is one launch accumulating into Y; the last runs in
// `parts` row parts recorded on part_done.  Returns the number of row parts, or 0 when the
// operator does not take this form (then nothing is launched).
int launch_kmatvec_colphased(Op& op, const double* V, double* Y, int s, cudaStream_t st,
                             const int64_t* cb, int ncp, const cudaEvent_t* vready, int parts,
                             cudaEvent_t* part_done);
// Whether launch_kmatvec_colphased applies (world 1, tensor-core operator, s <= 64, n large)
bool kmatvec_colphased_ok(const Op& op, int s, int parts);
void tc_build_operands(Op& op, DBuf<float>& XA, DBuf<float>& XB, const double* center,
                       cudaStream_t st);
int tc_k1(int dim, int precision, bool f16);
bool op_cross_tc(Op& op, const double* Xs, int64_t m, int dpad, const double* W, int s, double* Y,
                 cudaStream_t st);
bool tc_build_cross_rows(const Op& op, const double* Xs, int64_t m, int dpad, DBuf<float>& XAc,
                         cudaStream_t st);
// launch timing of the hot kernels (wgp_kernel_timer_*): event pairs on the launch stream,
// tagged by kernel ("kmatvec_tc", "kmatvec_f64", "krows", "kcols", "rff_eval", "rff_eval32")
struct KernelTimer {
  bool on = false;
  struct Entry {
    const char* tag;
    cudaEvent_t a, b;
  };
  std::vector<Entry> ev;
  void clear() {
    for (auto& e : ev) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    ev.clear();
  }
};
KernelTimer& kernel_timer();
// RAII: CUDA events around the launches in its scope when the timer is on
struct TimedScope {
  cudaEvent_t a = nullptr;
  cudaStream_t st;
  const char* tag;
  TimedScope(const char* t, cudaStream_t s) : st(s), tag(t) {
    if (kernel_timer().on) {
      cudaEventCreate(&a);
      cudaEventRecord(a, st);
    }
  }
  ~TimedScope() {
    if (!a) return;
    cudaEvent_t b = nullptr;
    cudaEventCreate(&b);
    cudaEventRecord(b, st);
    kernel_timer().ev.push_back({tag, a, b});
  }
};
bool tc_supported(int dim, int precision);  // false -> the fp32 CUDA-core kernel serves this dim

template <typename T>
void upload_problem(const Op& op, SolverWork<T>& w, const double* B, int64_t ldb, const double* U1,
                    int64_t ldu, int64_t n1, cudaStream_t st);
template <typename T>
void download_solution(SolverWork<T>& w, double* V, int64_t ldv, cudaStream_t st);
template <typename T>
void cg_solve_batched(Op& op, const wgp_solver_config& cfg, const PrecondDev& pd,
                      SolverWork<T>& w, SolveOutputs& out, cudaStream_t st);

void sgd_solve_batched(Op& op, const wgp_solver_config& cfg, const std::vector<uint64_t>& seeds,
                       SolverWork<double>& w, SolveOutputs& out, cudaStream_t st);
void ap_solve_batched(Op& op, const wgp_solver_config& cfg, SolverWork<double>& w,
                      SolveOutputs& out, cudaStream_t st);

// sgd_ap.cu
// g[c][i] = H[row_i] v_c - b[row_i] for batch rows this rank owns ([r0, r1); B holds those
// rows), 0 for the others
void launch_krows(const Op& op, const int* rows, int nb, const double* V, const double* B, int s,
                  const int* active, double* g, int64_t r0, int64_t r1, cudaStream_t st);
// R (rows r0 .. r0 + nrows) -= H[rows, B] delta
void launch_kcols(const Op& op, const int* blk, int bs, const double* delta, int s,
                  const int* active, double* R, int64_t r0, int64_t nrows, cudaStream_t st);
void launch_block_chol(const Op& op, int bs, int nblk, double* fac, double* inv, int* fail,
                       cudaStream_t st);
void launch_ap_block_solve(const double* inv, int bs, int64_t n, const int* blk, const int* active,
                           const double* R, const double* Rblk, int s, double* V, double* delta,
                           double* ybuf, cudaStream_t st);
void launch_seg_norms(const double* Rloc, int64_t r0, int64_t nloc, const int64_t* seg_start, int nseg,
                      int s, const int* active, double* segn, cudaStream_t st);
void launch_greedy_from_segments(const double* segn, const int* seg_block, int nseg, int nblk, int s,
                                 const int* active, int* blk, cudaStream_t st);
void launch_gather_block_rows(const double* Rloc, int64_t r0, int64_t nloc, int64_t n, int bs,
                              const int* blk, const int* active, int s, double* Rblk, cudaStream_t st);
void launch_set_cyclic(int* blk, int s, int value, cudaStream_t st);
void launch_sgd_update(double* V, double* vel, const int* rows, const double* g, int nb, int64_t n,
                       int s, const int* active, double momentum, double scale, double lr,
                       int64_t r0, cudaStream_t st);
void launch_copy_masked_cols(double* dst, const double* src, int64_t n, int s, const int* mask,
                             cudaStream_t st);

}  // namespace wgp
