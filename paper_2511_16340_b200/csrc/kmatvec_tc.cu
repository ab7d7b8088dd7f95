// kmatvec_tc.cu -- tcgen05 (5th-gen tensor core) fused kernel-matvec for sm_100a.
//
//   Y[i, :] = sum_j k(x_i, x_j) V[j, :] + sigma_n^2 V[i, :]      (gram, H = K + sigma_n^2 I)
//
// restating gram_matrix (kernel.cpp:48-72) + H*p (solvers.cpp:162) without materialising
// K.  One CTA owns 128 rows i and a contiguous range of j tiles (grid: row blocks x j
// splits); a tile is BJ_ = 64 columns (four TMEM tile buffers) or, when the RHS needs at
// most 32 accumulator columns, 128 (three buffers: half the pipeline rounds per pair):
//
//   GEMM1  S = XA_i . XB_j^T      (M=128, N=BJ_, K=K1)  tcgen05.mma SS, S (fp32) in TMEM.
//          The operands are pre-formatted so the contraction yields the squared distance
//          directly (the norm form |x|^2 + |y|^2 - 2 x.y of kernel.cpp:39-46, 65), as
//          3-way hi/lo splits: kind::f16 on x/l when the scaled coordinates fit fp16
//          comfortably (|x|/l <= 64), else kind::tf32 on x:
//            XA = [-2xh | -2xh | -2xl | sqh | sql | 1 | 1]
//            XB = [ xh  |  xl  |  xh  |  1  |  1  | sqh | sql]
//          (TF32 precision: XA = [-2xh | sqh | 1], XB = [xh | 1 | sqh], single pass, ~2^-11)
//   map    epilogue warps: tcgen05.ld S -> k(d2)/s^2 * 2^10 in registers (Matern-3/2 or RBF;
//          MUFU sqrt/ex2, packed FP32, one Matern exponential in eight as an FMA-pipe
//          polynomial) -> fp16 hi/lo split -> tcgen05.st back into the same TMEM columns (K
//          never leaves the SM).
//   GEMM2  Y += K_hi V_hi (chunk accumulator), C += K_hi V_lo + K_lo V_hi (correction
//          accumulator)  (M=128, N=s_pad, K=BJ_)  kind::f16, A from TMEM (TS form).  V is
//          pre-split into fp16 hi/lo with a per-column power-of-two scale, in 64-column
//          sub-tiles.
//   drain  every CH tiles the finished chunk accumulator is added (fp32 vector reductions)
//          into L2-resident partials; reduce_splits_kernel sums splits in fp64 and writes
//          Y * s^2 / (2^10 * scale_c) + sigma_n^2 V_i (or B - that: the true residual of
//          solvers.cpp:171) as fp64.
//
// Warp roles (32 warps): 28 = XB bulk-copy producer (TMA engine, UBLKCP) + XA load,
// 29 = GEMM1 issuer, 30 = V bulk-copy producer + TMEM allocator, 31 = GEMM2 issuer (whole
// warps run the schedules, one elected lane issues), 24..27 = drain warps (one per TMEM lane
// quadrant), 0..23 = epilogue: three sets of 8 warps taking j tiles round-robin (2 warps per
// TMEM lane quadrant, BJ_ / 2 columns each).  Pipelines:
// smem rings of XB_j (NSX) and V_j hi/lo (NSV); a ring of NB TMEM tile buffers (S written
// by GEMM1, overwritten in place by K for GEMM2); mbarriers + tcgen05.commit.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "solvers.h"

namespace wgp {
KernelTimer& kernel_timer() {
  static KernelTimer t;
  return t;
}

namespace tc {

constexpr int BM = 128;        // rows per CTA (UMMA M)
constexpr int BJ = 64;         // columns j per tile (GEMM1 N, GEMM2 K)
constexpr int EPIW = 24;       // epilogue warps
constexpr int SETW = 8;        // warps per epilogue set (2 per TMEM lane quadrant)
constexpr int NSET = EPIW / SETW;  // sets taking tiles round-robin
constexpr int CPW = 32;        // tile columns per epilogue warp
// One producer warp per smem ring: bulk copies issued by one warp are processed one at a
// time (~400-900 cycles each in isolation, tools/bulk_microbench2.cu), but two XB and three
// V producers measured no faster than one of each at C3 (the pipeline is paced by the
// epilogue, not by V arrival).  Role r (warp EPIW + r): 0 XB producer, 1 GEMM1, 2 V producer,
// 3 GEMM2.
// (Round-robin GEMM2 issue over several warps and 4-warp epilogue sets were tried and
// measured no faster / hung.)
// (Splitting GEMM2 over two issuing warps -- the leading product on role 3, the correction
// products on a fifth role warp, each with its own accumulators -- measured 2-7% slower: the
// MMAs of both issuers share one tensor pipe and GEMM1 then waits on two commits.)
constexpr int NROLE = 4;
// Four drain warps (one per TMEM lane quadrant, warps EPIW..EPIW+3) move each finished chunk
// accumulator into the partials, so the epilogue sets never drain (with the drain visits
// spread over the epilogue sets instead: 2.6% (C3) to 4.2% (C4-shape) slower).
constexpr int NDRAIN = 4;
constexpr int NTHREADS = 32 * (NROLE + NDRAIN + EPIW);  // role + drain + epilogue warps
constexpr int MAX_SPAD = 64;   // RHS columns per launch (wider RHS: column chunks)
constexpr int CH_DEFAULT = 16; // j tiles per TMEM accumulation chunk (drained after each)
// TMEM (512 columns): a ring of NB = 4 64-column tile buffers [0, 256) and the accumulators
// [256, 256 + 4 s_pad).  A buffer holds S(t) (fp32 d^2, written by GEMM1); the epilogue loads
// it into registers and writes K(t) back in place as packed fp16 (each warp into the 32
// columns it read: 16 hi + 16 lo), which GEMM2 then reads as its A operand; GEMM2's commit
// frees the buffer for GEMM1 of tile t + NB.  Accumulators per chunk parity a:
// [Y_a | C_a] adjacent, so one N = 2 s_pad MMA computes K_h [V_h | V_l] (the leading product
// into the chunk accumulator Y_a, the first correction product into C_a; V_h and V_l tiles
// are adjacent in shared memory) and one N = s_pad MMA adds K_l V_h into C_a: 8 MMAs per
// tile (12 with separate products measured 1-3% slower).  Every MMA accumulates; the drain
// warps zero the accumulators at the start and Y_a after draining it.  Each tcgen05.mma
// truncates its fp32 sum (a relative bias of about -2^-25 per instruction against the
// running accumulator), so Y_a covers only CH tiles before it is drained (alternating
// parities: GEMM2 fills one while the other drains); the correction products (2^-11 of the
// leading term) stay in C_a for the whole sweep.  Measured at the C3 shape
// (tools/probes/gpu_probe_ch_c3.py, vs the fp64 operator): CH = 16 -> 1.4e-6 (random V) /
// 5.8e-6 (positive V); 32 -> 2.6e-6 / 1.2e-5; 64 -> 4.9e-6 / 2.5e-5, each doubling ~1-2%
// faster.  WGP_TC_CH overrides.
constexpr int MAX_NB = 4;  // TMEM tile buffers (5 measured no faster)
constexpr int TRW = 14;  // trace slots per tile
constexpr float KSCALE_LOG2 = 10.0f;  // K stored as k/s^2 * 2^10 (fp16 normal range)

struct Params {
  const void* XA;       // tiled A operand rows (this launch's rows start at tile 0)
  const void* XB;       // tiled B operand rows (all columns j)
  int g1f16;            // GEMM1 operands fp16 (kind::f16, K = 16) instead of tf32 (K = 8)
  const __half* Vt;     // tiled V hi/lo per j tile (fp16, per-column scaled)
  const float* vscale;  // [s_pad] 2^-e_c: undo the per-column V scale
  int64_t nrows, row0, ncols;
  int64_t col0;         // global index of column 0 of this launch (diagonal detection)
  int ntiles;           // ceil(ncols / BJ)
  int tiles_per_split;  // j tiles per CTA along grid.y (2-D decomposition)
  int ch;               // j tiles per accumulation chunk
  float* Ypart;         // fp32 partial sums [gridDim.y][s_pad / 4][nrows][4] (unscaled)
  int s, s_pad, K1;
  int kind;
  float c1, neg_c_log2e;
  double out_scale;     // s^2 * 2^-10
  double noise2;
  int gram;
  unsigned long long* trace;  // debug: per-tile event clocks of CTA 0 (nullptr normally)
  unsigned long long* cta_trace;  // debug: per-CTA [start, loop end, end] globaltimer + smid
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cta_ev(const Params& p, int slot) {
  if (p.cta_trace) {
    const size_t c = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    p.cta_trace[c * 4 + slot] = gtimer();
    if (slot == 0) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
      p.cta_trace[c * 4 + 3] = sm;
    }
  }
}

__device__ __forceinline__ void trace_ev(const Params& p, int t, int slot) {
  if (p.trace && blockIdx.x == 0 && blockIdx.y == 0) p.trace[(size_t)t * TRW + slot] = clock64();
}

// round to the nearest tf32 (10 explicit mantissa bits; the tensor core ignores the low 13)
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

__device__ __forceinline__ uint32_t pack_h2(float lo_elem, float hi_elem) {
  const __half2 h = __floats2half2_rn(lo_elem, hi_elem);  // .x (low 16 bits) = lower k index
  return *reinterpret_cast<const uint32_t*>(&h);
}

// 2^10 * 2^a for a <= 0 on the FMA pipe (two values per packed instruction), for the share
// of the Matern map's exponentials moved off MUFU: a = j + f with j = round(a) (the 1.5 2^23
// magic add leaves j in the low mantissa bits of t), 2^f on [-1/2, 1/2] by a degree-5
// relative-minimax polynomial with its coefficients scaled by 2^10 (max relative error
// 2.3e-7 in fp32 Horner, like ex2.approx's ~2 ulp), 2^j added into the exponent field with
// an integer shift-add.  a is clamped at -100 so the exponent stays normal (2^-90 flushes to
// zero in the fp16 split anyway, as the MUFU path's value does).
// pairs of each 16-column group whose ex2 runs on the FMA pipe (even / odd 16-column groups
// of a warp's columns).  Short runs at the full clock: 2 of 8 pairs fastest (C3 5.62 ->
// 5.35 ms; 3 of 8 slower again); sustained 200-launch runs under the board power cap
// (~1700 MHz): 1 of 8 fastest (6.08-6.09 ms vs 6.14 at 2 of 8, 6.19 with none) -- the FMA
// path's energy competes with the clock there.  The bench is a sustained run.
#ifndef WGP_EXP_POLY_A
#define WGP_EXP_POLY_A 1
#endif
#ifndef WGP_EXP_POLY_RBF
#define WGP_EXP_POLY_RBF 0  // the same for the RBF map: not SFU-bound, 2 / 4 of 8 measured 3% / 11% slower
#endif
#ifndef WGP_EXP_POLY_B
#define WGP_EXP_POLY_B 1
#endif
#if defined(WGP_KSCALE_IN_EXP) && (WGP_EXP_POLY_A || WGP_EXP_POLY_B)
#error "WGP_EXP_POLY assumes the 2^10 scale outside the exponent argument"
#endif
__device__ __forceinline__ float2 ex2_poly_k(float2 a) {
  a.x = fmaxf(a.x, -100.0f);
  a.y = fmaxf(a.y, -100.0f);
  const float2 M = make_float2(0x1.8p23f, 0x1.8p23f);
  const float2 t = __fadd2_rn(a, M);
  const float2 j = __fadd2_rn(t, make_float2(-0x1.8p23f, -0x1.8p23f));
  const float2 f = __ffma2_rn(j, make_float2(-1.0f, -1.0f), a);
  float2 p = __ffma2_rn(make_float2(0x1.5c08e4p0f, 0x1.5c08e4p0f), f,
                        make_float2(0x1.3d0c52p3f, 0x1.3d0c52p3f));
  p = __ffma2_rn(p, f, make_float2(0x1.c6b6e4p5f, 0x1.c6b6e4p5f));
  p = __ffma2_rn(p, f, make_float2(0x1.ebf918p7f, 0x1.ebf918p7f));
  p = __ffma2_rn(p, f, make_float2(0x1.62e428p9f, 0x1.62e428p9f));
  p = __ffma2_rn(p, f, make_float2(0x1.000002p10f, 0x1.000002p10f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

// Kernel map of NCOL columns of a row: v = fp32 d^2 from TMEM, kv = k/s^2 * 2^10.  Pairs of
// columns go through the packed FP32 pipe, sqrt and exp2 through MUFU, except the first NPOLY
// pairs of the Matern map, whose exp2 runs on the FMA pipe (ex2_poly_k): the map is bound by
// the SFU (two MUFU ops per pair), the FMA pipe is mostly idle.  sqrt(|d2|): a tiny negative
// d2 from the norm-form cancellation maps to ~0 like the reference's max(.,0) clamp
// (kernel.cpp:44).
template <int NCOL, int NPOLY>
__device__ __forceinline__ void kernel_map(int kind, const uint32_t* v, float* kv, float c1,
                                           float nclog2e) {
#ifdef WGP_SKIP_MAP
  // timing-only probe build: no map (invalid results)
#pragma unroll
  for (int q = 0; q < NCOL; ++q) kv[q] = __uint_as_float(v[q]) * 0.5f;
  return;
#endif
  const float2 NC = make_float2(nclog2e, nclog2e);
#ifdef WGP_KSCALE_IN_EXP
  // (earlier form, kept for A/B probes) the 2^10 scale folded into the exponent argument:
  // one FFMA2 fewer, but the argument then carries |a| ~ 10 and its fp32 rounding puts
  // ~4e-7 relative error on the largest entries (d ~ 0)
  const float2 OFF = make_float2(KSCALE_LOG2, KSCALE_LOG2);
#else
  // the 2^10 scale is applied outside ex2 (exact power-of-two factors): the exponent
  // argument -z log2 e / -d2 log2 e / 2l^2 is ~0 for the largest entries, so its rounding
  // error (|a| 2^-24, x ln 2 on k) vanishes where k matters most
  const float2 SC = make_float2(0x1.0p10f, 0x1.0p10f);
#endif
  if (kind == WGP_MATERN32) {
    const float2 C1 = make_float2(c1, c1);
    // 2^10 (1 + z) with z = c1 r in one FFMA2 (2^10 c1 is exact): k = u e^{-z}, three
    // packed FP32 instructions per pair of columns besides the MUFU ops
    const float2 C1K = make_float2(c1 * 0x1.0p10f, c1 * 0x1.0p10f);
#pragma unroll
    for (int q = 0; q < NCOL / 2; ++q) {
      float2 r;
      r.x = ptx::sqrt_approx(fabsf(__uint_as_float(v[2 * q])));
      r.y = ptx::sqrt_approx(fabsf(__uint_as_float(v[2 * q + 1])));
#ifdef WGP_KSCALE_IN_EXP
      const float2 a = __ffma2_rn(r, NC, OFF);  // log2(2^10 e^{-z})
      float2 e;
      e.x = ptx::ex2_approx(a.x);
      e.y = ptx::ex2_approx(a.y);
      const float2 k = __ffma2_rn(__fmul2_rn(r, C1), e, e);
#else
      const float2 a = __fmul2_rn(r, NC);  // log2(e^{-z})
      float2 k;
      if (q < NPOLY) {
        const float2 e = ex2_poly_k(a);  // 2^10 e^{-z} on the FMA pipe
        k = __ffma2_rn(__fmul2_rn(r, C1), e, e);
      } else {
        float2 e;
        e.x = ptx::ex2_approx(a.x);
        e.y = ptx::ex2_approx(a.y);
        k = __fmul2_rn(__ffma2_rn(r, C1K, SC), e);  // 2^10 (1 + z) e^{-z}
      }
#endif
      kv[2 * q] = k.x;
      kv[2 * q + 1] = k.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < NCOL / 2; ++q) {
      const float2 d2 = make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
#ifdef WGP_KSCALE_IN_EXP
      const float2 a = __ffma2_rn(d2, NC, OFF);  // log2(2^10 e^{-d2/2l^2})
#else
      const float2 a = __fmul2_rn(d2, NC);  // log2(e^{-d2/2l^2})
#endif
      float2 e;
#ifndef WGP_KSCALE_IN_EXP
      if (q < WGP_EXP_POLY_RBF) {
        e = ex2_poly_k(a);
      } else {
        e.x = ptx::ex2_approx(a.x);
        e.y = ptx::ex2_approx(a.y);
        e = __fmul2_rn(e, SC);
      }
#else
      e.x = ptx::ex2_approx(a.x);
      e.y = ptx::ex2_approx(a.y);
#endif
      kv[2 * q] = e.x;
      kv[2 * q + 1] = e.y;
    }
  }
}

// BJ_ = j columns per tile: 64 (NB = 4 TMEM tile buffers, any s_pad <= 64) or 128 (NB = 3,
// s_pad <= 32: [0, 384) tile buffers + 4 s_pad accumulator columns).  A 128-column tile is two
// 64-column V sub-tiles (the global V layout is per 64 columns) and half as many pipeline
// rounds per pair: the GEMM2 issue loop (~900 cycles per round) then
// covers 16384 pairs instead of 8192, which is what bounds the one-MUFU RBF map.
// At BJ_ = 128 the three TMEM buffers leave no spare beyond the three epilogue sets: GEMM1 of
// a set's next tile waits for the GEMM2 of its current one (epilogue S wait ~1200 cycles per
// tile in the trace).  Two sets (16 epilogue warps, a spare buffer) measured slower still --
// the map then lacks warps -- with 32-column TMEM load batches slower again.
template <int BJ_>
__global__ void __launch_bounds__(NTHREADS, 1) kmatvec_tc_kernel(const Params p, int NSX, int NSV) {
  constexpr int NB = BJ_ == 64 ? MAX_NB : 3;
  constexpr int EPIW_ = EPIW;
  constexpr int NSET_ = NSET;
  constexpr int CPW_ = BJ_ / 2;           // tile columns per epilogue warp
  constexpr int NSUB = BJ_ / BJ;          // 64-column V sub-tiles per tile
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Epilogue warps 0..EPIW-1, drain warps EPIW..EPIW+3, role warps EPIW+4..EPIW+7 (role r on
  // SM sub-partition r): the issue arbiter favours the highest warp id, so the producers and
  // MMA issuers -- a few instructions per tile on the critical path -- win the issue slot over
  // the map warps they share a sub-partition with.
  const int role = warp - EPIW_ - NDRAIN;  // < 0 for epilogue (and drain) warps
  const uint32_t ESZ = p.g1f16 ? 2 : 4;     // GEMM1 operand element bytes
  const uint32_t XA_BYTES = BM * p.K1 * ESZ;
  const uint32_t XB_BYTES = BJ_ * p.K1 * ESZ;
  const uint32_t VT_BYTES = p.s_pad * BJ * 2;  // one of hi / lo (fp16) of a 64-column sub-tile
  const uint32_t VS_BYTES = NSUB * 2 * VT_BYTES;  // one V stage: NSUB x [hi | lo]
  unsigned char* sXA = smem;
  unsigned char* sXB = smem + XA_BYTES;                        // NSX stages of XB_j
  unsigned char* sV = sXB + (size_t)NSX * XB_BYTES;            // NSV stages of V_j hi | lo
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + (size_t)NSV * VS_BYTES);
  uint64_t* xb_full = bars;               // [NSX] bulk copy -> GEMM1
  uint64_t* xb_empty = xb_full + NSX;     // [NSX] GEMM1 -> XB producer
  uint64_t* v_full = xb_empty + NSX;      // [NSV] bulk copy -> GEMM2
  uint64_t* v_empty = v_full + NSV;       // [NSV] GEMM2 -> V producer
  uint64_t* xa_full = v_empty + NSV;
  // Per (TMEM buffer, column half) at BJ_ = 128 -- index 2 b + h -- so each half of a tile
  // flows on its own: the epilogue warps of column half h (their own warps) wait only for
  // S(t, h), GEMM2 issues the K-steps of half h as soon as K(t, h) is complete, and GEMM1 of
  // tile t + NB writes half h once GEMM2 has read K(t, h).  With three buffers for three
  // epilogue sets the set mapping tile t waits for the buffer of tile t itself: the halves
  // shorten that round trip.  At BJ_ = 64 only index 2 b is used (the whole tile).
  constexpr bool HALVES = BJ_ == 128;
  uint64_t* s_full = xa_full + 1;         // [2 MAX_NB] GEMM1 -> epilogue
  uint64_t* k_full = s_full + 2 * MAX_NB; // [2 MAX_NB] epilogue -> GEMM2
  uint64_t* b_free = k_full + 2 * MAX_NB; // [2 MAX_NB] GEMM2 -> GEMM1
  uint64_t* y_full = b_free + 2 * MAX_NB; // [2] chunk accumulator done (GEMM2 commit)
  uint64_t* y_free = y_full + 2;          // [2] chunk accumulator drained (drain warps)
  uint64_t* c_full = y_free + 2;          // correction accumulator final (last commit)
  uint64_t* acc_zero = c_full + 1;        // accumulators zeroed (drain warps, merged GEMM2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_zero + 1);
  // TMEM columns of the accumulators: [Y_0 | C_0 | Y_1 | C_1], s_pad each (see MAX_NB)
  const uint32_t TM_ACC = NB * BJ_;
  const uint32_t AW = (uint32_t)p.s_pad;
  // this CTA's j range: tiles [jt0, jt0 + T) of the column sweep
  const int jt0 = blockIdx.y * p.tiles_per_split;
  const int T = min(p.ntiles - jt0, p.tiles_per_split);
  const int CH = p.ch;
  const int NCH = (T + CH - 1) / CH;
  if (threadIdx.x == 0) cta_ev(p, 0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSX; ++i) {
      ptx::mbar_init(&xb_full[i], 1);
      ptx::mbar_init(&xb_empty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    ptx::mbar_init(xa_full, 1);
    ptx::mbar_init(c_full, 1);
    ptx::mbar_init(acc_zero, NDRAIN);
    for (int i = 0; i < MAX_NB; ++i) {
      for (int h = 0; h < 2; ++h) {
        ptx::mbar_init(&s_full[2 * i + h], 1);
        ptx::mbar_init(&k_full[2 * i + h], HALVES ? SETW / 2 : SETW);
        ptx::mbar_init(&b_free[2 * i + h], 1);
      }
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&y_full[i], 1);
      ptx::mbar_init(&y_free[i], NDRAIN);  // chunk accumulator drained (the drain warps)
    }
    ptx::fence_mbar_init();
  }
  if (role == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KS1 = p.K1 * ESZ / 32;          // GEMM1 K-steps (32 bytes of K per instruction)
  const uint32_t sbo1 = (p.K1 * ESZ / 16) * 128;  // 8-row group stride of XA/XB tiles

  if (role == 0 || role == 2) {
    // ------------------------------------------------------------ producers (TMA engine)
    // Two independent rings: XB_j is consumed by GEMM1 right away, V_j only by GEMM2 after
    // the kernel map, so V stays resident ~4x longer; separate rings let each be as deep as
    // its own lifetime needs.
    const bool leader = ptx::elect_one();
    if (role == 0 && leader) {
      ptx::mbar_arrive_expect_tx(xa_full, XA_BYTES);
      ptx::bulk_g2s(sXA, static_cast<const char*>(p.XA) + (size_t)blockIdx.x * XA_BYTES, XA_BYTES,
                    xa_full);
    }
    // (ring positions by counters: an integer division by a runtime ring size compiles to
    // MUFU.RCP, which queues behind the epilogue's SFU work on a loaded SM sub-partition)
    if (role == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = 0; t < T; ++t, st = (st + 1 == NSX) ? 0 : st + 1, ph ^= (st == 0)) {
        if (t >= NSX) ptx::mbar_wait(&xb_empty[st], ph ^ 1);
        if (leader) {
          trace_ev(p, t, 6);
          ptx::mbar_arrive_expect_tx(&xb_full[st], XB_BYTES);
          ptx::bulk_g2s(sXB + (size_t)st * XB_BYTES,
                        static_cast<const char*>(p.XB) + (size_t)(jt0 + t) * XB_BYTES, XB_BYTES,
                        &xb_full[st]);
        }
        __syncwarp();
      }
    } else {
      int st = 0;
      uint32_t ph = 0;
      for (int t = 0; t < T; ++t, st = (st + 1 == NSV) ? 0 : st + 1, ph ^= (st == 0)) {
        if (t >= NSV) ptx::mbar_wait(&v_empty[st], ph ^ 1);
        if (leader) {
          trace_ev(p, t, 8);
          ptx::mbar_arrive_expect_tx(&v_full[st], VS_BYTES);
          ptx::bulk_g2s(sV + (size_t)st * VS_BYTES, p.Vt + (size_t)(jt0 + t) * NSUB * 2 * p.s_pad * BJ,
                        VS_BYTES, &v_full[st]);
        }
        __syncwarp();
      }
    }
  } else if (role == 1 || role == 3) {
    // ------------------------------------------------------------ MMA issuers
    // tcgen05.mma issue blocks for about the instruction's execution time, so one thread
    // cannot keep two dependent streams fed.  Role 1 issues GEMM1 (distance tiles) and role 3
    // issues GEMM2 (K.V); each waits only on its own inputs and each tcgen05.commit tracks
    // its own thread's MMAs.  Whole warps run the schedules (uniform control flow, descriptors
    // in uniform registers: a single-lane loop measured 3x slower MMA issue); one elected lane
    // issues.
    if (role == 1) {
      constexpr int G1N = HALVES ? BJ_ / 2 : BJ_;  // GEMM1 N per instruction group
      const uint32_t idesc1 = p.g1f16 ? ptx::idesc_f16(BM, G1N) : ptx::idesc_tf32(BM, G1N);
      const uint64_t dXA = ptx::umma_desc(ptx::smem_u32(sXA), 128, sbo1);
      const uint64_t dXB0 = ptx::umma_desc(ptx::smem_u32(sXB), 128, sbo1);
      const uint64_t xb_step = (uint64_t)(XB_BYTES >> 4);  // descriptor start-address units
      ptx::mbar_wait(xa_full, 0);
      int st1 = 0, b1 = 0;
      uint32_t ph1 = 0, phb1 = 0;
      for (int t = 0; t < T; ++t) {
        ptx::mbar_wait(&xb_full[st1], ph1);
#pragma unroll
        for (int h = 0; h < (HALVES ? 2 : 1); ++h) {
          if (t >= NB) ptx::mbar_wait(&b_free[2 * b1 + h], phb1 ^ 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            if (h == 0) trace_ev(p, t, 0);
            // half h: XB rows 64 h.. (eight 8-row groups of sbo1 bytes further), S columns 64 h..
            const uint64_t dB = dXB0 + xb_step * st1 + (uint64_t)h * ((8 * sbo1) >> 4);
            const uint32_t dS = tmem + b1 * BJ_ + h * G1N;
            if (p.g1f16) {
              for (int ks = 0; ks < KS1; ++ks)
                ptx::mma_f16_ss(dS, dXA + 16 * ks, dB + 16 * ks, idesc1, ks > 0 ? 1u : 0u);
            } else {
              for (int ks = 0; ks < KS1; ++ks)
                ptx::mma_tf32_ss(dS, dXA + 16 * ks, dB + 16 * ks, idesc1, ks > 0 ? 1u : 0u);
            }
            ptx::mma_commit(&s_full[2 * b1 + h]);
            if (h == (HALVES ? 1 : 0)) ptx::mma_commit(&xb_empty[st1]);
          }
          __syncwarp();
        }
        if (++st1 == NSX) { st1 = 0; ph1 ^= 1; }
        if (++b1 == NB) { b1 = 0; phb1 ^= 1; }
      }
    } else {
      const uint32_t idesc2 = ptx::idesc_f16(BM, p.s_pad);
      const uint32_t idesc2w = ptx::idesc_f16(BM, 2 * p.s_pad);
      // fp16 V tile: rows c (N) in 8-row groups, K = 64 j in 8-element (16 B) chunks
      const uint64_t dV0 = ptx::umma_desc(ptx::smem_u32(sV), 128, (BJ / 8) * 128);
      const uint64_t v_step = (uint64_t)(VS_BYTES >> 4);
      const uint64_t sub_step = (uint64_t)((2 * VT_BYTES) >> 4);  // next 64-column sub-tile
      int st2 = 0, b2 = 0, c = 0, pos = 0;  // V stage, TMEM buffer, chunk, tile within chunk
      uint32_t ph2 = 0, phb2 = 0;
      for (int t = 0; t < T; ++t) {
        const int ya = c & 1;
        const bool first = pos == 0, last = t == T - 1 || pos == CH - 1;
        if (first && c >= 2) ptx::mbar_wait(&y_free[ya], ((c >> 1) - 1) & 1);
        if (lane == 0) trace_ev(p, t, 13);
        ptx::mbar_wait(&v_full[st2], ph2);
        if (lane == 0) trace_ev(p, t, 9);
        if (t == 0) ptx::mbar_wait(acc_zero, 0);  // drain warps zeroed the accumulators
        const uint64_t dVh = dV0 + v_step * st2;
        const uint32_t yacc = tmem + TM_ACC + 2 * AW * ya;
        const uint32_t kb = tmem + b2 * BJ_;
        // K-step ks: 16 j's of sub-tile ks / 4 (8 TMEM columns [hi] + 8 [lo] per step)
        auto issue = [&](int ks) {
          const uint64_t dv = dVh + sub_step * (ks / 4) + 16 * (ks % 4);
          ptx::mma_f16_ts(yacc, kb + ks * 16, dv, idesc2w, 1u);      // [Y|C] += Kh [Vh|Vl]
#ifndef WGP_PROBE_SKIP_CORR  // (timing-only probe: without the K_l V_h products)
          ptx::mma_f16_ts(yacc + AW, kb + ks * 16 + 8, dv, idesc2, 1u);  // C += Kl Vh
#endif
        };
        if (HALVES) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            ptx::mbar_wait(&k_full[2 * b2 + h], phb2);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
              if (h == 0) trace_ev(p, t, 1);
#pragma unroll
              for (int ks = 4 * h; ks < 4 * h + 4; ++ks) issue(ks);
              ptx::mma_commit(&b_free[2 * b2 + h]);  // K(t, h) read: GEMM1 may rewrite half h
            }
            __syncwarp();
          }
        } else {
          ptx::mbar_wait(&k_full[2 * b2], phb2);
          ptx::tc_fence_after();
        }
        if (ptx::elect_one()) {
          if (!HALVES) {
            trace_ev(p, t, 1);
#pragma unroll
            for (int ks = 0; ks < BJ_ / 16; ++ks) issue(ks);
            ptx::mma_commit(&b_free[2 * b2]);
          }
          trace_ev(p, t, 10);
          ptx::mma_commit(&v_empty[st2]);
          if (last) ptx::mma_commit(&y_full[ya]);
          if (t == T - 1) ptx::mma_commit(c_full);  // the correction accumulators are final
          trace_ev(p, t, 12);
        }
        __syncwarp();
        if (++st2 == NSV) { st2 = 0; ph2 ^= 1; }
        if (++b2 == NB) { b2 = 0; phb2 ^= 1; }
        if (++pos == CH) { pos = 0; ++c; }
      }
    }
  } else if (warp < EPIW_) {
    // ------------------------------------------------------------ kernel-map epilogue
    // NSET sets of 8 warps take tiles round-robin (set = t mod NSET); within a set, warp
    // (quadrant q, half) maps rows 32q.. and columns 32 half.. of the tile, 16 at a time.
    const int q = warp & 3;                   // TMEM lane quadrant accessible to this warp
    const int g = warp >> 2;                  // group of 4 warps (one per quadrant), 0..5
    const int set = g / (SETW / 4), half = g % (SETW / 4);
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int r = q * 32 + lane;              // row within the CTA tile
    const int64_t gi = p.row0 + (int64_t)blockIdx.x * BM + r;
    const int64_t grow0 = p.row0 + (int64_t)blockIdx.x * BM;
    const int64_t lr = (int64_t)blockIdx.x * BM + r;  // local output row
    const float kdiag = 1024.0f;              // k(x,x)/s^2 * 2^10
    for (int t = set; t < T; t += NSET_) {
      const int b = t % NB;                   // buffer and phase of tile t
      const uint32_t bph = (t / NB) & 1;
      const bool tr = lane == 0 && q == 0 && half == 0 && set == 0;
      if (tr) trace_ev(p, t, 2);
      ptx::mbar_wait(&s_full[2 * b + (HALVES ? half : 0)], bph);
      ptx::tc_fence_after();
      if (tr) trace_ev(p, t, 3);
      const int64_t gj_base = p.col0 + (int64_t)(jt0 + t) * BJ_ + half * CPW_;
      const bool diag = p.gram && gj_base < grow0 + BM && gj_base + CPW_ > grow0;
      // The warp's CPW_ columns in 16-column groups (GW) under the 64-register budget of 32
      // warps (issuing the next group's load before the current group's split measured no
      // faster).
      constexpr int GW = 16;
      const uint32_t col0 = tmem + lane_off + b * BJ_ + half * CPW_;
#pragma unroll
      for (int g0 = 0; g0 < CPW_; g0 += GW) {
        uint32_t v[GW];
#pragma unroll
        for (int u = 0; u < GW / 16; ++u)
          ptx::tmem_ld16(col0 + g0 + 16 * u, *reinterpret_cast<uint32_t(*)[16]>(v + 16 * u));
        ptx::tmem_wait_ld();
        if (tr && g0 == 0) trace_ev(p, t, 7);
        float kv[GW];
#pragma unroll
        for (int u = 0; u < GW / 16; ++u) {
          if (((g0 / 16) + u) % 2 == 0)
            kernel_map<16, WGP_EXP_POLY_A>(p.kind, v + 16 * u, kv + 16 * u, p.c1, p.neg_c_log2e);
          else
            kernel_map<16, WGP_EXP_POLY_B>(p.kind, v + 16 * u, kv + 16 * u, p.c1, p.neg_c_log2e);
        }
        if (diag) {  // tile touches the diagonal: k(x,x) = s^2 exactly
          const int64_t gj0 = gj_base + g0;
#pragma unroll
          for (int c = 0; c < GW; ++c)
            if (gj0 + c == gi) kv[c] = kdiag;
        }
#pragma unroll
        for (int u = 0; u < GW / 16; ++u) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            // hi = kv cut to fp16's 10 mantissa bits (exact in fp16 over its normal range; an
            // integer LOP on the ALU pipe), lo = kv - hi (FADD2, exact) rounded to fp16
            const float* k2 = kv + 16 * u + 2 * c;
            const float2 hf = make_float2(__uint_as_float(__float_as_uint(k2[0]) & 0xFFFFE000u),
                                          __uint_as_float(__float_as_uint(k2[1]) & 0xFFFFE000u));
            const float2 rem = __fadd2_rn(make_float2(k2[0], k2[1]), make_float2(-hf.x, -hf.y));
            hi[c] = pack_h2(hf.x, hf.y);
            lo[c] = pack_h2(rem.x, rem.y);
          }
          // K back into the 16 columns just read: [hi 8 | lo 8]
          const uint32_t col = col0 + g0 + 16 * u;
          ptx::tmem_st8(col, hi);
          ptx::tmem_st8(col + 8, lo);
        }
      }
      if (tr) trace_ev(p, t, 4);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&k_full[2 * b + (HALVES ? half : 0)]);
      if (tr) trace_ev(p, t, 5);
      if (lane == 0 && half == 0 && set == 0 && q == 3) trace_ev(p, t, 11);
    }
    if (warp == 0 && lane == 0) cta_ev(p, 1);
  }
  if (warp >= EPIW_ && warp < EPIW_ + NDRAIN) {
    // ------------------------------------------------------------ drain warps
    // Chunk c's accumulator (after its y_full) 16 columns at a time into this CTA's slice of
    // the partials [gy][s_pad/4][nrows][4] (4 columns of a row contiguous: one 16-byte vector
    // reduction per lane, a warp covering 512 contiguous bytes; L2-resident): the first chunk
    // stores, later chunks add with fire-and-forget reductions performed at L2 (fp32: ~50
    // chunk terms per sweep at C3, relative rounding ~1e-7).  Each address is only ever
    // touched by one thread, and same-address operations of one thread stay in program order,
    // so the summation order (chunk 0, 1, 2, ...) is deterministic.  A drain waits only on
    // GEMM2's commits, never on the pipeline, so it cannot deadlock; it must finish before
    // GEMM2 starts chunk c + 2 (y_free).  After the sweep: the correction accumulator.
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int64_t lr = (int64_t)blockIdx.x * BM + q * 32 + lane;
    const bool row_ok = lr < p.nrows;
    const int nquads = p.s_pad / 4;
    float* __restrict__ ypart = p.Ypart + ((size_t)blockIdx.y * nquads * p.nrows + lr) * 4;
    auto put4 = [&](int qd, const uint32_t* y, bool store) {
      if (!row_ok || 4 * qd >= p.s) return;
      float* dst = ypart + (size_t)qd * p.nrows * 4;
      if (store)
        asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(y[0]), "r"(y[1]),
                     "r"(y[2]), "r"(y[3]) : "memory");
      else
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(y[0]), "r"(y[1]),
                     "r"(y[2]), "r"(y[3]) : "memory");
    };
    const uint32_t zero16[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (uint32_t c16 = 0; c16 < 4 * AW; c16 += 16)  // [Y_0 | C_0 | Y_1 | C_1]
      ptx::tmem_st16(tmem + lane_off + TM_ACC + c16, zero16);
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(acc_zero);
    for (int c = 0; c < NCH; ++c) {
      const int ya = c & 1;
      const uint32_t ya_col = TM_ACC + 2 * AW * ya;
      ptx::mbar_wait(&y_full[ya], (c >> 1) & 1);
      ptx::tc_fence_after();
      for (int c16 = 0; c16 < p.s_pad; c16 += 16) {
        uint32_t y[16];
        ptx::tmem_ld16(tmem + lane_off + ya_col + c16, y);
        ptx::tmem_wait_ld();
        ptx::tmem_st16(tmem + lane_off + ya_col + c16, zero16);  // ready for chunk c + 2
#pragma unroll
        for (int k = 0; k < 4; ++k) put4(c16 / 4 + k, y + 4 * k, c == 0);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&y_free[ya]);
    }
    ptx::mbar_wait(c_full, 0);
    ptx::tc_fence_after();
    for (int a = 0; a < 2 && a < NCH; ++a)
      for (int c16 = 0; c16 < p.s_pad; c16 += 16) {
        uint32_t y[16];
        ptx::tmem_ld16(tmem + lane_off + TM_ACC + 2 * AW * a + AW + c16, y);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) put4(c16 / 4 + k, y + 4 * k, false);
      }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) cta_ev(p, 2);
  if (role == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// XA / XB operand rows in the tiled K-major "interleave" layout of 8-row x 16-byte core
// matrices: [row/8][k/CK][row%8][k%CK], CK = 16 / element size, from the centered fp64 rows
// scaled by `inv_l` (1 for tf32 operands; 1/l for fp16 so coordinates are O(1)).
template <typename E>
__device__ __forceinline__ E to_op(double v);
template <>
__device__ __forceinline__ float to_op<float>(double v) { return tf32_rn((float)v); }
template <>
__device__ __forceinline__ __half to_op<__half>(double v) { return __double2half(v); }
__device__ __forceinline__ double op_val(float v) { return (double)v; }
__device__ __forceinline__ double op_val(__half v) { return (double)__half2float(v); }

template <typename E>
__global__ void build_operands_kernel(const double* __restrict__ X, int dpad, int dim,
                                      const double* __restrict__ center, double inv_l, int64_t n,
                                      int K1, int split, E* __restrict__ XA, E* __restrict__ XB) {
  constexpr int CK = 16 / sizeof(E);
  const E one = to_op<E>(1.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i >> 3, ri = i & 7;
    auto at = [&](int k) -> int64_t { return ((g * (K1 / CK) + k / CK) * 8 + ri) * CK + (k % CK); };
    double sq = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double x = (X[i * dpad + k] - center[k]) * inv_l;
      sq += x * x;
      const E xh = to_op<E>(x);
      const E m2xh = to_op<E>(-2.0 * op_val(xh));
      XA[at(k)] = m2xh;
      if (XB) XB[at(k)] = xh;
      if (split) {
        const E xl = to_op<E>(x - op_val(xh));
        XA[at(dim + k)] = m2xh;
        XA[at(2 * dim + k)] = to_op<E>(-2.0 * op_val(xl));
        if (XB) XB[at(dim + k)] = xl;
        if (XB) XB[at(2 * dim + k)] = xh;
      }
    }
    const E sqh = to_op<E>(sq);
    int b = dim;
    if (split) {
      const E sql = to_op<E>(sq - op_val(sqh));
      b = 3 * dim;
      XA[at(b)] = sqh;
      XA[at(b + 1)] = sql;
      XA[at(b + 2)] = one;
      XA[at(b + 3)] = one;
      if (XB) XB[at(b)] = one;
      if (XB) XB[at(b + 1)] = one;
      if (XB) XB[at(b + 2)] = sqh;
      if (XB) XB[at(b + 3)] = sql;
      b += 4;
    } else {
      XA[at(b)] = sqh;
      XA[at(b + 1)] = one;
      if (XB) XB[at(b)] = one;
      if (XB) XB[at(b + 1)] = sqh;
      b += 2;
    }
    for (int k = b; k < K1; ++k) {
      XA[at(k)] = to_op<E>(0.0);
      if (XB) XB[at(k)] = to_op<E>(0.0);
    }
  }
}

// max over rows of |x - c|_inf / l and |x - c|^2 / l^2 (operand rebuilds only): grid-stride
// blocks, block maxima merged with atomicMax on the IEEE bits (ordered for non-negative
// doubles); out must be zeroed.
__global__ void scaled_extent_kernel(const double* __restrict__ X, int dpad, int dim,
                                     const double* __restrict__ center, double inv_l, int64_t n,
                                     unsigned long long* __restrict__ out) {
  __shared__ double red[2][256];
  double mx = 0.0, msq = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double sq = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double x = (X[i * dpad + k] - center[k]) * inv_l;
      sq += x * x;
      mx = fmax(mx, fabs(x));
    }
    msq = fmax(msq, sq);
  }
  red[0][threadIdx.x] = mx;
  red[1][threadIdx.x] = msq;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + o]);
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(red[0][0]));
    atomicMax(&out[1], (unsigned long long)__double_as_longlong(red[1][0]));
  }
}

// Per-column max |V|: blocks of 64 rows x all columns (coalesced row-major reads), block
// maxima merged with atomicMax on the IEEE bits (ordered for non-negative doubles).
// max_j |V[j, c]| per column (fp64 bits: non-negative doubles order like their bit
// patterns).  Block = 64 rows; threads = R row lanes x cp columns (cp = min(s, 256)), each
// lane striding the block's rows, lanes combined in shared memory, one atomic per column.
__global__ void __launch_bounds__(256) colmax_kernel(const double* __restrict__ V, int64_t n, int s,
                                                     unsigned long long* __restrict__ cmax) {
  __shared__ double red[256];
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int64_t r1 = min(n, r0 + 64);
  const int cp = min(s, 256);
  const int R = 256 / cp;
  const int lane_r = threadIdx.x / cp, cl = threadIdx.x % cp;
  for (int c0 = 0; c0 < s; c0 += cp) {
    const int c = c0 + cl;
    double a = 0.0;
    if (lane_r < R && c < s) {
#pragma unroll 4
      for (int64_t j = r0 + lane_r; j < r1; j += R) a = fmax(a, fabs(V[j * s + c]));
    }
    red[threadIdx.x] = a;
    __syncthreads();
    if (threadIdx.x < cp && c < s) {
      for (int k = 1; k < R; ++k) a = fmax(a, red[k * cp + cl]);
      atomicMax(&cmax[c], (unsigned long long)__double_as_longlong(a));
    }
    __syncthreads();
  }
}

__global__ void colscale_finish_kernel(const unsigned long long* __restrict__ cmax, int s, int s_pad,
                                       float* __restrict__ scale_up, float* __restrict__ scale_down) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= s_pad) return;
  const double mx = c < s ? __longlong_as_double((long long)cmax[c]) : 0.0;
  int e = 0;
  if (mx > 0.0) {
    int ex;
    frexp(mx, &ex);  // mx = f * 2^ex, f in [0.5, 1)
    e = max(-100, min(100, 14 - ex));
  }
  scale_up[c] = ldexpf(1.0f, e);
  scale_down[c] = ldexpf(1.0f, -e);
}

// V [ncols][s] fp64 -> per-64-row tile [hi|lo][s_pad/8][8 chunks][8 c][8 j] fp16.  One
// thread per (column c, 8-row group): a warp reads consecutive columns of each row
// (coalesced) and every thread writes its 8 hi and 8 lo halves as two 16-byte stores.
__global__ void split_v_kernel(const double* __restrict__ V, int64_t ncols, int s, int s_pad,
                               int64_t total_rows, const float* __restrict__ scale_up,
                               __half* __restrict__ Vt) {
  const int64_t total = (total_rows / 8) * s_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jg = e / s_pad;
    const int c = (int)(e - jg * s_pad);
    const int64_t j0 = jg * 8;
    const double su = (double)scale_up[c];
    __align__(16) __half hv[8];
    __align__(16) __half lv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t j = j0 + k;
      const double v = (j < ncols && c < s) ? V[j * s + c] * su : 0.0;
      hv[k] = __double2half(v);
      lv[k] = __double2half(v - (double)__half2float(hv[k]));
    }
    const int64_t t = j0 / BJ;
    const int jj0 = (int)(j0 % BJ);
    const int64_t idx = ((int64_t)((c >> 3) * (BJ / 8) + (jj0 >> 3)) * 8 + (c & 7)) * 8;
    __half* base = Vt + t * 2 * (int64_t)s_pad * BJ;
    *reinterpret_cast<uint4*>(base + idx) = *reinterpret_cast<const uint4*>(hv);
    *reinterpret_cast<uint4*>(base + (int64_t)s_pad * BJ + idx) = *reinterpret_cast<const uint4*>(lv);
  }
}

// Y = C + sgn ((sum over j-splits, fixed order) * s^2 2^-10 / scale_c + sigma^2 V_i (gram)),
// C optional (B - H V: C = B, sgn = -1).
// Partials are [nsplit][s_pad/4][nrows][4] fp32; a 32-row x 32-column tile is read as one
// float4 (4 columns of a row) per thread -- a warp reads 512 contiguous bytes -- summed over
// the splits in fp64, and transposed through shared memory so the row-major writes coalesce.
__global__ void reduce_splits_kernel(const float* __restrict__ Ypart, int nsplit, int64_t nrows,
                                     int64_t row0, int s, int s_pad, const float* __restrict__ vscale,
                                     double out_scale, const double* __restrict__ V64,
                                     int64_t vrow0, const double* __restrict__ C64, double sgn,
                                     double noise2, int gram, double* __restrict__ Y64) {
  __shared__ double tile[32][33];
  const int64_t rb = (int64_t)blockIdx.x * 32;
  const int cb = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  {
    const int c0 = cb + 4 * ty;  // this thread's 4 columns
    const int64_t r = rb + tx;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (c0 < s && r < nrows) {
      const size_t G = (size_t)(s_pad / 4);
      for (int q = 0; q < nsplit; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(Ypart + (((size_t)q * G + c0 / 4) * nrows + r) * 4);
        acc[0] += (double)v.x;
        acc[1] += (double)v.y;
        acc[2] += (double)v.z;
        acc[3] += (double)v.w;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c0 + k < s) acc[k] *= out_scale * (double)vscale[c0 + k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) tile[4 * ty + k][tx] = acc[k];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = rb + k;
    const int c = cb + tx;
    if (c < s && r < nrows) {
      const int64_t e = r * s + c;
      double acc = tile[tx][k];
      if (gram) acc += noise2 * V64[vrow0 * s + e];
      Y64[e] = C64 ? C64[e] + sgn * acc : sgn * acc;
    }
  }
}

inline int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

// Number of j splits: pad the grid to a near-integral number of waves of 148 SMs
// (one CTA per SM), keeping >= 32 tiles per split.
inline int choose_splits(int row_ctas, int ntiles) {
  int best = 1;
  double best_cost = 1e30;
  for (int k = 1; k <= 16; ++k) {
    if (k > 1 && ntiles / k < 32) break;
    const double w = (double)row_ctas * k / 148.0;
    const double cost = std::ceil(w) / w * (1.0 + 0.01 * (k - 1));
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = k;
    }
  }
  return best;
}

}  // namespace tc

int tc_k1(int dim, int precision, bool f16) {
  const int k = precision == WGP_TF32 ? dim + 2 : 3 * dim + 4;
  const int q = f16 ? 16 : 8;  // one MMA K-step
  return ((k + q - 1) / q) * q;
}

// Rebuild the tiled operand rows of an operator (after append).  XA/XB hold
// round_up(n, 128) rows so every CTA tile and every 64-row j tile is in bounds.  fp16
// operands (3xF16 split of x / l) are used when the scaled coordinates stay well inside the
// fp16 range (|x|/l <= 64, |x|^2/l^2 <= 8192); tf32 (x itself) otherwise.
void tc_build_operands(Op& op, DBuf<float>& XA, DBuf<float>& XB, const double* center,
                       cudaStream_t st) {
  const double inv_l = 1.0 / op.lengthscale;
  bool f16 = false;
  static const int force_tf32 = getenv("WGP_TC_TF32_GEMM1") ? atoi(getenv("WGP_TC_TF32_GEMM1")) : 0;
  if (op.precision == WGP_F32_3XTF32 && !force_tf32) {
    DBuf<unsigned long long> ext(2);
    WGP_CUDA(cudaMemsetAsync(ext.p, 0, sizeof(unsigned long long) * 2, st));
    tc::scaled_extent_kernel<<<tc::grid_for(op.n), 256, 0, st>>>(op.X64.p, op.dpad, op.dim, center,
                                                                inv_l, op.n, ext.p);
    WGP_CUDA(cudaGetLastError());
    unsigned long long hb[2];
    WGP_CUDA(cudaMemcpyAsync(hb, ext.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    double h[2];
    std::memcpy(h, hb, sizeof(h));
    f16 = h[0] <= 64.0 && h[1] <= 8192.0;
  }
  op.tc_f16 = f16;
  const int K1 = tc_k1(op.dim, op.precision, f16);
  const int64_t npad = ((op.n + tc::BM - 1) / tc::BM) * tc::BM;
  const size_t bytes = (size_t)npad * K1 * (f16 ? 2 : 4);
  XA.ensure(bytes / 4);
  XB.ensure(bytes / 4);
  WGP_CUDA(cudaMemsetAsync(XA.p, 0, bytes, st));
  WGP_CUDA(cudaMemsetAsync(XB.p, 0, bytes, st));
  const int split = op.precision == WGP_TF32 ? 0 : 1;
  if (f16)
    tc::build_operands_kernel<__half><<<tc::grid_for(op.n), 256, 0, st>>>(
        op.X64.p, op.dpad, op.dim, center, inv_l, op.n, K1, split,
        reinterpret_cast<__half*>(XA.p), reinterpret_cast<__half*>(XB.p));
  else
    tc::build_operands_kernel<float><<<tc::grid_for(op.n), 256, 0, st>>>(
        op.X64.p, op.dpad, op.dim, center, 1.0, op.n, K1, split, XA.p, XB.p);
  WGP_CUDA(cudaGetLastError());
}

// XA operand rows for arbitrary points (cross mode K(X*, X)): the operator's centring,
// scale and element format.  Returns false when the points leave the fp16 range of an
// fp16-operand operator (the caller then uses the fp64 CUDA-core path).
bool tc_build_cross_rows(const Op& op, const double* Xs, int64_t m, int dpad, DBuf<float>& XAc,
                         cudaStream_t st) {
  const bool f16 = op.tc_f16;
  const double inv_l = 1.0 / op.lengthscale;
  if (f16) {
    DBuf<unsigned long long> ext(2);
    WGP_CUDA(cudaMemsetAsync(ext.p, 0, sizeof(unsigned long long) * 2, st));
    tc::scaled_extent_kernel<<<tc::grid_for(m), 256, 0, st>>>(Xs, dpad, op.dim, op.center.p, inv_l, m,
                                                             ext.p);
    WGP_CUDA(cudaGetLastError());
    unsigned long long hb[2];
    WGP_CUDA(cudaMemcpyAsync(hb, ext.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    double h[2];
    std::memcpy(h, hb, sizeof(h));
    if (!(h[0] <= 64.0 && h[1] <= 8192.0)) return false;
  }
  const int K1 = tc_k1(op.dim, op.precision, f16);
  const int64_t mpad = ((m + tc::BM - 1) / tc::BM) * tc::BM;
  const size_t bytes = (size_t)mpad * K1 * (f16 ? 2 : 4);
  XAc.ensure(bytes / 4);
  WGP_CUDA(cudaMemsetAsync(XAc.p, 0, bytes, st));
  const int split = op.precision == WGP_TF32 ? 0 : 1;
  if (f16)
    tc::build_operands_kernel<__half><<<tc::grid_for(m), 256, 0, st>>>(
        Xs, dpad, op.dim, op.center.p, inv_l, m, K1, split, reinterpret_cast<__half*>(XAc.p), nullptr);
  else
    tc::build_operands_kernel<float><<<tc::grid_for(m), 256, 0, st>>>(
        Xs, dpad, op.dim, op.center.p, 1.0, m, K1, split, XAc.p, nullptr);
  WGP_CUDA(cudaGetLastError());
  return true;
}

// Shared memory: XA rows + NSX XB stages + NSV V stages + 1 KB of barriers.  XB lives from
// its copy to GEMM1 (~1 tile period), V until GEMM2 after the map (~4 periods), so the V
// ring gets the space first: NSX = 3 (2 if tight), NSV up to 8.
size_t tc_smem_bytes(int K1, int esz, int s_pad, int* nsx_out, int* nsv_out, int bj = tc::BJ) {
  const size_t xa = (size_t)tc::BM * K1 * esz;
  const size_t xb = (size_t)bj * K1 * esz;
  const size_t vb = 2 * (size_t)s_pad * bj * 2;
  const size_t avail = 227 * 1024 - 1024 - xa;
  static const int want_x = getenv("WGP_TC_NSX") ? atoi(getenv("WGP_TC_NSX")) : 5;
  int nsx = want_x, nsv = 0;
  for (; nsx >= 2; --nsx) {
    if (avail < nsx * xb) continue;
    nsv = (int)std::min<size_t>(8, (avail - nsx * xb) / vb);
    if (nsv >= 5 || nsx == 2) break;
  }
  *nsx_out = nsx;
  *nsv_out = nsv;
  return xa + nsx * xb + nsv * vb + 1024;
}

bool tc_supported(int dim, int precision) {
  int nsx = 0, nsv = 0;
  tc_smem_bytes(tc_k1(dim, precision, false), 4, tc::MAX_SPAD, &nsx, &nsv);
  return nsx >= 2 && nsv >= 2;
}

// Y = (K(Xr, Xc) [+ sigma^2 I]) V, rows [row0, row0 + nrows) of the operator.  V64 and
// Y64/B64 are fp64 row-major; RHS chunks of <= 128 columns per launch.
void launch_kmatvec_tc(const Op& op, const float* XA_all, const float* XB, int64_t nrows,
                       int64_t row0, int64_t ncols, const double* V64, int s, const double* B64,
                       double* Y64, bool gram, DBuf<float>& vt_scratch, DBuf<double>& vchunk,
                       DBuf<double>& ychunk, DBuf<double>& ysplit, cudaStream_t st, int row_parts,
                       cudaEvent_t* part_done, int64_t col0, const double* C64, double sgn,
                       int noise_mode, const double* noiseV) {
  if (nrows <= 0 || s <= 0 || ncols <= 0) return;
  WGP_REQUIRE(noise_mode != 1 || (noiseV && s <= tc::MAX_SPAD), "kmatvec_tc: bad noise operand");
  const double* Cin = B64 ? B64 : C64;
  const double csgn = B64 ? -1.0 : sgn;
  // Row parts (one RHS chunk only): the V preparation is shared, each part's rows finish
  // with their own reduce and an event, so a caller can start moving finished rows (e.g.
  // the device-to-host copy of the host API) while the next part computes.
  if (s > tc::MAX_SPAD || nrows < 2 * tc::BM) row_parts = 1;
  row_parts = std::max(1, row_parts);
  const bool f16 = op.tc_f16;
  const int esz = f16 ? 2 : 4;
  const int K1 = tc_k1(op.dim, op.precision, f16);
  const void* XA_rows = reinterpret_cast<const char*>(XA_all) + (size_t)row0 * K1 * esz;
  const KParams kp = op.kp();
  for (int c0 = 0; c0 < s; c0 += tc::MAX_SPAD) {
    const int sc = std::min(tc::MAX_SPAD, s - c0);
    const double* Vc = V64;
    const double* Bc = Cin;
    double* Yc = Y64;
    if (sc != s) {  // gather this column chunk (s > 128)
      vchunk.ensure((size_t)ncols * sc);
      ychunk.ensure((size_t)nrows * sc * (Cin ? 2 : 1));
      WGP_CUDA(cudaMemcpy2DAsync(vchunk.p, sizeof(double) * sc, V64 + c0, sizeof(double) * s,
                                 sizeof(double) * sc, ncols, cudaMemcpyDeviceToDevice, st));
      if (Cin)
        WGP_CUDA(cudaMemcpy2DAsync(ychunk.p + (size_t)nrows * sc, sizeof(double) * sc, Cin + c0,
                                   sizeof(double) * s, sizeof(double) * sc, nrows,
                                   cudaMemcpyDeviceToDevice, st));
      Vc = vchunk.p;
      Bc = Cin ? ychunk.p + (size_t)nrows * sc : nullptr;
      Yc = ychunk.p;
    }
    const int s_pad = ((sc + 15) / 16) * 16;
    // 128-column tiles where the accumulators leave TMEM room for three 128-column buffers
    // (s_pad <= 32; every column range starts on a 128-row boundary of XB, and XB holds
    // round_up(n, 128) rows, so the last tile stays in bounds)
    static const int forced_bj = getenv("WGP_TC_BJ") ? atoi(getenv("WGP_TC_BJ")) : 0;
    int bj = forced_bj == 64 || forced_bj == 128 ? (s_pad <= 32 ? forced_bj : 64)
                                                  : (s_pad <= 32 ? 128 : 64);
    if (bj == 128) {  // (large dim: the 64-column pipeline when 128-column stages do not fit)
      int nx = 0, nv = 0;
      tc_smem_bytes(K1, esz, s_pad, &nx, &nv, 128);
      if (nx < 2 || nv < 3) bj = 64;
    }
    const int ntiles = (int)((ncols + bj - 1) / bj);
    const int64_t nsub = (int64_t)ntiles * (bj / tc::BJ);  // 64-column V sub-tiles
    // scratch: fp16 tiles (2 x s_pad x 64 halves per sub-tile) + 2 x s_pad scales (floats)
    const size_t vt_halves = (size_t)nsub * tc::BJ * s_pad * 2;
    // (+ the per-column max bits, 8-byte aligned, after the scales)
    const size_t vt_floats = ((vt_halves + 1) / 2 + 1) & ~(size_t)1;
    vt_scratch.ensure_grow(vt_floats + 2 * (size_t)s_pad + 64 + 2 * (size_t)tc::MAX_SPAD);
    __half* vt = reinterpret_cast<__half*>(vt_scratch.p);
    float* sc_up = vt_scratch.p + vt_floats + 32;
    float* sc_down = sc_up + s_pad;
    unsigned long long* cmax =
        reinterpret_cast<unsigned long long*>(vt_scratch.p + vt_floats + 64 + 2 * (size_t)s_pad);
    WGP_CUDA(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * sc, st));
    tc::colmax_kernel<<<ceil_div(ncols, 64), 256, 0, st>>>(Vc, ncols, sc, cmax);
    tc::colscale_finish_kernel<<<1, 128, 0, st>>>(cmax, sc, s_pad, sc_up, sc_down);
    tc::split_v_kernel<<<tc::grid_for(nsub * (tc::BJ / 8) * s_pad), 256, 0, st>>>(
        Vc, ncols, sc, s_pad, nsub * tc::BJ, sc_up, vt);
    WGP_CUDA(cudaGetLastError());
    tc::Params prm;
    prm.XA = XA_rows;
    prm.g1f16 = f16 ? 1 : 0;
    prm.XB = XB;
    prm.Vt = vt;
    prm.vscale = sc_down;
    prm.nrows = nrows;
    prm.row0 = row0;
    prm.ncols = ncols;
    prm.col0 = col0;
    prm.ntiles = ntiles;
    static const int forced_ch = getenv("WGP_TC_CH") ? atoi(getenv("WGP_TC_CH")) : 0;
    // (the same number of MMA instructions per chunk accumulator for either tile width)
    prm.ch = forced_ch > 0 ? forced_ch : tc::CH_DEFAULT * tc::BJ / bj;
    for (int part = 0; part < row_parts; ++part) {
    // rows [pa, pb) of this launch, part boundaries on 128-row CTA tiles
    const int64_t pa = row_part_begin(nrows, part, row_parts);
    const int64_t pb = row_part_begin(nrows, part + 1, row_parts);
    const int64_t nrows_p = pb - pa;
    if (nrows_p <= 0) {
      if (part_done) WGP_CUDA(cudaEventRecord(part_done[part], st));
      continue;
    }
    prm.XA = static_cast<const char*>(XA_rows) + (size_t)pa * K1 * esz;
    prm.nrows = nrows_p;
    prm.row0 = row0 + pa;
    const int row_ctas = (int)((nrows_p + tc::BM - 1) / tc::BM);
    static const int forced_splits = getenv("WGP_TC_SPLITS") ? atoi(getenv("WGP_TC_SPLITS")) : 0;
    const int nsplit = forced_splits > 0 ? forced_splits : tc::choose_splits(row_ctas, ntiles);
    prm.tiles_per_split = (ntiles + nsplit - 1) / nsplit;
    const int gy = (ntiles + prm.tiles_per_split - 1) / prm.tiles_per_split;
    ysplit.ensure_grow(((size_t)gy * nrows_p * s_pad + 1) / 2);  // fp32 partials in fp64 storage
    prm.Ypart = reinterpret_cast<float*>(ysplit.p);
    prm.s = sc;
    prm.s_pad = s_pad;
    prm.K1 = K1;
    prm.kind = kp.kind;
    // fp16 operands are in units of l: z = sqrt(3) r' (Matern), r'^2 / 2 (RBF)
    const double c1 = f16 ? (kp.kind == WGP_MATERN32 ? kp.c1 * op.lengthscale
                                                     : kp.c1 * op.lengthscale * op.lengthscale)
                          : kp.c1;
    prm.c1 = (float)c1;
    prm.neg_c_log2e = (float)(-c1 * 1.4426950408889634);
    prm.out_scale = kp.s2 * 0x1.0p-10;
    prm.noise2 = kp.noise2;
    prm.gram = gram ? 1 : 0;
    prm.trace = nullptr;
    static const char* trace_path = getenv("WGP_TC_TRACE");
    prm.cta_trace = nullptr;
    DBuf<unsigned long long> trace_buf;
    const size_t nctas = (size_t)row_ctas * gy;
    if (trace_path) {
      trace_buf.alloc((size_t)ntiles * tc::TRW + nctas * 4);
      WGP_CUDA(cudaMemsetAsync(trace_buf.p, 0, sizeof(unsigned long long) * (ntiles * tc::TRW + nctas * 4), st));
      prm.trace = trace_buf.p;
      prm.cta_trace = trace_buf.p + (size_t)ntiles * tc::TRW;
    }
    int nsx = 0, nsv = 0;
    const size_t smem = tc_smem_bytes(K1, esz, s_pad, &nsx, &nsv, bj);
    WGP_REQUIRE(nsx >= 2 && nsv >= 2, "kmatvec_tc: dim %d too large for the shared-memory pipeline",
                op.dim);
    auto kern = bj == 64 ? tc::kmatvec_tc_kernel<64> : tc::kmatvec_tc_kernel<128>;
    const int nthreads = tc::NTHREADS;
    WGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {
      TimedScope ts("kmatvec_tc", st);
      kern<<<dim3(row_ctas, gy), nthreads, smem, st>>>(prm, nsx, nsv);
    }
    WGP_CUDA(cudaGetLastError());
    {
      // sigma^2 V_i: from this launch's V rows (default), from the full V (noise_mode 1: a
      // column-range launch whose rows' V lies outside its columns), or not at all (0)
      const double* nv = noise_mode == 1 ? noiseV : Vc;
      const int64_t nrow0 = noise_mode == 1 ? row0 + pa : row0 + pa - col0;
      const int add_noise = gram && noise_mode != 0 ? 1 : 0;
      tc::reduce_splits_kernel<<<dim3((unsigned)((nrows_p + 31) / 32), (sc + 31) / 32), 256, 0, st>>>(
          reinterpret_cast<const float*>(ysplit.p), gy, nrows_p, row0 + pa, sc, s_pad, sc_down, prm.out_scale, nv,
          nrow0, Bc ? Bc + pa * sc : nullptr, csgn, kp.noise2, add_noise, Yc + pa * sc);
      WGP_CUDA(cudaGetLastError());
    }
    if (trace_path) {
      std::vector<unsigned long long> h((size_t)ntiles * tc::TRW + nctas * 4);
      WGP_CUDA(cudaMemcpyAsync(h.data(), trace_buf.p, sizeof(unsigned long long) * h.size(),
                               cudaMemcpyDeviceToHost, st));
      WGP_CUDA(cudaStreamSynchronize(st));
      if (FILE* f = fopen(trace_path, "w")) {
        fprintf(f, "tile,g1_issue,g2_issue,epi_wait_s,epi_s_ready,epi_wait_k,epi_done,prod_issue,epi_ld_done,v_issue,g2_vready,g2_issued,done_q3,g2_committed,g2_yfree_ok\n");
        for (int t = 0; t < ntiles; ++t)
        {
          fprintf(f, "%d", t);
          for (int k = 0; k < tc::TRW; ++k) fprintf(f, ",%llu", h[(size_t)t * tc::TRW + k]);
          fprintf(f, "\n");
        }
        fclose(f);
      }
      if (FILE* f = fopen((std::string(trace_path) + ".ctas").c_str(), "w")) {
        fprintf(f, "cta_x,cta_y,start_ns,loop_end_ns,end_ns,smid\n");
        const unsigned long long* c = h.data() + (size_t)ntiles * tc::TRW;
        for (size_t i = 0; i < nctas; ++i)
          fprintf(f, "%zu,%zu,%llu,%llu,%llu,%llu\n", i % row_ctas, i / row_ctas, c[i * 4], c[i * 4 + 1],
                  c[i * 4 + 2], c[i * 4 + 3]);
        fclose(f);
      }
    }
      if (part_done) WGP_CUDA(cudaEventRecord(part_done[part], st));
    }  // row parts
    if (sc != s) {
      WGP_CUDA(cudaMemcpy2DAsync(Y64 + c0, sizeof(double) * s, Yc, sizeof(double) * sc,
                                 sizeof(double) * sc, nrows, cudaMemcpyDeviceToDevice, st));
    }
  }
}

}  // namespace wgp
