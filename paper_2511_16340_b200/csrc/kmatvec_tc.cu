// kmatvec_tc.cu -- tcgen05 (5th-gen tensor core) fused kernel-matvec for sm_100a.
//
//   Y[i, :] = sum_j k(x_i, x_j) V[j, :] + sigma_n^2 V[i, :]      (gram, H = K + sigma_n^2 I)
//
// restating gram_matrix (kernel.cpp:48-72) + H*p (solvers.cpp:162) without materialising
// K.  One CTA owns 128 rows i and streams all columns j in tiles of 64:
//
//   GEMM1  S = XA_i . XB_j^T      (M=128, N=64, K=K1)  tcgen05.mma kind::tf32, SS, S in TMEM.
//          The operands are pre-formatted so the contraction yields the squared distance
//          directly (the norm form |x|^2 + |y|^2 - 2 x.y of kernel.cpp:39-46, 65):
//            XA = [-2xh | -2xh | -2xl | sqh | sql | 1 | 1]   XB = [xh | xl | xh | 1 | 1 | sqh | sql]
//          (3xTF32: hi/lo splits of x and |x|^2, error ~2^-22 of the largest term).
//   map    epilogue warps: tcgen05.ld S -> k(d2)/s^2 * 2^10 in registers (Matern-3/2 or RBF;
//          MUFU sqrt/ex2) -> fp16 hi/lo split -> tcgen05.st into TMEM (K never leaves the SM).
//   GEMM2  Y += K_hi V_hi + K_hi V_lo + K_lo V_hi   (M=128, N=s_pad, K=64)  kind::f16, A from
//          TMEM (TS form), fp32 accumulator in TMEM for the whole j sweep.  V is pre-split
//          into fp16 hi/lo with a per-column power-of-two scale (3xFP16 ~ 2^-22 relative).
//   out    Y * s^2 / (2^10 * scale_c) + sigma_n^2 V_i in fp64 (or B - that: the true residual
//          of solvers.cpp:171) written as fp64.
//
// Warp roles (20 warps): 0 = bulk-copy producer (TMA engine, UBLKCP), 1 = GEMM1 issuer,
// 3 = GEMM2 issuer (whole warps run the schedules, one elected lane issues), 2 = TMEM
// allocator, 4..19 = epilogue:
// two sets of 8 warps taking alternate j tiles (2 warps per TMEM lane quadrant, 32 columns
// each).  Pipelines: smem stages (XB_j, V_j hi/lo) x NS; a ring of 6-7 TMEM tile buffers
// (S written by GEMM1, overwritten in place by K for GEMM2); mbarriers + tcgen05.commit.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace wgp {
namespace tc {

constexpr int BM = 128;        // rows per CTA (UMMA M)
constexpr int BJ = 64;         // columns j per tile (GEMM1 N, GEMM2 K)
constexpr int NTHREADS = 640;  // 4 role warps + 2 epilogue sets x 8 warps
constexpr int MAX_SPAD = 64;   // RHS columns per launch (wider RHS: column chunks)
constexpr int CH = 16;         // j tiles per TMEM accumulation chunk (fp64 drain after each)
// TMEM: a ring of NB 64-column tile buffers followed by the Y accumulator.  A buffer holds
// S(t) (fp32 d^2, written by GEMM1); the epilogue loads it into registers and writes K(t)
// back in place as packed fp16 (each warp into the 32 columns it read: 16 hi + 16 lo), which
// GEMM2 then reads as its A operand; GEMM2's commit frees the buffer for GEMM1 of tile
// t + NB.  Two 64-column Y accumulators alternate per chunk of CH tiles: the tensor core's
// fp32 accumulation error grows with the number of accumulated K-steps (measured 3.5e-4 at
// N = 101k in one accumulator), so every CH tiles the epilogue warps drain the finished
// accumulator into fp64 partial sums in shared memory (~4e-6 per chunk, summed in fp64).
// TMEM: NB = 6 buffers [0,384), Y0 [384,448), Y1 [448,512).
constexpr int MAX_NB = 6;
constexpr float KSCALE_LOG2 = 10.0f;  // K stored as k/s^2 * 2^10 (fp16 normal range)

struct Params {
  const float* XA;      // tiled A operand rows (this launch's rows start at tile 0)
  const float* XB;      // tiled B operand rows (all columns j)
  const __half* Vt;     // tiled V hi/lo per j tile (fp16, per-column scaled)
  const float* vscale;  // [s_pad] 2^-e_c: undo the per-column V scale
  const double* V64;    // [ncols][s] for the sigma^2 V_i term (gram) -- indexed by global row
  const double* B64;    // nullable: residual mode, [nrows][s]
  double* Y64;          // [nrows][s]
  int64_t nrows, row0, ncols;
  int ntiles;           // ceil(ncols / BJ)
  int tiles_per_split;  // j tiles per CTA along grid.y (2-D decomposition)
  double* Ysplit;       // nullptr: full output; else fp64 partials [gridDim.y][nrows][s]
  int s, s_pad, K1;
  int kind;
  float c1, neg_c_log2e;
  double out_scale;     // s^2 * 2^-10
  double noise2;
  int gram;
  unsigned long long* trace;  // debug: per-tile event clocks of CTA 0 (nullptr normally)
};

__device__ __forceinline__ void trace_ev(const Params& p, int t, int slot) {
  if (p.trace && blockIdx.x == 0 && blockIdx.y == 0) p.trace[(size_t)t * 8 + slot] = clock64();
}

__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

__device__ __forceinline__ uint32_t pack_h2(float lo_elem, float hi_elem) {
  const __half2 h = __floats2half2_rn(lo_elem, hi_elem);  // .x (low 16 bits) = lower k index
  return *reinterpret_cast<const uint32_t*>(&h);
}

__global__ void __launch_bounds__(NTHREADS, 1) kmatvec_tc_kernel(const Params p, int NS) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t XA_BYTES = BM * p.K1 * 4;
  const uint32_t XB_BYTES = BJ * p.K1 * 4;
  const uint32_t VT_BYTES = p.s_pad * BJ * 2;  // one of hi / lo (fp16)
  const uint32_t ST_BYTES = XB_BYTES + 2 * VT_BYTES;
  unsigned char* sXA = smem;
  unsigned char* sStage = smem + XA_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + (size_t)NS * ST_BYTES);
  uint64_t* stage_full = bars;
  uint64_t* stage_empty = bars + NS;
  uint64_t* xa_full = bars + 2 * NS;
  uint64_t* s_full = xa_full + 1;        // [MAX_NB] GEMM1 -> epilogue
  uint64_t* k_full = s_full + MAX_NB;    // [MAX_NB] epilogue -> GEMM2 (8 arrivals)
  uint64_t* b_free = k_full + MAX_NB;    // [MAX_NB] GEMM2 -> GEMM1
  uint64_t* y_full = b_free + MAX_NB;    // [2] chunk accumulator done (GEMM2 commit)
  uint64_t* y_free = y_full + 2;         // [2] chunk accumulator drained (16 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(y_free + 2);
  double* ypart = reinterpret_cast<double*>(smem + (size_t)(XA_BYTES + NS * ST_BYTES + 512));
  constexpr int NB = MAX_NB;
  constexpr uint32_t TM_Y = 384;         // Y accumulator a at TM_Y + 64 a
  // this CTA's j range: tiles [jt0, jt0 + T) of the column sweep
  const int jt0 = blockIdx.y * p.tiles_per_split;
  const int T = min(p.ntiles - jt0, p.tiles_per_split);
  const int NCH = (T + CH - 1) / CH;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&stage_full[i], 1);
      ptx::mbar_init(&stage_empty[i], 1);
    }
    ptx::mbar_init(xa_full, 1);
    for (int i = 0; i < MAX_NB; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&k_full[i], 8);
      ptx::mbar_init(&b_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&y_full[i], 1);
      ptx::mbar_init(&y_free[i], 16);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  for (int e = threadIdx.x; e < BM * p.s_pad; e += NTHREADS) ypart[e] = 0.0;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KS1 = p.K1 / 8;                 // GEMM1 K-steps (tf32: 8 per instruction)
  const uint32_t sbo1 = (p.K1 / 4) * 128;   // 8-row group stride of XA/XB tiles

  if (warp == 0) {
    // ------------------------------------------------------------ producer (TMA engine)
    const bool leader = ptx::elect_one();
    if (leader) {
      ptx::mbar_arrive_expect_tx(xa_full, XA_BYTES);
      ptx::bulk_g2s(sXA, p.XA + (size_t)blockIdx.x * BM * p.K1, XA_BYTES, xa_full);
    }
    int st = 0;
    uint32_t ph = 0;
    const float* xb_src = p.XB + (size_t)jt0 * BJ * p.K1;
    const __half* vt_src = p.Vt + (size_t)jt0 * 2 * p.s_pad * BJ;
    for (int t = 0; t < T; ++t) {
      if (t >= NS) ptx::mbar_wait(&stage_empty[st], ph ^ 1);
      if (leader) {
        trace_ev(p, t, 6);
        unsigned char* dst = sStage + (size_t)st * ST_BYTES;
        ptx::mbar_arrive_expect_tx(&stage_full[st], ST_BYTES);
        ptx::bulk_g2s(dst, xb_src, XB_BYTES, &stage_full[st]);
        ptx::bulk_g2s(dst + XB_BYTES, vt_src, 2 * VT_BYTES, &stage_full[st]);
      }
      __syncwarp();
      xb_src += (size_t)BJ * p.K1;
      vt_src += (size_t)2 * p.s_pad * BJ;
      if (++st == NS) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers
    // tcgen05.mma issue blocks for about the instruction's execution time, so one thread
    // cannot keep two dependent streams fed.  Warp 1 issues GEMM1 (distance tiles) and warp 3
    // issues GEMM2 (K.V); each waits only on its own inputs and each tcgen05.commit tracks
    // its own thread's MMAs.  Whole warps run the schedule (uniform control flow,
    // descriptors in uniform registers); one elected lane issues.
    const uint64_t st_step = (uint64_t)(ST_BYTES >> 4);  // descriptor start-address units
    if (warp == 1) {
      const uint32_t idesc1 = ptx::idesc_tf32(BM, BJ);
      const uint64_t dXA = ptx::umma_desc(ptx::smem_u32(sXA), 128, sbo1);
      const uint64_t dStage0 = ptx::umma_desc(ptx::smem_u32(sStage), 128, sbo1);
      ptx::mbar_wait(xa_full, 0);
      int st1 = 0, b1 = 0;
      uint32_t ph1 = 0, phb1 = 0;
      for (int t = 0; t < T; ++t) {
        ptx::mbar_wait(&stage_full[st1], ph1);
        if (t >= NB) ptx::mbar_wait(&b_free[b1], phb1 ^ 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          trace_ev(p, t, 0);
          const uint64_t dB = dStage0 + st_step * st1;
          for (int ks = 0; ks < KS1; ++ks)
            ptx::mma_tf32_ss(tmem + b1 * 64, dXA + 16 * ks, dB + 16 * ks, idesc1, ks > 0 ? 1u : 0u);
          ptx::mma_commit(&s_full[b1]);
        }
        __syncwarp();
        if (++st1 == NS) { st1 = 0; ph1 ^= 1; }
        if (++b1 == NB) { b1 = 0; phb1 ^= 1; }
      }
    } else {
      const uint32_t idesc2 = ptx::idesc_f16(BM, p.s_pad);
      // fp16 V tile: rows c (N) in 8-row groups, K = 64 j in 8-element (16 B) chunks
      const uint64_t dV0 = ptx::umma_desc(ptx::smem_u32(sStage + XB_BYTES), 128, (BJ / 8) * 128);
      const uint64_t vlo_step = (uint64_t)(VT_BYTES >> 4);
      int st2 = 0, b2 = 0;
      uint32_t phb2 = 0;
      for (int t = 0; t < T; ++t) {
        const int c = t / CH, ya = c & 1;
        const bool first = t == c * CH, last = t == T - 1 || t == c * CH + CH - 1;
        if (first && c >= 2) ptx::mbar_wait(&y_free[ya], ((c >> 1) - 1) & 1);
        ptx::mbar_wait(&k_full[b2], phb2);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          trace_ev(p, t, 1);
          const uint64_t dVh = dV0 + st_step * st2;
          const uint64_t dVl = dVh + vlo_step;
          const uint32_t yacc = tmem + TM_Y + ya * 64;
          // K layout in the buffer: [hi j0-31 | lo j0-31 | hi j32-63 | lo j32-63], 16 cols each
          const uint32_t kb = tmem + b2 * 64;
#pragma unroll
          for (int ks = 0; ks < BJ / 16; ++ks) {
            const uint32_t hcol = kb + (ks >> 1) * 32 + (ks & 1) * 8;
            ptx::mma_f16_ts(yacc, hcol, dVh + 16 * ks, idesc2, (!first || ks > 0) ? 1u : 0u);
          }
#pragma unroll
          for (int ks = 0; ks < BJ / 16; ++ks) {
            const uint32_t hcol = kb + (ks >> 1) * 32 + (ks & 1) * 8;
            ptx::mma_f16_ts(yacc, hcol, dVl + 16 * ks, idesc2, 1u);
          }
#pragma unroll
          for (int ks = 0; ks < BJ / 16; ++ks) {
            const uint32_t lcol = kb + (ks >> 1) * 32 + 16 + (ks & 1) * 8;
            ptx::mma_f16_ts(yacc, lcol, dVh + 16 * ks, idesc2, 1u);
          }
          ptx::mma_commit(&b_free[b2]);
          ptx::mma_commit(&stage_empty[st2]);
          if (last) ptx::mma_commit(&y_full[ya]);
        }
        __syncwarp();
        if (++st2 == NS) st2 = 0;
        if (++b2 == NB) { b2 = 0; phb2 ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ kernel-map epilogue
    const int q = warp & 3;                   // TMEM lane quadrant accessible to this warp
    const int g = (warp - 4) >> 2;            // 0..3
    const int set = g >> 1, half = g & 1;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int r = q * 32 + lane;              // row within the CTA tile
    const int64_t gi = p.row0 + (int64_t)blockIdx.x * BM + r;
    const int64_t grow0 = p.row0 + (int64_t)blockIdx.x * BM;
    const float kdiag = 1024.0f;              // k(x,x)/s^2 * 2^10
    // drain share of this warp: its quadrant's 32 rows x 16 accumulator columns
    const int dc0 = g * 16;
    int drained = 0;
    auto drain = [&](int c) {
      const int ya = c & 1;
      ptx::mbar_wait(&y_full[ya], (c >> 1) & 1);
      ptx::tc_fence_after();
      if (dc0 < p.s_pad) {
        uint32_t y[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15}, [%16];"
            : "=r"(y[0]), "=r"(y[1]), "=r"(y[2]), "=r"(y[3]), "=r"(y[4]), "=r"(y[5]), "=r"(y[6]),
              "=r"(y[7]), "=r"(y[8]), "=r"(y[9]), "=r"(y[10]), "=r"(y[11]), "=r"(y[12]),
              "=r"(y[13]), "=r"(y[14]), "=r"(y[15])
            : "r"(tmem + lane_off + TM_Y + ya * 64 + dc0));
        ptx::tmem_wait_ld();
        // column-major partials: lanes (rows) hit consecutive 8-byte words (no bank conflicts)
        double* colp = ypart + (size_t)dc0 * BM + r;
#pragma unroll
        for (int k = 0; k < 16; ++k) colp[(size_t)k * BM] += (double)__uint_as_float(y[k]);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&y_free[ya]);
    };
    int b = set;                              // buffer of tile t = t % NB
    uint32_t bph = 0;
    for (int t = set; t < T; t += 2) {
      // drain a finished chunk once this warp is well past its last tile
      while (drained < NCH - 1 && t >= (drained + 1) * CH + CH / 2) drain(drained++);
      const bool tr = lane == 0 && q == 0 && half == 0;
      if (tr) trace_ev(p, t, 2);
      ptx::mbar_wait(&s_full[b], bph);
      ptx::tc_fence_after();
      if (tr) trace_ev(p, t, 3);
      const uint32_t col = tmem + lane_off + b * 64 + half * 32;
      uint32_t v[32];
      ptx::tmem_ld32(col, v);
      ptx::tmem_wait_ld();
      float kv[32];
      if (p.kind == WGP_MATERN32) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float d2 = fmaxf(__uint_as_float(v[c]), 0.0f);
          const float rr = ptx::sqrt_approx(d2);
          const float e = ptx::ex2_approx(fmaf(rr, p.neg_c_log2e, KSCALE_LOG2));  // 2^10 e^{-z}
          const float z = rr * p.c1;
          kv[c] = fmaf(z, e, e);  // 2^10 (1+z) e^{-z}
        }
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float d2 = fmaxf(__uint_as_float(v[c]), 0.0f);
          kv[c] = ptx::ex2_approx(fmaf(d2, p.neg_c_log2e, KSCALE_LOG2));  // 2^10 e^{-d2/2l^2}
        }
      }
      const int64_t gj0 = (int64_t)(jt0 + t) * BJ + half * 32;
      if (p.gram && gj0 < grow0 + BM && gj0 + 32 > grow0) {  // tile touches the diagonal
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (gj0 + c == gi) kv[c] = kdiag;  // k(x,x) = s^2 exactly
      }
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        hi[c] = pack_h2(kv[2 * c], kv[2 * c + 1]);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hi[c]));
        lo[c] = pack_h2(kv[2 * c] - hf.x, kv[2 * c + 1] - hf.y);
      }
      if (tr) trace_ev(p, t, 4);
      // K back into the columns this warp read: [hi 16 | lo 16]
      ptx::tmem_st16(col, hi);
      ptx::tmem_st16(col + 16, lo);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&k_full[b]);
      if (tr) trace_ev(p, t, 5);
      b += 2;  // tile t + 2 -> buffer (t + 2) % NB, phase ((t + 2) / NB) & 1
      if (b >= NB) { b -= NB; bph ^= 1; }
    }
    // ------------------------------------------------------------ output
    while (drained < NCH) drain(drained++);
    const int64_t lr = (int64_t)blockIdx.x * BM + r;  // local output row
    if (lr < p.nrows && dc0 < p.s) {
      const int64_t base = lr * p.s;
      if (p.Ysplit) {  // partial over this CTA's j range; reduce_splits adds the rest
        double* dst = p.Ysplit + (size_t)blockIdx.y * p.nrows * p.s + base;
        for (int col = dc0; col < dc0 + 16 && col < p.s; ++col)
          dst[col] = ypart[(size_t)col * BM + r] * (p.out_scale * (double)p.vscale[col]);
      } else {
        for (int col = dc0; col < dc0 + 16 && col < p.s; ++col) {
          double acc = ypart[(size_t)col * BM + r] * (p.out_scale * (double)p.vscale[col]);
          if (p.gram) acc += p.noise2 * p.V64[gi * p.s + col];
          p.Y64[base + col] = p.B64 ? p.B64[base + col] - acc : acc;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// XA / XB operand rows in the tiled K-major "interleave" layout
// [row/8][k/4][row%8][k%4], from the centered fp64 rows.
__global__ void build_operands_kernel(const double* __restrict__ X, int dpad, int dim,
                                      const double* __restrict__ center, int64_t n, int K1,
                                      float* __restrict__ XA, float* __restrict__ XB) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i >> 3, ri = i & 7;
    auto at = [&](int k) -> int64_t { return ((g * (K1 / 4) + k / 4) * 8 + ri) * 4 + (k & 3); };
    double sq = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double x = X[i * dpad + k] - center[k];
      sq += x * x;
      const float xf = (float)x;
      const float xh = __uint_as_float(tf32_hi(xf));
      const float xl = (float)(x - (double)xh);
      XA[at(k)] = -2.0f * xh;
      XA[at(dim + k)] = -2.0f * xh;
      XA[at(2 * dim + k)] = -2.0f * xl;
      XB[at(k)] = xh;
      XB[at(dim + k)] = xl;
      XB[at(2 * dim + k)] = xh;
    }
    const float sqh = __uint_as_float(tf32_hi((float)sq));
    const float sql = (float)(sq - (double)sqh);
    const int b = 3 * dim;
    XA[at(b)] = sqh;
    XA[at(b + 1)] = sql;
    XA[at(b + 2)] = 1.0f;
    XA[at(b + 3)] = 1.0f;
    XB[at(b)] = 1.0f;
    XB[at(b + 1)] = 1.0f;
    XB[at(b + 2)] = sqh;
    XB[at(b + 3)] = sql;
    for (int k = b + 4; k < K1; ++k) {
      XA[at(k)] = 0.0f;
      XB[at(k)] = 0.0f;
    }
  }
}

// Per-column max |V| (one block per column) -> power-of-two scales 2^e_c, 2^-e_c with
// |V * 2^e_c| < 2^14 for the fp16 split.
__global__ void colscale_kernel(const double* __restrict__ V, int64_t n, int s, int s_pad,
                                float* __restrict__ scale_up, float* __restrict__ scale_down) {
  const int c = blockIdx.x;
  if (c >= s_pad) return;
  double m = 0.0;
  if (c < s)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, fabs(V[j * s + c]));
  __shared__ double red[256];
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int e = 0;
    if (red[0] > 0.0) {
      int ex;
      frexp(red[0], &ex);  // red = f * 2^ex, f in [0.5, 1)
      e = 14 - ex;         // |V| * 2^e < 2^14
      e = max(-100, min(100, e));
    }
    scale_up[c] = ldexpf(1.0f, e);
    scale_down[c] = ldexpf(1.0f, -e);
  }
}

// V [ncols][s] fp64 -> per-64-row tile [hi|lo][s_pad/8][8 chunks][8 c][8 j] fp16.
__global__ void split_v_kernel(const double* __restrict__ V, int64_t ncols, int s, int s_pad,
                               int64_t total_rows, const float* __restrict__ scale_up,
                               __half* __restrict__ Vt) {
  const int64_t total = total_rows * s_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / s_pad;
    const int c = (int)(e % s_pad);
    const double v = (j < ncols && c < s) ? V[j * s + c] * (double)scale_up[c] : 0.0;
    const __half vh = __double2half(v);
    const __half vl = __double2half(v - (double)__half2float(vh));
    const int64_t t = j / BJ;
    const int jj = (int)(j % BJ);
    const int64_t idx = ((int64_t)((c >> 3) * (BJ / 8) + (jj >> 3)) * 8 + (c & 7)) * 8 + (jj & 7);
    __half* base = Vt + t * 2 * (int64_t)s_pad * BJ;
    base[idx] = vh;
    base[(int64_t)s_pad * BJ + idx] = vl;
  }
}

// Y = sum over j-splits (fixed order) + sigma^2 V_i (gram), or B - that.
__global__ void reduce_splits_kernel(const double* __restrict__ Ysplit, int nsplit, int64_t nrows,
                                     int64_t row0, int s, const double* __restrict__ V64,
                                     const double* __restrict__ B64, double noise2, int gram,
                                     double* __restrict__ Y64) {
  const int64_t total = nrows * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < nsplit; ++q) acc += Ysplit[(size_t)q * total + e];
    if (gram) acc += noise2 * V64[row0 * s + e];
    Y64[e] = B64 ? B64[e] - acc : acc;
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

int tc_k1(int dim) { return ((3 * dim + 4 + 7) / 8) * 8; }

// Rebuild the tiled operand rows of an operator (after append).  XA/XB hold
// round_up(n, 128) rows so every CTA tile and every 64-row j tile is in bounds.
void tc_build_operands(const Op& op, DBuf<float>& XA, DBuf<float>& XB, const double* center,
                       cudaStream_t st) {
  const int K1 = tc_k1(op.dim);
  const int64_t npad = ((op.n + tc::BM - 1) / tc::BM) * tc::BM;
  XA.ensure((size_t)npad * K1);
  XB.ensure((size_t)npad * K1);
  WGP_CUDA(cudaMemsetAsync(XA.p, 0, sizeof(float) * npad * K1, st));
  WGP_CUDA(cudaMemsetAsync(XB.p, 0, sizeof(float) * npad * K1, st));
  tc::build_operands_kernel<<<tc::grid_for(op.n), 256, 0, st>>>(op.X64.p, op.dpad, op.dim, center,
                                                                op.n, K1, XA.p, XB.p);
  WGP_CUDA(cudaGetLastError());
}

size_t tc_smem_bytes(int K1, int s_pad, int* ns_out) {
  const size_t xa = (size_t)tc::BM * K1 * 4;
  const size_t stage = (size_t)tc::BJ * K1 * 4 + 2 * (size_t)s_pad * tc::BJ * 2;
  const size_t tail = 512 + (size_t)tc::BM * s_pad * 8;  // barriers + fp64 partial Y
  int ns = (int)((227 * 1024 - xa - tail) / stage);
  if (ns > 6) ns = 6;
  *ns_out = ns;
  return xa + ns * stage + tail;
}

bool tc_supported(int dim) {
  int ns = 0;
  tc_smem_bytes(tc_k1(dim), tc::MAX_SPAD, &ns);
  return ns >= 2;
}

// Y = (K(Xr, Xc) [+ sigma^2 I]) V, rows [row0, row0 + nrows) of the operator.  V64 and
// Y64/B64 are fp64 row-major; RHS chunks of <= 128 columns per launch.
void launch_kmatvec_tc(const Op& op, const float* XA_rows, const float* XB, int64_t nrows,
                       int64_t row0, int64_t ncols, const double* V64, int s, const double* B64,
                       double* Y64, bool gram, DBuf<float>& vt_scratch, DBuf<double>& vchunk,
                       DBuf<double>& ychunk, DBuf<double>& ysplit, cudaStream_t st) {
  if (nrows <= 0 || s <= 0) return;
  const int K1 = tc_k1(op.dim);
  const KParams kp = op.kp();
  for (int c0 = 0; c0 < s; c0 += tc::MAX_SPAD) {
    const int sc = std::min(tc::MAX_SPAD, s - c0);
    const double* Vc = V64;
    const double* Bc = B64;
    double* Yc = Y64;
    if (sc != s) {  // gather this column chunk (s > 128)
      vchunk.ensure((size_t)ncols * sc);
      ychunk.ensure((size_t)nrows * sc * (B64 ? 2 : 1));
      WGP_CUDA(cudaMemcpy2DAsync(vchunk.p, sizeof(double) * sc, V64 + c0, sizeof(double) * s,
                                 sizeof(double) * sc, ncols, cudaMemcpyDeviceToDevice, st));
      if (B64)
        WGP_CUDA(cudaMemcpy2DAsync(ychunk.p + (size_t)nrows * sc, sizeof(double) * sc, B64 + c0,
                                   sizeof(double) * s, sizeof(double) * sc, nrows,
                                   cudaMemcpyDeviceToDevice, st));
      Vc = vchunk.p;
      Bc = B64 ? ychunk.p + (size_t)nrows * sc : nullptr;
      Yc = ychunk.p;
    }
    const int s_pad = ((sc + 15) / 16) * 16;
    const int ntiles = (int)((ncols + tc::BJ - 1) / tc::BJ);
    // scratch: fp16 tiles (2 x s_pad x 64 halves per tile) + 2 x s_pad scales (floats)
    const size_t vt_halves = (size_t)ntiles * tc::BJ * s_pad * 2;
    vt_scratch.ensure((vt_halves + 1) / 2 + 2 * (size_t)s_pad + 64);
    __half* vt = reinterpret_cast<__half*>(vt_scratch.p);
    float* sc_up = vt_scratch.p + (vt_halves + 1) / 2 + 32;
    float* sc_down = sc_up + s_pad;
    tc::colscale_kernel<<<s_pad, 256, 0, st>>>(Vc, ncols, sc, s_pad, sc_up, sc_down);
    tc::split_v_kernel<<<tc::grid_for((int64_t)ntiles * tc::BJ * s_pad), 256, 0, st>>>(
        Vc, ncols, sc, s_pad, (int64_t)ntiles * tc::BJ, sc_up, vt);
    WGP_CUDA(cudaGetLastError());
    tc::Params prm;
    prm.XA = XA_rows;
    prm.XB = XB;
    prm.Vt = vt;
    prm.vscale = sc_down;
    prm.V64 = Vc;
    prm.B64 = Bc;
    prm.Y64 = Yc;
    prm.nrows = nrows;
    prm.row0 = row0;
    prm.ncols = ncols;
    prm.ntiles = ntiles;
    const int row_ctas = (int)((nrows + tc::BM - 1) / tc::BM);
    static const int forced_splits = getenv("WGP_TC_SPLITS") ? atoi(getenv("WGP_TC_SPLITS")) : 0;
    const int nsplit = forced_splits > 0 ? forced_splits : tc::choose_splits(row_ctas, ntiles);
    prm.tiles_per_split = (ntiles + nsplit - 1) / nsplit;
    const int gy = (ntiles + prm.tiles_per_split - 1) / prm.tiles_per_split;
    prm.Ysplit = nullptr;
    if (gy > 1) {
      ysplit.ensure((size_t)gy * nrows * sc);
      prm.Ysplit = ysplit.p;
    }
    prm.s = sc;
    prm.s_pad = s_pad;
    prm.K1 = K1;
    prm.kind = kp.kind;
    prm.c1 = (float)kp.c1;
    prm.neg_c_log2e = (float)(-kp.c1 * 1.4426950408889634);
    prm.out_scale = kp.s2 * 0x1.0p-10;
    prm.noise2 = kp.noise2;
    prm.gram = gram ? 1 : 0;
    prm.trace = nullptr;
    static const char* trace_path = getenv("WGP_TC_TRACE");
    DBuf<unsigned long long> trace_buf;
    if (trace_path) {
      trace_buf.alloc((size_t)ntiles * 8);
      WGP_CUDA(cudaMemsetAsync(trace_buf.p, 0, sizeof(unsigned long long) * ntiles * 8, st));
      prm.trace = trace_buf.p;
    }
    int ns = 0;
    const size_t smem = tc_smem_bytes(K1, s_pad, &ns);
    WGP_REQUIRE(ns >= 2, "kmatvec_tc: dim %d too large for the shared-memory pipeline", op.dim);
    WGP_CUDA(cudaFuncSetAttribute(tc::kmatvec_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    tc::kmatvec_tc_kernel<<<dim3(row_ctas, gy), tc::NTHREADS, smem, st>>>(prm, ns);
    WGP_CUDA(cudaGetLastError());
    if (gy > 1) {
      tc::reduce_splits_kernel<<<tc::grid_for(nrows * sc), 256, 0, st>>>(
          ysplit.p, gy, nrows, row0, sc, Vc, Bc, kp.noise2, gram ? 1 : 0, Yc);
      WGP_CUDA(cudaGetLastError());
    }
    if (trace_path) {
      std::vector<unsigned long long> h((size_t)ntiles * 8);
      WGP_CUDA(cudaMemcpyAsync(h.data(), trace_buf.p, sizeof(unsigned long long) * h.size(),
                               cudaMemcpyDeviceToHost, st));
      WGP_CUDA(cudaStreamSynchronize(st));
      if (FILE* f = fopen(trace_path, "w")) {
        fprintf(f, "tile,g1_issue,g2_issue,epi_wait_s,epi_s_ready,epi_wait_k,epi_done,prod_issue\n");
        for (int t = 0; t < ntiles; ++t)
          fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu,%llu\n", t, h[t * 8], h[t * 8 + 1], h[t * 8 + 2],
                  h[t * 8 + 3], h[t * 8 + 4], h[t * 8 + 5], h[t * 8 + 6]);
        fclose(f);
      }
    }
    if (sc != s) {
      WGP_CUDA(cudaMemcpy2DAsync(Y64 + c0, sizeof(double) * s, Yc, sizeof(double) * sc,
                                 sizeof(double) * sc, nrows, cudaMemcpyDeviceToDevice, st));
    }
  }
}

}  // namespace wgp
