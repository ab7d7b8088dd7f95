// kmatvec_tc.cu -- tcgen05 (5th-gen tensor core) fused kernel-matvec for sm_100a.
//
//   Y[i, :] = sum_j k(x_i, x_j) V[j, :] + sigma_n^2 V[i, :]      (gram, H = K + sigma_n^2 I)
//
// restating gram_matrix (kernel.cpp:48-72) + H*p (solvers.cpp:162) without materialising
// K.  One CTA owns 128 rows i and streams all columns j in tiles of 64:
//
//   GEMM1  S = XA_i . XB_j^T      (M=128, N=64,  K=K1)  tcgen05.mma kind::tf32, SS, S in TMEM
//          The operands are pre-formatted so the contraction yields the squared distance
//          directly (the norm form |x|^2 + |y|^2 - 2 x.y of kernel.cpp:39-46, 65):
//            XA = [-2xh | -2xh | -2xl | sqh | sql | 1 | 1]   XB = [xh | xl | xh | 1 | 1 | sqh | sql]
//          (3xTF32: hi/lo splits of x and |x|^2, error ~2^-22 of the largest term).
//   map    epilogue warps: tcgen05.ld S -> k(d2) in registers (Matern-3/2 or RBF, MUFU
//          sqrt/ex2) -> hi/lo TF32 split -> tcgen05.st into TMEM (K never leaves the SM).
//   GEMM2  Y += K_hi V_hi + K_hi V_lo + K_lo V_hi   (M=128, N=s_pad, K=64)  kind::tf32, A from
//          TMEM (TS form), accumulator in TMEM for the whole j sweep.
//   out    Y (fp32 accumulators) + sigma_n^2 V_i in fp64 (or B - that: the true residual of
//          solvers.cpp:171) written as fp64.
//
// Warp roles (12 warps): 0 = bulk-copy producer (TMA engine, UBLKCP), 1 = MMA issuer (one
// thread), 2 = TMEM allocator, 4..11 = kernel-map / output epilogue (two warps per TMEM
// lane quadrant, 32 columns each).  Pipelines: smem stages (XB_j, V_j hi/lo) x NS,
// S double buffer, K double buffer; all synchronised with mbarriers and tcgen05.commit.
#include "common.cuh"
#include "ptx.cuh"

namespace wgp {
namespace tc {

constexpr int BM = 128;       // rows per CTA (UMMA M)
constexpr int BJ = 64;        // columns j per tile (GEMM1 N, GEMM2 K)
constexpr int NTHREADS = 384;
constexpr uint32_t TM_S = 0;      // S double buffer: cols [0,128)
constexpr uint32_t TM_K = 128;    // K hi/lo double buffer: cols [128,384)
constexpr uint32_t TM_Y = 384;    // Y accumulator: cols [384, 384 + s_pad)
constexpr int MAX_SPAD = 128;

struct Params {
  const float* XA;      // tiled A operand rows (this launch's rows start at tile 0)
  const float* XB;      // tiled B operand rows (all columns j)
  const float* Vt;      // tiled V hi/lo per j tile
  const double* V64;    // [ncols][s] for the sigma^2 V_i term (gram) -- indexed by global row
  const double* B64;    // nullable: residual mode, [nrows][s]
  double* Y64;          // [nrows][s]
  int64_t nrows, row0, ncols;
  int ntiles;           // ceil(ncols / BJ)
  int s, s_pad, K1;
  int kind;
  float c1, neg_c_log2e, s2;
  double noise2;
  int gram;
};

__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

__global__ void __launch_bounds__(NTHREADS, 1) kmatvec_tc_kernel(const Params p, int NS) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t XA_BYTES = BM * p.K1 * 4;
  const uint32_t XB_BYTES = BJ * p.K1 * 4;
  const uint32_t VT_BYTES = p.s_pad * BJ * 4;  // one of hi / lo
  const uint32_t ST_BYTES = XB_BYTES + 2 * VT_BYTES;
  unsigned char* sXA = smem;
  unsigned char* sStage = smem + XA_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + (size_t)NS * ST_BYTES);
  uint64_t* stage_full = bars;
  uint64_t* stage_empty = bars + NS;
  uint64_t* xa_full = bars + 2 * NS;
  uint64_t* s_full = xa_full + 1;
  uint64_t* s_empty = s_full + 2;
  uint64_t* k_full = s_empty + 2;
  uint64_t* k_empty = k_full + 2;
  uint64_t* y_full = k_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(y_full + 1);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&stage_full[i], 1);
      ptx::mbar_init(&stage_empty[i], 1);
    }
    ptx::mbar_init(xa_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_empty[i], 8);
      ptx::mbar_init(&k_full[i], 8);
      ptx::mbar_init(&k_empty[i], 1);
    }
    ptx::mbar_init(y_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int T = p.ntiles;
  const int KS1 = p.K1 / 8;                 // GEMM1 K-steps
  const uint32_t sbo1 = (p.K1 / 4) * 128;   // 8-row group stride of XA/XB tiles

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(xa_full, XA_BYTES);
      ptx::bulk_g2s(sXA, p.XA + (size_t)blockIdx.x * BM * p.K1, XA_BYTES, xa_full);
      for (int t = 0; t < T; ++t) {
        const int st = t % NS;
        if (t >= NS) ptx::mbar_wait(&stage_empty[st], ((t / NS) - 1) & 1);
        unsigned char* dst = sStage + (size_t)st * ST_BYTES;
        ptx::mbar_arrive_expect_tx(&stage_full[st], ST_BYTES);
        ptx::bulk_g2s(dst, p.XB + (size_t)t * BJ * p.K1, XB_BYTES, &stage_full[st]);
        ptx::bulk_g2s(dst + XB_BYTES, p.Vt + (size_t)t * 2 * p.s_pad * BJ, 2 * VT_BYTES,
                      &stage_full[st]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc1 = ptx::idesc_tf32(BM, BJ);
      const uint32_t idesc2 = ptx::idesc_tf32(BM, p.s_pad);
      const uint32_t aXA = ptx::smem_u32(sXA);
      ptx::mbar_wait(xa_full, 0);
      auto gemm2 = [&](int u) {
        const int sb = u & 1, st = u % NS;
        ptx::mbar_wait(&k_full[sb], (u >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aV = ptx::smem_u32(sStage + (size_t)st * ST_BYTES + XB_BYTES);
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
          const uint32_t a_col = TM_K + sb * 128 + (pass == 2 ? 64 : 0);  // K_hi, K_hi, K_lo
          const uint32_t vb = aV + (pass == 1 ? VT_BYTES : 0);              // V_hi, V_lo, V_hi
#pragma unroll
          for (int ks = 0; ks < BJ / 8; ++ks) {
            const uint64_t bdesc = ptx::umma_desc(vb + ks * 256, 128, 16 * 128);
            ptx::mma_tf32_ts(tmem + TM_Y, tmem + a_col + ks * 8, bdesc, idesc2,
                             (u > 0 || pass > 0 || ks > 0) ? 1u : 0u);
          }
        }
        ptx::mma_commit(&k_empty[sb]);
        ptx::mma_commit(&stage_empty[st]);
      };
      for (int t = 0; t < T; ++t) {
        const int st = t % NS, sb = t & 1;
        ptx::mbar_wait(&stage_full[st], (t / NS) & 1);
        if (t >= 2) ptx::mbar_wait(&s_empty[sb], ((t - 2) >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aXB = ptx::smem_u32(sStage + (size_t)st * ST_BYTES);
        for (int ks = 0; ks < KS1; ++ks) {
          const uint64_t adesc = ptx::umma_desc(aXA + ks * 256, 128, sbo1);
          const uint64_t bdesc = ptx::umma_desc(aXB + ks * 256, 128, sbo1);
          ptx::mma_tf32_ss(tmem + TM_S + sb * 64, adesc, bdesc, idesc1, ks > 0 ? 1u : 0u);
        }
        ptx::mma_commit(&s_full[sb]);
        if (t >= 1) gemm2(t - 1);
      }
      gemm2(T - 1);
      ptx::mma_commit(y_full);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ kernel-map epilogue
    const int q = warp & 3;            // TMEM lane quadrant accessible to this warp
    const int half = (warp - 4) >> 2;  // which 32 of the 64 tile columns
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int r = q * 32 + lane;       // row within the CTA tile
    const int64_t gi = p.row0 + (int64_t)blockIdx.x * BM + r;
    const int64_t grow0 = p.row0 + (int64_t)blockIdx.x * BM;
    for (int t = 0; t < T; ++t) {
      const int sb = t & 1;
      ptx::mbar_wait(&s_full[sb], (t >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t v[32];
      ptx::tmem_ld32(tmem + lane_off + TM_S + sb * 64 + half * 32, v);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&s_empty[sb]);
      uint32_t hi[32];
      if (p.kind == WGP_MATERN32) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float d2 = fmaxf(__uint_as_float(v[c]), 0.0f);
          const float rr = ptx::sqrt_approx(d2);
          const float e = ptx::ex2_approx(rr * p.neg_c_log2e);
          const float z = rr * p.c1;
          v[c] = __float_as_uint(p.s2 * fmaf(z, e, e));
        }
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float d2 = fmaxf(__uint_as_float(v[c]), 0.0f);
          v[c] = __float_as_uint(p.s2 * ptx::ex2_approx(d2 * p.neg_c_log2e));
        }
      }
      const int64_t gj0 = (int64_t)t * BJ + half * 32;
      if (p.gram && gj0 < grow0 + BM && gj0 + 32 > grow0) {  // tile touches the diagonal
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (gj0 + c == gi) v[c] = __float_as_uint(p.s2);  // k(x,x) = s^2 exactly
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const uint32_t h = v[c] & 0xFFFFE000u;
        hi[c] = h;
        v[c] = __float_as_uint(__uint_as_float(v[c]) - __uint_as_float(h));  // lo
      }
      if (t >= 2) ptx::mbar_wait(&k_empty[sb], ((t - 2) >> 1) & 1);
      ptx::tc_fence_after();
      ptx::tmem_st32(tmem + lane_off + TM_K + sb * 128 + half * 32, hi);
      ptx::tmem_st32(tmem + lane_off + TM_K + sb * 128 + 64 + half * 32, v);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&k_full[sb]);
    }
    // ------------------------------------------------------------ output
    ptx::mbar_wait(y_full, 0);
    ptx::tc_fence_after();
    const bool valid = (int64_t)blockIdx.x * BM + r < p.nrows;
    const int64_t lr = (int64_t)blockIdx.x * BM + r;  // local output row
    for (int ch = half; ch * 32 < p.s_pad; ch += 2) {
      uint32_t y[32];
      ptx::tmem_ld32(tmem + lane_off + TM_Y + ch * 32, y);
      ptx::tmem_wait_ld();
      if (valid) {
#pragma unroll 4
        for (int c = 0; c < 32; ++c) {
          const int col = ch * 32 + c;
          if (col < p.s) {
            double acc = (double)__uint_as_float(y[c]);
            if (p.gram) acc += p.noise2 * p.V64[gi * p.s + col];
            p.Y64[lr * p.s + col] = p.B64 ? p.B64[lr * p.s + col] - acc : acc;
          }
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

// V [ncols][s] fp64 -> per-64-row tile [hi|lo][s_pad/8][16][8][4] fp32 (zero padded).
__global__ void split_v_kernel(const double* __restrict__ V, int64_t ncols, int s, int s_pad,
                               int64_t total_rows, float* __restrict__ Vt) {
  const int64_t total = total_rows * s_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / s_pad;
    const int c = (int)(e % s_pad);
    const double v = (j < ncols && c < s) ? V[j * s + c] : 0.0;
    const float vh = __uint_as_float(tf32_hi((float)v));
    const float vl = (float)(v - (double)vh);
    const int64_t t = j / BJ;
    const int jj = (int)(j % BJ);
    const int64_t idx = ((int64_t)((c >> 3) * (BJ / 4) + (jj >> 2)) * 8 + (c & 7)) * 4 + (jj & 3);
    float* base = Vt + t * 2 * (int64_t)s_pad * BJ;
    base[idx] = vh;
    base[(int64_t)s_pad * BJ + idx] = vl;
  }
}

inline int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
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
  const size_t stage = (size_t)tc::BJ * K1 * 4 + 2 * (size_t)s_pad * tc::BJ * 4;
  const size_t tail = 16 * 8 + 64;
  int ns = (int)((227 * 1024 - xa - tail) / stage);
  if (ns > 4) ns = 4;
  *ns_out = ns;
  return xa + ns * stage + tail;
}

// Y = (K(Xr, Xc) [+ sigma^2 I]) V, rows [row0, row0 + nrows) of the operator.  V64 and
// Y64/B64 are fp64 row-major; RHS chunks of <= 128 columns per launch.
void launch_kmatvec_tc(const Op& op, const float* XA_rows, const float* XB, int64_t nrows,
                       int64_t row0, int64_t ncols, const double* V64, int s, const double* B64,
                       double* Y64, bool gram, DBuf<float>& vt_scratch, DBuf<double>& vchunk,
                       DBuf<double>& ychunk, cudaStream_t st) {
  if (nrows <= 0 || s <= 0) return;
  const int K1 = tc_k1(op.dim);
  const KParams kp = op.kp();
  for (int c0 = 0; c0 < s; c0 += tc::MAX_SPAD) {
    const int sc = std::min(tc::MAX_SPAD, s - c0);
    const double* Vc = V64;
    const double* Bc = B64;
    double* Yc = Y64;
    if (sc != s) {  // gather this column chunk (rare: s > 128)
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
    vt_scratch.ensure((size_t)ntiles * tc::BJ * s_pad * 2);
    tc::split_v_kernel<<<tc::grid_for((int64_t)ntiles * tc::BJ * s_pad), 256, 0, st>>>(
        Vc, ncols, sc, s_pad, (int64_t)ntiles * tc::BJ, vt_scratch.p);
    WGP_CUDA(cudaGetLastError());
    tc::Params prm;
    prm.XA = XA_rows;
    prm.XB = XB;
    prm.Vt = vt_scratch.p;
    prm.V64 = Vc;
    prm.B64 = Bc;
    prm.Y64 = Yc;
    prm.nrows = nrows;
    prm.row0 = row0;
    prm.ncols = ncols;
    prm.ntiles = ntiles;
    prm.s = sc;
    prm.s_pad = s_pad;
    prm.K1 = K1;
    prm.kind = kp.kind;
    prm.c1 = (float)kp.c1;
    prm.neg_c_log2e = (float)(-kp.c1 * 1.4426950408889634);
    prm.s2 = (float)kp.s2;
    prm.noise2 = kp.noise2;
    prm.gram = gram ? 1 : 0;
    int ns = 0;
    const size_t smem = tc_smem_bytes(K1, s_pad, &ns);
    WGP_REQUIRE(ns >= 2, "kmatvec_tc: dim %d too large for the shared-memory pipeline", op.dim);
    WGP_CUDA(cudaFuncSetAttribute(tc::kmatvec_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    const int grid = (int)((nrows + tc::BM - 1) / tc::BM);
    tc::kmatvec_tc_kernel<<<grid, tc::NTHREADS, smem, st>>>(prm, ns);
    WGP_CUDA(cudaGetLastError());
    if (sc != s) {
      WGP_CUDA(cudaMemcpy2DAsync(Y64 + c0, sizeof(double) * s, Yc, sizeof(double) * sc,
                                 sizeof(double) * sc, nrows, cudaMemcpyDeviceToDevice, st));
    }
  }
}

}  // namespace wgp
