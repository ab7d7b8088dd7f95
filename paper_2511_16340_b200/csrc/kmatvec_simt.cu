// kmatvec_simt.cu -- CUDA-core fused kernel-matvec (fp64 path and fp32 validation path).
//
// Replaces gram_matrix (kernel.cpp:48-72) + the dense GEMV H*p (solvers.cpp:162) and
// b - H*v (solvers.cpp:150,171,...) with one tiled pass that never materialises K:
//   Y[r, c] = sum_j k(x_r, x_j) V[j, c]  (+ sigma_n^2 V[r, c] on the gram diagonal)
// Per 64x64 (row, col) tile: phase 1 evaluates the 4096 kernel entries into shared
// memory (the diagonal is set exactly to s^2 + sigma_n^2 like kernel.cpp:70), phase 2
// multiplies the tile into register accumulators for up to 64 RHS.
//
// Distances here use explicit differences sum_k (x_rk - x_jk)^2, which equals the
// reference's norm form to rounding and has no cancellation; the tensor-core path
// (kmatvec_tc.cu) uses the norm form as a contraction.
#include <cstdlib>

#include "solvers.h"

namespace wgp {
namespace {

constexpr int BM = 64, BN = 64, NT = 256;

template <typename T>
__device__ __forceinline__ T kmap(T d2, const KParams& p);

template <>
__device__ __forceinline__ double kmap<double>(double d2, const KParams& p) {
  d2 = d2 > 0.0 ? d2 : 0.0;
  if (p.kind == WGP_RBF) return p.s2 * exp_neg(-p.c1 * d2);
  const double z = p.c1 * sqrt(d2);
  return p.s2 * (1.0 + z) * exp_neg(-z);
}

template <>
__device__ __forceinline__ float kmap<float>(float d2, const KParams& p) {
  d2 = fmaxf(d2, 0.0f);
  const float s2 = (float)p.s2, c1 = (float)p.c1;
  if (p.kind == WGP_RBF) return s2 * exp2f(-c1 * 1.4426950408889634f * d2);
  const float z = c1 * sqrtf(d2);
  return s2 * (1.0f + z) * exp2f(-1.4426950408889634f * z);
}

// BS: RHS columns per block.  Phase-2 thread layout: 16 row groups x (BS/CN) column
// groups, 4 rows x CN columns per thread, j accumulated strictly in order -- every output
// column sees the same summation order whatever s is, so batched and single-RHS solves
// agree bitwise (test_solvers.cpp:397-413).  Threads beyond 16*BS/CN idle in phase 2.
template <typename T, int BS>
__global__ void __launch_bounds__(NT) kmatvec_simt_kernel(
    const T* __restrict__ Xr, int64_t nrows, int64_t row0, const T* __restrict__ Xc,
    int64_t ncols, int dpad, int dim, const double* __restrict__ V, int s,
    const double* __restrict__ B, double* __restrict__ Y, KParams p, int gram) {
  constexpr int CN = BS >= 64 ? 4 : (BS == 32 ? 2 : 1);
  constexpr int TXN = BS / CN;
  static_assert(16 * TXN <= NT, "bad layout");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sXr = reinterpret_cast<T*>(smem_raw);          // BM x (dim+1)
  T* sXc = sXr + BM * (dim + 1);                     // BN x (dim+1)
  T* sK = sXc + BN * (dim + 1);                      // BM x (BN+1)
  T* sV = sK + BM * (BN + 1);                        // BN x BS

  const int tid = threadIdx.x;
  const int64_t rbase = (int64_t)blockIdx.x * BM;
  const int c0 = blockIdx.y * BS;
  const int ds = dim + 1;

  for (int e = tid; e < BM * dim; e += NT) {
    const int r = e / dim, k = e % dim;
    const int64_t gr = rbase + r;
    sXr[r * ds + k] = gr < nrows ? Xr[gr * dpad + k] : T(0);
  }

  const int tx = tid % TXN;
  const int ty = (tid / TXN) % 16;
  const bool p2 = tid < 16 * TXN;
  T acc[4][CN];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < CN; ++b) acc[a][b] = T(0);

  const T kdiag = T(p.s2 + p.noise2);
  for (int64_t jb = 0; jb < ncols; jb += BN) {
    __syncthreads();
    for (int e = tid; e < BN * dim; e += NT) {
      const int j = e / dim, k = e % dim;
      const int64_t gj = jb + j;
      sXc[j * ds + k] = gj < ncols ? Xc[gj * dpad + k] : T(0);
    }
    for (int e = tid; e < BN * BS; e += NT) {
      const int j = e / BS, c = e % BS;
      const int64_t gj = jb + j;
      sV[j * BS + c] = (gj < ncols && c0 + c < s) ? (T)V[gj * s + c0 + c] : T(0);
    }
    __syncthreads();
    // phase 1: kernel tile
    {
      const int j = tid % BN;
      const int64_t gj = jb + j;
#pragma unroll 4
      for (int q = 0; q < BM * BN / NT; ++q) {
        const int r = tid / BN + q * (NT / BN);
        T d2 = T(0);
        for (int k = 0; k < dim; ++k) {
          const T df = sXr[r * ds + k] - sXc[j * ds + k];
          d2 = fma(df, df, d2);
        }
        T kv = kmap<T>(d2, p);
        if (gram && row0 + rbase + r == gj) kv = kdiag;
        if (gj >= ncols) kv = T(0);
        sK[r * (BN + 1) + j] = kv;
      }
    }
    __syncthreads();
    // phase 2: accumulate K_tile * V_tile
    if (!p2) continue;
#pragma unroll 4
    for (int jj = 0; jj < BN; ++jj) {
      T kv[4], vv[CN];
#pragma unroll
      for (int a = 0; a < 4; ++a) kv[a] = sK[(ty * 4 + a) * (BN + 1) + jj];
#pragma unroll
      for (int b = 0; b < CN; ++b) vv[b] = sV[jj * BS + tx + b * TXN];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < CN; ++b) acc[a][b] = fma(kv[a], vv[b], acc[a][b]);
    }
  }

  if (!p2) return;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gr = rbase + ty * 4 + a;
    if (gr >= nrows) continue;
#pragma unroll
    for (int b = 0; b < CN; ++b) {
      const int c = c0 + tx + b * TXN;
      if (c >= s) continue;
      const double y = (double)acc[a][b];
      Y[gr * s + c] = B ? B[gr * s + c] - y : y;
    }
  }
}

template <typename T, int BS>
void launch_bs(const Op& op, const T* Xr, int64_t nrows, int64_t row0, const T* Xc, int64_t ncols,
               const double* V, int s, const double* B, double* Y, bool gram, cudaStream_t st) {
  const int dim = op.dim;
  const size_t smem = sizeof(T) * ((size_t)(BM + BN) * (dim + 1) + BM * (BN + 1) + BN * BS);
  auto kern = kmatvec_simt_kernel<T, BS>;
  if (smem > 48 * 1024)
    WGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(ceil_div(nrows, BM), ceil_div(s, BS));
  kern<<<grid, NT, smem, st>>>(Xr, nrows, row0, Xc, ncols, op.dpad, dim, V, s, B, Y, op.kp(),
                               gram ? 1 : 0);
  WGP_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------------------------
// fp64 path on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64): per 64-row x 32-column
// tile, phase 1 evaluates the kernel entries into shared memory on the CUDA cores (the
// exp/sqrt sequences), phase 2 multiplies the tile into the accumulators with DMMA.  Warp w
// owns rows 8w..8w+7 and all NT 8-column RHS tiles; one A fragment (K) feeds NT DMMAs, so
// phase 2 moves ~1 byte of shared memory per FMA.  DMMA runs at the same 64 FMA/clk/SM as
// DFMA on B200 (tools/dmma_microbench.cu) with 1/8 of the instructions, leaving issue slots
// to phase 1.  Each output column's sum order is fixed and independent of s.
constexpr int DM = 64, DN = 32;

template <int NT>
__global__ void __launch_bounds__(256, NT <= 3 ? 4 : (NT <= 8 ? 3 : 2)) kmatvec_dmma_kernel(
    const double* __restrict__ Xr, int64_t nrows, int64_t row0, const double* __restrict__ Xc,
    int64_t ncols, int dpad, int dim, const double* __restrict__ V, int s,
    const double* __restrict__ B, double* __restrict__ Y, KParams p, int gram, int64_t jlen,
    double* __restrict__ part, int z0) {
  constexpr int BS = NT * 8;
  extern __shared__ double dsm[];
  const int ds = dim + 1;
  double* sXr = dsm;                   // [DM][ds]
  double* sXc = sXr + DM * ds;         // [DN][ds]
  double* sK = sXc + DN * ds;          // [DM][DN + 1]
  double* sV = sK + DM * (DN + 1);     // [DN][BS + 1]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rbase = (int64_t)blockIdx.x * DM;
  const int c0 = blockIdx.y * BS;
  for (int e = tid; e < DM * dim; e += 256) {
    const int r = e / dim, k = e % dim;
    const int64_t gr = rbase + r;
    sXr[r * ds + k] = gr < nrows ? Xr[gr * dpad + k] : 0.0;
  }
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const double kdiag = p.s2 + p.noise2;
  // this CTA's column range (grid.z splits the sweep into fixed-length ranges)
  const int zs = z0 + (int)blockIdx.z;  // column split of this CTA
  const int64_t j_lo = (int64_t)zs * jlen;
  const int64_t j_hi = min(ncols, j_lo + jlen);
  for (int64_t jb = j_lo; jb < j_hi; jb += DN) {
    __syncthreads();
    for (int e = tid; e < DN * dim; e += 256) {
      const int j = e / dim, k = e % dim;
      const int64_t gj = jb + j;
      sXc[j * ds + k] = gj < ncols ? Xc[gj * dpad + k] : 0.0;
    }
    for (int e = tid; e < DN * BS; e += 256) {
      const int j = e / BS, c = e % BS;
      const int64_t gj = jb + j;
      sV[j * (BS + 1) + c] = (gj < ncols && c0 + c < s) ? V[gj * s + c0 + c] : 0.0;
    }
    __syncthreads();
    // phase 1: 64 x 32 kernel entries, 8 per thread; the dimension loop runs outside the 8
    // entries so the eight distance and exp/sqrt chains interleave (ILP)
    {
      constexpr int NQ = DM * DN / 256;
      const int j = tid % DN;
      const int64_t gj = jb + j;
      double d2[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) d2[q] = 0.0;
      for (int k = 0; k < dim; ++k) {
        const double xc = sXc[j * ds + k];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const double df = sXr[(tid / DN + q * (256 / DN)) * ds + k] - xc;
          d2[q] = fma(df, df, d2[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = tid / DN + q * (256 / DN);
        double kv = kmap<double>(d2[q], p);
        if (gram && row0 + rbase + r == gj) kv = kdiag;
        if (gj >= ncols) kv = 0.0;
        sK[r * (DN + 1) + j] = kv;
      }
    }
    __syncthreads();
    // phase 2: Y[8w.., :] += K[8w.., 32] . V[32, BS] in 8 k-steps of 4
#pragma unroll
    for (int k0 = 0; k0 < DN; k0 += 4) {
      const double a = sK[(warp * 8 + (lane >> 2)) * (DN + 1) + k0 + (lane & 3)];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double b = sV[(k0 + (lane & 3)) * (BS + 1) + t * 8 + (lane >> 2)];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1])
                     : "d"(a), "d"(b));
      }
    }
  }
  const int64_t gr = rbase + warp * 8 + (lane >> 2);
  if (gr >= nrows) return;
  double* out = part ? part + (size_t)zs * nrows * s : Y;
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = c0 + t * 8 + (lane & 3) * 2 + u;
      if (c >= s) continue;
      const double y = acc[t][u];
      out[gr * s + c] = (B && !part) ? B[gr * s + c] - y : y;
    }
}

// Y = sum over the column splits in order (or B - that).
__global__ void sum_splits_kernel(const double* __restrict__ part, int nsplit, int64_t count,
                                  const double* __restrict__ B, double* __restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    double y = 0.0;
    for (int q = 0; q < nsplit; ++q) y += part[(size_t)q * count + e];
    Y[e] = B ? B[e] - y : y;
  }
}

// Column splits: the j sweep is cut into up to 16 equal ranges of at least 128 columns,
// summed in order by sum_splits_kernel, so small row counts still fill the GPU (config 1,
// N=2000: 32 row blocks x 16 splits instead of 32 CTAs each sweeping 2000 columns, 185 ->
// ~15 us per matvec).  The split depends on ncols only, so every rank of a row-sharded
// operator sums each output identically and the result is world-size independent.
constexpr int64_t kSplitCols = 128;
inline int f64_splits(int64_t ncols) { return (int)std::min<int64_t>(16, (ncols + kSplitCols - 1) / kSplitCols); }

// With a ColPhase (sharded matvec overlapping the V all-gather): the splits whose columns
// lie inside [c0, c1) run first, the others after ph->ready; every split is computed and
// summed exactly as in the single launch, so the result is bitwise the same.
template <int NT>
void launch_dmma(const double* Xr, int64_t nrows, int64_t row0, const double* Xc, int64_t ncols,
                 int dpad, int dim, const double* V, int s, const double* B, double* Y, KParams kp,
                 bool gram, DBuf<double>& split_buf, cudaStream_t st, const ColPhase* ph) {
  const int nsplit = std::max(1, f64_splits(ncols));
  const int64_t jlen = nsplit == 1 ? ncols : (((ncols + nsplit - 1) / nsplit + DN - 1) / DN) * DN;
  double* part = nullptr;
  if (nsplit > 1) {
    split_buf.ensure((size_t)nsplit * nrows * s);
    part = split_buf.p;
  }
  const size_t smem = sizeof(double) * ((size_t)(DM + DN) * (dim + 1) + DM * (DN + 1) +
                                        (size_t)DN * (NT * 8 + 1));
  if (smem > 48 * 1024)
    WGP_CUDA(cudaFuncSetAttribute(kmatvec_dmma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  auto run = [&](int za, int zb) {
    if (zb <= za) return;
    dim3 grid(ceil_div(nrows, DM), ceil_div(s, NT * 8), zb - za);
    kmatvec_dmma_kernel<NT><<<grid, 256, smem, st>>>(Xr, nrows, row0, Xc, ncols, dpad, dim, V, s, B, Y,
                                                     kp, gram ? 1 : 0, jlen, part, za);
    WGP_CUDA(cudaGetLastError());
  };
  if (!ph || !ph->ready) {
    run(0, nsplit);
  } else {
    int za = nsplit, zb = nsplit;  // splits inside [c0, c1)
    if (nsplit > 1) {
      za = (int)std::min<int64_t>(nsplit, (ph->c0 + jlen - 1) / jlen);
      zb = za;
      while (zb < nsplit && std::min<int64_t>(ncols, (int64_t)(zb + 1) * jlen) <= ph->c1) ++zb;
    }
    run(za, zb);
    WGP_CUDA(cudaStreamWaitEvent(st, ph->ready, 0));
    run(0, za);
    run(zb, nsplit);
  }
  if (part) {
    const int64_t count = nrows * s;
    sum_splits_kernel<<<(int)std::min<int64_t>(148 * 8, (count + 255) / 256), 256, 0, st>>>(part, nsplit, count,
                                                                                           B, Y);
    WGP_CUDA(cudaGetLastError());
  }
}

}  // namespace

// fp64 kernel-matvec: DMMA kernel (one RHS group up to 136 columns -- the kernel entries are
// evaluated once per group, so config 5's 129 columns run as one group -- else groups of
// 128); WGP_F64_SIMT=1 selects
// the all-CUDA-core kernel instead (validation).
static void launch_f64(const Op& op, const double* Xr, int64_t nrows, int64_t row0,
                       const double* Xc, int64_t ncols, const double* V, int s, const double* B,
                       double* Y, bool gram, cudaStream_t st, const ColPhase* ph) {
  WGP_REQUIRE(op.dim <= 32, "fp64 kmatvec: dim <= 32 supported, got %d", op.dim);
  const KParams kp = op.kp();
  const int dp = op.dpad, d = op.dim;
  if (s <= 8) return launch_dmma<1>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
  if (s <= 16) return launch_dmma<2>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
  if (s <= 24) return launch_dmma<3>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
  if (s <= 32) return launch_dmma<4>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
  if (s <= 64) return launch_dmma<8>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
  if (s <= 136) return launch_dmma<17>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
  return launch_dmma<16>(Xr, nrows, row0, Xc, ncols, dp, d, V, s, B, Y, kp, gram, op.f64split, st, ph);
}

template <typename T>
void launch_kmatvec_simt(const Op& op, const T* Xr, int64_t nrows, int64_t row0, const T* Xc,
                         int64_t ncols, const double* V, int s, const double* B, double* Y,
                         bool gram, cudaStream_t st, const ColPhase* ph) {
  if (nrows <= 0 || s <= 0) {
    if (ph && ph->ready) WGP_CUDA(cudaStreamWaitEvent(st, ph->ready, 0));
    return;
  }
  TimedScope ts_(sizeof(T) == 8 ? "kmatvec_f64" : "kmatvec_f32", st);
  if constexpr (sizeof(T) == 8) {
    static const bool simt = getenv("WGP_F64_SIMT") && atoi(getenv("WGP_F64_SIMT")) != 0;
    if (!simt) {
      return launch_f64(op, reinterpret_cast<const double*>(Xr), nrows, row0,
                        reinterpret_cast<const double*>(Xc), ncols, V, s, B, Y, gram, st, ph);
    }
  }
  if (ph && ph->ready) WGP_CUDA(cudaStreamWaitEvent(st, ph->ready, 0));  // no overlap here
  if (s <= 1) return launch_bs<T, 1>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
  if (s <= 2) return launch_bs<T, 2>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
  if (s <= 4) return launch_bs<T, 4>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
  if (s <= 8) return launch_bs<T, 8>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
  if (s <= 16) return launch_bs<T, 16>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
  if (s <= 32) return launch_bs<T, 32>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
  return launch_bs<T, 64>(op, Xr, nrows, row0, Xc, ncols, V, s, B, Y, gram, st);
}

template void launch_kmatvec_simt<double>(const Op&, const double*, int64_t, int64_t,
                                          const double*, int64_t, const double*, int,
                                          const double*, double*, bool, cudaStream_t,
                                          const ColPhase*);
template void launch_kmatvec_simt<float>(const Op&, const float*, int64_t, int64_t, const float*,
                                         int64_t, const double*, int, const double*, double*, bool,
                                         cudaStream_t, const ColPhase*);

}  // namespace wgp
