// dist.cpp -- NCCL plumbing for row-sharded operators (one process per GPU).
//
// Rank g owns rows wgp_shard_range(n, world, g) of every solver vector; the kernel-matvec
// needs the full direction vector, so each sharded iteration all-gathers the updated
// slice (ncclAllGather over NVLink/NVSwitch) and all-gathers the fixed-chunk fp64
// partials of the per-column dot products, which every rank then sums in chunk order --
// results are bit-identical for every world size.
#include <nccl.h>

#include <cstring>

#include "common.cuh"

namespace wgp {

struct Comm {
  ncclComm_t nccl = nullptr;
};

#define WGP_NCCL(call)                                                                  \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      ::wgp::throw_error(WGP_NCCL_ERROR, "%s: %s", #call, ncclGetErrorString(r_));     \
  } while (0)

void dist_init(Ctx& ctx, const void* uid) {
  WGP_REQUIRE(uid, "sharded context needs a NCCL unique id");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  Comm* c = new Comm();
  try {
    WGP_NCCL(ncclCommInitRank(&c->nccl, ctx.world, id, ctx.rank));
  } catch (...) {
    delete c;
    throw;
  }
  ctx.comm = c;
}

void dist_destroy(Ctx& ctx) {
  if (!ctx.comm) return;
  if (ctx.comm->nccl) ncclCommDestroy(ctx.comm->nccl);
  delete ctx.comm;
  ctx.comm = nullptr;
}

// Gather variable-size row slices (each rank's slice of an [n][s] array) into the full
// array on every rank: an NCCL group of broadcasts, one per owner (slices are contiguous
// and chunk-aligned, so their sizes differ by at most one 512-row chunk).
void dist_allgather_rows(const Ctx& ctx, void* full, int64_t n, int64_t row_elems, size_t esize,
                         cudaStream_t st) {
  if (ctx.world == 1) return;
  WGP_NCCL(ncclGroupStart());
  for (int r = 0; r < ctx.world; ++r) {
    int64_t a, b;
    wgp_shard_range(n, ctx.world, r, &a, &b);
    if (b <= a) continue;
    char* base = (char*)full + (size_t)a * row_elems * esize;
    WGP_NCCL(ncclBroadcast(base, base, (size_t)(b - a) * row_elems * esize, ncclChar, r,
                           ctx.comm->nccl, st));
  }
  WGP_NCCL(ncclGroupEnd());
}

// Same for per-chunk partial arrays [nch][per_chunk] fp64 (chunk c of rows [512c, 512c+512)).
void dist_allgather_chunks(const Ctx& ctx, double* part, int64_t n, int64_t per_chunk,
                           cudaStream_t st) {
  if (ctx.world == 1) return;
  WGP_NCCL(ncclGroupStart());
  for (int r = 0; r < ctx.world; ++r) {
    int64_t a, b;
    wgp_shard_range(n, ctx.world, r, &a, &b);
    if (b <= a) continue;
    const int64_t c0 = a / kChunkRows, c1 = (b + kChunkRows - 1) / kChunkRows;
    double* base = part + c0 * per_chunk;
    WGP_NCCL(ncclBroadcast(base, base, (size_t)(c1 - c0) * per_chunk, ncclDouble, r,
                           ctx.comm->nccl, st));
  }
  WGP_NCCL(ncclGroupEnd());
}

void dist_broadcast(const Ctx& ctx, void* buf, size_t bytes, int root, cudaStream_t st) {
  if (ctx.world == 1) return;
  WGP_NCCL(ncclBroadcast(buf, buf, bytes, ncclChar, root, ctx.comm->nccl, st));
}

// Every rank contributes `count` doubles; out holds world x count in rank order.
void dist_allgather(const Ctx& ctx, const double* in, double* out, size_t count, cudaStream_t st) {
  if (ctx.world == 1) {
    if (in != out) WGP_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    return;
  }
  WGP_NCCL(ncclAllGather(in, out, count, ncclDouble, ctx.comm->nccl, st));
}

int owner_rank(const Ctx& ctx, int64_t n, int64_t row) {
  for (int r = 0; r < ctx.world; ++r) {
    int64_t a, b;
    wgp_shard_range(n, ctx.world, r, &a, &b);
    if (row >= a && row < b) return r;
  }
  return ctx.world - 1;
}

}  // namespace wgp

extern "C" wgp_status wgp_allgather_rows_dev(wgp_ctx* ctx, void* dV, int64_t n, int s, void* stream) {
  if (!ctx || !dV || s < 1) return WGP_INVALID_ARGUMENT;
  try {
    wgp::Ctx* c = reinterpret_cast<wgp::Ctx*>(ctx);
    wgp::dist_allgather_rows(*c, dV, n, s, sizeof(double), stream ? (cudaStream_t)stream : c->stream);
  } catch (const wgp::Error& e) {
    return e.code;
  }
  return WGP_OK;
}

extern "C" wgp_status wgp_nccl_unique_id(void* out128) {
  if (!out128) return WGP_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return WGP_NCCL_ERROR;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof id);
  return WGP_OK;
}
