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
// array on every rank: ncclGroup of broadcasts from each owner (slices are contiguous).
void dist_allgather_rows(const Ctx& ctx, void* full, int64_t n, int s, size_t esize,
                         cudaStream_t st) {
  if (ctx.world == 1) return;
  WGP_NCCL(ncclGroupStart());
  for (int r = 0; r < ctx.world; ++r) {
    int64_t a, b;
    wgp_shard_range(n, ctx.world, r, &a, &b);
    if (b <= a) continue;
    char* base = (char*)full + (size_t)a * s * esize;
    WGP_NCCL(ncclBroadcast(base, base, (size_t)(b - a) * s * esize, ncclChar, r, ctx.comm->nccl, st));
  }
  WGP_NCCL(ncclGroupEnd());
}

}  // namespace wgp

extern "C" wgp_status wgp_nccl_unique_id(void* out128) {
  if (!out128) return WGP_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return WGP_NCCL_ERROR;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof id);
  return WGP_OK;
}
