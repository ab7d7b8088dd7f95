// dist.cpp -- collectives for row-sharded operators.
//
// Rank g owns the equal, chunk-aligned row slot wgp_shard_range(n, world, g) of every
// solver vector; the kernel-matvec needs the full direction vector, so each sharded
// iteration all-gathers the updated slices and all-gathers the fixed-chunk fp64 partials
// of the per-column dot products, which every rank then sums in chunk order -- results
// are bit-identical for every world size.  Full buffers are padded to world equal slots
// (padded_rows / padded_chunks, common.cuh) so both exchanges are ONE in-place
// ncclAllGather over NVLink/NVSwitch.
//
// Two transports behind the same five calls:
//  * NCCL (one process per GPU, wgp_ctx_create_sharded);
//  * loopback (wgp_ctx_create_loopback): the ranks are host threads of one process on one
//    device; a collective is "synchronise my stream, publish my buffer, barrier, copy the
//    other ranks' slices with cudaMemcpyAsync, synchronise, barrier".  No kernel waits on
//    another rank, so nothing depends on kernels of different ranks being co-resident.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace wgp {

struct LoopGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  std::vector<const void*> ptr;

  explicit LoopGroup(int w) : world(w), ptr(w, nullptr) {}

  // Barrier over the world ranks (generation counter).  A rank that waits longer than the
  // timeout marks the group broken (another rank failed before reaching this collective)
  // and every rank then throws instead of hanging.
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw_error(WGP_NCCL_ERROR, "loopback group broken (a rank failed)");
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return generation != gen || broken; }) ||
        broken) {
      broken = true;
      cv.notify_all();
      throw_error(WGP_NCCL_ERROR, "loopback collective timed out (a rank failed or diverged)");
    }
  }
};

struct Comm {
  ncclComm_t nccl = nullptr;
  LoopGroup* loop = nullptr;
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

void dist_init_loopback(Ctx& ctx, LoopGroup* g) {
  Comm* c = new Comm();
  c->loop = g;
  ctx.comm = c;
}

int loop_group_world(const LoopGroup* g) { return g->world; }

void dist_destroy(Ctx& ctx) {
  if (!ctx.comm) return;
  if (ctx.comm->nccl) ncclCommDestroy(ctx.comm->nccl);
  delete ctx.comm;
  ctx.comm = nullptr;
}

// Loopback exchange: every rank publishes `mine`; then for each other rank q, copies
// `bytes(q)` from src(q, ptr_q) into dst(q).  Both barriers bracket the copies so no rank
// overwrites a buffer another rank is still reading.
template <typename Src, typename Dst, typename Bytes>
static void loop_exchange(const Ctx& ctx, const void* mine, Src src, Dst dst, Bytes bytes,
                          cudaStream_t st) {
  LoopGroup& g = *ctx.comm->loop;
  WGP_CUDA(cudaStreamSynchronize(st));
  {
    std::lock_guard<std::mutex> lk(g.mu);
    g.ptr[ctx.rank] = mine;
  }
  g.barrier();
  for (int q = 0; q < ctx.world; ++q) {
    if (q == ctx.rank) continue;
    const size_t b = bytes(q);
    void* d = dst(q);
    if (b && d) WGP_CUDA(cudaMemcpyAsync(d, src(q, g.ptr[q]), b, cudaMemcpyDeviceToDevice, st));
  }
  WGP_CUDA(cudaStreamSynchronize(st));
  g.barrier();
}

// In-place all-gather of equal slots: `full` holds world slots of `slot_bytes`, rank r's
// own data in slot r.
static void allgather_slots(const Ctx& ctx, void* full, size_t slot_bytes, cudaStream_t st) {
  if (ctx.world == 1 || slot_bytes == 0) return;
  char* base = (char*)full;
  if (ctx.comm->loop) {
    loop_exchange(
        ctx, full, [&](int q, const void* pq) { return (const char*)pq + q * slot_bytes; },
        [&](int q) { return (void*)(base + q * slot_bytes); }, [&](int) { return slot_bytes; }, st);
    return;
  }
  WGP_NCCL(ncclAllGather(base + (size_t)ctx.rank * slot_bytes, base, slot_bytes, ncclChar,
                         ctx.comm->nccl, st));
}

// Full [padded_rows][row_elems] buffer: gather every rank's row slot.
void dist_allgather_rows(const Ctx& ctx, void* full, int64_t n, int64_t row_elems, size_t esize,
                         cudaStream_t st) {
  if (ctx.world == 1) return;
  allgather_slots(ctx, full, (size_t)shard_chunks(n, ctx.world) * kChunkRows * row_elems * esize, st);
}

cudaEvent_t dist_allgather_rows_begin(const Ctx& ctx, void* full, int64_t n, int64_t row_elems,
                                      size_t esize, cudaStream_t st) {
  if (ctx.world == 1) return nullptr;
  const size_t slot = (size_t)shard_chunks(n, ctx.world) * kChunkRows * row_elems * esize;
  if (ctx.comm->loop) {
    allgather_slots(ctx, full, slot, st);
    WGP_CUDA(cudaEventRecord(ctx.comm_ev[1], st));
    return ctx.comm_ev[1];
  }
  WGP_CUDA(cudaEventRecord(ctx.comm_ev[0], st));
  WGP_CUDA(cudaStreamWaitEvent(ctx.comm_stream, ctx.comm_ev[0], 0));
  allgather_slots(ctx, full, slot, ctx.comm_stream);
  WGP_CUDA(cudaEventRecord(ctx.comm_ev[1], ctx.comm_stream));
  return ctx.comm_ev[1];
}

// Per-chunk partial arrays [padded_chunks][per_chunk] fp64 (chunk c of rows [512c, 512c+512)).
void dist_allgather_chunks(const Ctx& ctx, double* part, int64_t n, int64_t per_chunk,
                           cudaStream_t st) {
  if (ctx.world == 1) return;
  allgather_slots(ctx, part, (size_t)shard_chunks(n, ctx.world) * per_chunk * sizeof(double), st);
}

void dist_broadcast(const Ctx& ctx, void* buf, size_t bytes, int root, cudaStream_t st) {
  if (ctx.world == 1) return;
  if (ctx.comm->loop) {
    const bool me = ctx.rank == root;
    loop_exchange(
        ctx, buf, [&](int, const void* pq) { return pq; },
        [&](int q) { return (!me && q == root) ? buf : (void*)nullptr; },
        [&](int q) { return q == root ? bytes : (size_t)0; }, st);
    return;
  }
  WGP_NCCL(ncclBroadcast(buf, buf, bytes, ncclChar, root, ctx.comm->nccl, st));
}

void dist_allreduce_sum(const Ctx& ctx, double* buf, size_t count, cudaStream_t st) {
  if (ctx.world == 1 || count == 0) return;
  if (ctx.comm->loop) {
    DBuf<double> slots((size_t)ctx.world * count);
    WGP_CUDA(cudaMemcpyAsync(slots.p + (size_t)ctx.rank * count, buf, sizeof(double) * count,
                             cudaMemcpyDeviceToDevice, st));
    loop_exchange(
        ctx, buf, [&](int, const void* pq) { return pq; },
        [&](int q) { return (void*)(slots.p + (size_t)q * count); },
        [&](int) { return sizeof(double) * count; }, st);
    launch_sum_slots(slots.p, ctx.world, count, buf, st);
    WGP_CUDA(cudaStreamSynchronize(st));  // slots is freed on return
    return;
  }
  WGP_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx.comm->nccl, st));
}

// Every rank contributes `count` doubles; out holds world x count in rank order.
void dist_allgather(const Ctx& ctx, const double* in, double* out, size_t count, cudaStream_t st) {
  if (in != out + (size_t)ctx.rank * count)
    WGP_CUDA(cudaMemcpyAsync(out + (size_t)ctx.rank * count, in, sizeof(double) * count,
                             cudaMemcpyDeviceToDevice, st));
  if (ctx.world == 1) return;
  allgather_slots(ctx, out, sizeof(double) * count, st);
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

extern "C" wgp_status wgp_loopback_group_create(int world, void** group) {
  if (!group || world < 1) return WGP_INVALID_ARGUMENT;
  *group = new wgp::LoopGroup(world);
  return WGP_OK;
}

extern "C" void wgp_loopback_group_destroy(void* group) {
  delete static_cast<wgp::LoopGroup*>(group);
}
