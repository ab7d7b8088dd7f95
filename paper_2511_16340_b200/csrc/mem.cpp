// mem.cpp -- the device block cache behind DBuf (common.cuh).
//
// Buckets: sizes rounded up to 1/8 of their power of two (at most 12.5% slack), minimum
// 4 KB.  A free synchronises the device (the implicit synchronisation cudaFree performed,
// so a block handed out again is never still read or written by queued work on any stream)
// and keeps the block; an allocation takes a cached block of its bucket or carves a new one
// from a chunk (below).  Thread-safe (loopback ranks are threads of one process).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace wgp {
namespace {

std::mutex g_mu;
std::map<std::pair<int, size_t>, std::vector<void*>>& cache() {
  static auto* m = new std::map<std::pair<int, size_t>, std::vector<void*>>();  // never destroyed
  return *m;
}

// WGP_PHASE_TIMING=1: report allocator calls slower than 5 ms on stderr (diagnostics)
bool slow_report() {
  static const bool on = getenv("WGP_PHASE_TIMING") && atoi(getenv("WGP_PHASE_TIMING")) != 0;
  return on;
}
struct SlowTimer {
  const char* what;
  size_t bytes;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~SlowTimer() {
    if (!slow_report()) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 5.0) fprintf(stderr, "[wgp mem] %s %zu bytes: %.1f ms\n", what, bytes, ms);
  }
};

size_t bucket(size_t bytes) {
  if (bytes <= 4096) return 4096;
  size_t top = 1;
  while ((top << 1) <= bytes) top <<= 1;
  const size_t step = top / 8;
  return (bytes + step - 1) / step * step;
}

// Blocks that are not in the cache come from per-device chunks of >= 256 MB carved by a bump
// pointer: cudaMalloc itself stalls sporadically on these boxes (5-135 ms even for 1 MB in
// WGP_PHASE_TIMING traces of the C2 growth sweep), so it is called a handful of times per
// process instead of once per new buffer size.  Chunks are never returned; freed blocks go to
// the bucket cache as before.
struct Chunk {
  int dev;
  char* base;
  size_t size, used;
};
std::vector<Chunk>& chunks() {
  static auto* v = new std::vector<Chunk>();  // never destroyed
  return *v;
}
constexpr size_t kChunk = (size_t)256 << 20;

}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  WGP_CUDA(cudaGetDevice(&dev));
  const size_t b = bucket(bytes);
  std::lock_guard<std::mutex> lk(g_mu);
  {
    auto it = cache().find({dev, b});
    if (it != cache().end() && !it->second.empty()) {
      void* q = it->second.back();
      it->second.pop_back();
      return q;
    }
  }
  for (Chunk& c : chunks())
    if (c.dev == dev && c.size - c.used >= b) {
      void* q = c.base + c.used;
      c.used += (b + 255) & ~(size_t)255;
      return q;
    }
  const size_t csz = b > kChunk ? b : kChunk;
  void* q = nullptr;
  cudaError_t e;
  {
    SlowTimer tm{"cudaMalloc", csz};
    e = cudaMalloc(&q, csz);
  }
  if (e == cudaErrorMemoryAllocation && csz > b) {  // no room for a whole chunk: just the block
    cudaGetLastError();
    SlowTimer tm{"cudaMalloc", b};
    e = cudaMalloc(&q, b);
    if (e == cudaSuccess) {
      chunks().push_back({dev, static_cast<char*>(q), b, b});
      return q;
    }
  }
  WGP_CUDA(e);
  chunks().push_back({dev, static_cast<char*>(q), csz, (b + 255) & ~(size_t)255});
  return q;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  // (called from destructors: never throws; after a device error the block is dropped --
  // blocks live inside chunks and are not the driver's to free individually)
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return;
  }
  {
    // synchronise the block's own device (a process may drive several)
    SlowTimer tm{"free-sync", bytes};
    int cur = a.device;
    cudaGetDevice(&cur);
    if (cur != a.device) cudaSetDevice(a.device);
    const cudaError_t e = cudaDeviceSynchronize();
    if (cur != a.device) cudaSetDevice(cur);
    if (e != cudaSuccess) return;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cache()[{a.device, bucket(bytes)}].push_back(p);  // the block's own device
}

}  // namespace wgp
