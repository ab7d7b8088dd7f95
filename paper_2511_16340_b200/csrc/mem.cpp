// mem.cpp -- the device block cache behind DBuf (common.cuh).
//
// Buckets: sizes rounded up to 1/8 of their power of two (at most 12.5% slack), minimum
// 4 KB.  A free synchronises the device (the implicit synchronisation cudaFree performed,
// so a block handed out again is never still read or written by queued work on any stream)
// and keeps the block; an allocation takes a cached block of its bucket or calls cudaMalloc,
// and on an out-of-memory error returns every cached block of the device to the driver and
// retries once.  Thread-safe (loopback ranks are threads of one process).
#include <cuda_runtime.h>

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

size_t bucket(size_t bytes) {
  if (bytes <= 4096) return 4096;
  size_t top = 1;
  while ((top << 1) <= bytes) top <<= 1;
  const size_t step = top / 8;
  return (bytes + step - 1) / step * step;
}

void release_device(int dev) {  // g_mu held
  auto& c = cache();
  for (auto it = c.begin(); it != c.end();) {
    if (it->first.first == dev) {
      for (void* q : it->second) cudaFree(q);
      it = c.erase(it);
    } else {
      ++it;
    }
  }
}

}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  WGP_CUDA(cudaGetDevice(&dev));
  const size_t b = bucket(bytes);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache().find({dev, b});
    if (it != cache().end() && !it->second.empty()) {
      void* q = it->second.back();
      it->second.pop_back();
      return q;
    }
  }
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, b);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();  // clear the sticky-free allocation error
    {
      std::lock_guard<std::mutex> lk(g_mu);
      release_device(dev);
    }
    e = cudaMalloc(&q, b);
  }
  WGP_CUDA(e);
  return q;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  // (called from destructors: never throws; on a device error the block goes back to the
  // driver instead of the cache)
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p);
    return;
  }
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cache()[{a.device, bucket(bytes)}].push_back(p);  // the block's own device
}

}  // namespace wgp
