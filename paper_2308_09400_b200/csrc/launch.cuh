// Launch bookkeeping shared by all translation units.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace b200ipc {

// defined in capi.cu
extern std::atomic<int64_t> g_launches;

// Count one kernel launch and fold the launch status into the ABI's return convention.
inline int post_launch(int launches = 1) {
  g_launches.fetch_add(launches, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

inline int cuda_rc(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e; }

// Per-call scratch from the device's stream-ordered pool (cudaMallocAsync).  The pool's release
// threshold is lifted once, so after the first call the buffers are recycled without touching the
// driver: cudaMalloc / cudaFree per buffer cost ~30 ms per narrow phase.
inline cudaError_t keep_pool_memory() {
  static bool done = false;
  if (done) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return e;
  uint64_t keep = ~0ull;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  done = e == cudaSuccess;
  return e;
}

}  // namespace b200ipc
