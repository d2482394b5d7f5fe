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

}  // namespace b200ipc
