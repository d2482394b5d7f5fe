// Library-level entry points and shared globals of libb200ipc.
#include "launch.cuh"
#include "../../include/b200ipc.h"

#define B200IPC_STR2(x) #x
#define B200IPC_STR(x) B200IPC_STR2(x)

namespace b200ipc {
std::atomic<int64_t> g_launches{0};
}

extern "C" int b200ipc_abi_version(void) { return B200IPC_ABI_VERSION; }

extern "C" const char* b200ipc_build_info(void) {
  return "libb200ipc: sm_100a, fp64, -fmad=false, CUDA " B200IPC_STR(CUDART_VERSION);
}

extern "C" int64_t b200ipc_launch_count(void) { return b200ipc::g_launches.load(std::memory_order_relaxed); }

// Row gather: dst[i] = src[idx[i]] for rows of `row_bytes` bytes (a multiple of 4), one thread per 4-, 8- or 16-byte
// word so that a warp moves consecutive words of consecutive destination rows.  (torch's 2-D index_select takes
// 0.55 ms for 1 M rows of 96 bytes; this takes the time of the copy.)
namespace b200ipc {
template <typename W>
__global__ void __launch_bounds__(256) gather_rows_kernel(int64_t n, int words, const W* __restrict__ src,
                                                          const int64_t* __restrict__ idx, W* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= n * words) return;
  const int64_t i = t / words;
  const int w = (int)(t - i * words);
  dst[t] = src[idx[i] * words + w];
}
}  // namespace b200ipc

extern "C" int b200ipc_gather_rows(int64_t n, int64_t row_bytes, const void* src, const int64_t* idx, void* dst,
                                   void* stream) {
  if (n < 0 || row_bytes <= 0 || (row_bytes & 3)) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!src || !idx || !dst) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const uintptr_t al = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)row_bytes;
  const int wb = (al & 15) == 0 ? 16 : ((al & 7) == 0 ? 8 : 4);
  const int words = (int)(row_bytes / wb);
  const int64_t total = n * words;
  if (total >= (1ll << 31) * 256) return B200IPC_EINVAL;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (wb == 16) b200ipc::gather_rows_kernel<uint4><<<grid, 256, 0, st>>>(n, words, (const uint4*)src, idx, (uint4*)dst);
  else if (wb == 8) b200ipc::gather_rows_kernel<uint2><<<grid, 256, 0, st>>>(n, words, (const uint2*)src, idx, (uint2*)dst);
  else b200ipc::gather_rows_kernel<uint32_t><<<grid, 256, 0, st>>>(n, words, (const uint32_t*)src, idx, (uint32_t*)dst);
  return b200ipc::post_launch();
}
