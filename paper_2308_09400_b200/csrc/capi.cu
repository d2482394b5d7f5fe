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
