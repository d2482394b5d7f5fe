// Scratch microbenchmark: read-only streaming bandwidth on B200.
//   mode 0: plain 16-byte loads, grid-stride, many CTAs
//   mode 1: persistent CTAs, cp.async.bulk ring (chunk bytes / stages from argv), consumers only wait
// Usage: read_bw <MB> <chunkKB> <stages>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256) plain_read(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
    const uint4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void __launch_bounds__(256) plain_read_u4x4(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * 256;
  size_t i = (size_t)blockIdx.x * 256 + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const uint4 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride), d = __ldg(p + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc ^= __ldg(p + i).x;
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void __launch_bounds__(256) plain_write(uint4* __restrict__ p, size_t n) {
  const uint4 v = make_uint4(1, 2, 3, 4);
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) p[i] = v;
}

__global__ void __launch_bounds__(128, 1) bulk_read(const char* __restrict__ p, size_t bytes, int chunk, int stages,
                                                    unsigned* sink) {
  extern __shared__ __align__(128) unsigned char dyn[];
  uint64_t* full = reinterpret_cast<uint64_t*>(dyn + (size_t)stages * chunk);
  const size_t nchunks = bytes / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(full + s)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned acc = 0;
  if (threadIdx.x == 0) {
    size_t issued = 0, done = 0;
    size_t mine = (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
    while (done < mine) {
      while (issued < mine && issued < done + stages) {
        const int s = issued % stages;
        const char* src = p + (blockIdx.x + issued * gridDim.x) * (size_t)chunk;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(full + s)), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s32(dyn + (size_t)s * chunk)),
                     "l"(src), "r"(chunk), "r"(s32(full + s))
                     : "memory");
        ++issued;
      }
      const int s = done % stages;
      const unsigned parity = (done / stages) & 1;
      asm volatile(
          "{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@q bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(
              s32(full + s)),
          "r"(parity)
          : "memory");
      acc ^= dyn[(size_t)s * chunk];
      ++done;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 1024;
  const size_t bytes = mb << 20;
  char* buf;
  unsigned* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int reps = 20;
  for (int grid : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    plain_read<<<grid, 256>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) plain_read<<<grid, 256>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("plain  grid %5d : %.1f GB/s\n", grid, bytes * reps / ms / 1e6);
    plain_read_u4x4<<<grid, 256>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) plain_read_u4x4<<<grid, 256>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("plain4 grid %5d : %.1f GB/s\n", grid, bytes * reps / ms / 1e6);
  }
  for (int grid : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    plain_write<<<grid, 256>>>((uint4*)buf, bytes / 16);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) plain_write<<<grid, 256>>>((uint4*)buf, bytes / 16);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("write  grid %5d : %.1f GB/s\n", grid, bytes * reps / ms / 1e6);
  }
  cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int chunkkb : {4, 8, 16, 32, 64}) {
    for (int stages : {2, 3, 4, 6, 8, 12, 16, 24, 48}) {
      const int chunk = chunkkb * 1024;
      const size_t smem = (size_t)chunk * stages + 8 * stages;
      if (smem > 216 * 1024) continue;
      bulk_read<<<148, 128, smem>>>(buf, bytes, chunk, stages, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) bulk_read<<<148, 128, smem>>>(buf, bytes, chunk, stages, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("bulk chunk %2d KB stages %2d (%3d KB in flight/SM): %.1f GB/s  %s\n", chunkkb, stages, chunkkb * stages,
             bytes * reps / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
