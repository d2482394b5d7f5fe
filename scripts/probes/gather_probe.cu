// Scratch microbenchmark: achievable bandwidth of warp-wide reads of CHUNK-double runs at random vs
// sequential run indices from a ~0.9 GB array (the access pattern of the row-wise assembly).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>
#include <random>

template <int CHUNK, int PF>
__global__ void gather(const double* __restrict__ src, const unsigned* __restrict__ idx, long n, double* out) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (long j = warp * PF; j < n; j += nwarps * PF) {
    double v0[PF], v1[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const long jj = j + u < n ? j + u : n - 1;
      const double* p = src + (long)CHUNK * idx[jj];
      v0[u] = lane < CHUNK ? p[lane] : 0.0;
      v1[u] = lane + 32 < CHUNK ? p[lane + 32] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) acc += v0[u] + v1[u];
  }
  if (acc == 1.2345e-300) out[0] = acc;
}

template <int CHUNK, int PF>
void run(const char* name, const double* src, const unsigned* idx, long n, double* out, int ctas_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = 148 * ctas_per_sm;
  for (int i = 0; i < 3; ++i) gather<CHUNK, PF><<<grid, 256>>>(src, idx, n, out);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) gather<CHUNK, PF><<<grid, 256>>>(src, idx, n, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  printf("%-28s chunk %3d B  pf %d  ctas/sm %d : %.3f ms  %.0f GB/s\n", name, CHUNK * 8, PF, ctas_per_sm, ms,
         n * (CHUNK * 8.0 + 4.0) / ms / 1e6);
}

int main() {
  const long n = 3'300'000;  // runs
  const int CH = 36;
  double* src; unsigned *idx_r, *idx_s; double* out;
  cudaMalloc(&src, n * CH * 8); cudaMemset(src, 0, n * CH * 8);
  cudaMalloc(&idx_r, n * 4); cudaMalloc(&idx_s, n * 4); cudaMalloc(&out, 8);
  std::vector<unsigned> h(n);
  for (long i = 0; i < n; ++i) h[i] = (unsigned)i;
  cudaMemcpy(idx_s, h.data(), n * 4, cudaMemcpyHostToDevice);
  std::mt19937 rng(1); std::shuffle(h.begin(), h.end(), rng);
  cudaMemcpy(idx_r, h.data(), n * 4, cudaMemcpyHostToDevice);
  for (int c : {2, 4, 8}) {
    run<36, 1>("random 288B", src, idx_r, n, out, c);
    run<36, 2>("random 288B", src, idx_r, n, out, c);
    run<36, 4>("random 288B", src, idx_r, n, out, c);
    run<36, 8>("random 288B", src, idx_r, n, out, c);
    run<36, 4>("sequential 288B", src, idx_s, n, out, c);
  }
  run<27, 4>("random 216B", src, idx_r, n, out, 8);
  run<18, 4>("random 144B", src, idx_r, n, out, 8);
  run<9, 4>("random 72B", src, idx_r, n, out, 8);
  return 0;
}
