// FP64 throughput probe: the denominator of the fp64 rooflines bench.py reports for the kernels that are
// compute- rather than HBM-bound (accd_kernel, elastic_blocks_kernel).  SURVEY.md 8d: "fp64 peak to be
// measured on-box with a DFMA microbenchmark".
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kProbeChains = 8;      // independent DFMA chains per thread: covers the pipe latency at 8 warps/SM-part
constexpr int kProbeIters = 4096;    // DFMAs per chain
constexpr int kProbeThreads = 256;

__global__ void __launch_bounds__(kProbeThreads) fp64_probe_kernel(double* sink, double a, double b) {
  double acc[kProbeChains];
#pragma unroll
  for (int k = 0; k < kProbeChains; ++k) acc[k] = (double)(threadIdx.x + k);
#pragma unroll 1
  for (int it = 0; it < kProbeIters; it += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < kProbeChains; ++k) acc[k] = fma(acc[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kProbeChains; ++k) s += acc[k];
  if (s == 123.456) sink[0] = s;   // never true for the probe's constants; keeps the chains alive
}

}  // namespace b200ipc

extern "C" int b200ipc_fp64_probe(double* tflops, void* stream) {
  using namespace b200ipc;
  if (!tflops) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_rc(e);
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_rc(e);
  double* sink = nullptr;
  e = cudaMalloc(&sink, sizeof(double));
  if (e != cudaSuccess) return cuda_rc(e);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ctas = sms * 8 * 4;   // four waves of eight resident CTAs per SM
  float best = 1e30f;
  int rc = 0;
  for (int rep = 0; rep < 6 && rc == 0; ++rep) {   // first pass warms up
    cudaEventRecord(e0, st);
    fp64_probe_kernel<<<ctas, kProbeThreads, 0, st>>>(sink, 1.0000001, 1e-9);
    rc = post_launch();
    cudaEventRecord(e1, st);
    e = cudaEventSynchronize(e1);
    if (e != cudaSuccess) rc = cuda_rc(e);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (rc != 0) return rc;
  const double flops = 2.0 * (double)ctas * kProbeThreads * kProbeChains * kProbeIters;
  *tflops = flops / ((double)best * 1e-3) / 1e12;
  return 0;
}
