// matvec_blocks twin (kernels/_core.pyx:222-247): out += scatter(H_b . gather(x)) over one
// size family.  A sub-warp of D = 3s lanes owns a block: lane r streams row r of H_b
// (contiguous D doubles), multiplies with the gathered x held in shared memory, and adds its
// y_r into out with one fp64 reduction per (block,row).  The assembled BSR SpMV (spmv.cu) is the
// production path for PCG; this twin keeps the reference's matrix-free entry point alive.
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kMvThreads = 192;  // multiple of 6, 9 (x: 189 used) and 12

template <int S>
__global__ void __launch_bounds__(kMvThreads) matvec_blocks_kernel(int64_t nb, const double* __restrict__ hess,
                                                                   const int64_t* __restrict__ vids,
                                                                   const double* __restrict__ x,
                                                                   double* __restrict__ out) {
  constexpr int D = 3 * S;
  constexpr int BPC = kMvThreads / D;  // blocks per CTA per pass
  __shared__ double xs[BPC * D];
  const int tid = threadIdx.x;
  const int lb = tid / D, r = tid - lb * D;
  for (int64_t b0 = (int64_t)blockIdx.x * BPC; b0 < nb; b0 += (int64_t)gridDim.x * BPC) {
    const int64_t b = b0 + lb;
    const bool on = lb < BPC && b < nb;
    int64_t gi = 0;
    if (on) {
      gi = vids[b * S + r / 3];
      xs[lb * D + r] = x[3 * gi + (r % 3)];
    }
    __syncthreads();
    if (on) {
      const double* row = hess + (b * D + r) * D;
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) acc += row[c] * xs[lb * D + c];
      atomicAdd(out + 3 * gi + (r % 3), acc);
    }
    __syncthreads();
  }
}

// matvec_matrix_free prologue/epilogue (solver.py:255-261): vin = v with fixed rows zeroed,
// out = m * vin; afterwards out[fixed] = v[fixed].
__global__ void __launch_bounds__(256) matvec_begin_kernel(int64_t n, const double* __restrict__ masses,
                                                           const uint8_t* __restrict__ fixed,
                                                           const double* __restrict__ v, double* __restrict__ vin,
                                                           double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= 3 * n) return;
  const int64_t i = t / 3;
  const double x = fixed[i] ? 0.0 : v[t];
  vin[t] = x;
  out[t] = masses[i] * x;
}

__global__ void __launch_bounds__(256) matvec_end_kernel(int64_t n, const uint8_t* __restrict__ fixed,
                                                         const double* __restrict__ v, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= 3 * n) return;
  if (fixed[t / 3]) out[t] = v[t];
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_matvec_begin(int64_t n, const double* masses, const uint8_t* fixed, const double* v,
                                    double* vin, double* out, void* stream) {
  if (n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!masses || !fixed || !v || !vin || !out) return B200IPC_EINVAL;
  matvec_begin_kernel<<<(unsigned)((3 * n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, masses, fixed, v, vin, out);
  return post_launch();
}

extern "C" int b200ipc_matvec_end(int64_t n, const uint8_t* fixed, const double* v, double* out, void* stream) {
  if (n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!fixed || !v || !out) return B200IPC_EINVAL;
  matvec_end_kernel<<<(unsigned)((3 * n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, fixed, v, out);
  return post_launch();
}

extern "C" int b200ipc_matvec_blocks(int64_t nb, int32_t s, const double* hess, const int64_t* vids, const double* x,
                                     double* out, void* stream) {
  if (nb < 0 || s < 2 || s > 4) return B200IPC_EINVAL;
  if (nb == 0) return 0;
  if (!hess || !vids || !x || !out) return B200IPC_EINVAL;
  const int bpc = kMvThreads / (3 * s);
  int64_t grid = (nb + bpc - 1) / bpc;
  if (grid > 148 * 16) grid = 148 * 16;
  cudaStream_t st = (cudaStream_t)stream;
  if (s == 2) matvec_blocks_kernel<2><<<(unsigned)grid, kMvThreads, 0, st>>>(nb, hess, vids, x, out);
  else if (s == 3) matvec_blocks_kernel<3><<<(unsigned)grid, kMvThreads, 0, st>>>(nb, hess, vids, x, out);
  else matvec_blocks_kernel<4><<<(unsigned)grid, kMvThreads, 0, st>>>(nb, hess, vids, x, out);
  return post_launch();
}
