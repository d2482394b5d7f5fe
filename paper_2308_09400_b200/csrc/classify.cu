// tetipc.kernels twins: pt_classify_batch, ee_classify_batch, cross_sq_batch
// (kernels/_core.pyx:46-219).  Thread-per-query; inputs are four (n,3) row-major arrays.
// A CTA reads its queries' coordinates as flat contiguous spans (coalesced), evaluates in
// registers, and writes grad (n,4,3) through shared memory so the 96-byte rows leave as
// full-width consecutive stores.
#include "geom.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kCT = 128;

enum { OP_PT = 0, OP_EE = 1, OP_CROSS = 2 };

struct ClassifyArgs {
  int64_t n;
  const double* in[4];
  int64_t* codes;
  double* d2;
  double* grad;
  double* w;
};

template <int OP>
__global__ void __launch_bounds__(kCT) classify_kernel(const ClassifyArgs a) {
  __shared__ double sm[kCT * 12 + 4];
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kCT;
  const int64_t left = a.n - base;
  const int cnt = left < kCT ? (int)left : kCT;

  // stage the four coordinate spans through shared memory: coalesced global reads
  V3 x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double* src = a.in[j] + 3 * base;
    for (int e = tid; e < 3 * cnt; e += kCT) sm[e] = __ldg(src + e);
    __syncthreads();
    if (tid < cnt) x[j] = {sm[3 * tid], sm[3 * tid + 1], sm[3 * tid + 2]};
    __syncthreads();
  }

  V3 g[4];
  if (tid < cnt) {
    const int64_t i = base + tid;
    if (OP == OP_CROSS) {
      const double c = cross_sq_one(x[0], x[1], x[2], x[3], g);
      if (a.d2) a.d2[i] = c;
    } else {
      double d2, w1, w2;
      const int code = OP == OP_PT ? pt_one(x[0], x[1], x[2], x[3], d2, g, w1, w2)
                                   : ee_one(x[0], x[1], x[2], x[3], d2, g, w1, w2);
      if (a.codes) a.codes[i] = code;
      if (a.d2) a.d2[i] = d2;
      if (a.w) *reinterpret_cast<double2*>(a.w + 2 * i) = make_double2(w1, w2);
    }
    if (a.grad) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        sm[12 * tid + 3 * v + 0] = g[v].x;
        sm[12 * tid + 3 * v + 1] = g[v].y;
        sm[12 * tid + 3 * v + 2] = g[v].z;
      }
    }
  }
  if (a.grad) {
    __syncthreads();
    double* out = a.grad + 12 * base;
    for (int e = 2 * tid; e < 12 * cnt; e += 2 * kCT)
      *reinterpret_cast<double2*>(out + e) = make_double2(sm[e], sm[e + 1]);
  }
}

template <int OP>
static int launch_classify(int64_t n, const double* i0, const double* i1, const double* i2, const double* i3,
                           int64_t* codes, double* d2, double* grad, double* w, void* stream) {
  if (n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!i0 || !i1 || !i2 || !i3) return B200IPC_EINVAL;
  if (((uintptr_t)grad | (uintptr_t)w) & 15) return B200IPC_EINVAL;
  ClassifyArgs a{n, {i0, i1, i2, i3}, codes, d2, grad, w};
  const unsigned grid = (unsigned)((n + kCT - 1) / kCT);
  classify_kernel<OP><<<grid, kCT, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_pt_classify(int64_t n, const double* p, const double* t1, const double* t2, const double* t3,
                                   int64_t* codes, double* d2, double* grad, double* w, void* stream) {
  return launch_classify<OP_PT>(n, p, t1, t2, t3, codes, d2, grad, w, stream);
}

extern "C" int b200ipc_ee_classify(int64_t n, const double* a1, const double* a2, const double* b1, const double* b2,
                                   int64_t* codes, double* d2, double* grad, double* w, void* stream) {
  return launch_classify<OP_EE>(n, a1, a2, b1, b2, codes, d2, grad, w, stream);
}

extern "C" int b200ipc_cross_sq(int64_t n, const double* a1, const double* a2, const double* b1, const double* b2,
                                double* c, double* grad, void* stream) {
  return launch_classify<OP_CROSS>(n, a1, a2, b1, b2, nullptr, c, grad, nullptr, stream);
}
