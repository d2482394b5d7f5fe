// Per-stencil entry points of the reference kept as batched kernels (n is usually small):
//   b200ipc_diagonal_jacobian    <- stencil_distance + parallel_measure + build_diagonal_jacobian
//   b200ipc_blocks_from_jacobian <- build_local_quadratic / build_mollified_local_quadratic
//   b200ipc_barrier_scalars      <- barrier_value/dg/d2g, lambda1, lambda23, filtered_lambda1
//   b200ipc_mollified_eigensystem<- mollified_eigensystem
// They reuse the device functions of the fused kernel, so the shims and the hot path cannot
// drift apart.  Thread-per-row with direct stores: these are API-parity paths, not the hot path.
#include "stencil_math.cuh"
#include "launch.cuh"

namespace b200ipc {

constexpr int kDT = 128;

__device__ __forceinline__ void store_rows(double* dst, const V3 g[4]) {
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    dst[3 * v + 0] = g[v].x;
    dst[3 * v + 1] = g[v].y;
    dst[3 * v + 2] = g[v].z;
  }
}

struct JacArgs {
  b200ipc_params prm;
  const double* positions;
  int64_t n;
  const uint8_t* kind;
  const int32_t* verts;
  const uint8_t* sub;
  double *d2, *grad_d2, *witness, *f, *grad_f, *c, *grad_c, *sqrt_c, *grad_sqrt_c;
  uint8_t* status;
};

__global__ void __launch_bounds__(kDT) diagonal_jacobian_kernel(const JacArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kDT + threadIdx.x;
  if (i >= a.n) return;
  const int kind = a.kind[i];
  const int4 vid = reinterpret_cast<const int4*>(a.verts)[i];
  const int s = (kind == B200IPC_PP) ? 2 : (kind == B200IPC_PE ? 3 : 4);
  V3 x[4];
  x[0] = load3(a.positions, vid.x);
  x[1] = load3(a.positions, vid.y);
  x[2] = s >= 3 ? load3(a.positions, vid.z) : vzero();
  x[3] = s >= 4 ? load3(a.positions, vid.w) : vzero();
  const int sb = a.sub ? a.sub[i] : 0;
  V3 gd[4];
  double d2, w0, w1;
  switch (kind) {
    case B200IPC_EE: d2 = eval_distance<B200IPC_EE>(x, sb, gd, w0, w1); break;
    case B200IPC_EEP: d2 = eval_distance<B200IPC_EEP>(x, sb, gd, w0, w1); break;
    case B200IPC_PE: d2 = eval_distance<B200IPC_PE>(x, sb, gd, w0, w1); break;
    case B200IPC_PEP: d2 = eval_distance<B200IPC_PEP>(x, sb, gd, w0, w1); break;
    case B200IPC_PP: d2 = eval_distance<B200IPC_PP>(x, sb, gd, w0, w1); break;
    case B200IPC_PPP: d2 = eval_distance<B200IPC_PPP>(x, sb, gd, w0, w1); break;
    default: d2 = eval_distance<B200IPC_PT>(x, sb, gd, w0, w1); break;
  }
  if (a.d2) a.d2[i] = d2;
  if (a.grad_d2) store_rows(a.grad_d2 + 12 * i, gd);
  if (a.witness) {
    a.witness[2 * i] = w0;
    a.witness[2 * i + 1] = w1;
  }
  // gap.py:61-64 compares against d_hat*d_hat
  if (a.status)
    a.status[i] = d2 <= 0.0 ? B200IPC_PENETRATION : (d2 >= a.prm.d_hat_sq ? B200IPC_INACTIVE : B200IPC_ACTIVE);
  const double d = sqrt(d2);
  if (a.f) a.f[i] = d / a.prm.d_hat;
  if (a.grad_f) {
    // gap.py:67: grad_d2 / (2 d d_hat), a true division per entry
    const double den = 2.0 * d * a.prm.d_hat;
    V3 gf[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) gf[v] = {gd[v].x / den, gd[v].y / den, gd[v].z / den};
    store_rows(a.grad_f + 12 * i, gf);
  }
  const bool par = kind == B200IPC_EEP || kind == B200IPC_PEP || kind == B200IPC_PPP;
  if (par) {
    V3 gc[4];
    const double c = cross_sq_one(x[0], x[1], x[2], x[3], gc);
    const double sc = sqrt(c);
    if (a.c) a.c[i] = c;
    if (a.grad_c) store_rows(a.grad_c + 12 * i, gc);
    if (a.sqrt_c) a.sqrt_c[i] = sc;
    if (a.grad_sqrt_c) {
      V3 gs[4];
      const double den = 2.0 * sc;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        gs[v] = sc > 0.0 ? V3{gc[v].x / den, gc[v].y / den, gc[v].z / den} : vzero();
      store_rows(a.grad_sqrt_c + 12 * i, gs);
    }
  }
}

struct BlkArgs {
  b200ipc_params prm;
  int64_t n;
  const uint8_t* kind;
  const double *f, *grad_f, *sqrt_c, *grad_sqrt_c, *eps_x;
  double *grad, *hess;
};

// One CTA row of 144 threads per stencil: thread (r,c) writes hess[r][c]; reference op order
// lam * (u_r*u_c) then * dt2, so the n = 1 shims agree with the reference to the last bits.
__global__ void __launch_bounds__(144) blocks_from_jacobian_kernel(const BlkArgs a) {
  const int64_t i = blockIdx.x;
  const int kind = a.kind[i];
  const bool par = kind == B200IPC_EEP || kind == B200IPC_PEP || kind == B200IPC_PPP;
  const double f = a.f[i];
  Coef k;
  if (!par) {
    k = a.prm.form == 0 ? coef_plain<0>(a.prm, f) : coef_plain<1>(a.prm, f);
  } else {
    const double sc = a.sqrt_c[i], eps = a.eps_x[i];
    k = a.prm.form == 0 ? coef_parallel<0>(a.prm, f, sc, eps) : coef_parallel<1>(a.prm, f, sc, eps);
  }
  const int r = threadIdx.x / 12, c = threadIdx.x % 12;
  const double* uf = a.grad_f + 12 * i;
  const double* uc = par ? a.grad_sqrt_c + 12 * i : nullptr;
  const double wr = par ? k.cw_c * uc[r] + k.cw_f * uf[r] : uf[r];
  const double wc = par ? k.cw_c * uc[c] + k.cw_f * uf[c] : uf[c];
  if (a.hess) a.hess[144 * i + threadIdx.x] = a.prm.dt2 * (k.lam * (wr * wc));
  if (a.grad && threadIdx.x < 12) {
    const int q = threadIdx.x;
    const double gr = par ? k.cg_c * uc[q] + k.cg_f * uf[q] : k.cg_f * uf[q];
    a.grad[12 * i + q] = a.prm.dt2 * gr;
  }
}

__global__ void __launch_bounds__(kDT) barrier_scalars_kernel(b200ipc_params prm, int64_t n,
                                                              const double* __restrict__ g, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kDT + threadIdx.x;
  if (i >= n) return;
  const double gi = g[i];
  const Barrier s = prm.form == 0 ? barrier_scalars<0>(gi, prm.scale) : barrier_scalars<1>(gi, prm.scale);
  const double l1 = lambda1_of(gi, s);
  double lf = l1;
  if (prm.use_filter && !(gi >= prm.eps_g)) {
    const Barrier t = prm.form == 0 ? barrier_scalars<0>(prm.eps_g, prm.scale) : barrier_scalars<1>(prm.eps_g, prm.scale);
    lf = lambda1_of(prm.eps_g, t);
  }
  double* o = out + 6 * i;
  o[0] = s.b;
  o[1] = s.bg;
  o[2] = s.bgg;
  o[3] = l1;
  o[4] = 2.0 * s.bg;
  o[5] = lf;
}

__global__ void __launch_bounds__(kDT) mollified_eig_kernel(b200ipc_params prm, int64_t n, const double* __restrict__ g,
                                                            const double* __restrict__ c,
                                                            const double* __restrict__ eps, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kDT + threadIdx.x;
  if (i >= n) return;
  const MollEig m = prm.form == 0 ? mollified_eig<0>(prm.scale, g[i], c[i], eps[i])
                                  : mollified_eig<1>(prm.scale, g[i], c[i], eps[i]);
  double e, de, d2e;
  mollifier_eval(c[i], eps[i], e, de, d2e);
  double* o = out + 12 * i;
  o[0] = m.lg1; o[1] = m.lf1; o[2] = m.t; o[3] = m.p; o[4] = m.lam7; o[5] = m.lam8;
  o[6] = m.q_c; o[7] = m.q_f; o[8] = m.b_gamma; o[9] = m.b_g; o[10] = e; o[11] = de;
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_diagonal_jacobian(const b200ipc_params* params, int64_t nverts, const double* positions,
                                         int64_t n, const uint8_t* kind, const int32_t* verts, const uint8_t* sub,
                                         double* d2, double* grad_d2, double* witness, double* f, double* grad_f,
                                         double* c, double* grad_c, double* sqrt_c, double* grad_sqrt_c,
                                         uint8_t* status, void* stream) {
  if (!params || n < 0 || nverts < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!positions || !kind || !verts || ((uintptr_t)verts & 15)) return B200IPC_EINVAL;
  JacArgs a{*params, positions, n, kind, verts, sub, d2, grad_d2, witness, f, grad_f, c, grad_c, sqrt_c,
            grad_sqrt_c, status};
  diagonal_jacobian_kernel<<<(unsigned)((n + kDT - 1) / kDT), kDT, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}

extern "C" int b200ipc_blocks_from_jacobian(const b200ipc_params* params, int64_t n, const uint8_t* kind,
                                            const double* f, const double* grad_f, const double* sqrt_c,
                                            const double* grad_sqrt_c, const double* eps_x, double* grad,
                                            double* hess, void* stream) {
  if (!params || n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!kind || !f || !grad_f) return B200IPC_EINVAL;
  BlkArgs a{*params, n, kind, f, grad_f, sqrt_c, grad_sqrt_c, eps_x, grad, hess};
  blocks_from_jacobian_kernel<<<(unsigned)n, 144, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}

extern "C" int b200ipc_barrier_scalars(const b200ipc_params* params, int64_t n, const double* g, double* out,
                                       void* stream) {
  if (!params || n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!g || !out) return B200IPC_EINVAL;
  barrier_scalars_kernel<<<(unsigned)((n + kDT - 1) / kDT), kDT, 0, (cudaStream_t)stream>>>(*params, n, g, out);
  return post_launch();
}

extern "C" int b200ipc_mollified_eigensystem(const b200ipc_params* params, int64_t n, const double* g,
                                             const double* c, const double* eps_x, double* out, void* stream) {
  if (!params || n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!g || !c || !eps_x || !out) return B200IPC_EINVAL;
  mollified_eig_kernel<<<(unsigned)((n + kDT - 1) / kDT), kDT, 0, (cudaStream_t)stream>>>(*params, n, g, c, eps_x, out);
  return post_launch();
}
