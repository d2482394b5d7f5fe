// Lagged smooth Coulomb friction (friction.py), batched over the contact table.
//
//   friction_state_kernel  update_friction_state (friction.py:148-171): once per time step, per
//     stencil: distance branch + witness weights (_witness_coefficients, :85-117), contact normal
//     from the one-sided gradient of d2 and the tangent frame (build_basis, :128-145; _tangent_frame,
//     :120-125), lambda_n = |sum of side A's raw barrier gradient|.  The sliding basis T (3s x 2) has
//     T[3v:3v+3, k] = cn_v t_k with cn = coeffs / |coeffs|, so a "frame" of 12 doubles per datum
//     (cn[4], t1[3], t2[3], lambda_n, 0) holds it without materialising T.
//   friction_blocks_kernel<S>  per Newton iteration, per datum: u = T^T (x - x_start)
//     (tangential_displacement, :174-178), the potential mu lambda_n f0(|u|) (:49-52), the gradient
//     -dt^2 force = dt^2 mu lambda_n f1/|u| T u (:55-61, solver.py:210-213) and the PSD block
//     dt^2 mu lambda_n T core T^T (:64-82).  The 2x2 core has eigenpairs (max(f1',0), u^) and
//     (max(f1/|u|,0), u^perp), so the block is w_p p p^T + w_q q q^T with p = T u^, q = T u^perp
//     -- closed form, rank 2, no eigendecomposition.  Thread per datum for the scalars, then the tile's
//     (ntile, D, D) blocks leave as one contiguous span with consecutive lanes on consecutive doubles.
//   friction_explicit_kernel  the per-datum entry points potential / friction_force /
//     friction_hessian_psd(datum, u) with an explicit basis and u (parity twins, n rows).
#include "stencil_math.cuh"
#include "launch.cuh"

namespace b200ipc {

constexpr int kFT = 128;

struct FrictionStateArgs {
  int64_t n;
  int64_t kind_off[B200IPC_NKINDS + 1];
  const int32_t* verts;        // (n,4)
  const uint8_t* sub;
  const double* positions;
  const double* grad[B200IPC_NKINDS];   // raw barrier gradient, first row of each kind inside its family array
  double* frame;               // (n,12)
  uint8_t* status;             // 0 datum, 1 skipped (d2 <= 0 or lambda_n <= 0), 3 undefined normal
};

__device__ __forceinline__ int kind_of_row(const int64_t* off, int64_t i) {
  int k = 0;
#pragma unroll
  for (int q = 1; q < B200IPC_NKINDS; ++q)
    if (i >= off[q]) k = q;
  return k;
}

template <int KIND>
__device__ __forceinline__ void friction_state_row(const FrictionStateArgs& a, int64_t i, int64_t local_row) {
  constexpr int S = (KIND == B200IPC_PP) ? 2 : (KIND == B200IPC_PE ? 3 : 4);
  const int4 id = reinterpret_cast<const int4*>(a.verts)[i];
  const int v[4] = {id.x, id.y, id.z, id.w};
  V3 x[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = k < S ? load3(a.positions, v[k]) : vzero();
  const int sb = a.sub[i];
  V3 gd[4];
  double w0, w1;
  const double d2 = eval_distance<KIND>(x, sb, gd, w0, w1);
  double* fr = a.frame + 12 * i;
#pragma unroll
  for (int k = 0; k < 12; ++k) fr[k] = 0.0;
  if (!(d2 > 0.0)) {
    a.status[i] = 1;
    return;
  }
  // witness coefficients and side A (friction.py:85-117)
  double co[4] = {0.0, 0.0, 0.0, 0.0};
  bool side[4] = {false, false, false, false};
  if (KIND == B200IPC_PP) {
    co[0] = 1.0; co[1] = -1.0; side[0] = true;
  } else if (KIND == B200IPC_PE) {
    co[0] = 1.0; co[1] = -(1.0 - w0); co[2] = -w0; side[0] = true;
  } else if (KIND == B200IPC_PT) {
    co[0] = 1.0; co[1] = -(1.0 - w0 - w1); co[2] = -w0; co[3] = -w1; side[0] = true;
  } else if (KIND == B200IPC_EE) {
    co[0] = 1.0 - w0; co[1] = w0; co[2] = -(1.0 - w1); co[3] = -w1; side[0] = side[1] = true;
  } else {
    const int loc[4] = {sb & 3, (sb >> 2) & 3, (sb >> 4) & 3, (sb >> 6) & 3};
    double lc[4] = {0.0, 0.0, 0.0, 0.0};
    int nl;
    if (KIND == B200IPC_EEP) {
      lc[0] = 1.0 - w0; lc[1] = w0; lc[2] = -(1.0 - w1); lc[3] = -w1; nl = 4;
    } else if (KIND == B200IPC_PEP) {
      lc[0] = 1.0; lc[1] = -(1.0 - w0); lc[2] = -w0; nl = 3;
    } else {
      lc[0] = 1.0; lc[1] = -1.0; nl = 2;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (r < nl) {
#pragma unroll
        for (int l = 0; l < 4; ++l)
          if (loc[r] == l) {
            co[l] = lc[r];
            if (lc[r] > 0.0) side[l] = true;
          }
      }
  }
  V3 one = vzero(), gs = vzero();
  const double* g = a.grad[KIND] + (int64_t)(3 * S) * local_row;
#pragma unroll
  for (int k = 0; k < S; ++k)
    if (side[k]) {
      one = one + gd[k];
      gs = gs + V3{g[3 * k], g[3 * k + 1], g[3 * k + 2]};
    }
  const double d = sqrt(d2);
  V3 nrm = {one.x / (2.0 * d), one.y / (2.0 * d), one.z / (2.0 * d)};
  const double nn = sqrt(dot3(nrm, nrm));
  if (nn == 0.0) {
    a.status[i] = 3;
    return;
  }
  nrm = {nrm.x / nn, nrm.y / nn, nrm.z / nn};
  // _tangent_frame: reference axis = the smallest |component| (first on ties)
  const double ax = fabs(nrm.x), ay = fabs(nrm.y), az = fabs(nrm.z);
  int m = 0;
  double best = ax;
  if (ay < best) { best = ay; m = 1; }
  if (az < best) { m = 2; }
  const V3 ref = {m == 0 ? 1.0 : 0.0, m == 1 ? 1.0 : 0.0, m == 2 ? 1.0 : 0.0};
  V3 t1 = cross3(nrm, ref);
  const double n1 = sqrt(dot3(t1, t1));
  t1 = {t1.x / n1, t1.y / n1, t1.z / n1};
  const V3 t2 = cross3(nrm, t1);
  const double lam = sqrt(dot3(gs, gs));
  if (!(lam > 0.0)) {
    a.status[i] = 1;
    return;
  }
  const double cnorm = sqrt(co[0] * co[0] + co[1] * co[1] + co[2] * co[2] + co[3] * co[3]);
#pragma unroll
  for (int k = 0; k < 4; ++k) fr[k] = co[k] / cnorm;
  fr[4] = t1.x; fr[5] = t1.y; fr[6] = t1.z;
  fr[7] = t2.x; fr[8] = t2.y; fr[9] = t2.z;
  fr[10] = lam;
  a.status[i] = 0;
}

__global__ void __launch_bounds__(kFT) friction_state_kernel(const __grid_constant__ FrictionStateArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kFT + threadIdx.x;
  if (i >= a.n) return;
  const int k = kind_of_row(a.kind_off, i);
  const int64_t lr = i - a.kind_off[k];
  switch (k) {
    case B200IPC_EE: friction_state_row<B200IPC_EE>(a, i, lr); break;
    case B200IPC_EEP: friction_state_row<B200IPC_EEP>(a, i, lr); break;
    case B200IPC_PE: friction_state_row<B200IPC_PE>(a, i, lr); break;
    case B200IPC_PEP: friction_state_row<B200IPC_PEP>(a, i, lr); break;
    case B200IPC_PP: friction_state_row<B200IPC_PP>(a, i, lr); break;
    case B200IPC_PPP: friction_state_row<B200IPC_PPP>(a, i, lr); break;
    default: friction_state_row<B200IPC_PT>(a, i, lr); break;
  }
}

// f0_f1 (friction.py:33-46)
__device__ __forceinline__ void f0_f1(double un, double h, double& f0, double& f1, double& f1p) {
  if (un >= h) {
    f0 = un; f1 = 1.0; f1p = 0.0;
    return;
  }
  f1 = -un * un / (h * h) + 2.0 * un / h;
  f1p = -2.0 * un / (h * h) + 2.0 / h;
  f0 = -(un * un * un) / (3.0 * h * h) + un * un / h + h / 3.0;
}

// weights of the rank-2 block and direction pair (u^, u^perp); returns the gradient factor f1/|u|
__device__ __forceinline__ double friction_core(double u0, double u1, double h, double& f0, double& wp, double& wq,
                                                double& c0, double& c1) {
  const double un = sqrt(u0 * u0 + u1 * u1);
  double f1, f1p;
  f0_f1(un, h, f0, f1, f1p);
  if (un == 0.0) {  // isotropic core 2/(eps_v dt) I (friction.py:71-72); no force
    wp = wq = 2.0 / h;
    c0 = 1.0;
    c1 = 0.0;
    return 0.0;
  }
  c0 = u0 / un;
  c1 = u1 / un;
  wp = fmax(f1p, 0.0);
  wq = fmax(f1 / un, 0.0);
  return f1 / un;
}

struct Segs {
  int32_t nseg;
  int64_t start[5];   // first table row of each segment
  int64_t count[5];
};

struct FrictionBlockArgs {
  int64_t nb;                // rows of this family
  Segs segs;                 // family row -> table row
  const int32_t* verts;      // (n,4)
  const double* frame;       // (n,12)
  const double* x;
  const double* x_start;
  double mu, h, dt2;         // h = dt * eps_v
  double* energy;            // (n) by table row, may be NULL
  double* grad;              // (nb, D) may be NULL
  double* hess;              // (nb, D, D) may be NULL
};

template <int S>
__global__ void __launch_bounds__(kFT) friction_blocks_kernel(const __grid_constant__ FrictionBlockArgs a) {
  constexpr int D = 3 * S;
  __shared__ double sp[D][kFT + 1], sq[D][kFT + 1], sg[D][kFT + 1];
  const int64_t tile0 = (int64_t)blockIdx.x * kFT;
  const int ntile = (int)min((int64_t)kFT, a.nb - tile0);
  const int t = threadIdx.x;
  if (t < ntile) {
    int64_t r = tile0 + t, row = 0;
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (q < a.segs.nseg) {
        if (r >= 0 && r < a.segs.count[q]) { row = a.segs.start[q] + r; r = -1; }
        else if (r >= 0) r -= a.segs.count[q];
      }
    const int4 id = reinterpret_cast<const int4*>(a.verts)[row];
    const int v[4] = {id.x, id.y, id.z, id.w};
    const double* fr = a.frame + 12 * row;
    const V3 t1 = {fr[4], fr[5], fr[6]}, t2 = {fr[7], fr[8], fr[9]};
    const double lam = fr[10];
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const V3 rel = load3(a.x, v[k]) - load3(a.x_start, v[k]);
      u0 += fr[k] * dot3(t1, rel);
      u1 += fr[k] * dot3(t2, rel);
    }
    double f0, wp, wq, c0, c1;
    const double gf = friction_core(u0, u1, a.h, f0, wp, wq, c0, c1);
    const double ml = a.mu * lam;
    if (a.energy) a.energy[row] = ml * f0;
    const double sp_ = sqrt(a.dt2 * ml * wp), sq_ = sqrt(a.dt2 * ml * wq);
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const V3 tu = {t1.x * u0 + t2.x * u1, t1.y * u0 + t2.y * u1, t1.z * u0 + t2.z * u1};   // T u (per vertex / cn)
      const V3 pv = {t1.x * c0 + t2.x * c1, t1.y * c0 + t2.y * c1, t1.z * c0 + t2.z * c1};   // T u^
      const V3 qv = {t2.x * c0 - t1.x * c1, t2.y * c0 - t1.y * c1, t2.z * c0 - t1.z * c1};   // T u^perp
      const double cn = fr[k];
      sp[3 * k][t] = sp_ * cn * pv.x; sp[3 * k + 1][t] = sp_ * cn * pv.y; sp[3 * k + 2][t] = sp_ * cn * pv.z;
      sq[3 * k][t] = sq_ * cn * qv.x; sq[3 * k + 1][t] = sq_ * cn * qv.y; sq[3 * k + 2][t] = sq_ * cn * qv.z;
      const double gk = a.dt2 * ml * gf * cn;
      sg[3 * k][t] = gk * tu.x; sg[3 * k + 1][t] = gk * tu.y; sg[3 * k + 2][t] = gk * tu.z;
    }
  }
  __syncthreads();
  if (a.hess) {
    double* out = a.hess + tile0 * (D * D);
    for (int e = t; e < ntile * D * D; e += kFT) {
      const int i = e / (D * D), rc = e - i * (D * D);
      const int r = rc / D, c = rc - r * D;
      out[e] = sp[r][i] * sp[c][i] + sq[r][i] * sq[c][i];
    }
  }
  if (a.grad) {
    double* out = a.grad + tile0 * D;
    for (int e = t; e < ntile * D; e += kFT) {
      const int i = e / D, r = e - i * D;
      out[e] = sg[r][i];
    }
  }
}

// potential / friction_force / friction_hessian_psd with an explicit basis T (n, 3s, 2) and u (n, 2)
struct FrictionExplicitArgs {
  int64_t n;
  int32_t s;
  const double* basis;     // (n, 3s, 2)
  const double* u;         // (n, 2)
  const double* lambda_n;  // (n)
  double mu, h;
  double* potential;       // (n)
  double* force;           // (n, 3s)
  double* hess;            // (n, 3s, 3s)
};

__global__ void __launch_bounds__(kFT) friction_explicit_kernel(const __grid_constant__ FrictionExplicitArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kFT + threadIdx.x;
  if (i >= a.n) return;
  const int D = 3 * a.s;
  const double u0 = a.u[2 * i], u1 = a.u[2 * i + 1];
  double f0, wp, wq, c0, c1;
  const double gf = friction_core(u0, u1, a.h, f0, wp, wq, c0, c1);
  const double ml = a.mu * a.lambda_n[i];
  if (a.potential) a.potential[i] = ml * f0;
  const double* T = a.basis + (int64_t)i * D * 2;
  if (a.force)
    for (int r = 0; r < D; ++r) a.force[i * D + r] = -ml * gf * (T[2 * r] * u0 + T[2 * r + 1] * u1);
  if (a.hess)
    for (int r = 0; r < D; ++r) {
      const double pr = T[2 * r] * c0 + T[2 * r + 1] * c1, qr = T[2 * r + 1] * c0 - T[2 * r] * c1;
      for (int c = 0; c < D; ++c) {
        const double pc = T[2 * c] * c0 + T[2 * c + 1] * c1, qc = T[2 * c + 1] * c0 - T[2 * c] * c1;
        a.hess[(i * D + r) * D + c] = ml * (wp * pr * pc + wq * qr * qc);
      }
    }
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_friction_state(int64_t n, const int64_t* kind_off, const int32_t* verts, const uint8_t* sub,
                                      const double* positions, const double* grad2, const double* grad3,
                                      const double* grad4, double* frame, uint8_t* status, void* stream) {
  if (n < 0 || !kind_off) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!verts || !sub || !positions || !frame || !status) return B200IPC_EINVAL;
  if (((uintptr_t)verts) & 15) return B200IPC_EINVAL;
  FrictionStateArgs a;
  a.n = n;
  for (int k = 0; k <= B200IPC_NKINDS; ++k) a.kind_off[k] = kind_off[k];
  if (kind_off[0] != 0 || kind_off[B200IPC_NKINDS] != n) return B200IPC_EINVAL;
  a.verts = verts; a.sub = sub; a.positions = positions; a.frame = frame; a.status = status;
  // family layout of group_blocks: s = 2: PP; s = 3: PE; s = 4: EE, EEP, PEP, PPP, PT in that order
  const int fam4[5] = {B200IPC_EE, B200IPC_EEP, B200IPC_PEP, B200IPC_PPP, B200IPC_PT};
  for (int k = 0; k < B200IPC_NKINDS; ++k) a.grad[k] = nullptr;
  a.grad[B200IPC_PP] = grad2;
  a.grad[B200IPC_PE] = grad3;
  int64_t row4 = 0;
  for (int q = 0; q < 5; ++q) {
    const int k = fam4[q];
    const int64_t cnt = kind_off[k + 1] - kind_off[k];
    if (cnt < 0) return B200IPC_EINVAL;
    a.grad[k] = grad4 ? grad4 + 12 * row4 : nullptr;
    row4 += cnt;
  }
  for (int k = 0; k < B200IPC_NKINDS; ++k)
    if (kind_off[k + 1] > kind_off[k] && !a.grad[k]) return B200IPC_EINVAL;
  friction_state_kernel<<<(unsigned)((n + kFT - 1) / kFT), kFT, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}

extern "C" int b200ipc_friction_blocks(int64_t n, const int64_t* kind_off, const int32_t* verts, const double* frame,
                                       const double* x, const double* x_start, double mu, double eps_v, double dt,
                                       double* energy, double* grad2, double* hess2, double* grad3, double* hess3,
                                       double* grad4, double* hess4, void* stream) {
  if (n < 0 || !kind_off) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!verts || !frame || !x || !x_start || !(mu >= 0.0) || !(eps_v > 0.0) || !(dt > 0.0)) return B200IPC_EINVAL;
  if (((uintptr_t)verts) & 15) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int fam_kinds[3][5] = {{B200IPC_PP, -1, -1, -1, -1},
                               {B200IPC_PE, -1, -1, -1, -1},
                               {B200IPC_EE, B200IPC_EEP, B200IPC_PEP, B200IPC_PPP, B200IPC_PT}};
  double* grads[3] = {grad2, grad3, grad4};
  double* hesss[3] = {hess2, hess3, hess4};
  for (int f = 0; f < 3; ++f) {
    FrictionBlockArgs a;
    a.segs.nseg = 0;
    a.nb = 0;
    for (int q = 0; q < 5; ++q) {
      const int k = fam_kinds[f][q];
      if (k < 0) continue;
      a.segs.start[a.segs.nseg] = kind_off[k];
      a.segs.count[a.segs.nseg] = kind_off[k + 1] - kind_off[k];
      a.nb += a.segs.count[a.segs.nseg];
      ++a.segs.nseg;
    }
    for (int q = a.segs.nseg; q < 5; ++q) a.segs.start[q] = a.segs.count[q] = 0;
    if (a.nb == 0) continue;
    a.verts = verts; a.frame = frame; a.x = x; a.x_start = x_start;
    a.mu = mu; a.h = dt * eps_v; a.dt2 = dt * dt;
    a.energy = energy; a.grad = grads[f]; a.hess = hesss[f];
    const unsigned grid = (unsigned)((a.nb + kFT - 1) / kFT);
    if (f == 0) friction_blocks_kernel<2><<<grid, kFT, 0, st>>>(a);
    else if (f == 1) friction_blocks_kernel<3><<<grid, kFT, 0, st>>>(a);
    else friction_blocks_kernel<4><<<grid, kFT, 0, st>>>(a);
    int rc = post_launch();
    if (rc) return rc;
  }
  return 0;
}

extern "C" int b200ipc_friction_explicit(int64_t n, int32_t s, const double* basis, const double* u,
                                         const double* lambda_n, double mu, double eps_v, double dt,
                                         double* potential, double* force, double* hess, void* stream) {
  if (n < 0 || s < 2 || s > 4) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!basis || !u || !lambda_n || !(eps_v > 0.0) || !(dt > 0.0)) return B200IPC_EINVAL;
  FrictionExplicitArgs a{n, s, basis, u, lambda_n, mu, dt * eps_v, potential, force, hess};
  friction_explicit_kernel<<<(unsigned)((n + kFT - 1) / kFT), kFT, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}
