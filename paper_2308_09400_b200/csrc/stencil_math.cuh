// Per-stencil math shared by the fused hot kernel (stencil.cu) and the per-stencil
// entry-point kernels (diag.cu): distance branch per kind, barrier / mollified coefficients.
#pragma once

#include "geom.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

__device__ __forceinline__ V3 pick(const V3 x[4], int loc) {
  V3 r = x[0];
  if (loc == 1) r = x[1];
  if (loc == 2) r = x[2];
  if (loc == 3) r = x[3];
  return r;
}

// full[l] = rows[j] where loc[j] == l, else zero (proximity.py:219-221)
template <int NR>
__device__ __forceinline__ void unpick(const V3* rows, const int* loc, V3 full[4]) {
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    V3 v = vzero();
#pragma unroll
    for (int j = NR - 1; j >= 0; --j)
      if (loc[j] == l) v = rows[j];
    full[l] = v;
  }
}

// d2 and its gradient padded to four rows (stencil_distance, proximity.py:183-222); wit = the
// branch witness ((w1,w2), (s,t) or (t,-)).
template <int KIND>
__device__ __forceinline__ double eval_distance(const V3 x[4], int sb, V3 gd[4], double& wit0, double& wit1) {
  double d2;
  wit0 = wit1 = 0.0;
  gd[2] = gd[3] = vzero();
  if (KIND == B200IPC_PP) {
    d2 = pp_one(x[0], x[1], gd);
  } else if (KIND == B200IPC_PE) {
    d2 = pe_one(x[0], x[1], x[2], gd, wit0);
  } else if (KIND == B200IPC_PT) {
    pt_one(x[0], x[1], x[2], x[3], d2, gd, wit0, wit1);
  } else if (KIND == B200IPC_EE) {
    ee_one(x[0], x[1], x[2], x[3], d2, gd, wit0, wit1);
  } else {
    const int loc[4] = {sb & 3, (sb >> 2) & 3, (sb >> 4) & 3, (sb >> 6) & 3};
    V3 rows[4];
    if (KIND == B200IPC_EEP) {
      ee_one(pick(x, loc[0]), pick(x, loc[1]), pick(x, loc[2]), pick(x, loc[3]), d2, rows, wit0, wit1);
      unpick<4>(rows, loc, gd);
    } else if (KIND == B200IPC_PEP) {
      d2 = pe_one(pick(x, loc[0]), pick(x, loc[1]), pick(x, loc[2]), rows, wit0);
      unpick<3>(rows, loc, gd);
    } else {
      d2 = pp_one(pick(x, loc[0]), pick(x, loc[1]), rows);
      unpick<2>(rows, loc, gd);
    }
  }
  return d2;
}

// Scalars of the local quadratic: block = lam * w w^T, gradient = cg_c * grad sqrt(c) + cg_f * grad f,
// w = cw_c * grad sqrt(c) + cw_f * grad f.
struct Coef {
  double lam, cw_f, cw_c, cg_f, cg_c;
};

// Plain kinds: build_local_quadratic (barrier.py:172-176) with the proximal filter (:114-120).
template <int FORM>
__device__ __forceinline__ Coef coef_plain(const b200ipc_params& prm, double f) {
  const double g = f * f;
  const Barrier bs = barrier_scalars<FORM>(g, prm.scale);
  double l1 = lambda1_of(g, bs);
  if (prm.use_filter && !(g >= prm.eps_g)) l1 = lambda1_of(prm.eps_g, barrier_scalars<FORM>(prm.eps_g, prm.scale));
  Coef k;
  k.lam = fmax(l1, 0.0);
  k.cg_f = 2.0 * f * bs.bg;
  k.cw_f = 1.0;
  k.cg_c = k.cw_c = 0.0;
  return k;
}

// mollifier_eval (mollifier.py:55-67)
__device__ __forceinline__ void mollifier_eval(double c, double eps, double& e, double& de, double& d2e) {
  e = 1.0;
  de = 0.0;
  d2e = 0.0;
  if (c < eps) {
    e = -(c * c) / (eps * eps) + 2.0 * c / eps;
    de = -2.0 * c / (eps * eps) + 2.0 / eps;
    d2e = -2.0 / (eps * eps);
  }
}

struct MollEig {
  double lg1, lf1, t, p, lam7, lam8, q_c, q_f, b_gamma, b_g;
};

// _channel_derivatives + mollified_eigensystem (mollifier.py:74-86, :106-127); c = sqrt_c^2.
template <int FORM>
__device__ __forceinline__ MollEig mollified_eig(double scale, double g, double cc, double eps) {
  const Barrier bs = barrier_scalars<FORM>(g, scale);
  double e, de, d2e;
  mollifier_eval(cc, eps, e, de, d2e);
  MollEig m;
  m.b_gamma = de * bs.b;
  const double b_gamma2 = d2e * bs.b;
  m.b_g = e * bs.bg;
  const double b_g2 = e * bs.bgg, b_gamma_g = de * bs.bg;
  m.lg1 = 2.0 * (m.b_gamma + 2.0 * cc * b_gamma2);
  m.lf1 = 2.0 * (m.b_g + 2.0 * g * b_g2);
  m.t = b_gamma_g * sqrt(cc) * sqrt(g);
  const double dl = m.lg1 - m.lf1;
  m.p = 0.5 * sqrt(dl * dl + 64.0 * m.t * m.t);
  const double mean = 0.5 * (m.lg1 + m.lf1);
  m.lam7 = mean - m.p;
  m.lam8 = mean + m.p;
  if (fabs(8.0 * m.t) < 1e-12 * (fabs(m.lg1) + fabs(m.lf1)) || m.t == 0.0) {
    // decoupled limit: the 2x2 block is diagonal, k2 is 0/0 (mollifier.py:120-122)
    m.q_c = m.lg1 >= m.lf1 ? 1.0 : 0.0;
    m.q_f = m.lg1 >= m.lf1 ? 0.0 : 1.0;
  } else {
    const double k2 = (dl + 2.0 * m.p) / (8.0 * m.t);
    const double nrm = sqrt(k2 * k2 + 1.0);
    m.q_c = k2 / nrm;
    m.q_f = 1.0 / nrm;
  }
  return m;
}

// Parallel kinds: build_mollified_local_quadratic + mollified_gradient (mollifier.py:89-103, :191-210).
template <int FORM>
__device__ __forceinline__ Coef coef_parallel(const b200ipc_params& prm, double f, double sqrt_c, double eps) {
  const MollEig m = mollified_eig<FORM>(prm.scale, f * f, sqrt_c * sqrt_c, eps);
  Coef k;
  k.lam = fmax(m.lam8, 0.0);
  k.cw_c = m.q_c;
  k.cw_f = m.q_f;
  k.cg_c = m.b_gamma * 2.0 * sqrt_c;
  k.cg_f = m.b_g * 2.0 * f;
  return k;
}

}  // namespace b200ipc
