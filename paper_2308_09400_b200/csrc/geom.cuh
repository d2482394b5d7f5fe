// Device-side geometry and barrier math shared by the kernels of the barrier hot path.
//
// Compile with -fmad=false: the discrete results (region codes, d2 < d_hat^2, c < eps_x)
// must round like the reference's compiled backend, which is scalar x86-64 code without
// FMA (kernels/_core.pyx, setup.py: -O3 only).  Operation order below is the left-to-right
// order of that file.  dot3_blas() is the one deliberate exception.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b200ipc {

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 vzero() { return {0.0, 0.0, 0.0}; }

// _dot3 (_core.pyx:22-23)
__device__ __forceinline__ double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// np.dot on a 3-vector as the reference's Python call sites evaluate it (proximity.py:172-176,
// :189, :218, :257-259): OpenBLAS ddot's sequential tail loop with FMA contraction.
__device__ __forceinline__ double dot3_blas(V3 a, V3 b) {
  return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x));
}

// _cross3 (_core.pyx:32-35)
__device__ __forceinline__ V3 cross3(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

__device__ __forceinline__ V3 load3(const double* __restrict__ base, int64_t i) {
  const double* p = base + 3 * i;
  return {__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}

// Point-triangle closest feature: _pt_one (_core.pyx:46-106).
// g[0..3] = gradient of d2 over (p, t1, t2, t3); returns the region code.
__device__ __forceinline__ int pt_one(V3 p, V3 t1, V3 t2, V3 t3, double& d2, V3 g[4], double& w1,
                                      double& w2) {
  const V3 ab = t2 - t1, ac = t3 - t1, ap = p - t1;
  const double d1 = dot3(ab, ap), d2_ = dot3(ac, ap);
  const V3 bp = p - t2;
  const double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  const V3 cp = p - t3;
  const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  const double vc = d1 * d4 - d3 * d2_;
  const double vb = d5 * d2_ - d1 * d6;
  const double va = d3 * d6 - d5 * d4;
  int code;
  w1 = 0.0;
  w2 = 0.0;
  if (d1 <= 0.0 && d2_ <= 0.0) {
    code = 1;
  } else if (d3 >= 0.0 && d4 <= d3) {
    code = 2;
    w1 = 1.0;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    code = 4;
    w1 = d1 / (d1 - d3);
  } else if (d6 >= 0.0 && d5 <= d6) {
    code = 3;
    w2 = 1.0;
  } else if (vb <= 0.0 && d2_ >= 0.0 && d6 <= 0.0) {
    code = 6;
    w2 = d2_ / (d2_ - d6);
  } else if (va <= 0.0 && d4 - d3 >= 0.0 && d5 - d6 >= 0.0) {
    code = 5;
    const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    w1 = 1.0 - t;
    w2 = t;
  } else {
    code = 0;
    const double denom = va + vb + vc;
    w1 = vb / denom;
    w2 = vc / denom;
  }
  const double w0 = 1.0 - w1 - w2;
  const V3 closest = {w0 * t1.x + w1 * t2.x + w2 * t3.x, w0 * t1.y + w1 * t2.y + w2 * t3.y,
                      w0 * t1.z + w1 * t2.z + w2 * t3.z};
  const V3 r = p - closest;
  d2 = dot3(r, r);
  g[0] = 2.0 * r;
  g[1] = (-2.0 * w0) * r;
  g[2] = (-2.0 * w1) * r;
  g[3] = (-2.0 * w2) * r;
  return code;
}

// Clamped segment-segment closest pair: _ee_one (_core.pyx:109-150).  Returns 3*ra+rb.
__device__ __forceinline__ int ee_one(V3 a1, V3 a2, V3 b1, V3 b2, double& d2, V3 g[4], double& s_out,
                                      double& t_out) {
  const V3 da = a2 - a1, db = b2 - b1, r = a1 - b1;
  const double a = dot3(da, da), e = dot3(db, db), f = dot3(db, r);
  const double b = dot3(da, db), c = dot3(da, r);
  const double denom = a * e - b * b;
  double s = denom > 0.0 ? clamp01((b * f - c * e) / denom) : 0.0;
  double t = (b * s + f) / e;
  if (t < 0.0) {
    t = 0.0;
    s = clamp01(-c / a);
  } else if (t > 1.0) {
    t = 1.0;
    s = clamp01((b - c) / a);
  }
  const int ra = s <= 0.0 ? 0 : (s >= 1.0 ? 1 : 2);
  const int rb = t <= 0.0 ? 0 : (t >= 1.0 ? 1 : 2);
  const V3 rv = {(a1.x + s * da.x) - (b1.x + t * db.x), (a1.y + s * da.y) - (b1.y + t * db.y),
                 (a1.z + s * da.z) - (b1.z + t * db.z)};
  d2 = dot3(rv, rv);
  g[0] = (2.0 * (1.0 - s)) * rv;
  g[1] = (2.0 * s) * rv;
  g[2] = (-2.0 * (1.0 - t)) * rv;
  g[3] = (-2.0 * t) * rv;
  s_out = s;
  t_out = t;
  return 3 * ra + rb;
}

// c = |(a2-a1) x (b2-b1)|^2 and its gradient: cross_sq_batch (_core.pyx:195-219).
__device__ __forceinline__ double cross_sq_one(V3 a1, V3 a2, V3 b1, V3 b2, V3 g[4]) {
  const V3 u = a2 - a1, v = b2 - b1;
  const V3 w = cross3(u, v);
  const V3 gu = cross3(v, w), gv = cross3(w, u);
  g[0] = -2.0 * gu;
  g[1] = 2.0 * gu;
  g[2] = -2.0 * gv;
  g[3] = 2.0 * gv;
  return dot3(w, w);
}

// Point-segment distance: _point_edge_eval (proximity.py:170-180); np.dot -> dot3_blas.
__device__ __forceinline__ double pe_one(V3 p, V3 e1, V3 e2, V3 g[3], double& t_out) {
  const V3 e = e2 - e1;
  const double ee = dot3_blas(e, e);
  const V3 pe = p - e1;
  const double t = clamp01(dot3_blas(pe, e) / ee);
  t_out = t;
  const V3 r = pe - t * e;
  g[0] = 2.0 * r;
  g[1] = (-2.0 * (1.0 - t)) * r;
  g[2] = (-2.0 * t) * r;
  return dot3_blas(r, r);
}

// Point-point: stencil_distance (proximity.py:187-190).
__device__ __forceinline__ double pp_one(V3 a, V3 b, V3 g[2]) {
  const V3 r = a - b;
  g[0] = 2.0 * r;
  g[1] = -2.0 * r;
  return dot3_blas(r, r);
}

// Barrier scalars b, b', b'' (barrier.py:76-101); S = kappa d_hat^4.
struct Barrier {
  double b, bg, bgg;
};

template <int FORM>
__device__ __forceinline__ Barrier barrier_scalars(double g, double S) {
  const double lg = log(g);
  const double om = 1.0 - g;
  Barrier r;
  if (FORM == 0) {  // qlog
    r.b = S * (om * om) * lg * lg;
    r.bg = S * (-2.0 * om * lg * lg + 2.0 * (om * om) * lg / g);
    r.bgg = S * (2.0 * lg * lg - 8.0 * om * lg / g + 2.0 * (om * om) * (1.0 - lg) / (g * g));
  } else {  // single log
    r.b = -S * (om * om) * lg;
    r.bg = S * (2.0 * om * lg - (om * om) / g);
    r.bgg = S * (-2.0 * lg + om * (3.0 * g + 1.0) / (g * g));
  }
  return r;
}

// lambda1 = 4 g b'' + 2 b' (barrier.py:104-106)
__device__ __forceinline__ double lambda1_of(double g, const Barrier& s) { return 4.0 * g * s.bgg + 2.0 * s.bg; }

}  // namespace b200ipc
