// Additive CCD step bound (accd_max_step, kernels/_core.pyx:250-325) for whole candidate lists, and
// the global step filter built on it (global_ccd_filter, proximity.py:424-432).
//
// One thread per pair, everything in registers: mean-free displacement q, the motion bound lp, the
// conservative-advancement loop t += (d(t) - gap) / lp with the reference's three exits (step <= 0,
// t + step >= 1 -> 1.0, step < 1e-14) and its iteration cap.  The arithmetic follows the compiled
// reference operation by operation (no FMA: the library is built with -fmad=false; sqrt and / are
// IEEE on both sides), so every per-pair bound is bit-identical to tetipc's.  The filter takes the
// minimum over all pairs with an ordered-bits atomicMin: min is exact and order-free, hence still
// deterministic.
#include "geom.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kCT = 128;

// _pair_dist2_c (_core.pyx:250-269)
__device__ __forceinline__ double pair_dist2(const V3 (&x)[4], int pair_kind) {
  double d2, w1, w2;
  V3 g[4];
  if (pair_kind == B200IPC_PAIR_PT) {
    pt_one(x[0], x[1], x[2], x[3], d2, g, w1, w2);
    return d2;
  }
  if (pair_kind == B200IPC_PAIR_EE) {
    ee_one(x[0], x[1], x[2], x[3], d2, g, w1, w2);
    return d2;
  }
  if (pair_kind == B200IPC_PAIR_PE) {
    const V3 e = x[2] - x[1];
    const double ee = dot3(e, e);
    V3 r = x[0] - x[1];
    const double t = clamp01(dot3(r, e) / ee);
    r.x = r.x - t * e.x;
    r.y = r.y - t * e.y;
    r.z = r.z - t * e.z;
    return dot3(r, r);
  }
  const V3 r = x[0] - x[1];
  return dot3(r, r);
}

// Returns the step fraction; *bad = true when the initial distance is not positive (the reference
// raises ValueError there, _core.pyx:307-308).
//
// `bound` (step filter only): the running minimum over all pairs.  t only grows along the iteration and
// the result is >= the current t, so a pair whose t has reached the running minimum cannot lower it and
// stops (returning 1); the minimum itself -- the only thing the filter reports -- is unchanged, bit for bit.
__device__ __forceinline__ double accd_one(const V3 (&x0)[4], const V3 (&dx)[4], int s, int pair_kind, double slack,
                                           int max_iter, bool* bad, const unsigned long long* bound = nullptr) {
  *bad = false;
  V3 mean = vzero();
  for (int v = 0; v < s; ++v) mean = mean + dx[v];
  mean.x /= s;
  mean.y /= s;
  mean.z /= s;
  V3 q[4];
  double norms[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    q[v] = v < s ? dx[v] - mean : vzero();
    norms[v] = sqrt(q[v].x * q[v].x + q[v].y * q[v].y + q[v].z * q[v].z);
  }
  double lp;
  if (pair_kind == B200IPC_PAIR_PT) lp = norms[0] + fmax(norms[1], fmax(norms[2], norms[3]));
  else if (pair_kind == B200IPC_PAIR_EE) lp = fmax(norms[0], norms[1]) + fmax(norms[2], norms[3]);
  else if (pair_kind == B200IPC_PAIR_PE) lp = norms[0] + fmax(norms[1], norms[2]);
  else lp = norms[0] + norms[1];
  if (lp == 0.0) return 1.0;
  const double d0 = sqrt(pair_dist2(x0, pair_kind));
  if (!(d0 > 0.0)) {
    *bad = true;
    return 0.0;
  }
  const double gap = (1.0 - slack) * d0;
  double t = 0.0;
  for (int it = 0; it < max_iter; ++it) {
    V3 xt[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) xt[v] = {x0[v].x + t * q[v].x, x0[v].y + t * q[v].y, x0[v].z + t * q[v].z};
    const double d = sqrt(pair_dist2(xt, pair_kind));
    const double step = (d - gap) / lp;
    if (step <= 0.0) break;
    if (t + step >= 1.0) return 1.0;
    t += step;
    if (step < 1e-14) break;
    if (bound && (it & 3) == 3 &&
        t >= __longlong_as_double((long long)*reinterpret_cast<const volatile unsigned long long*>(bound)))
      return 1.0;
  }
  return t;
}

__device__ __forceinline__ int pair_size(int pair_kind) {
  return pair_kind == B200IPC_PAIR_PE ? 3 : (pair_kind == B200IPC_PAIR_PP ? 2 : 4);
}

struct AccdArgs {
  int64_t n;
  const int32_t* ids;         // (n,4) global vertex ids, -1 padded
  const uint8_t* pair_kind;   // per pair, or NULL: uniform_kind
  int32_t uniform_kind;
  const double* positions;
  const double* directions;
  double slack;
  int32_t max_iter;
  double* step;               // (n) or NULL
  uint8_t* status;            // (n) or NULL
  unsigned long long* alpha_bits;  // running minimum (ordered bits of a non-negative double) or NULL
  unsigned long long* n_invalid;   // pairs with a non-positive initial distance, or NULL
  const unsigned long long* n_dev; // when set: the pair count lives on the device (a list compacted there), n = its capacity
};

__global__ void __launch_bounds__(kCT) accd_kernel(const __grid_constant__ AccdArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kCT + threadIdx.x;
  double t = 1.0;
  bool bad = false;
  const int64_t n = a.n_dev ? (int64_t)*a.n_dev : a.n;
  if (i < n) {
    const int kind = a.pair_kind ? a.pair_kind[i] : a.uniform_kind;
    const int s = pair_size(kind);
    const int4 id = reinterpret_cast<const int4*>(a.ids)[i];
    const int v[4] = {id.x, id.y, id.z, id.w};
    V3 x0[4], dx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool on = k < s;
      x0[k] = on ? load3(a.positions, v[k]) : vzero();
      dx[k] = on ? load3(a.directions, v[k]) : vzero();
    }
    t = accd_one(x0, dx, s, kind, a.slack, a.max_iter, &bad, a.step ? nullptr : a.alpha_bits);
    if (a.step) a.step[i] = t;
    if (a.status) a.status[i] = bad ? 2 : 0;
    // non-negative doubles order like their bit patterns; a bad pair does not take part in the min.
    // Published per lane as soon as it is known (and only when it lowers the minimum), so that the
    // pairs still iterating can stop against it.
    if (a.alpha_bits && !bad && t < 1.0 &&
        t < __longlong_as_double((long long)*reinterpret_cast<const volatile unsigned long long*>(a.alpha_bits)))
      atomicMin(a.alpha_bits, (unsigned long long)__double_as_longlong(t));
  }
  if (a.alpha_bits && a.n_invalid) {
    const unsigned nbad = __popc(__ballot_sync(0xffffffffu, bad));
    if ((threadIdx.x & 31) == 0 && nbad) atomicAdd(a.n_invalid, (unsigned long long)nbad);
  }
}

// sweep_candidates' own predicate (proximity.py:388-421) on a candidate pair: the swept boxes of its two
// primitives -- pose at x and at x + d, grown by `margin` -- overlap.  Corners are formed exactly like broad.cu
// forms them (min / max over both poses, then -margin / +margin), so a SUPERSET of the reference's candidate
// list filtered by this test is the reference's list.  Pairs that pass are appended to `out` (one atomic per warp;
// the order is arbitrary, the minimum taken over them afterwards is order-free).
struct SweptFilterArgs {
  int64_t n;
  const int32_t* ids;      // (n,4)
  int32_t na;              // vertices of the first primitive: 1 (point-triangle) or 2 (edge-edge)
  const double* positions;
  const double* directions;
  double margin;
  int32_t* out;            // (n,4)
  unsigned long long* count;
};

__global__ void __launch_bounds__(kCT) swept_filter_kernel(const __grid_constant__ SweptFilterArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kCT + threadIdx.x;
  bool pass = false;
  int4 id = make_int4(0, 0, 0, 0);
  if (i < a.n) {
    id = reinterpret_cast<const int4*>(a.ids)[i];
    const int v[4] = {id.x, id.y, id.z, id.w};
    double lo[2][3], hi[2][3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int b = k < a.na ? 0 : 1;
      const bool first = k == 0 || k == a.na;
      const V3 x = load3(a.positions, v[k]), d = load3(a.directions, v[k]);
      const double p0[3] = {x.x, x.y, x.z}, p1[3] = {x.x + d.x, x.y + d.y, x.z + d.z};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double l = fmin(p0[c], p1[c]), h = fmax(p0[c], p1[c]);
        lo[b][c] = first ? l : fmin(lo[b][c], l);
        hi[b][c] = first ? h : fmax(hi[b][c], h);
      }
    }
    pass = true;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      pass = pass && (lo[0][c] - a.margin <= hi[1][c] + a.margin) && (lo[1][c] - a.margin <= hi[0][c] + a.margin);
  }
  const unsigned m = __ballot_sync(0xffffffffu, pass);
  if (m) {
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(a.count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (pass) reinterpret_cast<int4*>(a.out)[base + __popc(m & ((1u << lane) - 1u))] = id;
  }
}

__global__ void accd_init_kernel(unsigned long long* alpha_bits, unsigned long long* n_invalid) {
  *alpha_bits = (unsigned long long)__double_as_longlong(1.0);
  if (n_invalid) *n_invalid = 0ull;
}

}  // namespace b200ipc

using namespace b200ipc;

static int accd_args_ok(int64_t n, const int32_t* ids, const uint8_t* pair_kind, int32_t uniform_kind,
                        const double* positions, const double* directions, double slack, int32_t max_iter) {
  if (n < 0 || max_iter < 0 || !(slack > 0.0 && slack < 1.0)) return B200IPC_EINVAL;
  if (n && (!ids || !positions || !directions)) return B200IPC_EINVAL;
  if (((uintptr_t)ids) & 15) return B200IPC_EINVAL;
  if (!pair_kind && (uniform_kind < 0 || uniform_kind > 3)) return B200IPC_EINVAL;
  return 0;
}

extern "C" int b200ipc_accd_max_step(int64_t n, const int32_t* ids, const uint8_t* pair_kind, int32_t uniform_kind,
                                     const double* positions, const double* directions, double slack,
                                     int32_t max_iter, double* step, uint8_t* status, void* stream) {
  int rc = accd_args_ok(n, ids, pair_kind, uniform_kind, positions, directions, slack, max_iter);
  if (rc) return rc;
  if (n == 0) return 0;
  if (!step) return B200IPC_EINVAL;
  AccdArgs a{n, ids, pair_kind, uniform_kind, positions, directions, slack, max_iter, step, status, nullptr, nullptr, nullptr};
  accd_kernel<<<(unsigned)((n + kCT - 1) / kCT), kCT, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}

extern "C" int b200ipc_ccd_filter(int64_t n_vt, const int32_t* vt, int64_t n_ee, const int32_t* ee,
                                  const double* positions, const double* directions, double slack, int32_t max_iter,
                                  double* alpha, int64_t* n_invalid, void* stream) {
  if (!alpha) return B200IPC_EINVAL;
  int rc = accd_args_ok(n_vt, vt, nullptr, B200IPC_PAIR_PT, positions, directions, slack, max_iter);
  if (rc) return rc;
  rc = accd_args_ok(n_ee, ee, nullptr, B200IPC_PAIR_EE, positions, directions, slack, max_iter);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(alpha);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(n_invalid);
  accd_init_kernel<<<1, 1, 0, st>>>(bits, bad);
  rc = post_launch();
  if (rc) return rc;
  if (n_vt) {
    AccdArgs a{n_vt, vt, nullptr, B200IPC_PAIR_PT, positions, directions, slack, max_iter, nullptr, nullptr, bits, bad, nullptr};
    accd_kernel<<<(unsigned)((n_vt + kCT - 1) / kCT), kCT, 0, st>>>(a);
    rc = post_launch();
    if (rc) return rc;
  }
  if (n_ee) {
    AccdArgs a{n_ee, ee, nullptr, B200IPC_PAIR_EE, positions, directions, slack, max_iter, nullptr, nullptr, bits, bad, nullptr};
    accd_kernel<<<(unsigned)((n_ee + kCT - 1) / kCT), kCT, 0, st>>>(a);
    rc = post_launch();
    if (rc) return rc;
  }
  return 0;
}

// global_ccd_filter over ANY superset of sweep_candidates' lists: every pair is first put to the reference's
// swept-box test at `sweep_margin`, the survivors (compacted on the device, no host round trip) go through ACCD.
// `scratch`: device, 16 (n_vt + n_ee) + 16 bytes, 16-byte aligned.
extern "C" int b200ipc_ccd_filter_swept(int64_t n_vt, const int32_t* vt, int64_t n_ee, const int32_t* ee,
                                        const double* positions, const double* directions, double sweep_margin,
                                        double slack, int32_t max_iter, void* scratch, double* alpha, int64_t* n_invalid,
                                        void* stream) {
  if (!alpha || !scratch || !(sweep_margin >= 0.0) || (((uintptr_t)scratch) & 15)) return B200IPC_EINVAL;
  int rc = accd_args_ok(n_vt, vt, nullptr, B200IPC_PAIR_PT, positions, directions, slack, max_iter);
  if (rc) return rc;
  rc = accd_args_ok(n_ee, ee, nullptr, B200IPC_PAIR_EE, positions, directions, slack, max_iter);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* counts = static_cast<unsigned long long*>(scratch);   // [vt kept, ee kept]
  int32_t* keep_vt = reinterpret_cast<int32_t*>(counts + 2);
  int32_t* keep_ee = keep_vt + 4 * n_vt;
  cudaError_t e = cudaMemsetAsync(counts, 0, 16, st);
  if (e != cudaSuccess) return -(int)e;
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(alpha);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(n_invalid);
  accd_init_kernel<<<1, 1, 0, st>>>(bits, bad);
  rc = post_launch();
  if (rc) return rc;
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t n = pass == 0 ? n_vt : n_ee;
    if (!n) continue;
    const int32_t* ids = pass == 0 ? vt : ee;
    int32_t* keep = pass == 0 ? keep_vt : keep_ee;
    SweptFilterArgs f{n, ids, pass == 0 ? 1 : 2, positions, directions, sweep_margin, keep, counts + pass};
    swept_filter_kernel<<<(unsigned)((n + kCT - 1) / kCT), kCT, 0, st>>>(f);
    rc = post_launch();
    if (rc) return rc;
    AccdArgs a{n, keep, nullptr, pass == 0 ? B200IPC_PAIR_PT : B200IPC_PAIR_EE, positions, directions, slack, max_iter,
               nullptr, nullptr, bits, bad, counts + pass};
    accd_kernel<<<(unsigned)((n + kCT - 1) / kCT), kCT, 0, st>>>(a);
    rc = post_launch();
    if (rc) return rc;
  }
  return 0;
}
