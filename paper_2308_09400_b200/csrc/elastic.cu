// Stable neo-Hookean tetrahedra (elasticity.py): per-tet energy, gradient and
// PSD-projected 12x12 Hessian, the opaque block family the barrier blocks are assembled next to.
//
//   Psi = mu/2 (tr F^T F - 3) + lam/2 (J - a)^2,  a = 1 + mu/lam           (elasticity.py:103-108)
//   P   = mu F + lam (J - a) dJ/dF                                           (:111-115)
//   H9  = mu I + lam g g^T + lam (J - a) d2J/dF2,  g = vec(dJ/dF)           (:118-125)
// The reference projects H9 with LAPACK eigh (9x9, numerical).  Here the projection is ANALYTIC, in the
// spirit of the paper's barrier blocks: with the rotation-variant SVD F = U diag(s) V^T the nine
// eigenpairs of H9 are known in closed form -- three twists (mu + k s_k), three flips (mu - k s_k),
// k = lam (J - a), and the eigenpairs of the 3x3 "scaling" matrix A = mu I + lam g^ g^^T + k B(s) -- so
//   H_psd = H9 - sum over negative eigenvalues of  w q q^T,
// and after the change of basis every 3x3 block (v,u) of the 12x12 is
//   vol [ mu (w_v.w_u) I + lam p_v p_u^T - k skew(F (w_v x w_u)) - U K(v,u) U^T ]
// with K built from the negative parts only.  Everything lives in registers: a one-sided Jacobi SVD
// of the 3x3 F and a Jacobi eigensolve of the 3x3 A are the only iterations (tests: 2e-15 of the
// reference's eigh projection, including inverted and strongly compressed elements).  The change of
// basis uses the structure of dvec(F)/dx (rest_data, :39-56): F_ic = sum_v w_vc x_vi with
// w_0c = -sum_r Dm^-1_rc, w_vc = Dm^-1_(v-1)c, so no 9x12 map is stored.  `project = 0` (the
// reference's diagnostic switch) keeps the raw Hessian.
//
// Two phases (the first version did everything in one thread per tet: 255 registers, 8 warps per SM, the
// dependent fp64 chains of the two Jacobi iterations at no occupancy, 0.43 ms for 400 k tets):
//   elastic_state_kernel    thread per tet: F, energy, gradient, the eigensystem -> 53 doubles of state
//   elastic_hessian_kernel  thread per 3x3 block (v,u): 16 x more threads with a fifth of the registers form
//                           the blocks from that state; tiles of 16 tets leave through shared memory so that
//                           the (16, 12, 12) span is written with consecutive lanes on consecutive doubles.
#include "geom.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kET = 64;

__global__ void __launch_bounds__(kET) elastic_rest_kernel(int64_t nt, const int32_t* __restrict__ tets,
                                                           const double* __restrict__ rest, double* __restrict__ rest_inv,
                                                           double* __restrict__ vols) {
  const int64_t t = (int64_t)blockIdx.x * kET + threadIdx.x;
  if (t >= nt) return;
  const int4 id = reinterpret_cast<const int4*>(tets)[t];
  const V3 x0 = load3(rest, id.x);
  const V3 e1 = load3(rest, id.y) - x0, e2 = load3(rest, id.z) - x0, e3 = load3(rest, id.w) - x0;
  // Dm columns = edges: Dm[r][k] = e_k[r]
  const double m[3][3] = {{e1.x, e2.x, e3.x}, {e1.y, e2.y, e3.y}, {e1.z, e2.z, e3.z}};
  const double c00 = m[1][1] * m[2][2] - m[1][2] * m[2][1], c01 = m[1][2] * m[2][0] - m[1][0] * m[2][2],
               c02 = m[1][0] * m[2][1] - m[1][1] * m[2][0];
  const double det = m[0][0] * c00 + m[0][1] * c01 + m[0][2] * c02;
  const double r = 1.0 / det;
  double* o = rest_inv + 9 * t;
  o[0] = c00 * r;
  o[1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) * r;
  o[2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) * r;
  o[3] = c01 * r;
  o[4] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) * r;
  o[5] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) * r;
  o[6] = c02 * r;
  o[7] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) * r;
  o[8] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) * r;
  vols[t] = det / 6.0;
}

// One-sided Jacobi SVD of a 3x3: F = U diag(s) V^T with U, V rotations (det +1), |s0| >= |s1| >= |s2|,
// s0, s1 >= 0 and s2 carrying the sign of det F.  Column rotations orthogonalise B = F V (relative
// accuracy also for small singular values); columns are then ordered and U completed by a cross product.
__device__ __forceinline__ void svd3_rot(const double (&f)[3][3], double (&U)[3][3], double (&sg)[3], double (&V)[3][3]) {
  double b[3][3], v[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      b[i][j] = f[i][j];
      v[i][j] = i == j ? 1.0 : 0.0;
    }
#pragma unroll 1
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double aa = b[0][p] * b[0][p] + b[1][p] * b[1][p] + b[2][p] * b[2][p];
      const double bb = b[0][q] * b[0][q] + b[1][q] * b[1][q] + b[2][q] * b[2][q];
      const double cc = b[0][p] * b[0][q] + b[1][p] * b[1][q] + b[2][p] * b[2][q];
      // converged when |cc| <= 1e-15 sqrt(aa bb) for every pair: compared as squares, no sqrt / divide
      if (cc * cc > 1e-30 * (aa * bb)) off = 1.0;
      if (cc != 0.0) {
        // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (bb - aa) / (2 cc), rearranged to ONE square root and
        // ONE divide; cs by rsqrt.  fp64 divide and sqrt are ~30-instruction sequences and this loop was bound by them.
        const double d = bb - aa, c2 = 2.0 * cc;
        const double t = d == 0.0 ? 1.0 : ((d > 0.0) == (c2 > 0.0) ? fabs(c2) : -fabs(c2)) / (fabs(d) + sqrt(d * d + c2 * c2));
        const double cs = rsqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double bp = b[k][p], bq = b[k][q];
          b[k][p] = cs * bp - sn * bq;
          b[k][q] = sn * bp + cs * bq;
          const double vp = v[k][p], vq = v[k][q];
          v[k][p] = cs * vp - sn * vq;
          v[k][q] = sn * vp + cs * vq;
        }
      }
    }
    if (off == 0.0) break;
  }
  // order columns by norm (each swap flips the orientation; an odd count is undone by negating column 2)
  double n2[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) n2[j] = b[0][j] * b[0][j] + b[1][j] * b[1][j] + b[2][j] * b[2][j];
  bool odd = false;
  auto swap_cols = [&](int p, int q) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double t = b[k][p]; b[k][p] = b[k][q]; b[k][q] = t;
      t = v[k][p]; v[k][p] = v[k][q]; v[k][q] = t;
    }
    const double t = n2[p]; n2[p] = n2[q]; n2[q] = t;
    odd = !odd;
  };
  if (n2[0] < n2[1]) swap_cols(0, 1);
  if (n2[1] < n2[2]) swap_cols(1, 2);
  if (n2[0] < n2[1]) swap_cols(0, 1);
  if (odd) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      b[k][2] = -b[k][2];
      v[k][2] = -v[k][2];
    }
  }
  const double n0 = sqrt(n2[0]);
  V3 u0 = n0 > 0.0 ? V3{b[0][0] / n0, b[1][0] / n0, b[2][0] / n0} : V3{1.0, 0.0, 0.0};
  const V3 b1 = {b[0][1], b[1][1], b[2][1]}, b2 = {b[0][2], b[1][2], b[2][2]};
  const double d01 = dot3(b1, u0);
  V3 u1 = {b1.x - d01 * u0.x, b1.y - d01 * u0.y, b1.z - d01 * u0.z};
  const double n1 = sqrt(dot3(u1, u1));
  if (n1 > 0.0) {
    u1 = {u1.x / n1, u1.y / n1, u1.z / n1};
  } else {  // rank <= 1: any unit vector orthogonal to u0
    const V3 e = fabs(u0.x) < 0.9 ? V3{1.0, 0.0, 0.0} : V3{0.0, 1.0, 0.0};
    u1 = cross3(u0, e);
    const double m = sqrt(dot3(u1, u1));
    u1 = {u1.x / m, u1.y / m, u1.z / m};
  }
  const V3 u2 = cross3(u0, u1);
  U[0][0] = u0.x; U[1][0] = u0.y; U[2][0] = u0.z;
  U[0][1] = u1.x; U[1][1] = u1.y; U[2][1] = u1.z;
  U[0][2] = u2.x; U[1][2] = u2.y; U[2][2] = u2.z;
  sg[0] = n0;
  sg[1] = dot3(u1, b1);
  sg[2] = dot3(u2, b2);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = v[i][j];
}

// Negative part of a symmetric 3x3: S = sum_k min(w_k, 0) q_k q_k^T (two-sided Jacobi, in registers).
__device__ __forceinline__ void negative_part3(double (&a)[3][3], double (&S)[3][3]) {
  double q[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  const double tr = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
#pragma unroll 1
  for (int sweep = 0; sweep < 20; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    if (off <= 1e-32 * tr * tr) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, r = pq == 0 ? 1 : 2;
      const double apr = a[p][r];
      if (apr != 0.0) {
        const double d = a[r][r] - a[p][p], a2 = 2.0 * apr;   // theta = d / a2; same rearrangement as in svd3_rot
        const double t = ((d >= 0.0) == (a2 > 0.0) ? fabs(a2) : -fabs(a2)) / (fabs(d) + sqrt(d * d + a2 * a2));
        const double c = rsqrt(t * t + 1.0), s = t * c;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akr = a[k][r];
          a[k][p] = c * akp - s * akr;
          a[k][r] = s * akp + c * akr;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], ark = a[r][k];
          a[p][k] = c * apk - s * ark;
          a[r][k] = s * apk + c * ark;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double qkp = q[k][p], qkr = q[k][r];
          q[k][p] = c * qkp - s * qkr;
          q[k][r] = s * qkp + c * qkr;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      S[i][j] = fmin(a[0][0], 0.0) * q[i][0] * q[j][0] + fmin(a[1][1], 0.0) * q[i][1] * q[j][1] +
                fmin(a[2][2], 0.0) * q[i][2] * q[j][2];
}

struct ElasticArgs {
  int64_t nt;
  const int32_t* tets;
  const double* positions;
  const double* rest_inv;
  const double* vols;
  const double* mu;
  const double* lam;
  double scale;     // dt^2 for grad / hess (energy is not scaled)
  int32_t project;
  double* energy;
  double* grad;     // (nt, 12)
  double* hess;     // (nt, 12, 12)
  double* state;    // (nt, kState): hand-off between the two phases (null when no Hessian is wanted)
};

// Per-tet state handed from the eigen phase to the write-out phase (doubles):
//   0-8 F (row-major)   9-17 Dm^-1   18-26 U   27-35 V   36-41 S (00 01 02 11 12 22)   42-44 (cT+cL)/2
//   45-47 (cL-cT)/2   48 mu   49 lam   50 k = lam (J - a)   51 dt^2 vol   52 any negative eigenvalue (0/1)
// stored as a structure of arrays, state[k nt + t]: phase 1 writes and phase 2 reads whole 128-byte segments.
constexpr int kState = 53;

// Phase 1, one thread per tet: deformation gradient, energy, gradient, and -- when the Hessian is wanted -- the
// analytic eigensystem (the two small Jacobi iterations), written to `state`.  Small live state and no
// 12x12 in flight: 128-thread CTAs at several per SM instead of 64 threads holding 255 registers each.
constexpr int kES = 128;
__global__ void __launch_bounds__(kES, 4) elastic_state_kernel(const __grid_constant__ ElasticArgs a) {
  const int64_t t = (int64_t)blockIdx.x * kES + threadIdx.x;
  if (t >= a.nt) return;
  const int4 id = reinterpret_cast<const int4*>(a.tets)[t];
  const V3 x0 = load3(a.positions, id.x);
  const V3 d1 = load3(a.positions, id.y) - x0, d2 = load3(a.positions, id.z) - x0, d3 = load3(a.positions, id.w) - x0;
  const double ds[3][3] = {{d1.x, d2.x, d3.x}, {d1.y, d2.y, d3.y}, {d1.z, d2.z, d3.z}};
  double ri[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) ri[r][c] = a.rest_inv[9 * t + 3 * r + c];
  double f[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < 3; ++c) f[i][c] = ds[i][0] * ri[0][c] + ds[i][1] * ri[1][c] + ds[i][2] * ri[2][c];
  const double mu = a.mu[t], lam = a.lam[t], vol = a.vols[t];
  const double alpha = 1.0 + mu / lam;
  // columns of F and the cofactor columns dJ/dF = [f1 x f2, f2 x f0, f0 x f1]
  const V3 c0 = {f[0][0], f[1][0], f[2][0]}, c1 = {f[0][1], f[1][1], f[2][1]}, c2 = {f[0][2], f[1][2], f[2][2]};
  const V3 g0 = cross3(c1, c2), g1 = cross3(c2, c0), g2 = cross3(c0, c1);
  const double J = dot3(c0, g0);
  const double ic = dot3(c0, c0) + dot3(c1, c1) + dot3(c2, c2);
  if (a.energy) a.energy[t] = (0.5 * mu * (ic - 3.0) + 0.5 * lam * (J - alpha) * (J - alpha)) * vol;
  const double k1 = lam * (J - alpha);
  if (a.grad) {
    // w_v: dvec(F)/dx weights, p_v = (dJ/dF) w_v
    V3 w[4];
    w[0] = {-(ri[0][0] + ri[1][0] + ri[2][0]), -(ri[0][1] + ri[1][1] + ri[2][1]), -(ri[0][2] + ri[1][2] + ri[2][2])};
    w[1] = {ri[0][0], ri[0][1], ri[0][2]};
    w[2] = {ri[1][0], ri[1][1], ri[1][2]};
    w[3] = {ri[2][0], ri[2][1], ri[2][2]};
    double* g = a.grad + 12 * t;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const V3 pg = {g0.x * w[v].x + g1.x * w[v].y + g2.x * w[v].z, g0.y * w[v].x + g1.y * w[v].y + g2.y * w[v].z,
                     g0.z * w[v].x + g1.z * w[v].y + g2.z * w[v].z};
      // F w_v and (dJ/dF) w_v
      const V3 fw = {c0.x * w[v].x + c1.x * w[v].y + c2.x * w[v].z, c0.y * w[v].x + c1.y * w[v].y + c2.y * w[v].z,
                     c0.z * w[v].x + c1.z * w[v].y + c2.z * w[v].z};
      g[3 * v] = a.scale * vol * (mu * fw.x + k1 * pg.x);
      g[3 * v + 1] = a.scale * vol * (mu * fw.y + k1 * pg.y);
      g[3 * v + 2] = a.scale * vol * (mu * fw.z + k1 * pg.z);
    }
  }
  if (!a.state) return;
  // negative parts of the analytic eigensystem
  double U[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}}, V[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  double sg[3], S[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  double cs_[3] = {0.0, 0.0, 0.0}, cd_[3] = {0.0, 0.0, 0.0};  // (cT + cL)/2 and (cL - cT)/2 per axis
  bool any = false;
  if (a.project) {
    svd3_rot(f, U, sg, V);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double cT = fmin(mu + k1 * sg[k], 0.0), cL = fmin(mu - k1 * sg[k], 0.0);
      cs_[k] = 0.5 * (cT + cL);
      cd_[k] = 0.5 * (cL - cT);
      any = any || cT < 0.0 || cL < 0.0;
    }
    const double gh[3] = {sg[1] * sg[2], sg[0] * sg[2], sg[0] * sg[1]};
    double A[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) A[i][j] = lam * gh[i] * gh[j] + (i == j ? mu : k1 * sg[3 - i - j]);
    negative_part3(A, S);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) any = any || S[i][j] != 0.0;
  }
  double* st = a.state + t;   // structure of arrays: word k of tet t at state[k nt + t] (coalesced across the warp)
  const int64_t nt = a.nt;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      st[(3 * i + j) * nt] = f[i][j];
      st[(9 + 3 * i + j) * nt] = ri[i][j];
      st[(18 + 3 * i + j) * nt] = U[i][j];
      st[(27 + 3 * i + j) * nt] = V[i][j];
    }
  st[(36) * nt] = S[0][0]; st[(37) * nt] = S[0][1]; st[(38) * nt] = S[0][2]; st[(39) * nt] = S[1][1]; st[(40) * nt] = S[1][2]; st[(41) * nt] = S[2][2];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    st[(42 + k) * nt] = cs_[k];
    st[(45 + k) * nt] = cd_[k];
  }
  st[(48) * nt] = mu; st[(49) * nt] = lam; st[(50) * nt] = k1; st[(51) * nt] = a.scale * vol; st[(52) * nt] = any ? 1.0 : 0.0;
}

// Phase 2, one thread per 3x3 block (v,u) of a tet's 12x12, sixteen tets per CTA: the block is formed from the
// tet's state (broadcast loads: the sixteen threads of a tet read the same words), dropped into a
// shared-memory tile and the tile's (16, 12, 12) span leaves with consecutive lanes on consecutive doubles.
constexpr int kEPad = 145;      // odd row stride of the staging tile
constexpr int kTileTets = 16;
__global__ void __launch_bounds__(16 * kTileTets, 4) elastic_hessian_kernel(const __grid_constant__ ElasticArgs a) {
  __shared__ double tile[kTileTets * kEPad];
  __shared__ double sst[kTileTets][kState + 2];   // the tile's state, one row per tet (row stride 55: odd)
  const int64_t tile0 = (int64_t)blockIdx.x * kTileTets;
  const int lt = threadIdx.x >> 4, blkid = threadIdx.x & 15;
  const int v = blkid >> 2, u = blkid & 3;
  const int64_t t = tile0 + lt;
  const int ntile = (int)min((int64_t)kTileTets, a.nt - tile0);
  {   // 128-byte segments: word k of 16 tets; all four loads of a thread in flight before the first store
    constexpr int kPasses = (kState * kTileTets + 16 * kTileTets - 1) / (16 * kTileTets);
    double w[kPasses];
#pragma unroll
    for (int q = 0; q < kPasses; ++q) {
      const int e = threadIdx.x + q * 16 * kTileTets;
      const int k = e >> 4, i = e & 15;
      w[q] = (e < kState * kTileTets && i < ntile) ? a.state[(int64_t)k * a.nt + tile0 + i] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kPasses; ++q) {
      const int e = threadIdx.x + q * 16 * kTileTets;
      if (e < kState * kTileTets) sst[e & 15][e >> 4] = w[q];
    }
  }
  __syncthreads();
  if (t < a.nt) {
    const double* __restrict__ st = sst[lt];
    auto weight = [&](int k) -> V3 {   // w_0 = -(sum of the rows of Dm^-1), w_k = row k-1
      if (k == 0) return V3{-(st[9] + st[12] + st[15]), -(st[10] + st[13] + st[16]), -(st[11] + st[14] + st[17])};
      const double* r = st + 6 + 3 * k;
      return V3{r[0], r[1], r[2]};
    };
    const V3 wv = weight(v), wu = weight(u);
    const V3 c0 = {st[0], st[3], st[6]}, c1 = {st[1], st[4], st[7]}, c2 = {st[2], st[5], st[8]};
    const V3 g0 = cross3(c1, c2), g1 = cross3(c2, c0), g2 = cross3(c0, c1);
    const double pv[3] = {g0.x * wv.x + g1.x * wv.y + g2.x * wv.z, g0.y * wv.x + g1.y * wv.y + g2.y * wv.z,
                          g0.z * wv.x + g1.z * wv.y + g2.z * wv.z};
    const double pu[3] = {g0.x * wu.x + g1.x * wu.y + g2.x * wu.z, g0.y * wu.x + g1.y * wu.y + g2.y * wu.z,
                          g0.z * wu.x + g1.z * wu.y + g2.z * wu.z};
    const double mu = st[48], lam = st[49], k1 = st[50], sv = st[51];
    const double wd = mu * dot3(wv, wu);
    const V3 wx = cross3(wv, wu);
    const V3 fx = {c0.x * wx.x + c1.x * wx.y + c2.x * wx.z, c0.y * wx.x + c1.y * wx.y + c2.y * wx.z,
                   c0.z * wx.x + c1.z * wx.y + c2.z * wx.z};
    double blk[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) blk[i][j] = lam * pv[i] * pu[j] + (i == j ? wd : 0.0);
    // - k1 skew(F (w_v x w_u))
    blk[0][1] += k1 * fx.z; blk[0][2] -= k1 * fx.y;
    blk[1][0] -= k1 * fx.z; blk[1][2] += k1 * fx.x;
    blk[2][0] += k1 * fx.y; blk[2][1] -= k1 * fx.x;
    if (st[52] != 0.0) {
      double U[3][3], S[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) U[i][j] = st[18 + 3 * i + j];
      S[0][0] = st[36]; S[0][1] = S[1][0] = st[37]; S[0][2] = S[2][0] = st[38];
      S[1][1] = st[39]; S[1][2] = S[2][1] = st[40]; S[2][2] = st[41];
      double avv[3], avu[3];   // a_vc = V[:,c] . w_v
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        avv[c] = st[27 + c] * wv.x + st[30 + c] * wv.y + st[33 + c] * wv.z;
        avu[c] = st[27 + c] * wu.x + st[30 + c] * wu.y + st[33 + c] * wu.z;
      }
      // K(v,u): scaling part S_cd a_vc a_ud, plus the twist / flip pair of each axis k with plane (i,j)
      double K[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) K[c][d] = S[c][d] * avv[c] * avu[d];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int i = (k + 1) % 3, j = (k + 2) % 3;
        const double cs = st[42 + k], cd = st[45 + k];
        K[j][j] += cs * avv[i] * avu[i];
        K[i][i] += cs * avv[j] * avu[j];
        K[j][i] += cd * avv[i] * avu[j];
        K[i][j] += cd * avv[j] * avu[i];
      }
      // blk -= U K U^T
      double UK[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) UK[i][d] = U[i][0] * K[0][d] + U[i][1] * K[1][d] + U[i][2] * K[2][d];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) blk[i][j] -= UK[i][0] * U[j][0] + UK[i][1] * U[j][1] + UK[i][2] * U[j][2];
    }
    double* row = tile + lt * kEPad;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) row[(3 * v + i) * 12 + 3 * u + j] = sv * blk[i][j];
  }
  __syncthreads();
  double* out = a.hess + tile0 * 144;
  for (int e = threadIdx.x; e < ntile * 144; e += 16 * kTileTets) {
    const int i = e / 144, k = e - 144 * i;
    out[e] = tile[i * kEPad + k];
  }
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_elastic_rest(int64_t ntets, const int32_t* tets, const double* rest_positions, double* rest_inv,
                                    double* vols, void* stream) {
  if (ntets < 0) return B200IPC_EINVAL;
  if (ntets == 0) return 0;
  if (!tets || !rest_positions || !rest_inv || !vols || (((uintptr_t)tets) & 15)) return B200IPC_EINVAL;
  elastic_rest_kernel<<<(unsigned)((ntets + kET - 1) / kET), kET, 0, (cudaStream_t)stream>>>(ntets, tets, rest_positions,
                                                                                           rest_inv, vols);
  return post_launch();
}

extern "C" int b200ipc_elastic_blocks(int64_t ntets, const int32_t* tets, const double* positions, const double* rest_inv,
                                      const double* vols, const double* mu, const double* lam, double scale,
                                      int32_t project, double* energy, double* grad, double* hess, void* stream) {
  if (ntets < 0) return B200IPC_EINVAL;
  if (ntets == 0) return 0;
  if (!tets || !positions || !rest_inv || !vols || !mu || !lam || (((uintptr_t)tets) & 15)) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  ElasticArgs a{ntets, tets, positions, rest_inv, vols, mu, lam, scale, project, energy, grad, hess, nullptr};
  if (hess) {   // hand-off buffer of the two phases, from the stream-ordered pool
    cudaError_t e0 = keep_pool_memory();
    if (e0 != cudaSuccess) return -(int)e0;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&a.state), sizeof(double) * kState * (size_t)ntets, st);
    if (e != cudaSuccess) return -(int)e;
  }
  elastic_state_kernel<<<(unsigned)((ntets + kES - 1) / kES), kES, 0, st>>>(a);
  int rc = post_launch();
  if (hess && rc == 0) {
    elastic_hessian_kernel<<<(unsigned)((ntets + kTileTets - 1) / kTileTets), 16 * kTileTets, 0, st>>>(a);
    rc = post_launch();
  }
  if (a.state) {
    cudaError_t e = cudaFreeAsync(a.state, st);
    if (e != cudaSuccess && rc == 0) rc = -(int)e;
  }
  return rc;
}
