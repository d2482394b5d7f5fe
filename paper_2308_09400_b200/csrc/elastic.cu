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
// reference's diagnostic switch) keeps the raw Hessian.  Tiles of 64 tets are staged through shared
// memory so that the (ntile, 12, 12) span leaves with consecutive lanes on consecutive doubles.
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
      off = fmax(off, fabs(cc) / fmax(sqrt(aa * bb), 1e-300));
      if (cc != 0.0) {
        const double zeta = (bb - aa) / (2.0 * cc);
        const double t = zeta == 0.0 ? 1.0 : (zeta > 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
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
    if (off < 1e-15) break;
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
        const double theta = (a[r][r] - a[p][p]) / (2.0 * apr);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
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
};

constexpr int kEPad = 145;  // odd row stride: thread t writes row t, the copy-out reads consecutive entries

#ifndef B200IPC_ELASTIC_MINB
#define B200IPC_ELASTIC_MINB 1
#endif
__global__ void __launch_bounds__(kET, B200IPC_ELASTIC_MINB) elastic_blocks_kernel(const __grid_constant__ ElasticArgs a) {
  extern __shared__ double tile[];  // (kET, kEPad)
  const int64_t tile0 = (int64_t)blockIdx.x * kET;
  const int64_t t = tile0 + threadIdx.x;
  const int ntile = (int)min((int64_t)kET, a.nt - tile0);
  if (t < a.nt) {
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
    // w_v: dvec(F)/dx weights, p_v = (dJ/dF) w_v
    V3 w[4];
    w[0] = {-(ri[0][0] + ri[1][0] + ri[2][0]), -(ri[0][1] + ri[1][1] + ri[2][1]), -(ri[0][2] + ri[1][2] + ri[2][2])};
    w[1] = {ri[0][0], ri[0][1], ri[0][2]};
    w[2] = {ri[1][0], ri[1][1], ri[1][2]};
    w[3] = {ri[2][0], ri[2][1], ri[2][2]};
    V3 pg[4];
#pragma unroll
    for (int v = 0; v < 4; ++v)
      pg[v] = {g0.x * w[v].x + g1.x * w[v].y + g2.x * w[v].z, g0.y * w[v].x + g1.y * w[v].y + g2.y * w[v].z,
               g0.z * w[v].x + g1.z * w[v].y + g2.z * w[v].z};
    if (a.grad) {
      double* g = a.grad + 12 * t;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        // F w_v and (dJ/dF) w_v
        const V3 fw = {c0.x * w[v].x + c1.x * w[v].y + c2.x * w[v].z, c0.y * w[v].x + c1.y * w[v].y + c2.y * w[v].z,
                       c0.z * w[v].x + c1.z * w[v].y + c2.z * w[v].z};
        g[3 * v] = a.scale * vol * (mu * fw.x + k1 * pg[v].x);
        g[3 * v + 1] = a.scale * vol * (mu * fw.y + k1 * pg[v].y);
        g[3 * v + 2] = a.scale * vol * (mu * fw.z + k1 * pg[v].z);
      }
    }
    if (a.hess) {
      // negative parts of the analytic eigensystem
      double U[3][3], V[3][3], sg[3], S[3][3];
      double cs_[3] = {0.0, 0.0, 0.0}, cd_[3] = {0.0, 0.0, 0.0};  // (cT + cL)/2 and (cL - cT)/2 per axis
      double av[4][3];                                             // a_vc = V[:,c] . w_v
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
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          av[v][0] = V[0][0] * w[v].x + V[1][0] * w[v].y + V[2][0] * w[v].z;
          av[v][1] = V[0][1] * w[v].x + V[1][1] * w[v].y + V[2][1] * w[v].z;
          av[v][2] = V[0][2] * w[v].x + V[1][2] * w[v].y + V[2][2] * w[v].z;
        }
      }
      double* row = tile + threadIdx.x * kEPad;
      const double sv = a.scale * vol;
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double wd = mu * dot3(w[v], w[u]);
          const V3 wx = cross3(w[v], w[u]);
          const V3 fx = {c0.x * wx.x + c1.x * wx.y + c2.x * wx.z, c0.y * wx.x + c1.y * wx.y + c2.y * wx.z,
                         c0.z * wx.x + c1.z * wx.y + c2.z * wx.z};
          double blk[3][3];
          const double pv[3] = {pg[v].x, pg[v].y, pg[v].z}, pu[3] = {pg[u].x, pg[u].y, pg[u].z};
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) blk[i][j] = lam * pv[i] * pu[j] + (i == j ? wd : 0.0);
          // - k1 skew(F (w_v x w_u))
          blk[0][1] += k1 * fx.z; blk[0][2] -= k1 * fx.y;
          blk[1][0] -= k1 * fx.z; blk[1][2] += k1 * fx.x;
          blk[2][0] += k1 * fx.y; blk[2][1] -= k1 * fx.x;
          if (any) {
            // K(v,u): scaling part S_cd a_vc a_ud, plus the twist / flip pair of each axis k with plane (i,j)
            double K[3][3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int d = 0; d < 3; ++d) K[c][d] = S[c][d] * av[v][c] * av[u][d];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              const int i = (k + 1) % 3, j = (k + 2) % 3;
              K[j][j] += cs_[k] * av[v][i] * av[u][i];
              K[i][i] += cs_[k] * av[v][j] * av[u][j];
              K[j][i] += cd_[k] * av[v][i] * av[u][j];
              K[i][j] += cd_[k] * av[v][j] * av[u][i];
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
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) row[(3 * v + i) * 12 + 3 * u + j] = sv * blk[i][j];
        }
    }
  }
  if (!a.hess) return;
  __syncthreads();
  double* out = a.hess + tile0 * 144;
  for (int e = threadIdx.x; e < ntile * 144; e += kET) {
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
  ElasticArgs a{ntets, tets, positions, rest_inv, vols, mu, lam, scale, project, energy, grad, hess};
  const size_t smem = (size_t)kET * kEPad * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(elastic_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return -(int)e;
    attr = true;
  }
  elastic_blocks_kernel<<<(unsigned)((ntets + kET - 1) / kET), kET, smem, (cudaStream_t)stream>>>(a);
  return post_launch();
}
