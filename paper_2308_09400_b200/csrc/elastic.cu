// Stable neo-Hookean tetrahedra (elasticity.py): per-tet energy, gradient and
// PSD-projected 12x12 Hessian, the opaque block family the barrier blocks are assembled next to.
//
//   Psi = mu/2 (tr F^T F - 3) + lam/2 (J - a)^2,  a = 1 + mu/lam           (elasticity.py:103-108)
//   P   = mu F + lam (J - a) dJ/dF                                           (:111-115)
//   H9  = mu I + lam g g^T + lam (J - a) d2J/dF2,  g = vec(dJ/dF)           (:118-125)
// The reference projects H9 with LAPACK eigh; here each thread diagonalises its 9x9 with cyclic
// Jacobi rotations (the projection sum_k max(w_k, 0) q_k q_k^T is unique, so the algorithm only has to
// be accurate: off-diagonal mass below 1e-30 of the trace after <= 12 sweeps).  The change of basis to
// vertex coordinates uses the structure of dvec(F)/dx (rest_data, :39-56): F_ic = sum_v w_vc x_vi with
// w_0c = -sum_r Dm^-1_rc, w_vc = Dm^-1_(v-1)c, so no 9x12 map is stored.  Column-major vec throughout.
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

// In-place projection of a symmetric 9x9 onto the PSD cone: A <- sum_k max(w_k, 0) q_k q_k^T.
__device__ void project_psd9(double (&a)[9][9]) {
  double v[9][9];
#pragma unroll 1
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j < 9; ++j) v[i][j] = i == j ? 1.0 : 0.0;
  double tr = 0.0;
  for (int i = 0; i < 9; ++i) tr += fabs(a[i][i]);
#pragma unroll 1
  for (int sweep = 0; sweep < 12; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 8; ++p)
      for (int q = p + 1; q < 9; ++q) off += a[p][q] * a[p][q];
    if (off <= 1e-30 * tr * tr) break;
#pragma unroll 1
    for (int p = 0; p < 8; ++p)
#pragma unroll 1
      for (int q = p + 1; q < 9; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
        for (int k = 0; k < 9; ++k) {  // columns p, q
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 9; ++k) {  // rows p, q
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 9; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  double w[9];
  for (int k = 0; k < 9; ++k) w[k] = fmax(a[k][k], 0.0);
#pragma unroll 1
  for (int i = 0; i < 9; ++i)
    for (int j = i; j < 9; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 9; ++k) acc += v[i][k] * w[k] * v[j][k];
      a[i][j] = a[j][i] = acc;
    }
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

__global__ void __launch_bounds__(kET) elastic_blocks_kernel(const __grid_constant__ ElasticArgs a) {
  const int64_t t = (int64_t)blockIdx.x * kET + threadIdx.x;
  if (t >= a.nt) return;
  const int4 id = reinterpret_cast<const int4*>(a.tets)[t];
  const V3 x0 = load3(a.positions, id.x);
  const V3 d1 = load3(a.positions, id.y) - x0, d2 = load3(a.positions, id.z) - x0, d3 = load3(a.positions, id.w) - x0;
  const double ds[3][3] = {{d1.x, d2.x, d3.x}, {d1.y, d2.y, d3.y}, {d1.z, d2.z, d3.z}};
  double ri[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) ri[r][c] = a.rest_inv[9 * t + 3 * r + c];
  double f[3][3];
  for (int i = 0; i < 3; ++i)
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
  // vec(P), column-major: entry 3c + i
  const double gj[9] = {g0.x, g0.y, g0.z, g1.x, g1.y, g1.z, g2.x, g2.y, g2.z};
  const double fv[9] = {c0.x, c0.y, c0.z, c1.x, c1.y, c1.z, c2.x, c2.y, c2.z};
  // w_vc: dvec(F)/dx weights
  double w[4][3];
  for (int c = 0; c < 3; ++c) {
    w[0][c] = -(ri[0][c] + ri[1][c] + ri[2][c]);
    w[1][c] = ri[0][c];
    w[2][c] = ri[1][c];
    w[3][c] = ri[2][c];
  }
  if (a.grad) {
    double* g = a.grad + 12 * t;
    for (int v = 0; v < 4; ++v)
      for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
        for (int c = 0; c < 3; ++c) acc += w[v][c] * (mu * fv[3 * c + i] + k1 * gj[3 * c + i]);
        g[3 * v + i] = a.scale * vol * acc;
      }
  }
  if (!a.hess) return;
  double h[9][9];
#pragma unroll 1
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j < 9; ++j) h[i][j] = lam * gj[i] * gj[j] + (i == j ? mu : 0.0);
  // + k1 * d2J/dF2: block (c, d) of the 9x9 is +-skew(f_e) (elasticity.py:87-100)
  const V3 cols[3] = {c0, c1, c2};
  auto add_skew = [&](int br, int bc, const V3& u, double sgn) {
    const double s = sgn * k1;
    h[3 * br + 0][3 * bc + 1] += -s * u.z;
    h[3 * br + 0][3 * bc + 2] += s * u.y;
    h[3 * br + 1][3 * bc + 0] += s * u.z;
    h[3 * br + 1][3 * bc + 2] += -s * u.x;
    h[3 * br + 2][3 * bc + 0] += -s * u.y;
    h[3 * br + 2][3 * bc + 1] += s * u.x;
  };
  add_skew(0, 1, cols[2], -1.0);
  add_skew(0, 2, cols[1], 1.0);
  add_skew(1, 0, cols[2], 1.0);
  add_skew(1, 2, cols[0], -1.0);
  add_skew(2, 0, cols[1], -1.0);
  add_skew(2, 1, cols[0], 1.0);
  if (a.project) project_psd9(h);
  // hess[(3v+i), (3u+j)] = scale vol sum_{c,d} w_vc w_ud H9[3c+i][3d+j]
  double* out = a.hess + 144 * t;
  const double sv = a.scale * vol;
#pragma unroll 1
  for (int v = 0; v < 4; ++v)
    for (int i = 0; i < 3; ++i)
      for (int u = 0; u < 4; ++u)
        for (int j = 0; j < 3; ++j) {
          double acc = 0.0;
          for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) acc += w[v][c] * w[u][d] * h[3 * c + i][3 * d + j];
          out[(3 * v + i) * 12 + 3 * u + j] = sv * acc;
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
  elastic_blocks_kernel<<<(unsigned)((ntets + kET - 1) / kET), kET, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}
