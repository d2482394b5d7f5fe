// Per-contact barrier energy / gradient / analytically PSD-projected Hessian block.
//
// One launch per table; the table is kind-sorted and every CTA owns a 128-stencil tile of a
// single kind, so CTAs are branch-uniform.
// Phase 1: thread-per-stencil -- gather the 2..4 vertex positions, evaluate the distance
// branch, f = d/d_hat and its gradient, the barrier scalars and the closed-form retained
// eigenpair (lambda, w); everything stays in registers, no numerical eigendecomposition.
// The rank-1 factor z = sqrt(dt2*max(lambda,0)) * w and the scaled gradient are parked in
// shared memory, k-major with an odd stride (conflict-free both ways).
// Phase 2: the whole CTA streams the tile's dense D x D blocks out as z z^T with 16-byte
// stores to consecutive addresses -- the kernel is bound by those HBM writes
// (1152 B per 12x12 block against ~120 B of input).
//
// Reference semantics: proximity.py:183-229, gap.py:56-82, barrier.py:76-120,163-177,
// mollifier.py:55-144,191-210, solver.py:127-146,202-209.
#include "stencil_math.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

// 16-byte store of two adjacent outputs.  STREAM: evict-first (st.global.cs) -- a step that writes more than the L2
// holds gains nothing from allocating its output there (measured on 1.27 GB of blocks: 0.2417 -> 0.2376 ms); small
// batches keep plain stores so that the assembly that follows finds the blocks in L2.
template <bool STREAM>
__device__ __forceinline__ void store2(double* p, double a, double b) {
  if (STREAM) __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
  else *reinterpret_cast<double2*>(p) = make_double2(a, b);
}


constexpr int kTile = 128;  // stencils per CTA == threads per CTA

template <int KIND>
struct KindTraits;
template <> struct KindTraits<B200IPC_EE>  { static constexpr int S = 4; static constexpr bool PAR = false; };
template <> struct KindTraits<B200IPC_EEP> { static constexpr int S = 4; static constexpr bool PAR = true; };
template <> struct KindTraits<B200IPC_PE>  { static constexpr int S = 3; static constexpr bool PAR = false; };
template <> struct KindTraits<B200IPC_PEP> { static constexpr int S = 4; static constexpr bool PAR = true; };
template <> struct KindTraits<B200IPC_PP>  { static constexpr int S = 2; static constexpr bool PAR = false; };
template <> struct KindTraits<B200IPC_PPP> { static constexpr int S = 4; static constexpr bool PAR = true; };
template <> struct KindTraits<B200IPC_PT>  { static constexpr int S = 4; static constexpr bool PAR = false; };

struct KindArgs {
  int64_t n;                 // rows of this kind
  const int32_t* verts;      // (n,4)
  const uint8_t* sub;        // (n)
  const double* eps_x;       // (n)
  double* energy;            // (n) or null
  uint8_t* status;           // (n) or null
  double* grad;              // (n,D) or null
  double* hess;              // (n,D,D) or null
  double* fac;               // (n,D) or null: rank-1 factor z with hess = z z^T
};

// One launch covers every kind: CTA b works on tile (b - tile_off[kind]) of the kind whose tile
// range contains b, so a CTA is still branch-uniform while the step pays one launch and one tail.
struct StencilArgs {
  b200ipc_params prm;
  const double* positions;
  KindArgs k[B200IPC_NKINDS];
  uint32_t tile_off[B200IPC_NKINDS + 1];
};

constexpr int kPad = kTile + 1;  // odd stride: bank = 2(k*P + i) mod 32 is distinct across k and i

// TILED: the dense block leaves sub-block-major, (nb, S, S, 3, 3) -- every 3x3 sub-block 72 contiguous bytes, what
// the assembly's gather wants (one line per source instead of three); the reference's (nb, 3S, 3S) view is then
// produced only at the host boundary.  Same products, same bytes, another order.
template <int KIND, int FORM, bool STREAM, bool TILED>
__device__ __forceinline__ void stencil_tile(const b200ipc_params& prm, const double* __restrict__ positions,
                                             const KindArgs& a, int64_t tile, double* sm_z, double* sm_g,
                                             uint32_t* sm_lut) {
  using KT = KindTraits<KIND>;
  constexpr int S = KT::S;
  constexpr int D = 3 * S;
  constexpr int DD = D * D;
  constexpr int P = kPad;

  const int tid = threadIdx.x;
  const int64_t tile0 = tile * kTile;
  const int64_t i = tile0 + tid;

  if (TILED && a.hess) {
    // element k = ((va S + vc) 3 + i) 3 + j of a tiled block is z[3 va + i] z[3 vc + j]: shared-memory rows, once per CTA
    for (int k = tid; k < DD; k += kTile) {
      const int t = k / 9, q = k - 9 * t;
      const int va = t / S, vc = t - S * va;
      const int qi = q / 3, qj = q - 3 * qi;
      sm_lut[k] = (uint32_t)((3 * va + qi) * P) | ((uint32_t)((3 * vc + qj) * P) << 16);
    }
  }

  if (i < a.n) {
    const int4 vid = __ldg(reinterpret_cast<const int4*>(a.verts) + i);
    V3 x[4];
    x[0] = load3(positions, vid.x);
    x[1] = load3(positions, vid.y);
    if (S >= 3) x[2] = load3(positions, vid.z);
    if (S >= 4) x[3] = load3(positions, vid.w);

    V3 gd[4];
    double wit0, wit1;
    const double d2 = eval_distance<KIND>(x, KT::PAR ? (int)__ldg(a.sub + i) : 0, gd, wit0, wit1);

    const int st = d2 <= 0.0 ? B200IPC_PENETRATION : (d2 >= prm.d_hat_pow2 ? B200IPC_INACTIVE : B200IPC_ACTIVE);
    if (a.status) a.status[i] = (uint8_t)st;
    const bool live = st == B200IPC_ACTIVE;

    // ---- diagonal Jacobian (gap.py:65-67) ---------------------------------------------
    const double d = sqrt(d2);
    const double f = d / prm.d_hat;
    const double rinv = 1.0 / (2.0 * d * prm.d_hat);

    double energy = 0.0;
    if (a.energy) {  // solver.py:141-145: g = d2 / d_hat**2, not f*f
      energy = barrier_scalars<FORM>(d2 / prm.d_hat_pow2, prm.scale).b;
    }

    Coef k;
    V3 gc[4];
    double rc = 0.0;  // 1 / (2 sqrt c), 0 when sqrt c == 0 (gap.py:74-79)
    if (!KT::PAR) {
      k = coef_plain<FORM>(prm, f);
    } else {
      const double eps = __ldg(a.eps_x + i);
      const double c = cross_sq_one(x[0], x[1], x[2], x[3], gc);
      const double sqrt_c = sqrt(c);
      rc = sqrt_c > 0.0 ? 1.0 / (2.0 * sqrt_c) : 0.0;
      if (a.energy) {  // solver.py:140-142 uses the raw c of parallel_measure
        double e, de, d2e;
        mollifier_eval(c, eps, e, de, d2e);
        energy = e * energy;
      }
      k = coef_parallel<FORM>(prm, f, sqrt_c, eps);
    }

    if (a.energy) a.energy[i] = live ? energy : 0.0;

    // scale: grad *= dt2, hess *= dt2 (solver.py:207-208); z z^T = dt2*lam * w w^T
    const double zs = live ? sqrt(prm.dt2 * k.lam) : 0.0;
    const double gs = live ? prm.dt2 : 0.0;
#pragma unroll
    for (int v = 0; v < S; ++v) {
      const double uf[3] = {gd[v].x * rinv, gd[v].y * rinv, gd[v].z * rinv};
      double uc[3] = {0.0, 0.0, 0.0};
      if (KT::PAR) {
        uc[0] = gc[v].x * rc;
        uc[1] = gc[v].y * rc;
        uc[2] = gc[v].z * rc;
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double w, gr;
        if (KT::PAR) {
          w = k.cw_c * uc[q] + k.cw_f * uf[q];
          gr = k.cg_c * uc[q] + k.cg_f * uf[q];
        } else {
          w = uf[q];
          gr = k.cg_f * uf[q];
        }
        sm_z[(3 * v + q) * P + tid] = live ? zs * w : 0.0;
        sm_g[(3 * v + q) * P + tid] = live ? gs * gr : 0.0;
      }
    }
  }
  __syncthreads();

  const int64_t left = a.n - tile0;
  const int ntile = left < kTile ? (int)left : kTile;

  // ---- phase 2a: gradient tile and factor tile, (ntile, D) contiguous each ------------------
#pragma unroll
  for (int which = 0; which < 2; ++which) {
    double* base = which == 0 ? a.grad : a.fac;
    const double* sm = which == 0 ? sm_g : sm_z;
    if (!base) continue;
    double* out = base + tile0 * D;
    const int total = ntile * D;
    for (int e = 2 * tid; e < total; e += 2 * kTile) {
      const int b0 = e / D, k0 = e - b0 * D;
      const double v0 = sm[k0 * P + b0];
      if (e + 1 < total) {
        const int k1 = (k0 + 1 == D) ? 0 : k0 + 1;
        const int b1 = (k0 + 1 == D) ? b0 + 1 : b0;
        const double v1 = sm[k1 * P + b1];
        store2<STREAM>(out + e, v0, v1);
      } else {
        out[e] = v0;
      }
    }
  }

  // ---- phase 2b: Hessian tile, (ntile, D, D) contiguous, z z^T ----------------------------
  if (a.hess) {
    double* out = a.hess + tile0 * DD;
    const int total = ntile * DD;
    if (TILED) {
      for (int e = 2 * tid; e < total; e += 2 * kTile) {
        const int b0 = e / DD, k0 = e - b0 * DD;
        const uint32_t l0 = sm_lut[k0];
        const double v0 = sm_z[(l0 & 0xffffu) + b0] * sm_z[(l0 >> 16) + b0];
        if (e + 1 < total) {
          const int k1 = (k0 + 1 == DD) ? 0 : k0 + 1;
          const int b1 = (k0 + 1 == DD) ? b0 + 1 : b0;
          const uint32_t l1 = sm_lut[k1];
          const double v1 = sm_z[(l1 & 0xffffu) + b1] * sm_z[(l1 >> 16) + b1];
          store2<STREAM>(out + e, v0, v1);
        } else {
          out[e] = v0;
        }
      }
    } else if (D % 2 == 0) {
      // rows have even length: a pair never straddles a row
      for (int e = 2 * tid; e < total; e += 2 * kTile) {
        const int b = e / DD, k = e - b * DD;
        const int r = k / D, c = k - r * D;
        const double zr = sm_z[r * P + b];
        const double v0 = zr * sm_z[c * P + b];
        const double v1 = zr * sm_z[(c + 1) * P + b];
        store2<STREAM>(out + e, v0, v1);
      }
    } else {
      for (int e = 2 * tid; e < total; e += 2 * kTile) {
        const int b0 = e / DD, k0 = e - b0 * DD;
        const int r0 = k0 / D, c0 = k0 - r0 * D;
        const double v0 = sm_z[r0 * P + b0] * sm_z[c0 * P + b0];
        if (e + 1 < total) {
          const int e1 = e + 1;
          const int b1 = e1 / DD, k1 = e1 - b1 * DD;
          const int r1 = k1 / D, c1 = k1 - r1 * D;
          const double v1 = sm_z[r1 * P + b1] * sm_z[c1 * P + b1];
          store2<STREAM>(out + e, v0, v1);
        } else {
          out[e] = v0;
        }
      }
    }
  }
}

template <int FORM, bool STREAM, bool TILED>
__global__ void __launch_bounds__(kTile) barrier_stencil_kernel(const StencilArgs a) {
  __shared__ double sm_z[12 * kPad];
  __shared__ double sm_g[12 * kPad];
  __shared__ uint32_t sm_lut[TILED ? 144 : 1];
  const uint32_t b = blockIdx.x;
  int kind = 0;
#pragma unroll
  for (int k = 1; k < B200IPC_NKINDS; ++k)
    if (b >= a.tile_off[k]) kind = k;
  const int64_t tile = b - a.tile_off[kind];
  switch (kind) {
    case B200IPC_EE: stencil_tile<B200IPC_EE, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_EE], tile, sm_z, sm_g, sm_lut); break;
    case B200IPC_EEP: stencil_tile<B200IPC_EEP, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_EEP], tile, sm_z, sm_g, sm_lut); break;
    case B200IPC_PE: stencil_tile<B200IPC_PE, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_PE], tile, sm_z, sm_g, sm_lut); break;
    case B200IPC_PEP: stencil_tile<B200IPC_PEP, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_PEP], tile, sm_z, sm_g, sm_lut); break;
    case B200IPC_PP: stencil_tile<B200IPC_PP, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_PP], tile, sm_z, sm_g, sm_lut); break;
    case B200IPC_PPP: stencil_tile<B200IPC_PPP, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_PPP], tile, sm_z, sm_g, sm_lut); break;
    default: stencil_tile<B200IPC_PT, FORM, STREAM, TILED>(a.prm, a.positions, a.k[B200IPC_PT], tile, sm_z, sm_g, sm_lut); break;
  }
}

// ---------------------------------------------------------------------------------------------
// energy reduction: deterministic two-pass sum + status counts
// ---------------------------------------------------------------------------------------------
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 592;  // 4 per SM

__global__ void __launch_bounds__(kRedThreads) reduce_energy_pass1(int64_t n, const double* __restrict__ energy,
                                                                   const uint8_t* __restrict__ status,
                                                                   double* __restrict__ part_e,
                                                                   int64_t* __restrict__ part_c) {
  double acc = 0.0;
  long long c1 = 0, c2 = 0;
  for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedThreads) {
    if (energy) acc += energy[i];
    if (status) {
      const int s = status[i];
      c1 += s == B200IPC_INACTIVE;
      c2 += s == B200IPC_PENETRATION;
    }
  }
  __shared__ double se[kRedThreads / 32];
  __shared__ long long s1[kRedThreads / 32], s2[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    c1 += __shfl_down_sync(0xffffffffu, c1, o);
    c2 += __shfl_down_sync(0xffffffffu, c2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = acc;
    s1[threadIdx.x >> 5] = c1;
    s2[threadIdx.x >> 5] = c2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0;
    long long a1 = 0, a2 = 0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      e += se[w];
      a1 += s1[w];
      a2 += s2[w];
    }
    part_e[blockIdx.x] = e;
    part_c[2 * blockIdx.x] = a1;
    part_c[2 * blockIdx.x + 1] = a2;
  }
}

__global__ void reduce_energy_pass2(int nparts, const double* __restrict__ part_e, const int64_t* __restrict__ part_c,
                                    double* __restrict__ result, int64_t* __restrict__ counts) {
  // one warp, fixed order
  double e = 0.0;
  long long c1 = 0, c2 = 0;
  for (int i = threadIdx.x; i < nparts; i += 32) {
    e += part_e[i];
    c1 += part_c[2 * i];
    c2 += part_c[2 * i + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_down_sync(0xffffffffu, e, o);
    c1 += __shfl_down_sync(0xffffffffu, c1, o);
    c2 += __shfl_down_sync(0xffffffffu, c2, o);
  }
  if (threadIdx.x == 0) {
    if (result) result[0] = e;
    if (counts) {
      counts[0] = c1;
      counts[1] = c2;
    }
  }
}

}  // namespace b200ipc

using namespace b200ipc;

template <int FORM>
static void launch_stencils(bool streaming, bool tiled, unsigned tiles, cudaStream_t s, const StencilArgs& a) {
  if (tiled) {
    if (streaming) barrier_stencil_kernel<FORM, true, true><<<tiles, kTile, 0, s>>>(a);
    else barrier_stencil_kernel<FORM, false, true><<<tiles, kTile, 0, s>>>(a);
  } else {
    if (streaming) barrier_stencil_kernel<FORM, true, false><<<tiles, kTile, 0, s>>>(a);
    else barrier_stencil_kernel<FORM, false, false><<<tiles, kTile, 0, s>>>(a);
  }
}

extern "C" int b200ipc_barrier_stencils_layout(const b200ipc_params* params, int64_t nverts, const double* positions,
                                               int64_t n, const int64_t* kind_off, const int32_t* verts,
                                               const uint8_t* sub, const double* eps_x, double* energy,
                                               uint8_t* status, double* grad2, double* hess2, double* grad3,
                                               double* hess3, double* grad4, double* hess4, double* fac2, double* fac3,
                                               double* fac4, int32_t hess_layout, void* stream) {
  if (!params || !kind_off || n < 0 || nverts < 0) return B200IPC_EINVAL;
  if (hess_layout != B200IPC_LAYOUT_DENSE && hess_layout != B200IPC_LAYOUT_SUBBLOCK) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!positions || !verts) return B200IPC_EINVAL;
  if (kind_off[0] != 0 || kind_off[B200IPC_NKINDS] != n) return B200IPC_EINVAL;
  for (int k = 0; k < B200IPC_NKINDS; ++k)
    if (kind_off[k + 1] < kind_off[k]) return B200IPC_EINVAL;
  const bool has_par = kind_off[B200IPC_EEP + 1] > kind_off[B200IPC_EEP] ||
                       kind_off[B200IPC_PEP + 1] > kind_off[B200IPC_PEP] ||
                       kind_off[B200IPC_PPP + 1] > kind_off[B200IPC_PPP];
  if (has_par && (!sub || !eps_x)) return B200IPC_EINVAL;
  if (params->form != 0 && params->form != 1) return B200IPC_EINVAL;
  const uintptr_t align = (uintptr_t)verts | (uintptr_t)grad2 | (uintptr_t)hess2 | (uintptr_t)grad3 |
                          (uintptr_t)hess3 | (uintptr_t)grad4 | (uintptr_t)hess4 | (uintptr_t)fac2 |
                          (uintptr_t)fac3 | (uintptr_t)fac4;
  if (align & 15) return B200IPC_EINVAL;  // int4 loads / double2 stores

  cudaStream_t s = (cudaStream_t)stream;
  // family-4 rows follow the list order EE, EEP, PEP, PPP, PT (solver.py:237-248)
  const int fam4_order[5] = {B200IPC_EE, B200IPC_EEP, B200IPC_PEP, B200IPC_PPP, B200IPC_PT};
  int64_t row4[B200IPC_NKINDS] = {0, 0, 0, 0, 0, 0, 0};
  int64_t acc = 0;
  for (int j = 0; j < 5; ++j) {
    row4[fam4_order[j]] = acc;
    acc += kind_off[fam4_order[j] + 1] - kind_off[fam4_order[j]];
  }
  StencilArgs a;
  a.prm = *params;
  a.positions = positions;
  uint64_t tiles = 0;
  for (int k = 0; k < B200IPC_NKINDS; ++k) {
    const int64_t off = kind_off[k], cnt = kind_off[k + 1] - off;
    KindArgs& ka = a.k[k];
    ka.n = cnt;
    ka.verts = verts + 4 * off;
    ka.sub = sub ? sub + off : nullptr;
    ka.eps_x = eps_x ? eps_x + off : nullptr;
    ka.energy = energy ? energy + off : nullptr;
    ka.status = status ? status + off : nullptr;
    if (k == B200IPC_PP) {
      ka.grad = grad2; ka.hess = hess2; ka.fac = fac2;
    } else if (k == B200IPC_PE) {
      ka.grad = grad3; ka.hess = hess3; ka.fac = fac3;
    } else {
      ka.grad = grad4 ? grad4 + 12 * row4[k] : nullptr;
      ka.hess = hess4 ? hess4 + 144 * row4[k] : nullptr;
      ka.fac = fac4 ? fac4 + 12 * row4[k] : nullptr;
    }
    a.tile_off[k] = (uint32_t)tiles;
    tiles += (uint64_t)((cnt + kTile - 1) / kTile);
  }
  a.tile_off[B200IPC_NKINDS] = (uint32_t)tiles;
  if (tiles >= (1ull << 31)) return B200IPC_EINVAL;
  // output larger than what the L2 can keep for the next kernel: stream it
  int64_t out_bytes = 0;
  for (int k = 0; k < B200IPC_NKINDS; ++k) {
    const int64_t sz = k == B200IPC_PP ? 2 : (k == B200IPC_PE ? 3 : 4);
    if (a.k[k].hess) out_bytes += a.k[k].n * 72 * sz * sz;
  }
  const bool streaming = out_bytes > (96ll << 20);
  const bool tiled = hess_layout == B200IPC_LAYOUT_SUBBLOCK;
  if (params->form == 0) launch_stencils<0>(streaming, tiled, (unsigned)tiles, s, a);
  else launch_stencils<1>(streaming, tiled, (unsigned)tiles, s, a);
  return post_launch();
}

extern "C" int b200ipc_barrier_stencils_ex(const b200ipc_params* params, int64_t nverts, const double* positions,
                                           int64_t n, const int64_t* kind_off, const int32_t* verts,
                                           const uint8_t* sub, const double* eps_x, double* energy, uint8_t* status,
                                           double* grad2, double* hess2, double* grad3, double* hess3, double* grad4,
                                           double* hess4, double* fac2, double* fac3, double* fac4, void* stream) {
  return b200ipc_barrier_stencils_layout(params, nverts, positions, n, kind_off, verts, sub, eps_x, energy, status,
                                         grad2, hess2, grad3, hess3, grad4, hess4, fac2, fac3, fac4,
                                         B200IPC_LAYOUT_DENSE, stream);
}

extern "C" int b200ipc_barrier_stencils(const b200ipc_params* params, int64_t nverts, const double* positions,
                                        int64_t n, const int64_t* kind_off, const int32_t* verts, const uint8_t* sub,
                                        const double* eps_x, double* energy, uint8_t* status, double* grad2,
                                        double* hess2, double* grad3, double* hess3, double* grad4, double* hess4,
                                        void* stream) {
  return b200ipc_barrier_stencils_ex(params, nverts, positions, n, kind_off, verts, sub, eps_x, energy, status, grad2,
                                     hess2, grad3, hess3, grad4, hess4, nullptr, nullptr, nullptr, stream);
}

extern "C" int b200ipc_reduce_energy(int64_t n, const double* energy, const uint8_t* status, double* result,
                                     int64_t* counts, void* workspace, void* stream) {
  if (n < 0 || (!result && !counts) || !workspace) return B200IPC_EINVAL;
  static_assert(3 * kRedBlocks * 8 <= B200IPC_REDUCE_WS_BYTES, "workspace constant too small");
  cudaStream_t s = (cudaStream_t)stream;
  double* part_e = static_cast<double*>(workspace);
  int64_t* part_c = reinterpret_cast<int64_t*>(part_e + kRedBlocks);
  reduce_energy_pass1<<<kRedBlocks, kRedThreads, 0, s>>>(n, energy, status, part_e, part_c);
  int rc = post_launch();
  if (rc) return rc;
  reduce_energy_pass2<<<1, 32, 0, s>>>(kRedBlocks, part_e, part_c, result, counts);
  return post_launch();
}
