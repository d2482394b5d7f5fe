// Multilevel additive Schwarz (MAS) preconditioner for the assembled Newton matrix, and the PCG loop that
// uses it -- SURVEY.md section 8(f) row N4, second half; PAPER.md:683-685 ("we incorporate the Multilevel
// Additive Schwarz preconditioner [Wu et al. 2022] ... we trial the CG solver with both preconditioners per
// simulation and choose the one that is most efficient").  The reference package has block-Jacobi only
// (solver.py:265-276), which stays the default; nothing below exists in /root/reference.
//
//   order   vertices are sorted by the Morton code of their positions, quantised ISOTROPICALLY (10 bits per
//           axis over the largest extent), so that a thin stack of cloth layers falls into the same cells and
//           a run of 32 consecutive vertices is a spatial patch ACROSS the layers in contact.  (Measured on
//           the 1 M-contact cloth stack: index order or per-axis quantisation keep the layers apart and the
//           domains then contain none of the contact coupling -- 239-308 iterations, no better than
//           block-Jacobi's 244; isotropic Morton order: 73.)
//   level 0 domains = runs of 32 vertices (96 x 96); level l nodes = runs of 32^l vertices, 32 nodes per
//           domain; the level-l matrix is the Galerkin product with piecewise-constant (per coordinate)
//           prolongation, restricted to the domain.
//   setup   one CTA per domain gathers its 96 x 96 matrix from the BSR rows into shared memory, inverts it in
//           place (register-tiled block Gauss-Jordan, no pivoting: principal sub-matrices of an SPD matrix) and
//           stores one half of the symmetrised inverse in fp32, as node-block diagonals laid out so that a warp
//           applying it reads 128 consecutive bytes per instruction.  (The preconditioner only has to be a
//           fixed SPD operator; fp32 and the symmetric half quarter its HBM traffic -- 48 MB per application at
//           78 k vertices -- and leave the iteration count unchanged: measured 73 vs 73.)
//   apply   M^-1 r = sum_l P_l D_l^-1 P_l^T r; one warp per domain, lane k holds vertex k's three components.
//
// pcg_mas_kernel is pcg_stream_kernel (pcg.cu) with this operator in the place of the 3x3 inverses: the level-0
// application needs only the residual of the domain's own 32 vertices, so it is fused into the update phase --
// a warp per domain forms r' = r - alpha q for its vertices and multiplies straight away -- and the iteration
// keeps its TWO grid barriers.  A second level adds a coarse phase and a fix-up pass (two more barriers).
// The loop stops on the REFERENCE's rule: delta_bj = r . P_bj r <= tol * delta_bj0 with the block-Jacobi
// inverses P_bj (solver.py:302), so a caller gets a direction that meets the same criterion whichever
// preconditioner drove the iteration.  Deterministic: fixed summation orders, no atomics.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cub/cub.cuh>

#include "spmv_stream.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace cg = cooperative_groups;

namespace b200ipc {
namespace mas {

constexpr int kDom = 32;            // vertices (nodes) per domain
constexpr int kDim = 3 * kDom;      // 96
constexpr int kLd = kDim + 1;       // shared-memory row stride of the matrix being inverted (odd: no bank conflicts down a column)
constexpr int kInvThreads = 256;
constexpr int kMaxLevels = 2;
constexpr int kMaxParts = 4096;
// Matrix bytes fetched with evict-last priority in the PCG loop; everything else streams evict-first, which is what
// keeps the stored inverses (48 MB at 78 k vertices, evict-last loads) L2-resident from one iteration to the next:
// measured 56.0 -> 47.7 us per iteration, DRAM reads 162 -> 102 MB per iteration.
constexpr double kMasPinMb = 1.0;
constexpr int kOffsets = kDom / 2 + 1;   // stored node-block diagonals: block (k, (k + o) mod 32), o = 0..16
constexpr int64_t kInvFloats = (int64_t)kOffsets * 9 * kDom;   // fp32 entries of one stored inverse (symmetric half)

template <typename T>
struct Buf {
  T* ptr = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, n * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

}  // namespace mas
}  // namespace b200ipc

struct b200ipc_mas {
  int64_t nverts = 0;
  int32_t levels = 0;                 // levels built by the last setup
  int64_t ndom[b200ipc::mas::kMaxLevels] = {0, 0};    // domains per level
  int64_t nnode[b200ipc::mas::kMaxLevels] = {0, 0};   // nodes per level (level 0: vertices)
  bool ordered = false, ready = false;
  const uint8_t* fixed = nullptr;     // caller's array of the last setup (must outlive the solves)
  b200ipc::mas::Buf<int32_t> perm;    // (32 ndom0): vertex of each rank, -1 = padding
  b200ipc::mas::Buf<int32_t> rank;    // (nverts): rank of each vertex
  b200ipc::mas::Buf<float> inv[b200ipc::mas::kMaxLevels];   // stored inverses, (ndom, 17, 9, 32)
  b200ipc::mas::Buf<double> coarse;   // level-1 node residuals and corrections: 2 x 3 x nnode1
  b200ipc::mas::Buf<int32_t> colrank;  // column indices renamed to ranks (the PCG loop's vectors are in domain order)
  b200ipc::mas::Buf<uint32_t> keys_a, keys_b, val_a, val_b;
  b200ipc::mas::Buf<unsigned long long> box;   // 6 order-preserving encodings: min xyz, max xyz
  b200ipc::mas::Buf<uint8_t> temp;
};

namespace b200ipc {
namespace mas {

// ---- order ----------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long encode_ordered(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double decode_ordered(unsigned long long e) {
  const unsigned long long b = (e >> 63) ? (e & 0x7fffffffffffffffull) : ~e;
  return __longlong_as_double((long long)b);
}

__global__ void box_init_kernel(unsigned long long* box) {
  if (threadIdx.x < 3) box[threadIdx.x] = ~0ull;
  else if (threadIdx.x < 6) box[threadIdx.x] = 0ull;
}

__global__ void __launch_bounds__(256) box_kernel(int64_t n, const double* __restrict__ x, unsigned long long* box) {
  const int64_t v = (int64_t)blockIdx.x * 256 + threadIdx.x;
  for (int k = 0; k < 3; ++k) {
    unsigned long long lo = ~0ull, hi = 0ull;
    if (v < n) lo = hi = encode_ordered(x[3 * v + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_down_sync(0xffffffffu, lo, o), h2 = __shfl_down_sync(0xffffffffu, hi, o);
      lo = l2 < lo ? l2 : lo;
      hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {   // min / max are exact and order-free: deterministic
      atomicMin(box + k, lo);
      atomicMax(box + 3 + k, hi);
    }
  }
}

__device__ __forceinline__ uint32_t spread3(uint32_t v) {   // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// code = interleave(qx, qy, qz), q = floor((p - lo) / ext * 1023) with ext the LARGEST extent (isotropic cells)
__global__ void __launch_bounds__(256) morton_kernel(int64_t n, const double* __restrict__ x,
                                                     const unsigned long long* __restrict__ box,
                                                     uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t v = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (v >= n) return;
  double lo[3], ext = 0.0;
  for (int k = 0; k < 3; ++k) {
    lo[k] = decode_ordered(box[k]);
    const double e = decode_ordered(box[3 + k]) - lo[k];
    ext = e > ext ? e : ext;
  }
  uint32_t code = 0;
  if (ext > 0.0) {
    uint32_t q[3];
    for (int k = 0; k < 3; ++k) {
      const double t = (x[3 * v + k] - lo[k]) / ext * 1023.0;
      q[k] = (uint32_t)t;   // 0 <= t <= 1023
    }
    code = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
  }
  keys[v] = code;
  vals[v] = (uint32_t)v;
}

__global__ void __launch_bounds__(256) iota_kernel(int64_t n, uint32_t* vals) {
  const int64_t v = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (v < n) vals[v] = (uint32_t)v;
}

__global__ void __launch_bounds__(256) perm_kernel(int64_t n, int64_t npad, const uint32_t* __restrict__ sorted,
                                                   int32_t* __restrict__ perm, int32_t* __restrict__ rank) {
  const int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (r >= npad) return;
  if (r < n) {
    const int32_t v = (int32_t)sorted[r];
    perm[r] = v;
    rank[v] = (int32_t)r;
  } else {
    perm[r] = -1;
  }
}

// ---- setup: gather + invert -------------------------------------------------------------------------------
struct SetupArgs {
  int64_t n;
  int64_t nnode;            // nodes of this level
  int level;                // 0 or 1
  const int32_t* rowptr;
  const int32_t* colidx;
  const double* vals;
  const int32_t* perm;
  const int32_t* rank;
  const uint8_t* fixed;     // Dirichlet vertices stay out of the coarse spaces
  float* inv;               // (ndom, 17, 9, 32)
};

// In-place inverse of the SPD matrix in shared memory (row stride kLd) by BLOCK Gauss-Jordan over the 32
// node blocks (3x3 pivots, no pivoting: principal sub-matrices of an SPD matrix), register-tiled: the 256
// threads form a 16 x 16 grid and thread (ty, tx) keeps the 6 x 6 tile of rows 6ty.., columns 6tx.. in
// registers for all 32 steps.  Step K: the pivot's owner inverts it (P); the 16 threads of its tile row publish
// R' = P A[K,:] with P itself in the pivot columns, the 16 of its tile column publish C' = A[:,K] with -I in
// the pivot rows; then every thread does A' = B - C'^T R' on its tile, B = A with the pivot rows and columns
// zeroed -- one uniform rank-3 update, 108 FMAs from 36 shared-memory loads, which also lands the scaled
// pivot rows, -C P in the pivot columns and P in the pivot block.  (The first version updated the matrix in
// shared memory element by element, 96 scalar steps: 2.9 ms for 2450 domains, instruction-bound on index
// arithmetic.)
__device__ __forceinline__ void invert_in_place(double* A, double* Rp, double* Cp, double* Pp) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double a[6][6];
  __syncthreads();   // the gather that filled A
#pragma unroll
  for (int s = 0; s < 6; ++s)
#pragma unroll
    for (int t = 0; t < 6; ++t) a[s][t] = A[(6 * ty + s) * kLd + 6 * tx + t];
  for (int K = 0; K < kDom; ++K) {
    const int tK = K >> 1;
    const bool hi = K & 1;
    if (ty == tK && tx == tK) {   // the pivot block: closed-form 3x3 inverse
      double p[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) p[i][j] = hi ? a[3 + i][3 + j] : a[i][j];
      const double c00 = p[1][1] * p[2][2] - p[1][2] * p[2][1], c01 = p[1][2] * p[2][0] - p[1][0] * p[2][2],
                   c02 = p[1][0] * p[2][1] - p[1][1] * p[2][0];
      const double inv = 1.0 / (p[0][0] * c00 + p[0][1] * c01 + p[0][2] * c02);
      Pp[0] = c00 * inv;
      Pp[1] = (p[0][2] * p[2][1] - p[0][1] * p[2][2]) * inv;
      Pp[2] = (p[0][1] * p[1][2] - p[0][2] * p[1][1]) * inv;
      Pp[3] = c01 * inv;
      Pp[4] = (p[0][0] * p[2][2] - p[0][2] * p[2][0]) * inv;
      Pp[5] = (p[0][2] * p[1][0] - p[0][0] * p[1][2]) * inv;
      Pp[6] = c02 * inv;
      Pp[7] = (p[0][1] * p[2][0] - p[0][0] * p[2][1]) * inv;
      Pp[8] = (p[0][0] * p[1][1] - p[0][1] * p[1][0]) * inv;
    }
    __syncthreads();
    if (ty == tK) {   // R'[i][j] = (P A[K,:])[i][j]; pivot columns: P
      double P[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) P[e] = Pp[e];
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const double r0 = hi ? a[3][t] : a[0][t], r1 = hi ? a[4][t] : a[1][t], r2 = hi ? a[5][t] : a[2][t];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double v = fma(P[3 * i + 2], r2, fma(P[3 * i + 1], r1, P[3 * i] * r0));
          if (tx == tK && (t >= 3) == hi) v = P[3 * i + (t % 3)];
          Rp[i * kDim + 6 * tx + t] = v;
        }
      }
    }
    if (tx == tK) {   // C'[j][i] = A[i][K-column j]; pivot rows: -I
#pragma unroll
      for (int s2 = 0; s2 < 6; ++s2)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double v = hi ? a[s2][3 + j] : a[s2][j];
          if (ty == tK && (s2 >= 3) == hi) v = (s2 % 3) == j ? -1.0 : 0.0;
          Cp[j * kDim + 6 * ty + s2] = v;
        }
    }
    __syncthreads();
    double r[3][6];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int t = 0; t < 6; ++t) r[i][t] = Rp[i * kDim + 6 * tx + t];
    const bool row_lo = 2 * ty == K, row_hi = 2 * ty + 1 == K, col_lo = 2 * tx == K, col_hi = 2 * tx + 1 == K;
#pragma unroll
    for (int s2 = 0; s2 < 6; ++s2) {
      const double c0 = Cp[6 * ty + s2], c1 = Cp[kDim + 6 * ty + s2], c2 = Cp[2 * kDim + 6 * ty + s2];
      const bool rowp = s2 < 3 ? row_lo : row_hi;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const bool colp = t < 3 ? col_lo : col_hi;
        const double base = (rowp || colp) ? 0.0 : a[s2][t];
        a[s2][t] = fma(-c2, r[2][t], fma(-c1, r[1][t], fma(-c0, r[0][t], base)));
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 6; ++s)
#pragma unroll
    for (int t = 0; t < 6; ++t) A[(6 * ty + s) * kLd + 6 * tx + t] = a[s][t];
  __syncthreads();
}

__global__ void __launch_bounds__(kInvThreads, 2) mas_setup_kernel(const __grid_constant__ SetupArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                       // kDim x kLd
  double* Rp = sm + kDim * kLd;         // 3 x kDim
  double* Cp = Rp + 3 * kDim;           // 3 x kDim
  double* Pp = Cp + 3 * kDim;           // 9
  const int64_t D = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < kDim * kLd; e += kInvThreads) A[e] = 0.0;
  __syncthreads();
  if (a.level == 0) {
    // node k of the domain = vertex perm[32 D + k]; every BSR block of its row whose column lies in the domain
    // is one 3x3 of the domain matrix -- distinct blocks, distinct targets: plain stores
    for (int k = w; k < kDom; k += kInvThreads / 32) {
      const int32_t i = a.perm[kDom * D + k];
      if (i < 0) {   // padding: identity
        if (lane < 3) A[(3 * k + lane) * kLd + 3 * k + lane] = 1.0;
        continue;
      }
      const int32_t b0 = a.rowptr[i], b1 = a.rowptr[i + 1];
      for (int32_t b = b0 + lane; b < b1; b += 32) {
        const int32_t rj = a.rank[a.colidx[b]];
        if ((rj >> 5) == D) {
          const int m = rj & 31;
          const double* v = a.vals + 9ll * b;
#pragma unroll
          for (int t = 0; t < 9; ++t) A[(3 * k + t / 3) * kLd + 3 * m + t % 3] = v[t];
        }
      }
    }
  } else {
    // node g = 32 D + k of level 1 = the 32 vertices of ranks [32 g, 32 g + 32); entry (k, m) of the domain
    // matrix sums every BSR block between the two nodes.  Lane m owns column node m; the warp walks the
    // rows and blocks of node k one after the other (fixed order: deterministic sums, no atomics).  Dirichlet
    // vertices are not part of the coarse space (their prolongation rows are zero, so the correction leaves
    // them exactly at rest); a node made of such vertices only gets the identity.
    for (int k = w; k < kDom; k += kInvThreads / 32) {
      const int64_t g = (int64_t)kDom * D + k;
      double acc[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[t] = 0.0;
      if (g >= a.nnode) {
        if (lane < 3) A[(3 * k + lane) * kLd + 3 * k + lane] = 1.0;
        continue;
      }
      bool any = false;
      for (int rr = 0; rr < kDom; ++rr) {
        const int64_t r = kDom * g + rr;
        if (r >= a.n) break;
        const int32_t i = a.perm[r];
        if (a.fixed[i]) continue;
        any = true;
        const int32_t b0 = a.rowptr[i], b1 = a.rowptr[i + 1];
        for (int32_t bb = b0; bb < b1; bb += 32) {
          const int32_t b = bb + lane;
          int32_t gj = -1;
          if (b < b1) gj = a.rank[a.colidx[b]] >> 5;             // level-1 node of the block's column
          const bool mine_dom = gj >= 0 && (gj >> 5) == D;
          unsigned todo = __ballot_sync(0xffffffffu, mine_dom);
          while (todo) {                                          // blocks of this trip inside the domain, in order
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int m = __shfl_sync(0xffffffffu, gj, src) & 31;
            if (lane == m) {
              const double* v = a.vals + 9ll * (bb + src);
#pragma unroll
              for (int t = 0; t < 9; ++t) acc[t] += v[t];
            }
          }
        }
      }
#pragma unroll
      for (int t = 0; t < 9; ++t) A[(3 * k + t / 3) * kLd + 3 * lane + t % 3] = acc[t];
      if (!any && lane < 3) A[(3 * k + lane) * kLd + 3 * k + lane] = 1.0;
    }
  }
  invert_in_place(A, Rp, Cp, Pp);
  // stored: the node-block diagonals o = 0..16 of the symmetrised inverse, fp32, S[o][e][k] = entry e = 3a+b of
  // block (k, (k+o) mod 32) -- every unordered pair of nodes once (o = 16 holds both orientations), and lane k
  // of the applying warp reads S[o][e][k]: 128 consecutive bytes per instruction
  float* out = a.inv + D * kInvFloats;
  for (int e2 = threadIdx.x; e2 < kOffsets * 9 * kDom; e2 += kInvThreads) {
    const int o = e2 / (9 * kDom), rem = e2 - o * 9 * kDom, e = rem / kDom, k = rem - e * kDom;
    const int row = 3 * k + e / 3, col = 3 * ((k + o) & 31) + e % 3;
    out[e2] = (float)(0.5 * (A[row * kLd + col] + A[col * kLd + row]));
  }
}

// ---- apply ------------------------------------------------------------------------------------------------
// z = Minv r for one domain: lane k holds r (3k..3k+2) and receives z (3k..3k+2).  Offset o pairs lane k with
// node m = k + o: the lane adds B_km r_m to its own z and hands B_km^T r_k to lane m -- every lane receives exactly
// one such term per offset, so there is no conflict and the order is fixed.  153 coalesced 128-byte loads.
// the stored inverses are re-read every iteration: evict-last keeps them in L2 under the matrix stream
__device__ __forceinline__ float ld_keep(const float* p) {
#ifdef B200IPC_MAS_NO_HINT
  return __ldg(p);
#else
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(0x14F0000000000000ull));
  return v;
#endif
}

__device__ __forceinline__ void domain_apply(const float* __restrict__ S, int lane, double r0, double r1, double r2,
                                             double& z0, double& z1, double& z2) {
  const float* s = S + lane;
  {
    const float b0 = ld_keep(s), b1 = ld_keep(s + 32), b2 = ld_keep(s + 64), b3 = ld_keep(s + 96), b4 = ld_keep(s + 128),
                b5 = ld_keep(s + 160), b6 = ld_keep(s + 192), b7 = ld_keep(s + 224), b8 = ld_keep(s + 256);
    z0 = fma((double)b2, r2, fma((double)b1, r1, (double)b0 * r0));
    z1 = fma((double)b5, r2, fma((double)b4, r1, (double)b3 * r0));
    z2 = fma((double)b8, r2, fma((double)b7, r1, (double)b6 * r0));
  }
#pragma unroll 3
  for (int o = 1; o < kDom / 2; ++o) {
    const float* so = s + o * 9 * kDom;
    const float b0 = ld_keep(so), b1 = ld_keep(so + 32), b2 = ld_keep(so + 64), b3 = ld_keep(so + 96), b4 = ld_keep(so + 128),
                b5 = ld_keep(so + 160), b6 = ld_keep(so + 192), b7 = ld_keep(so + 224), b8 = ld_keep(so + 256);
    const int m = (lane + o) & 31, from = (lane - o) & 31;
    const double x0 = __shfl_sync(0xffffffffu, r0, m), x1 = __shfl_sync(0xffffffffu, r1, m),
                 x2 = __shfl_sync(0xffffffffu, r2, m);
    z0 = fma((double)b2, x2, fma((double)b1, x1, fma((double)b0, x0, z0)));
    z1 = fma((double)b5, x2, fma((double)b4, x1, fma((double)b3, x0, z1)));
    z2 = fma((double)b8, x2, fma((double)b7, x1, fma((double)b6, x0, z2)));
    const double t0 = fma((double)b6, r2, fma((double)b3, r1, (double)b0 * r0));
    const double t1 = fma((double)b7, r2, fma((double)b4, r1, (double)b1 * r0));
    const double t2 = fma((double)b8, r2, fma((double)b5, r1, (double)b2 * r0));
    z0 += __shfl_sync(0xffffffffu, t0, from);
    z1 += __shfl_sync(0xffffffffu, t1, from);
    z2 += __shfl_sync(0xffffffffu, t2, from);
  }
  {
    const float* so = s + (kDom / 2) * 9 * kDom;
    const float b0 = ld_keep(so), b1 = ld_keep(so + 32), b2 = ld_keep(so + 64), b3 = ld_keep(so + 96), b4 = ld_keep(so + 128),
                b5 = ld_keep(so + 160), b6 = ld_keep(so + 192), b7 = ld_keep(so + 224), b8 = ld_keep(so + 256);
    const double x0 = __shfl_xor_sync(0xffffffffu, r0, 16), x1 = __shfl_xor_sync(0xffffffffu, r1, 16),
                 x2 = __shfl_xor_sync(0xffffffffu, r2, 16);
    z0 = fma((double)b2, x2, fma((double)b1, x1, fma((double)b0, x0, z0)));
    z1 = fma((double)b5, x2, fma((double)b4, x1, fma((double)b3, x0, z1)));
    z2 = fma((double)b8, x2, fma((double)b7, x1, fma((double)b6, x0, z2)));
  }
}

struct Hierarchy {
  int64_t n;
  int32_t levels;
  int64_t ndom0, ndom1, nnode1;
  const int32_t* perm;
  const int32_t* rank;
  const uint8_t* fixed;
  const float* inv0;
  const float* inv1;
  double* r1;        // (nnode1, 3) level-1 residuals
  double* y1;        // (nnode1, 3) level-1 corrections
  int32_t debug;     // B200IPC_MAS_DEBUG: 1 = skip the domain products (z = r), 2 = skip the gathers' stores too (timing probes)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;   // lane 0
}

// standalone application (tests, and callers that run their own Krylov loop): three small launches
__global__ void __launch_bounds__(256) apply_level0_kernel(const __grid_constant__ Hierarchy h, const double* __restrict__ r,
                                                           double* __restrict__ z) {
  const int64_t D = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (D >= h.ndom0) return;
  const int32_t v = h.perm[kDom * D + lane];
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  if (v >= 0) {
    r0 = r[3 * v]; r1 = r[3 * v + 1]; r2 = r[3 * v + 2];
  }
  double z0, z1, z2;
  domain_apply(h.inv0 + D * kInvFloats, lane, r0, r1, r2, z0, z1, z2);
  if (v >= 0) {
    z[3 * v] = z0; z[3 * v + 1] = z1; z[3 * v + 2] = z2;
  }
  if (h.levels > 1) {
    const bool in = v >= 0 && !h.fixed[v];
    const double s0 = warp_sum(in ? r0 : 0.0), s1 = warp_sum(in ? r1 : 0.0), s2 = warp_sum(in ? r2 : 0.0);
    if (lane == 0) {
      h.r1[3 * D] = s0; h.r1[3 * D + 1] = s1; h.r1[3 * D + 2] = s2;
    }
  }
}

__global__ void __launch_bounds__(256) apply_level1_kernel(const __grid_constant__ Hierarchy h) {
  const int64_t D = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (D >= h.ndom1) return;
  const int64_t g = kDom * D + lane;
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  if (g < h.nnode1) {
    r0 = h.r1[3 * g]; r1 = h.r1[3 * g + 1]; r2 = h.r1[3 * g + 2];
  }
  double z0, z1, z2;
  domain_apply(h.inv1 + D * kInvFloats, lane, r0, r1, r2, z0, z1, z2);
  if (g < h.nnode1) {
    h.y1[3 * g] = z0; h.y1[3 * g + 1] = z1; h.y1[3 * g + 2] = z2;
  }
}

__global__ void __launch_bounds__(256) apply_prolong_kernel(const __grid_constant__ Hierarchy h, double* __restrict__ z) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= 3 * h.n) return;
  const int64_t v = t / 3;
  if (!h.fixed[v]) z[t] += h.y1[3 * (int64_t)(h.rank[v] >> 5) + (t - 3 * v)];
}

// ---- the PCG loop ---------------------------------------------------------------------------------------
struct PcgMasArgs {
  int64_t n;
  const double* pinv;       // block-Jacobi inverses: the stopping rule's norm
  const uint8_t* fixed;
  const double* rhs;
  double* d;
  // every working vector lives in DOMAIN ORDER (position p = rank of the vertex), so that the update phase of a
  // domain touches 32 consecutive vertices; the product reaches them through the renamed column indices
  double* buf[2];           // (n, 3, 2): (s_j, c_j) pairs, as in pcg_stream_kernel
  double* rbuf[2];
  double* q;
  double* dm;               // the solution in domain order (scattered to d at the end)
  double* pinvm;            // block-Jacobi inverses in domain order
  uint8_t* fixedm;          // Dirichlet flags in domain order
  double* part;             // 4 * kMaxParts partial sums
  double rel_tol;
  int32_t max_iters;
  b200ipc_pcg_result* result;  // device
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;  // valid in thread 0
}

// every CTA sums all partials in the same order -> identical value everywhere
__device__ __forceinline__ double sum_parts(const double* part, int nparts, double* sh, double* bc) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += part[i];
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) *bc = t;
  __syncthreads();
  const double out = *bc;
  __syncthreads();
  return out;
}

__global__ void __launch_bounds__(kStreamThreads, 1) pcg_mas_kernel(const __grid_constant__ PcgMasArgs a,
                                                                     const __grid_constant__ StreamMatrix m,
                                                                     const __grid_constant__ Hierarchy h) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ double sh[kStreamThreads / 32];
  __shared__ double bc;
  const StreamSmem sm = stream_smem(dyn);
  StreamState st;
  stream_init(m, sm, st);
  const uint32_t unbounded = 0xffffffffu;

  const int64_t tid = (int64_t)blockIdx.x * kStreamThreads + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * kStreamThreads;
  const int64_t gwarp = tid >> 5, nwarps = nthreads >> 5;
  const int lane = threadIdx.x & 31;
  const int nparts = gridDim.x;
  const int j = lane % 3;  // x component of this lane inside the product (lane = 9 r + 3 i + j)
  double* part_cq = a.part;
  double* part_mas = a.part + kMaxParts;
  double* part_bj = a.part + 2 * kMaxParts;
  double* part_co = a.part + 3 * kMaxParts;

  // The update phase, one warp per level-0 domain: r' = r - alpha q (first call: the masked right-hand side),
  // d += alpha c, s = level-0 correction of r', partial sums of r'.s and of the block-Jacobi norm r'.P_bj r'.
  auto update = [&](bool first, double alpha, const double* rold, double* rnew, double* bnew) {
    double acc_mas = 0.0, acc_bj = 0.0;
    // domains dealt round-robin over the CTAs first: every SM streams its share of the stored inverses
    for (int64_t D = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x; D < h.ndom0; D += nwarps) {
      const int64_t p = kDom * D + lane;
      const bool in = p < a.n;
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
      bool fx = false;
      if (in) {
        double* pm = a.pinvm + 9 * p;
        if (first) {   // bring the caller's arrays into domain order
          const int32_t v = h.perm[p];
          fx = a.fixed[v];
          a.fixedm[p] = fx;
          r0 = fx ? 0.0 : a.rhs[3 * v]; r1 = fx ? 0.0 : a.rhs[3 * v + 1]; r2 = fx ? 0.0 : a.rhs[3 * v + 2];
          a.dm[3 * p] = a.dm[3 * p + 1] = a.dm[3 * p + 2] = 0.0;
#pragma unroll
          for (int e = 0; e < 9; ++e) pm[e] = a.pinv[9 * v + e];
        } else {
          fx = a.fixedm[p];
          r0 = rold[3 * p] - alpha * a.q[3 * p];
          r1 = rold[3 * p + 1] - alpha * a.q[3 * p + 1];
          r2 = rold[3 * p + 2] - alpha * a.q[3 * p + 2];
          a.dm[3 * p] += alpha * bnew[6 * p + 1];
          a.dm[3 * p + 1] += alpha * bnew[6 * p + 3];
          a.dm[3 * p + 2] += alpha * bnew[6 * p + 5];
        }
        rnew[3 * p] = r0; rnew[3 * p + 1] = r1; rnew[3 * p + 2] = r2;
        acc_bj += r0 * (pm[0] * r0 + pm[1] * r1 + pm[2] * r2) + r1 * (pm[3] * r0 + pm[4] * r1 + pm[5] * r2) +
                  r2 * (pm[6] * r0 + pm[7] * r1 + pm[8] * r2);
      }
      double z0 = r0, z1 = r1, z2 = r2;
      if (h.debug != 1) domain_apply(h.inv0 + D * kInvFloats, lane, r0, r1, r2, z0, z1, z2);
      if (in) {
        bnew[6 * p] = z0; bnew[6 * p + 2] = z1; bnew[6 * p + 4] = z2;
        if (first) bnew[6 * p + 1] = bnew[6 * p + 3] = bnew[6 * p + 5] = 0.0;   // beta = 0 makes the first direction s
        acc_mas += r0 * z0 + r1 * z1 + r2 * z2;
      }
      if (h.levels > 1) {
        const bool use = in && !fx;
        const double s0 = warp_sum(use ? r0 : 0.0), s1 = warp_sum(use ? r1 : 0.0), s2 = warp_sum(use ? r2 : 0.0);
        if (lane == 0) {
          h.r1[3 * D] = s0; h.r1[3 * D + 1] = s1; h.r1[3 * D + 2] = s2;
        }
      }
    }
    const double t = block_sum(acc_mas, sh);
    if (threadIdx.x == 0) part_mas[blockIdx.x] = t;
    const double u = block_sum(acc_bj, sh);
    if (threadIdx.x == 0) part_bj[blockIdx.x] = u;
  };
  // Second level: coarse solves (a warp per level-1 domain), then the corrections are added to s.  Returns
  // (in every thread) the coarse part of r.s.
  auto coarse = [&](double* bnew) {
    double acc = 0.0;
    for (int64_t D = gwarp; D < h.ndom1; D += nwarps) {
      const int64_t g = kDom * D + lane;
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
      if (g < h.nnode1) {
        r0 = h.r1[3 * g]; r1 = h.r1[3 * g + 1]; r2 = h.r1[3 * g + 2];
      }
      double z0, z1, z2;
      domain_apply(h.inv1 + D * kInvFloats, lane, r0, r1, r2, z0, z1, z2);
      if (g < h.nnode1) {
        h.y1[3 * g] = z0; h.y1[3 * g + 1] = z1; h.y1[3 * g + 2] = z2;
        acc += r0 * z0 + r1 * z1 + r2 * z2;
      }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part_co[blockIdx.x] = t;
    grid.sync();
    for (int64_t t3 = tid; t3 < 3 * a.n; t3 += nthreads) {
      const int64_t p = t3 / 3;
      const int k = (int)(t3 - 3 * p);
      if (!a.fixedm[p]) bnew[6 * p + 2 * k] += h.y1[3 * (p >> 5) + k];
    }
    const double co = sum_parts(part_co, nparts, sh, &bc);
    grid.sync();
    return co;
  };

  update(true, 0.0, nullptr, a.rbuf[0], a.buf[0]);
  grid.sync();
  double delta0 = sum_parts(part_mas, nparts, sh, &bc);
  const double bj0 = sum_parts(part_bj, nparts, sh, &bc);
  if (h.levels > 1) delta0 += coarse(a.buf[0]);
  double delta_new = delta0, bj_new = bj0;
  double beta = 0.0;
  int iters = 0, cur = 0;

#ifdef B200IPC_PCG_TIMING
  unsigned long long tm[4] = {0, 0, 0, 0}, t0, t1;
#define MAS_TICK(k)                                            \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));     \
  tm[k] += t1 - t0;                                            \
  t0 = t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#else
#define MAS_TICK(k)
#endif
  if (bj0 > 0.0 && delta0 > 0.0) {
    while (iters < a.max_iters && bj_new > a.rel_tol * bj0) {
      const double* bold = a.buf[cur];
      double* bnew = a.buf[cur ^ 1];
      // ---- c = s + beta c (on the fly); q = A c; denom = c.q -----------------------------------------
      double acc = 0.0;
      const double2* wj = reinterpret_cast<const double2*>(bold) + j;
      stream_product(
          m, sm, st, unbounded,
          [&](int col) {
            const double2 w = wj[3ll * col];
            return w.x + beta * w.y;
          },
          [&](int64_t row, int i, double yi) {
            const int64_t p = h.rank[row];   // rows stream in matrix order; their vector entries sit at the rank
            const double2 w = reinterpret_cast<const double2*>(bold)[3 * p + i];
            const double cn = w.x + beta * w.y;
            bnew[6 * p + 2 * i + 1] = cn;
            a.q[3 * p + i] = yi;
            acc += cn * yi;
          });
      {
        const double t = block_sum(acc, sh);
        if (threadIdx.x == 0) part_cq[blockIdx.x] = t;
      }
      MAS_TICK(0)
      grid.sync();
      const double denom = sum_parts(part_cq, nparts, sh, &bc);
      if (denom <= 0.0) break;  // solver.py:305-306
      const double alpha = delta_new / denom;
      MAS_TICK(1)
      update(false, alpha, a.rbuf[cur], a.rbuf[cur ^ 1], bnew);
      MAS_TICK(2)
      grid.sync();
      const double delta_old = delta_new;
      delta_new = sum_parts(part_mas, nparts, sh, &bc);
      bj_new = sum_parts(part_bj, nparts, sh, &bc);
      if (h.levels > 1) delta_new += coarse(bnew);
      beta = delta_new / delta_old;
      cur ^= 1;
      ++iters;
      MAS_TICK(3)
    }
  }
  stream_drain(sm, st);
#ifdef B200IPC_PCG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 512)   // [product, barrier 1 + sums, update, barrier 2 + sums] ns per CTA
    for (int k = 0; k < 4; ++k) part_co[512 * k + blockIdx.x] = (double)tm[k];
#endif
  for (int64_t t3 = tid; t3 < 3 * a.n; t3 += nthreads) {   // back to the caller's order
    const int64_t p = t3 / 3;
    a.d[3 * (int64_t)h.perm[p] + (t3 - 3 * p)] = a.dm[t3];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result->iters = iters;
    a.result->converged = (bj0 <= 0.0) || (bj_new <= a.rel_tol * bj0);
    a.result->delta0 = bj0;
    a.result->delta_new = bj_new;
  }
}

}  // namespace mas

int stream_rows_per_chunk(int64_t n, int64_t nnzb);  // spmv.cu
int64_t stream_pin_rows(int64_t n, int64_t nnzb, double budget_mb);  // spmv.cu

}  // namespace b200ipc

using namespace b200ipc;
using namespace b200ipc::mas;

#define CK(expr)                                  \
  do {                                            \
    cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return -(int)_e;       \
  } while (0)
#define RC(expr)            \
  do {                      \
    int _r = (expr);        \
    if (_r) return _r;      \
  } while (0)

static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

extern "C" int b200ipc_mas_create(b200ipc_mas** out) {
  if (!out) return B200IPC_EINVAL;
  *out = new (std::nothrow) b200ipc_mas();
  return *out ? 0 : B200IPC_EINVAL;
}

extern "C" int b200ipc_mas_destroy(b200ipc_mas* h) {
  if (!h) return 0;
  h->perm.release(); h->rank.release(); h->inv[0].release(); h->inv[1].release(); h->coarse.release();
  h->colrank.release(); h->keys_a.release(); h->keys_b.release(); h->val_a.release(); h->val_b.release(); h->box.release(); h->temp.release();
  delete h;
  return 0;
}

extern "C" int b200ipc_mas_order(b200ipc_mas* h, int64_t nverts, const double* positions, void* stream) {
  if (!h || nverts <= 0 || nverts >= (1ll << 31)) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  h->ready = false;
  h->nverts = nverts;
  const int64_t ndom0 = (nverts + kDom - 1) / kDom;
  CK(h->perm.reserve(kDom * ndom0)); CK(h->rank.reserve(nverts));
  CK(h->val_a.reserve(nverts)); CK(h->val_b.reserve(nverts));
  const uint32_t* sorted = h->val_a.ptr;
  if (positions) {
    CK(h->keys_a.reserve(nverts)); CK(h->keys_b.reserve(nverts)); CK(h->box.reserve(6));
    box_init_kernel<<<1, 32, 0, st>>>(h->box.ptr);
    RC(post_launch());
    box_kernel<<<nblk(nverts), 256, 0, st>>>(nverts, positions, h->box.ptr);
    RC(post_launch());
    morton_kernel<<<nblk(nverts), 256, 0, st>>>(nverts, positions, h->box.ptr, h->keys_a.ptr, h->val_a.ptr);
    RC(post_launch());
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, h->keys_a.ptr, h->keys_b.ptr, h->val_a.ptr, h->val_b.ptr, (int)nverts,
                                       0, 30, st));
    CK(h->temp.reserve(tb));
    CK(cub::DeviceRadixSort::SortPairs(h->temp.ptr, tb, h->keys_a.ptr, h->keys_b.ptr, h->val_a.ptr, h->val_b.ptr,
                                       (int)nverts, 0, 30, st));   // stable: ties keep index order
    g_launches.fetch_add(1, std::memory_order_relaxed);
    sorted = h->val_b.ptr;
  } else {
    iota_kernel<<<nblk(nverts), 256, 0, st>>>(nverts, h->val_a.ptr);
    RC(post_launch());
  }
  perm_kernel<<<nblk(kDom * ndom0), 256, 0, st>>>(nverts, kDom * ndom0, sorted, h->perm.ptr, h->rank.ptr);
  RC(post_launch());
  h->ordered = true;
  return 0;
}

extern "C" int b200ipc_mas_get_order(b200ipc_mas* h, int32_t* rank, void* stream) {
  if (!h || !h->ordered) return B200IPC_ESTATE;
  if (!rank) return B200IPC_EINVAL;
  CK(cudaMemcpyAsync(rank, h->rank.ptr, h->nverts * sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return 0;
}

extern "C" int b200ipc_mas_setup(b200ipc_mas* h, int64_t nverts, int64_t nnzb, const int32_t* rowptr, const int32_t* colidx,
                                 const double* vals, const uint8_t* fixed, int32_t levels, void* stream) {
  if (!h || !h->ordered) return B200IPC_ESTATE;
  if (nverts != h->nverts || nnzb < nverts || !rowptr || !colidx || !vals || !fixed || levels < 1 || levels > kMaxLevels)
    return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  h->ready = false;
  h->nnode[0] = nverts;
  h->ndom[0] = (nverts + kDom - 1) / kDom;
  h->nnode[1] = h->ndom[0];
  h->ndom[1] = (h->nnode[1] + kDom - 1) / kDom;
  if (levels > 1 && h->ndom[0] < 2) levels = 1;   // one domain already holds the whole matrix
  const size_t smem = sizeof(double) * (kDim * kLd + 6 * kDim + 16);
  CK(cudaFuncSetAttribute(mas_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int l = 0; l < levels; ++l) {
    CK(h->inv[l].reserve((size_t)(h->ndom[l] * kInvFloats)));
    SetupArgs a{nverts, h->nnode[l], l, rowptr, colidx, vals, h->perm.ptr, h->rank.ptr, fixed, h->inv[l].ptr};
    mas_setup_kernel<<<(unsigned)h->ndom[l], kInvThreads, smem, st>>>(a);
    RC(post_launch());
  }
  if (levels > 1) CK(h->coarse.reserve((size_t)(6 * h->nnode[1])));
  h->fixed = fixed;
  h->levels = levels;
  h->ready = true;
  return 0;
}

static Hierarchy hierarchy_of(const b200ipc_mas* h) {
  Hierarchy y;
  y.n = h->nverts;
  y.levels = h->levels;
  y.ndom0 = h->ndom[0];
  y.ndom1 = h->ndom[1];
  y.nnode1 = h->nnode[1];
  y.perm = h->perm.ptr;
  y.rank = h->rank.ptr;
  y.fixed = h->fixed;
  y.inv0 = h->inv[0].ptr;
  y.inv1 = h->inv[1].ptr;
  y.r1 = h->coarse.ptr;
  y.y1 = h->coarse.ptr ? h->coarse.ptr + 3 * h->nnode[1] : nullptr;
  const char* dbg = getenv("B200IPC_MAS_DEBUG");
  y.debug = dbg ? atoi(dbg) : 0;
  return y;
}

extern "C" int b200ipc_mas_apply(b200ipc_mas* h, const double* r, double* z, void* stream) {
  if (!h || !h->ready) return B200IPC_ESTATE;
  if (!r || !z) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const Hierarchy y = hierarchy_of(h);
  apply_level0_kernel<<<nblk(32 * y.ndom0), 256, 0, st>>>(y, r, z);
  RC(post_launch());
  if (y.levels > 1) {
    apply_level1_kernel<<<nblk(32 * y.ndom1), 256, 0, st>>>(y);
    RC(post_launch());
    apply_prolong_kernel<<<nblk(3 * y.n), 256, 0, st>>>(y, z);
    RC(post_launch());
  }
  return 0;
}

extern "C" int64_t b200ipc_pcg_mas_workspace_bytes(int64_t n) {
  if (n < 0) return 0;
  // 2 x (n,6) pairs, 2 r, q, d and the 3x3 inverses in domain order, the flags, the partial sums
  return (int64_t)sizeof(double) * (8 * 3 * n + 9 * n + 4 * kMaxParts) + ((n + 255) & ~255ll) + 256;
}

namespace b200ipc {
namespace mas {
__global__ void __launch_bounds__(256) rename_columns_kernel(int64_t nnzb, const int32_t* __restrict__ colidx,
                                                             const int32_t* __restrict__ rank, int32_t* __restrict__ out) {
  const int64_t b = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (b < nnzb) out[b] = rank[colidx[b]];
}
}  // namespace mas
}  // namespace b200ipc

extern "C" int b200ipc_pcg_mas(b200ipc_mas* h, int64_t n, int64_t nnzb, const int32_t* rowptr, const int32_t* colidx,
                               const double* vals, const double* pinv, const uint8_t* fixed, const double* rhs, double* d,
                               double rel_tol, int32_t max_iters, void* workspace, int64_t workspace_bytes,
                               b200ipc_pcg_result* result, void* stream) {
  if (!h || !h->ready) return B200IPC_ESTATE;
  if (n != h->nverts || nnzb < n || !rowptr || !colidx || !vals || !pinv || !fixed || !rhs || !d || !workspace || !result)
    return B200IPC_EINVAL;
  if (workspace_bytes < b200ipc_pcg_mas_workspace_bytes(n) || max_iters < 0) return B200IPC_EINVAL;
  if ((((uintptr_t)vals | (uintptr_t)colidx | (uintptr_t)rowptr) & 15) != 0) return B200IPC_EINVAL;   // bulk copies
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // the product gathers from vectors kept in domain order: stream the column indices renamed to ranks
  CK(h->colrank.reserve((size_t)nnzb));
  rename_columns_kernel<<<nblk(nnzb), 256, 0, st>>>(nnzb, colidx, h->rank.ptr, h->colrank.ptr);
  RC(post_launch());
  StreamMatrix m{n, nnzb, b200ipc::stream_rows_per_chunk(n, nnzb), 0, rowptr, h->colrank.ptr, vals, nullptr,
                 b200ipc::stream_pin_rows(n, nnzb, kMasPinMb)};
  CK(cudaFuncSetAttribute(pcg_mas_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmemBytes));
  const int64_t nchunks = (n + m.rows_per_chunk - 1) / m.rows_per_chunk;
  int64_t grid = nchunks < sms ? nchunks : sms;
  if (grid < 1) grid = 1;
  double* w = static_cast<double*>(workspace);
  PcgMasArgs a;
  a.n = n; a.pinv = pinv; a.fixed = fixed; a.rhs = rhs; a.d = d;
  a.buf[0] = w; a.buf[1] = w + 6 * n; a.rbuf[0] = w + 12 * n; a.rbuf[1] = w + 15 * n; a.q = w + 18 * n;
  a.dm = w + 21 * n; a.pinvm = w + 24 * n;
  a.part = w + 33 * n;
  a.result = reinterpret_cast<b200ipc_pcg_result*>(a.part + 4 * kMaxParts);
  a.fixedm = reinterpret_cast<uint8_t*>(a.part + 4 * kMaxParts) + 64;
  a.rel_tol = rel_tol; a.max_iters = max_iters;
  Hierarchy y = hierarchy_of(h);
  void* args[] = {(void*)&a, (void*)&m, (void*)&y};
  CK(cudaLaunchCooperativeKernel((const void*)pcg_mas_kernel, dim3((unsigned)grid), dim3(kStreamThreads), args,
                                 kStreamSmemBytes, st));
  RC(post_launch());
  CK(cudaMemcpyAsync(result, a.result, sizeof(b200ipc_pcg_result), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}
