// Scatter-assembly of the 6x6 / 9x9 / 12x12 local blocks into the 3x3-block sparse global
// matrix (BSR), and the gradient scatter -- both WITHOUT atomics.
//
// The reference never assembles (matvec is matrix-free, solver.py:251-262); the assembled matrix
// is defined by its test oracle (tests/test_solver.py:71-84): A = diag(m_i I3) + sum of blocks at
// ix_(idx, idx), fixed rows/cols zeroed with a unit diagonal.
//
// symbolic (once per contact set): every (block, a, b) sub-block slot and every diagonal mass
//   slot gets the key row*N+col; a stable LSD radix sort (CUB) of (key, slot) gives, per unique
//   key, a contiguous run of source slots in list order; run heads -> colidx / rowptr.
// numeric (once per Newton iteration): one thread per (unique block, entry) walks its run and sums
//   the 3x3 sub-blocks in list order -- a segmented reduction by gather, deterministic, bitwise
//   reproducible, no contention.  Threads of a warp write consecutive doubles of vals.
// The gradient scatter (SimState.gradient, solver.py:218-226) reuses the same machinery keyed by
// vertex.
#include <cub/cub.cuh>

#include "launch.cuh"
#include "../../include/b200ipc.h"

#include "assembly.cuh"

namespace b200ipc {

__device__ __forceinline__ void decode_slot(const FamDesc& fd, int64_t q, int& f, int64_t& b, int& a, int& c) {
  f = 0;
#pragma unroll
  for (int k = 1; k < kMaxFam; ++k)
    if (k < fd.nfam && q >= fd.ent_off[k]) f = k;
  const int s = fd.s[f];
  const int64_t r = q - fd.ent_off[f];
  b = r / (s * s);
  const int rem = (int)(r - b * (s * s));
  a = rem / s;
  c = rem - a * s;
}

// keys for matrix slots: slot < N is the diagonal mass slot of vertex `slot`
__global__ void __launch_bounds__(kAT) matrix_keys_kernel(FamDesc fd, int64_t nverts, int64_t nslots,
                                                          const uint8_t* __restrict__ fixed,
                                                          uint64_t* __restrict__ keys, uint32_t* __restrict__ slots) {
  const int64_t e = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (e >= nslots) return;
  int64_t row, col;
  if (e < nverts) {
    row = col = e;
  } else {
    int f, a, c;
    int64_t b;
    decode_slot(fd, e - nverts, f, b, a, c);
    const int64_t* v = fd.vids[f] + b * fd.s[f];
    row = v[a];
    col = v[c];
  }
  uint64_t key = (uint64_t)row * (uint64_t)nverts + (uint64_t)col;
  // Dirichlet: an off-diagonal slot with a fixed end is dropped (sorts last), and so are the block slots on the
  // diagonal of a fixed row -- its block is the unit matrix whatever they hold; only the mass slot stays, as in
  // the row-wise phase (same run contents and the same source count in both phases)
  if ((row != col && (fixed[row] | fixed[col])) || (row == col && e >= nverts && fixed[row]))
    key = (uint64_t)nverts * (uint64_t)nverts;
  keys[e] = key;
  slots[e] = (uint32_t)e;
}

__global__ void __launch_bounds__(kAT) head_flags_kernel(int64_t n, uint64_t sentinel,
                                                         const uint64_t* __restrict__ keys,
                                                         int32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  head[i] = (k != sentinel && (i == 0 || keys[i - 1] != k)) ? 1 : 0;
}

// keys are sorted with the sentinel last: index of the first sentinel = number of kept slots
__global__ void first_sentinel_kernel(int64_t n, uint64_t sentinel, const uint64_t* keys, int64_t* out) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] != sentinel) lo = mid + 1;
    else hi = mid;
  }
  out[0] = lo;
}

// scan[i] = inclusive count of heads; heads write colidx / run start; count valid slots
__global__ void __launch_bounds__(kAT) emit_pattern_kernel(int64_t n, int64_t nverts, const uint64_t* __restrict__ keys,
                                                           const int32_t* __restrict__ scan,
                                                           int32_t* __restrict__ colidx, int32_t* __restrict__ useg,
                                                           int32_t* __restrict__ rowmark) {
  const int64_t i = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  if (k == (uint64_t)nverts * (uint64_t)nverts) return;
  const bool is_head = i == 0 || keys[i - 1] != k;
  if (is_head) {
    const int32_t u = scan[i] - 1;
    const int64_t row = (int64_t)(k / (uint64_t)nverts);
    colidx[u] = (int32_t)(k - (uint64_t)row * (uint64_t)nverts);
    useg[u] = (int32_t)i;
    // first block of a row: every row has its diagonal, so each row owns >= 1 block
    const bool row_head = i == 0 || (int64_t)(keys[i - 1] / (uint64_t)nverts) != row;
    if (row_head) rowmark[row] = u;
  }
}

__global__ void finish_pattern_kernel(int64_t nverts, int64_t nnzb, int64_t nvalid, int32_t* rowptr, int32_t* useg) {
  rowptr[nverts] = (int32_t)nnzb;
  useg[nnzb] = (int32_t)nvalid;
}

// sorted sources are contiguous: run u ends where run u+1 starts
__global__ void __launch_bounds__(kAT) run_ends_kernel(int64_t nnzb, const int32_t* __restrict__ useg, int32_t* __restrict__ uend) {
  const int64_t u = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (u < nnzb) uend[u] = useg[u + 1];
}

// Source descriptors, written once per pattern in sorted order, 32 bits each: the numeric phase then
// needs no integer division, no family search and a single address computation per source.
//   block source : family (2 bits) << 30 | (element offset of the 3x3 sub-block) / 3
//   mass slot    : 3 << 30 | vertex          (always the first source of a diagonal block's run)
// (needs nfam <= 3 and family arrays below 2^30 * 24 bytes; otherwise the row-wise kernel is used)
__global__ void __launch_bounds__(kAT) source_desc_kernel(FamDesc fd, int64_t nverts, int64_t nvalid,
                                                          const uint32_t* __restrict__ perm,
                                                          uint32_t* __restrict__ desc) {
  const int64_t j = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (j >= nvalid) return;
  const int64_t slot = perm[j];
  if (slot < nverts) {
    desc[j] = 0xC0000000u | (uint32_t)slot;
  } else {
    int f, a, c;
    int64_t b;
    decode_slot(fd, slot - nverts, f, b, a, c);
    const int64_t s = fd.s[f];
    // row-major: ((b*D + 3a)*D + 3c) / 3 with D = 3s; sub-block-major: 9 (b s^2 + a s + c) / 3
    desc[j] = ((uint32_t)f << 30) | (uint32_t)((b * 3 * s + 3 * a) * s + fd.cmul[f] * c);
  }
}

struct NumericArgs {
  HessPtrs hp;
  int32_t ld[4];        // row stride of a 3x3 sub-block in families 0..2: D row-major, 3 sub-block-major (slot 3 unused)
  int64_t nnzb;
  const uint8_t* fixed;
  const double* masses;
  const int32_t* useg;      // run u = sources [useg[u], uend[u])
  const int32_t* uend;
  const uint32_t* desc;
  double* vals;
};

#ifndef B200IPC_ASM_BLOCKS_PER_WARP
#define B200IPC_ASM_BLOCKS_PER_WARP 8
#endif
#ifndef B200IPC_ASM_WARPS
#define B200IPC_ASM_WARPS 8
#endif
constexpr int kNumWarps = B200IPC_ASM_WARPS;
constexpr int kBlocksPerWarp = B200IPC_ASM_BLOCKS_PER_WARP;   // consecutive output blocks per warp (one descriptor prefetch for all)

__device__ __forceinline__ double gather_entry(const NumericArgs& a, uint32_t d, int er, int ec) {
  const uint32_t f = d >> 30;
  const uint32_t e = (d & 0x3fffffffu) * 3u + (uint32_t)(er * a.ld[f] + ec);
  return __ldg(a.hp.p[f] + e);
}

__device__ __forceinline__ void touch_l1(const void* p) {
  unsigned tmp;
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(tmp) : "l"(p));
  (void)tmp;
}

// Shared walker of the per-block runs.  A warp owns kBlocksPerWarp consecutive output blocks, whose
// sources are one contiguous span of descriptors: the span is pulled into L1 with coalesced loads up
// front (one DRAM latency for the whole warp instead of one dependent miss per block), then each
// block is reduced with lanes (g, e) = (lane / 9, lane % 9), g < 3: entry e of every third source,
// twelve sub-blocks of loads in flight before the adds, three partial sums combined in fixed order by
// two shuffles.  Lanes 0..8 write the block: nine consecutive doubles.  32 registers, no shared
// memory: 64 resident warps per SM.  ENTRY(desc, er, ec) returns one entry of one source.
template <typename ARGS, typename ENTRY>
__device__ __forceinline__ void walk_runs(const ARGS& a, const uint32_t* __restrict__ desc, ENTRY entry) {
  const int64_t u0 = ((int64_t)blockIdx.x * kNumWarps + (threadIdx.x >> 5)) * kBlocksPerWarp;
  if (u0 >= a.nnzb) return;
  const int lane = threadIdx.x & 31;
  const int nb = (int)min((int64_t)kBlocksPerWarp, a.nnzb - u0);
  const int32_t mine = a.useg[u0 + min(lane, nb - 1)], mine_end = a.uend[u0 + min(lane, nb - 1)];
  const int32_t span0 = __shfl_sync(0xffffffffu, mine, 0), span1 = __shfl_sync(0xffffffffu, mine_end, nb - 1);
  for (int32_t t = span0 + lane; t < span1; t += 32) touch_l1(desc + t);  // 128-byte lines, fire and forget
  const int g = lane / 9, e = lane - 9 * g;
  const int er = e / 3, ec = e - 3 * er;
  for (int i = 0; i < nb; ++i) {
    int32_t j0 = __shfl_sync(0xffffffffu, mine, i);
    const int32_t j1 = __shfl_sync(0xffffffffu, mine_end, i);
    const int64_t u = u0 + i;
    double acc = 0.0;
    const uint32_t first = desc[j0];
    if (first >= 0xC0000000u) {  // diagonal block: mass slot first
      const uint32_t v = first & 0x3fffffffu;
      if (a.fixed[v]) {  // Dirichlet vertex: unit diagonal, nothing else
        if (lane < 9) a.vals[9 * u + lane] = er == ec ? 1.0 : 0.0;
        continue;
      }
      if (g == 0 && er == ec) acc = a.masses[v];
      ++j0;
    }
    if (g < 3) {
      int32_t j = j0 + g;
      for (; j + 9 < j1; j += 12) {
        const uint32_t d0 = desc[j], d1 = desc[j + 3], d2 = desc[j + 6], d3 = desc[j + 9];
        const double v0 = entry(d0, er, ec), v1 = entry(d1, er, ec);
        const double v2 = entry(d2, er, ec), v3 = entry(d3, er, ec);
        acc += v0;
        acc += v1;
        acc += v2;
        acc += v3;
      }
      for (; j < j1; j += 3) acc += entry(desc[j], er, ec);
    }
    const double s1 = __shfl_down_sync(0xffffffffu, acc, 9);   // group 1's partial sum (lanes 0..8)
    const double s2 = __shfl_down_sync(0xffffffffu, acc, 18);  // group 2's
    if (lane < 9) a.vals[9 * u + lane] = (acc + s1) + s2;
  }
}

// Second walker: THREE output blocks per warp trip, nine lanes per block (lane = 9 r + e), each lane walking its
// block's whole run, four sources per step.  The per-block overhead of walk_runs (run bounds by shuffle, head
// test, two-shuffle tail: ~100 warp instructions against ~36 for an average run of nine sources) is shared by
// three blocks and the three-group split disappears; the price is that a trio runs as long as its longest run.
#ifndef B200IPC_ASM_TRIOS
#define B200IPC_ASM_TRIOS 4
#endif
constexpr int kTriosPerWarp = B200IPC_ASM_TRIOS;

template <typename ARGS, typename ENTRY>
__device__ __forceinline__ void walk_trios(const ARGS& a, const uint32_t* __restrict__ desc, ENTRY entry) {
  const int lane = threadIdx.x & 31;
  const int r = lane / 9, e = lane - 9 * r;
  const int er = e / 3, ec = e - 3 * er;
  const int64_t first_trio = ((int64_t)blockIdx.x * kNumWarps + (threadIdx.x >> 5)) * kTriosPerWarp;
#pragma unroll 1
  for (int t = 0; t < kTriosPerWarp; ++t) {
    const int64_t u = (first_trio + t) * 3 + r;
    const bool valid = r < 3 && u < a.nnzb;
    if (!__any_sync(0xffffffffu, valid)) return;
    int32_t j0 = 0, j1 = 0;
    double acc = 0.0;
    bool unit = false;
    if (valid) {
      j0 = a.useg[u];
      j1 = a.uend[u];
      const uint32_t head = desc[j0];
      if (head >= 0xC0000000u) {  // diagonal block: mass slot first
        const uint32_t v = head & 0x3fffffffu;
        unit = a.fixed[v];        // Dirichlet vertex: unit diagonal, nothing else
        if (er == ec) acc = unit ? 1.0 : a.masses[v];
        ++j0;
        if (unit) j1 = j0;
      }
    }
    const int len = j1 - j0;
    const int maxlen = __reduce_max_sync(0xffffffffu, len);
    const uint32_t* dj = desc + j0;
    int k = 0;
    for (; k + 4 <= maxlen; k += 4) {
      const bool p0 = k < len, p1 = k + 1 < len, p2 = k + 2 < len, p3 = k + 3 < len;
      const uint32_t d0 = p0 ? dj[k] : 0u, d1 = p1 ? dj[k + 1] : 0u, d2 = p2 ? dj[k + 2] : 0u, d3 = p3 ? dj[k + 3] : 0u;
      const double v0 = p0 ? entry(d0, er, ec) : 0.0, v1 = p1 ? entry(d1, er, ec) : 0.0;
      const double v2 = p2 ? entry(d2, er, ec) : 0.0, v3 = p3 ? entry(d3, er, ec) : 0.0;
      if (p0) acc += v0;
      if (p1) acc += v1;
      if (p2) acc += v2;
      if (p3) acc += v3;
    }
    for (; k < maxlen; ++k)
      if (k < len) acc += entry(dj[k], er, ec);
    if (valid) a.vals[9 * u + e] = acc;
  }
}

__global__ void __launch_bounds__(32 * kNumWarps, 8) assemble_numeric_kernel(const __grid_constant__ NumericArgs a) {
  walk_runs(a, a.desc, [&](uint32_t d, int er, int ec) { return gather_entry(a, d, er, ec); });
}

// ---- numeric assembly straight from the rank-1 factors ---------------------------------------------
// Barrier blocks are z z^T (stencil.cu), so sub-block (a,c) of block b is z_a z_c^T: instead of the
// dense block (72 s^2 bytes) the gather reads two 3-vectors of the factor array (24 s bytes per block,
// ~0.1 GB for 1M contacts: L2-resident).  Entries are the same products the dense block holds, summed
// in the same order as assemble_numeric_kernel, so both paths give bitwise identical matrices.
//   fdesc : family (2 bits) << 30 | (c - a + 3) << 27 | element index of z_a = b*D + 3a   (27 bits)
__global__ void __launch_bounds__(kAT) factor_desc_kernel(FamDesc fd, int64_t nverts, int64_t nvalid,
                                                          const uint32_t* __restrict__ perm,
                                                          uint32_t* __restrict__ fdesc) {
  const int64_t j = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (j >= nvalid) return;
  const int64_t slot = perm[j];
  if (slot < nverts) {
    fdesc[j] = 0xC0000000u | (uint32_t)slot;
  } else {
    int f, a, c;
    int64_t b;
    decode_slot(fd, slot - nverts, f, b, a, c);
    const int64_t D = 3 * fd.s[f];
    fdesc[j] = ((uint32_t)f << 30) | ((uint32_t)(c - a + 3) << 27) | (uint32_t)(b * D + 3 * a);
  }
}

struct FactorArgs {
  HessPtrs fp;          // factor arrays (nb, D) per family
  int64_t nnzb;
  const uint8_t* fixed;
  const double* masses;
  const int32_t* useg;
  const int32_t* uend;
  const uint32_t* fdesc;
  double* vals;
};

__device__ __forceinline__ double factor_entry(const FactorArgs& a, uint32_t d, int er, int ec) {
  const double* z = a.fp.p[d >> 30] + (d & 0x07ffffffu);
  const int dc = 3 * ((int)((d >> 27) & 7u) - 3);
  return __ldg(z + er) * __ldg(z + dc + ec);
}

__global__ void __launch_bounds__(32 * kNumWarps, 8) assemble_factors_kernel(const __grid_constant__ FactorArgs a) {
  walk_runs(a, a.fdesc, [&](uint32_t d, int er, int ec) { return factor_entry(a, d, er, ec); });
}

__global__ void __launch_bounds__(32 * kNumWarps, 8) assemble_factors_trio_kernel(const __grid_constant__ FactorArgs a) {
  walk_trios(a, a.fdesc, [&](uint32_t d, int er, int ec) { return factor_entry(a, d, er, ec); });
}

__global__ void __launch_bounds__(32 * kNumWarps, 8) assemble_numeric_trio_kernel(const __grid_constant__ NumericArgs a) {
  walk_trios(a, a.desc, [&](uint32_t d, int er, int ec) { return gather_entry(a, d, er, ec); });
}

// ---- row-wise numeric assembly ------------------------------------------------------------------
// A "row-source" is (block b of family f, local vertex a): rows 3a..3a+2 of the dense block are ONE
// contiguous run of 3*D doubles.  For output block-row i the row-sources are the gradient runs
// (vertex i's incidences in list order).  rs_desc = (element offset of the run << 3) | family,
// rs_dst = four u16: index of column vertex v_c inside row i's block list (0xffff = dropped).
__global__ void __launch_bounds__(kAT) row_source_kernel(FamDesc fd, int64_t nverts, int64_t ng,
                                                         const uint32_t* __restrict__ gperm,
                                                         const uint8_t* __restrict__ fixed,
                                                         const int32_t* __restrict__ rowptr,
                                                         const int32_t* __restrict__ colidx,
                                                         uint64_t* __restrict__ rs_desc, uint64_t* __restrict__ rs_dst) {
  const int64_t j = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (j >= ng) return;
  const int64_t q = gperm[j];
  int f = 0;
#pragma unroll
  for (int k = 1; k < kMaxFam; ++k)
    if (k < fd.nfam && q >= fd.vert_off[k]) f = k;
  const int s = fd.s[f];
  const int64_t r = q - fd.vert_off[f];
  const int64_t b = r / s;
  const int a = (int)(r - b * s);
  const int64_t D = 3 * s;
  const int64_t* v = fd.vids[f] + b * s;
  const int64_t row = v[a];
  rs_desc[j] = ((uint64_t)((b * D + 3 * a) * D) << 3) | (uint64_t)f;
  uint64_t dst = 0;
  const int32_t r0 = rowptr[row], r1 = rowptr[row + 1];
  for (int c = 0; c < 4; ++c) {
    uint64_t rel = 0xffffull;
    if (c < s && !fixed[row]) {
      const int64_t col = v[c];
      if (col == row || !fixed[col]) {
        int32_t lo = r0, hi = r1;
        while (lo < hi) {
          const int32_t mid = (lo + hi) >> 1;
          if (colidx[mid] < col) lo = mid + 1;
          else hi = mid;
        }
        rel = (uint64_t)(lo - r0);
      }
    }
    dst |= rel << (16 * c);
  }
  rs_dst[j] = dst;
}

struct RowArgs {
  HessPtrs hp;
  int32_t fs[kMaxFam + 1];   // stencil size s per family; fs[7] = 0 tags an absent source
  int64_t nverts;
  const uint8_t* fixed;
  const double* masses;
  const int32_t* rowptr;
  const int32_t* colidx;
  const int32_t* gseg;
  const uint64_t* rs_desc;
  const uint64_t* rs_dst;
  double* vals;
};

constexpr int kRowWarps = 8;
constexpr int kRowWin = 64;   // blocks of one row accumulated per pass in shared memory

// Per-lane constants of the element -> (sub-block, entry) map of a run of 3*D doubles.
template <int D>
struct LaneMap {
  int k0, sh0, k1, sh1;  // entry index er*3+ec and shift 16*c for elements lane and lane+32
  __device__ __forceinline__ explicit LaneMap(int lane) {
    const int t0 = lane < 3 * D ? lane : 0;
    const int er0 = t0 / D, cc0 = t0 - er0 * D;
    k0 = er0 * 3 + cc0 % 3;
    sh0 = 16 * (cc0 / 3);
    const int t1 = lane + 32 < 3 * D ? lane + 32 : 0;
    const int er1 = t1 / D, cc1 = t1 - er1 * D;
    k1 = er1 * 3 + cc1 % 3;
    sh1 = 16 * (cc1 / 3);
  }
};

template <int D>
__device__ __forceinline__ void row_add(double* acc, const LaneMap<D>& m, int lane, uint64_t dst, int win, int wlen,
                                        double v0, double v1) {
  if (lane < 3 * D) {
    const unsigned rel = (unsigned)((dst >> m.sh0) & 0xffff) - (unsigned)win;
    if (rel < (unsigned)wlen) acc[rel * 9 + m.k0] += v0;
  }
  if (3 * D > 32) {
    if (lane + 32 < 3 * D) {
      const unsigned rel = (unsigned)((dst >> m.sh1) & 0xffff) - (unsigned)win;
      if (rel < (unsigned)wlen) acc[rel * 9 + m.k1] += v1;
    }
  }
}

// One warp per block-row.  Every row-source is read as one contiguous run (full sectors, each dense
// block is read exactly once over the whole kernel) and its s sub-blocks are added into the row's
// accumulators in shared memory in list order -- no atomics, bitwise reproducible.  The finished
// row (72 bytes per block, contiguous) is written with consecutive lanes on consecutive doubles.
__global__ void __launch_bounds__(32 * kRowWarps) assemble_rows_kernel(const __grid_constant__ RowArgs a) {
  __shared__ double sm[kRowWarps][kRowWin * 9];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowWarps + w;
  if (row >= a.nverts) return;
  double* acc = sm[w];
  const int32_t r0 = a.rowptr[row], len = a.rowptr[row + 1] - r0;
  double* out = a.vals + 9ll * r0;
  if (a.fixed[row]) {  // Dirichlet row: identity diagonal only
    if (lane < 9) out[lane] = (lane == 0 || lane == 4 || lane == 8) ? 1.0 : 0.0;
    return;
  }
  // diagonal block position inside the row
  int32_t lo = 0, hi = len;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (a.colidx[r0 + mid] < row) lo = mid + 1;
    else hi = mid;
  }
  const int drel = lo;
  const double mass = a.masses[row];
  const int32_t j0 = a.gseg[row], j1 = a.gseg[row + 1];
  const LaneMap<6> m6(lane);
  const LaneMap<9> m9(lane);
  const LaneMap<12> m12(lane);

  for (int win = 0; win < len; win += kRowWin) {
    const int wlen = min(kRowWin, len - win);
    for (int t = lane; t < 9 * wlen; t += 32) acc[t] = 0.0;
    __syncwarp();
    if (lane < 3 && drel >= win && drel < win + wlen) acc[(drel - win) * 9 + 4 * lane] = mass;
    __syncwarp();
    // Software pipeline over pairs of row-sources: descriptors are loaded two pairs ahead and the
    // dense runs one pair ahead of the accumulation, so neither memory latency sits on the
    // critical path of the (ordered) shared-memory adds.
    auto load_desc = [&](int32_t j, uint64_t& d, uint64_t& m) {
      const bool ok = j < j1;
      d = ok ? a.rs_desc[j] : 7ull;
      m = ok ? a.rs_dst[j] : ~0ull;
    };
    auto fetch = [&](uint64_t d, int& sz, double& v0, double& v1) {
      sz = a.fs[d & 7];
      const double* p = a.hp.p[d & 7] + (d >> 3);
      v0 = lane < 9 * sz ? __ldg(p + lane) : 0.0;
      v1 = lane + 32 < 9 * sz ? __ldg(p + lane + 32) : 0.0;
    };
    auto add = [&](int sz, uint64_t m, double v0, double v1) {
      if (sz == 4) row_add<12>(acc, m12, lane, m, win, wlen, v0, v1);
      else if (sz == 3) row_add<9>(acc, m9, lane, m, win, wlen, v0, v1);
      else if (sz == 2) row_add<6>(acc, m6, lane, m, win, wlen, v0, v1);
    };
    uint64_t dA, mA, dB, mB, ndA, nmA, ndB, nmB;
    load_desc(j0, dA, mA);
    load_desc(j0 + 1, dB, mB);
    load_desc(j0 + 2, ndA, nmA);
    load_desc(j0 + 3, ndB, nmB);
    int sA, sB;
    double vA0, vA1, vB0, vB1;
    fetch(dA, sA, vA0, vA1);
    fetch(dB, sB, vB0, vB1);
    for (int32_t j = j0; j < j1; j += 2) {
      uint64_t fdA, fmA, fdB, fmB;  // two pairs ahead
      load_desc(j + 4, fdA, fmA);
      load_desc(j + 5, fdB, fmB);
      int nsA, nsB;                 // one pair ahead
      double nA0, nA1, nB0, nB1;
      fetch(ndA, nsA, nA0, nA1);
      fetch(ndB, nsB, nB0, nB1);
      add(sA, mA, vA0, vA1);
      __syncwarp();
      add(sB, mB, vB0, vB1);
      __syncwarp();
      sA = nsA; mA = nmA; vA0 = nA0; vA1 = nA1;
      sB = nsB; mB = nmB; vB0 = nB0; vB1 = nB1;
      ndA = fdA; nmA = fmA; ndB = fdB; nmB = fmB;
    }
    for (int t = lane; t < 9 * wlen; t += 32) out[9 * win + t] = acc[t];
    __syncwarp();
  }
}

// ---- gradient ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(kAT) gradient_keys_kernel(FamDesc fd, int64_t ngslots, uint32_t* __restrict__ keys,
                                                            uint32_t* __restrict__ slots) {
  const int64_t q = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (q >= ngslots) return;
  int f = 0;
#pragma unroll
  for (int k = 1; k < kMaxFam; ++k)
    if (k < fd.nfam && q >= fd.vert_off[k]) f = k;
  keys[q] = (uint32_t)fd.vids[f][q - fd.vert_off[f]];
  slots[q] = (uint32_t)q;
}

__global__ void __launch_bounds__(kAT) lower_bound_kernel(int64_t nverts, int64_t n, const uint32_t* __restrict__ keys,
                                                          int32_t* __restrict__ seg) {
  const int64_t v = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (v > nverts) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)keys[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  seg[v] = (int32_t)lo;
}

struct GradArgs {
  FamDesc fd;
  HessPtrs gp;
  int64_t nverts;
  const uint8_t* fixed;
  const double *masses, *x, *x_tilde;
  const int32_t* gseg;
  const uint32_t* gperm;
  double* out;
};

// thread = (vertex, component): m (x - x~) + contributions in list order; fixed rows -> 0
__global__ void __launch_bounds__(kAT) scatter_gradient_kernel(const __grid_constant__ GradArgs a) {
  const int64_t t = (int64_t)blockIdx.x * kAT + threadIdx.x;
  if (t >= 3 * a.nverts) return;
  const int64_t v = t / 3;
  const int k = (int)(t - 3 * v);
  if (a.fixed[v]) {
    a.out[t] = 0.0;
    return;
  }
  double acc = a.masses[v] * (a.x[t] - a.x_tilde[t]);
  for (int32_t j = a.gseg[v]; j < a.gseg[v + 1]; ++j) {
    const int64_t q = a.gperm[j];
    int f = 0;
#pragma unroll
    for (int kk = 1; kk < kMaxFam; ++kk)
      if (kk < a.fd.nfam && q >= a.fd.vert_off[kk]) f = kk;
    // slot q - vert_off[f] = b*s + a  ->  grad_f[b][3a + k] = base[3*(b*s+a) + k]
    acc += __ldg(a.gp.p[f] + 3 * (q - a.fd.vert_off[f]) + k);
  }
  a.out[t] = acc;
}

__global__ void __launch_bounds__(kAT) max_row_kernel(int64_t nverts, const int32_t* __restrict__ rowptr, int64_t* out) {
  const int64_t v = (int64_t)blockIdx.x * kAT + threadIdx.x;
  int len = v < nverts ? rowptr[v + 1] - rowptr[v] : 0;
  len = __reduce_max_sync(0xffffffffu, len);
  if ((threadIdx.x & 31) == 0 && len > 0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)len);
}

static inline unsigned blocks_for(int64_t n) { return (unsigned)((n + kAT - 1) / kAT); }

static int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b)) ++b;
  return b;
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_assembly_create(b200ipc_assembly** out) {
  if (!out) return B200IPC_EINVAL;
  *out = new (std::nothrow) b200ipc_assembly();
  return *out ? 0 : B200IPC_EINVAL;
}

extern "C" int b200ipc_assembly_set_variant(b200ipc_assembly* h, int32_t variant) {
  if (!h || !(variant == 0 || variant == 1 || variant == 2 || variant == 4)) return B200IPC_EINVAL;
  h->variant = variant;
  return 0;
}

extern "C" int b200ipc_assembly_destroy(b200ipc_assembly* h) {
  if (!h) return 0;
  h->fixed.release(); h->keys_a.release(); h->keys_b.release(); h->slot_a.release(); h->slot_b.release();
  h->head.release(); h->useg.release(); h->desc.release(); h->fdesc.release(); h->rowptr.release(); h->colidx.release();
  h->gkeys_a.release(); h->gkeys_b.release(); h->gslot_a.release(); h->gslot_b.release(); h->gseg.release(); h->rs_desc.release(); h->rs_dst.release();
  h->temp.release(); h->scalars.release(); h->uend.release(); h->row_len.release(); h->slab_col.release(); h->slab_beg.release(); h->slab_end.release();
  delete h;
  return 0;
}

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

namespace b200ipc {
int symbolic_by_rows(b200ipc_assembly* h, bool want_desc, bool want_fdesc, bool* overflow, cudaStream_t st);  // symbolic_rows.cu

// Sort-based symbolic phase: every sub-block slot keyed by row*N+col, one stable LSD radix sort, run heads
// -> colidx / rowptr / run starts.  Handles rows of any length; the row-wise phase falls back to it.
static int symbolic_by_sort(b200ipc_assembly* h, cudaStream_t st) {
  const FamDesc& fd = h->fam;
  const int64_t nverts = h->nverts, n = h->nslots;
  CK(h->keys_a.reserve(n)); CK(h->keys_b.reserve(n)); CK(h->slot_a.reserve(n)); CK(h->slot_b.reserve(n));
  CK(h->head.reserve(n)); CK(h->rowptr.reserve(nverts + 1)); CK(h->scalars.reserve(4));

  matrix_keys_kernel<<<blocks_for(n), kAT, 0, st>>>(fd, nverts, n, h->fixed.ptr, h->keys_a.ptr, h->slot_a.ptr);
  RC(post_launch());

  // stable LSD radix sort over the significant bits only; the sentinel N*N is the largest key
  const uint64_t sentinel = (uint64_t)nverts * (uint64_t)nverts;
  const int end_bit = bits_for(sentinel);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, h->keys_a.ptr, h->keys_b.ptr, h->slot_a.ptr, h->slot_b.ptr, (int)n,
                                     0, end_bit, st));
  size_t tb2 = 0;
  CK(cub::DeviceScan::InclusiveSum(nullptr, tb2, h->head.ptr, h->head.ptr, (int)n, st));
  CK(h->temp.reserve(tb > tb2 ? tb : tb2));
  CK(cub::DeviceRadixSort::SortPairs(h->temp.ptr, tb, h->keys_a.ptr, h->keys_b.ptr, h->slot_a.ptr, h->slot_b.ptr,
                                     (int)n, 0, end_bit, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);

  head_flags_kernel<<<blocks_for(n), kAT, 0, st>>>(n, sentinel, h->keys_b.ptr, h->head.ptr);
  RC(post_launch());
  CK(cub::DeviceScan::InclusiveSum(h->temp.ptr, tb2, h->head.ptr, h->head.ptr, (int)n, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  // nnzb = scan[n-1] and the number of kept slots, both with one synchronisation
  first_sentinel_kernel<<<1, 1, 0, st>>>(n, sentinel, h->keys_b.ptr, h->scalars.ptr);
  RC(post_launch());
  int32_t nnzb32 = 0;
  int64_t nvalid = 0;
  CK(cudaMemcpyAsync(&nnzb32, h->head.ptr + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nvalid, h->scalars.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->nnzb = nnzb32;
  h->nvalid = nvalid;
  CK(h->colidx.reserve(h->nnzb)); CK(h->useg.reserve(h->nnzb + 1));
  emit_pattern_kernel<<<blocks_for(n), kAT, 0, st>>>(n, nverts, h->keys_b.ptr, h->head.ptr, h->colidx.ptr,
                                                     h->useg.ptr, h->rowptr.ptr);
  RC(post_launch());
  finish_pattern_kernel<<<1, 1, 0, st>>>(nverts, h->nnzb, h->nvalid, h->rowptr.ptr, h->useg.ptr);
  RC(post_launch());
  CK(h->uend.reserve(h->nnzb + 1));
  run_ends_kernel<<<blocks_for(h->nnzb), kAT, 0, st>>>(h->nnzb, h->useg.ptr, h->uend.ptr);
  RC(post_launch());
  h->have_desc = h->have_fdesc = false;   // built from the slot permutation on first use
  h->max_row = -1;
  return 0;
}

// 32-bit source descriptors apply: <= 3 families (2-bit family field), element offsets inside the fields
static bool dense_desc_fits(const FamDesc& fd) {
  if (fd.nfam > 3) return false;
  for (int f = 0; f < fd.nfam; ++f)
    if (fd.nb[f] * 9 * fd.s[f] * fd.s[f] >= (3ll << 30)) return false;
  return true;
}
static bool factor_desc_fits(const FamDesc& fd) {
  if (fd.nfam > 3) return false;
  for (int f = 0; f < fd.nfam; ++f)
    if (fd.nb[f] * 3 * fd.s[f] >= (1ll << 27)) return false;
  return true;
}

}  // namespace b200ipc

extern "C" int b200ipc_assembly_set_symbolic(b200ipc_assembly* h, int32_t mode) {
  if (!h || !(mode == 0 || mode == 1)) return B200IPC_EINVAL;
  h->symbolic_mode = mode;
  return 0;
}

extern "C" int b200ipc_assembly_set_layout(b200ipc_assembly* h, uint32_t tiled_mask) {
  if (!h || tiled_mask >= (1u << kMaxFam)) return B200IPC_EINVAL;
  h->tiled_next = tiled_mask;   // descriptors are written by the symbolic phase: takes effect at the next pattern
  return 0;
}

extern "C" int b200ipc_assembly_stats(b200ipc_assembly* h, int64_t* out) {
  if (!h || !out) return B200IPC_EINVAL;
  if (!h->ready) return B200IPC_ESTATE;
  out[0] = h->symbolic_used;
  out[1] = h->max_row;
  out[2] = h->nnzb;
  out[3] = h->nvalid;
  return 0;
}

extern "C" int b200ipc_assemble_symbolic(b200ipc_assembly* h, int64_t nverts, const uint8_t* fixed, int32_t nfam,
                                         const int32_t* fam_s, const int64_t* fam_nb, const int64_t* const* fam_vids,
                                         int64_t* nnzb_out, void* stream) {
  if (!h || nverts <= 0 || nfam < 0 || nfam > kMaxFam || !fixed) return B200IPC_EINVAL;
  if (nfam && (!fam_s || !fam_nb || !fam_vids)) return B200IPC_EINVAL;
  if (nverts >= (1ll << 31)) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  h->ready = false;
  FamDesc& fd = h->fam;
  fd.nfam = nfam;
  fd.ent_off[0] = fd.vert_off[0] = 0;
  for (int f = 0; f < nfam; ++f) {
    if (fam_s[f] < 2 || fam_s[f] > 4 || fam_nb[f] < 0 || (fam_nb[f] && !fam_vids[f])) return B200IPC_EINVAL;
    fd.s[f] = fam_s[f];
    fd.nb[f] = fam_nb[f];
    fd.vids[f] = fam_vids[f];
    fd.ent_off[f + 1] = fd.ent_off[f] + fam_nb[f] * fam_s[f] * fam_s[f];
    fd.vert_off[f + 1] = fd.vert_off[f] + fam_nb[f] * fam_s[f];
    fd.cmul[f] = (h->tiled_next >> f) & 1u ? 3 : 1;
  }
  h->tiled = nfam ? h->tiled_next & ((1u << nfam) - 1u) : 0u;
  h->nverts = nverts;
  h->nslots = nverts + fd.ent_off[nfam];
  h->ngslots = fd.vert_off[nfam];
  if (h->nslots >= (1ll << 31)) return B200IPC_EINVAL;  // int32 run offsets

  CK(h->fixed.reserve(nverts));
  CK(cudaMemcpyAsync(h->fixed.ptr, fixed, nverts, cudaMemcpyDeviceToDevice, st));

  // incidence runs: the (block, local vertex) slots sorted by vertex, in list order inside a vertex.  The
  // gradient scatter, the row-wise numeric kernel and the row-wise symbolic phase all walk them.
  const int64_t ng = h->ngslots;
  CK(h->gseg.reserve(nverts + 1));
  if (ng > 0) {
    CK(h->gkeys_a.reserve(ng)); CK(h->gkeys_b.reserve(ng)); CK(h->gslot_a.reserve(ng)); CK(h->gslot_b.reserve(ng));
    gradient_keys_kernel<<<blocks_for(ng), kAT, 0, st>>>(fd, ng, h->gkeys_a.ptr, h->gslot_a.ptr);
    RC(post_launch());
    size_t tg = 0;
    const int vbits = bits_for((uint64_t)nverts);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tg, h->gkeys_a.ptr, h->gkeys_b.ptr, h->gslot_a.ptr, h->gslot_b.ptr,
                                       (int)ng, 0, vbits, st));
    CK(h->temp.reserve(tg));
    CK(cub::DeviceRadixSort::SortPairs(h->temp.ptr, tg, h->gkeys_a.ptr, h->gkeys_b.ptr, h->gslot_a.ptr,
                                       h->gslot_b.ptr, (int)ng, 0, vbits, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  lower_bound_kernel<<<blocks_for(nverts + 1), kAT, 0, st>>>(nverts, ng, h->gkeys_b.ptr, h->gseg.ptr);
  RC(post_launch());

  bool by_rows = h->symbolic_mode == 0;
  if (by_rows) {
    bool overflow = false;
    RC(symbolic_by_rows(h, dense_desc_fits(fd), factor_desc_fits(fd), &overflow, st));
    if (overflow) by_rows = false;   // some row has more distinct columns than the per-warp set holds
  }
  if (!by_rows) RC(symbolic_by_sort(h, st));
  h->symbolic_used = by_rows ? 2 : 1;
  h->have_rows = false;
  h->ready = true;
  if (nnzb_out) *nnzb_out = h->nnzb;
  return 0;
}

// Descriptor tables of the numeric kernels, built on first use after a symbolic phase (a Newton
// iteration uses one numeric path, so the other tables are never built).
static int ensure_desc(b200ipc_assembly* h, cudaStream_t st) {
  if (h->have_desc) return 0;
  CK(h->desc.reserve(h->nvalid));
  source_desc_kernel<<<blocks_for(h->nvalid), kAT, 0, st>>>(h->fam, h->nverts, h->nvalid, h->slot_b.ptr, h->desc.ptr);
  RC(post_launch());
  h->have_desc = true;
  return 0;
}

static int ensure_fdesc(b200ipc_assembly* h, cudaStream_t st) {
  if (h->have_fdesc) return 0;
  CK(h->fdesc.reserve(h->nvalid));
  factor_desc_kernel<<<blocks_for(h->nvalid), kAT, 0, st>>>(h->fam, h->nverts, h->nvalid, h->slot_b.ptr, h->fdesc.ptr);
  RC(post_launch());
  h->have_fdesc = true;
  return 0;
}

static int ensure_rows(b200ipc_assembly* h, cudaStream_t st) {
  if (h->have_rows) return 0;
  if (h->max_row < 0) {   // pattern from the sort path: measure the longest row once
    CK(h->scalars.reserve(4));
    CK(cudaMemsetAsync(h->scalars.ptr, 0, sizeof(int64_t), st));
    max_row_kernel<<<blocks_for(h->nverts), kAT, 0, st>>>(h->nverts, h->rowptr.ptr, h->scalars.ptr);
    RC(post_launch());
    int64_t m = 0;
    CK(cudaMemcpyAsync(&m, h->scalars.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h->max_row = m;
  }
  // rs_dst packs the position of a destination block inside its row into 16 bits (0xffff = dropped)
  if (h->max_row >= 0xffff) return B200IPC_EINVAL;
  const int64_t ng = h->ngslots;
  if (ng > 0) {
    CK(h->rs_desc.reserve(ng)); CK(h->rs_dst.reserve(ng));
    row_source_kernel<<<blocks_for(ng), kAT, 0, st>>>(h->fam, h->nverts, ng, h->gslot_b.ptr, h->fixed.ptr, h->rowptr.ptr,
                                                     h->colidx.ptr, h->rs_desc.ptr, h->rs_dst.ptr);
    RC(post_launch());
  }
  h->have_rows = true;
  return 0;
}

extern "C" int b200ipc_assembly_pattern(b200ipc_assembly* h, int32_t* rowptr, int32_t* colidx, void* stream) {
  if (!h || !h->ready) return B200IPC_ESTATE;
  cudaStream_t st = (cudaStream_t)stream;
  if (rowptr) CK(cudaMemcpyAsync(rowptr, h->rowptr.ptr, (h->nverts + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  if (colidx) CK(cudaMemcpyAsync(colidx, h->colidx.ptr, h->nnzb * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  return 0;
}

extern "C" int b200ipc_assemble_numeric(b200ipc_assembly* h, const double* masses, const double* const* fam_hess,
                                        double* vals, void* stream) {
  if (!h || !h->ready) return B200IPC_ESTATE;
  if (!masses || !vals || (h->fam.nfam && !fam_hess)) return B200IPC_EINVAL;
  NumericArgs a;
  for (int f = 0; f <= kMaxFam; ++f) a.hp.p[f] = nullptr;
  for (int f = 0; f < 4; ++f) a.ld[f] = 0;
  bool packed_ok = h->fam.nfam <= 3;
  for (int f = 0; f < h->fam.nfam; ++f) {
    if (h->fam.nb[f] && !fam_hess[f]) return B200IPC_EINVAL;
    a.hp.p[f] = fam_hess[f];
    if (f < 3) a.ld[f] = h->fam.cmul[f] == 3 ? 3 : 3 * h->fam.s[f];
    if (h->fam.nb[f] * 9 * h->fam.s[f] * h->fam.s[f] >= (3ll << 30)) packed_ok = false;
  }
  a.nnzb = h->nnzb; a.fixed = h->fixed.ptr; a.masses = masses;
  a.useg = h->useg.ptr; a.uend = h->uend.ptr; a.desc = h->desc.ptr; a.vals = vals;
  // automatic choice between the two per-block-run walkers: trios win while runs are short (cloth on sphere,
  // 2.5 sources per block: 48 vs 60 us), the three-group walker when the diagonal runs are long (cloth stack,
  // 9 per block, 46 on the diagonal: 299 vs 320 us); b200ipc_assemble_numeric_factors makes the same choice, so
  // the two paths stay bitwise equal
  const bool short_runs = h->nvalid < 4 * h->nnzb;
  if ((h->variant == 1 || (h->variant == 0 && !short_runs)) && packed_ok) {  // per-block runs (gather of 3x3 sub-blocks)
    RC(ensure_desc(h, (cudaStream_t)stream));
    a.desc = h->desc.ptr;
    const unsigned grid = (unsigned)((h->nnzb + kNumWarps * kBlocksPerWarp - 1) / (kNumWarps * kBlocksPerWarp));
    assemble_numeric_kernel<<<grid, 32 * kNumWarps, 0, (cudaStream_t)stream>>>(a);
    return post_launch();
  }
  if ((h->variant == 2 || h->variant == 0) && packed_ok) {  // per-block runs, three blocks per warp trip
    RC(ensure_desc(h, (cudaStream_t)stream));
    a.desc = h->desc.ptr;
    const int64_t per_cta = (int64_t)kNumWarps * kTriosPerWarp * 3;
    assemble_numeric_trio_kernel<<<(unsigned)((h->nnzb + per_cta - 1) / per_cta), 32 * kNumWarps, 0, (cudaStream_t)stream>>>(a);
    return post_launch();
  }
  if (h->tiled) return B200IPC_EINVAL;   // the row-wise kernel reads whole rows of row-major blocks
  RC(ensure_rows(h, (cudaStream_t)stream));
  RowArgs r;
  r.hp = a.hp;
  for (int f = 0; f <= kMaxFam; ++f) r.fs[f] = f < h->fam.nfam ? h->fam.s[f] : 0;
  r.nverts = h->nverts; r.fixed = h->fixed.ptr; r.masses = masses; r.rowptr = h->rowptr.ptr; r.colidx = h->colidx.ptr;
  r.gseg = h->gseg.ptr; r.rs_desc = h->rs_desc.ptr; r.rs_dst = h->rs_dst.ptr; r.vals = vals;
  const unsigned grid = (unsigned)((h->nverts + kRowWarps - 1) / kRowWarps);
  assemble_rows_kernel<<<grid, 32 * kRowWarps, 0, (cudaStream_t)stream>>>(r);
  return post_launch();
}

extern "C" int b200ipc_assemble_numeric_factors(b200ipc_assembly* h, const double* masses,
                                                const double* const* fam_fac, double* vals, void* stream) {
  if (!h || !h->ready) return B200IPC_ESTATE;
  if (!masses || !vals || (h->fam.nfam && !fam_fac)) return B200IPC_EINVAL;
  if (h->fam.nfam > 3) return B200IPC_EINVAL;  // 2-bit family field
  FactorArgs a;
  for (int f = 0; f <= kMaxFam; ++f) a.fp.p[f] = nullptr;
  for (int f = 0; f < h->fam.nfam; ++f) {
    if (h->fam.nb[f] && !fam_fac[f]) return B200IPC_EINVAL;
    if (h->fam.nb[f] * 3 * h->fam.s[f] >= (1ll << 27)) return B200IPC_EINVAL;  // 27-bit element index
    a.fp.p[f] = fam_fac[f];
  }
  RC(ensure_fdesc(h, (cudaStream_t)stream));
  a.nnzb = h->nnzb; a.fixed = h->fixed.ptr; a.masses = masses; a.useg = h->useg.ptr; a.uend = h->uend.ptr; a.fdesc = h->fdesc.ptr;
  a.vals = vals;
  const bool short_runs = h->nvalid < 4 * h->nnzb;
  if (h->variant == 1 || (h->variant != 2 && !short_runs)) {   // same walker as b200ipc_assemble_numeric: bitwise equal to it
    const unsigned grid = (unsigned)((h->nnzb + kNumWarps * kBlocksPerWarp - 1) / (kNumWarps * kBlocksPerWarp));
    assemble_factors_kernel<<<grid, 32 * kNumWarps, 0, (cudaStream_t)stream>>>(a);
    return post_launch();
  }
  const int64_t per_cta = (int64_t)kNumWarps * kTriosPerWarp * 3;
  assemble_factors_trio_kernel<<<(unsigned)((h->nnzb + per_cta - 1) / per_cta), 32 * kNumWarps, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}

extern "C" int b200ipc_scatter_gradient(b200ipc_assembly* h, const double* masses, const double* x,
                                        const double* x_tilde, const double* const* fam_grad, double* out,
                                        void* stream) {
  if (!h || !h->ready) return B200IPC_ESTATE;
  if (!masses || !x || !x_tilde || !out || (h->fam.nfam && !fam_grad)) return B200IPC_EINVAL;
  GradArgs a;
  a.fd = h->fam;
  for (int f = 0; f < h->fam.nfam; ++f) {
    if (h->fam.nb[f] && !fam_grad[f]) return B200IPC_EINVAL;
    a.gp.p[f] = fam_grad[f];
  }
  a.nverts = h->nverts; a.fixed = h->fixed.ptr; a.masses = masses; a.x = x; a.x_tilde = x_tilde;
  a.gseg = h->gseg.ptr; a.gperm = h->gslot_b.ptr; a.out = out;
  scatter_gradient_kernel<<<blocks_for(3 * h->nverts), kAT, 0, (cudaStream_t)stream>>>(a);
  return post_launch();
}
