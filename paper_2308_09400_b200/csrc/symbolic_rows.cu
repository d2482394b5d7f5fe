// Row-wise symbolic assembly: the pattern and the source runs of the BSR matrix built per block-row
// from the vertex-incidence runs, without a global sort of the 16 n_c (row, col) slots.
//
// The sort-based phase (assembly.cu) keys every sub-block slot by row*N+col and radix-sorts all of
// them: five passes over 16.5 M 64-bit keys for 1 M contacts, 1.26 ms, four times the numeric phase.
// But the slots of row i are exactly the sub-blocks (a, c) of the blocks incident to vertex i with
// v[a] = i, and the incidence runs -- (block, local vertex) pairs per vertex in list order -- already
// exist for the gradient scatter (one 17-bit sort of 4 n_c keys).  So:
//
//   count  one warp per row walks the row's incidences, eight per trip (lane = 4 jj + c handles
//          sub-block c of incidence jj), and drops the kept column ids into a per-warp hash set in
//          shared memory: U_i unique columns, C_i kept sources.
//   scan   one exclusive sum over the packed (U_i << 32 | C_i) gives every row its first block and
//          its first source.
//   emit   the warp rebuilds the set, ranks its U_i columns (all distinct: rank = number of smaller
//          ones, U_i^2 / 32 compares per lane, U_i ~ 17), turns the per-column source counts into run
//          starts and walks the incidences once more: a source's position inside its run is the run's
//          cursor plus the number of earlier lanes of the trip with the same column
//          (__match_any_sync), so every run lists its sources in list order, the mass slot first --
//          the order the sort-based phase produces, hence bitwise the same matrices.  It writes
//          colidx, the run starts and BOTH 32-bit source descriptor tables of the numeric kernels
//          directly (they need no slot permutation any more).
//
// A row with more than kSymMaxU distinct columns raises a flag and the caller rebuilds the pattern
// with the sort-based phase.  No atomics on global data except that flag and a max: deterministic.
#include <cub/cub.cuh>

#include "launch.cuh"
#include "../../include/b200ipc.h"

#include "assembly.cuh"

namespace b200ipc {

constexpr int kSymHT = 512;      // hash slots per warp (power of two)
constexpr int kSymMaxU = 256;    // distinct columns per row this path handles
constexpr int kCountWarps = 8;
constexpr int kEmitWarps = 4;

struct SymArgs {
  FamDesc fd;
  int64_t nverts;
  const uint8_t* fixed;
  const int32_t* gseg;                // (N+1) incidence runs per vertex
  const uint32_t* gperm;              // gradient slots b*s+a (family offset included), sorted by vertex
  unsigned long long* counts;         // (N+1): U << 32 | C, entry N = 0
  const unsigned long long* base;     // exclusive sum of counts
  int32_t* rowptr;
  int32_t* colidx;
  int32_t* useg;
  uint32_t* desc;                     // may be null (families that do not fit the 32-bit descriptors)
  uint32_t* fdesc;                    // may be null
  int64_t* scalars;                   // [0] nnzb, [1] sources kept, [2] overflow flag, [3] longest row
};

struct Candidate {
  int32_t col;
  uint32_t desc, fdesc;
  bool keep;
};

// sub-block c of incidence j of `row` (j1 = end of the row's run)
__device__ __forceinline__ Candidate make_candidate(const SymArgs& a, int64_t row, int32_t j, int32_t j1, int c) {
  Candidate k;
  k.col = -1;
  k.desc = k.fdesc = 0;
  k.keep = false;
  if (j < j1) {
    const int64_t q = a.gperm[j];
    int f = 0;
#pragma unroll
    for (int t = 1; t < kMaxFam; ++t)
      if (t < a.fd.nfam && q >= a.fd.vert_off[t]) f = t;
    const int s = a.fd.s[f];
    if (c < s) {
      const int64_t r = q - a.fd.vert_off[f];
      const int64_t b = r / s;
      const int la = (int)(r - b * s);
      const int64_t col = a.fd.vids[f][b * s + c];
      k.col = (int32_t)col;
      k.keep = col == row || !a.fixed[col];
      const int64_t za = b * 3 * s + 3 * la;    // element index of z_a / first row of the sub-block row
      k.desc = ((uint32_t)f << 30) | (uint32_t)(za * s + c);
      k.fdesc = ((uint32_t)f << 30) | ((uint32_t)(c - la + 3) << 27) | (uint32_t)za;
    }
  }
  return k;
}

__device__ __forceinline__ int hash_home(int32_t col) { return (int)(((uint32_t)col * 2654435761u) >> 23); }  // 9 bits

// insert into the warp's set; returns the slot, fresh = this call created it
__device__ __forceinline__ int set_insert(int32_t* keys, int32_t col, bool& fresh) {
  int h = hash_home(col);
  for (;;) {
    const int32_t prev = atomicCAS(&keys[h], -1, col);
    if (prev == -1) {
      fresh = true;
      return h;
    }
    if (prev == col) {
      fresh = false;
      return h;
    }
    h = (h + 1) & (kSymHT - 1);
  }
}

__device__ __forceinline__ int set_find(const int32_t* keys, int32_t col) {
  int h = hash_home(col);
  while (keys[h] != col) h = (h + 1) & (kSymHT - 1);
  return h;
}

__global__ void __launch_bounds__(32 * kCountWarps) row_count_kernel(const __grid_constant__ SymArgs a) {
  __shared__ int32_t keys[kCountWarps][kSymHT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kCountWarps + w;
  if (row > a.nverts) return;
  if (row == a.nverts) {
    if (lane == 0) a.counts[row] = 0ull;
    return;
  }
  if (a.fixed[row]) {   // Dirichlet row: the unit diagonal, one (mass) source
    if (lane == 0) a.counts[row] = (1ull << 32) | 1ull;
    return;
  }
  int32_t* ht = keys[w];
  for (int t = lane; t < kSymHT; t += 32) ht[t] = -1;
  __syncwarp();
  int nu = 0, nc = 0;
  if (lane == 0) {
    bool fresh;
    set_insert(ht, (int32_t)row, fresh);   // the diagonal block always exists; its first source is the mass slot
    nu = nc = 1;
  }
  __syncwarp();
  const int32_t j0 = a.gseg[row], j1 = a.gseg[row + 1];
  bool over = false;
  for (int32_t j = j0; j < j1; j += 8) {
    const Candidate k = make_candidate(a, row, j + (lane >> 2), j1, lane & 3);
    if (k.keep) {
      bool fresh;
      set_insert(ht, k.col, fresh);
      nu += fresh ? 1 : 0;
      nc += 1;
    }
    if (__reduce_add_sync(0xffffffffu, nu) > kSymMaxU) {   // the set never fills: at most 32 new columns per trip
      over = true;
      break;
    }
  }
  nu = __reduce_add_sync(0xffffffffu, nu);
  nc = __reduce_add_sync(0xffffffffu, nc);
  if (lane == 0) {
    if (over) {
      a.scalars[2] = 1;                       // the caller rebuilds this pattern with the sort-based phase
      a.counts[row] = (1ull << 32) | 1ull;
    } else {
      a.counts[row] = ((unsigned long long)nu << 32) | (unsigned long long)nc;
      atomicMax(reinterpret_cast<unsigned long long*>(a.scalars + 3), (unsigned long long)nu);
    }
  }
}

__global__ void __launch_bounds__(32 * kEmitWarps) row_emit_kernel(const __grid_constant__ SymArgs a) {
  __shared__ int32_t keys[kEmitWarps][kSymHT];     // column of each occupied slot, -1 = empty
  __shared__ int32_t cnt[kEmitWarps][kSymHT];      // sources per slot
  __shared__ uint16_t rank_of[kEmitWarps][kSymHT]; // rank of the slot's column among the row's columns
  __shared__ int32_t ucol[kEmitWarps][kSymMaxU];   // the row's distinct columns (unordered)
  __shared__ uint16_t uslot[kEmitWarps][kSymMaxU]; // their slots
  __shared__ int32_t cur[kEmitWarps][kSymMaxU];    // per rank: source count -> run start -> write cursor
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kEmitWarps + w;
  if (row > a.nverts) return;
  const unsigned long long pre = a.base[row];
  const int64_t rowbase = (int64_t)(pre >> 32), srcbase = (int64_t)(pre & 0xffffffffull);
  if (row == a.nverts) {   // totals: closes rowptr and the run starts, reports to the host
    if (lane == 0) {
      a.rowptr[row] = (int32_t)rowbase;
      a.useg[rowbase] = (int32_t)srcbase;
      a.scalars[0] = rowbase;
      a.scalars[1] = srcbase;
    }
    return;
  }
  if (lane == 0) a.rowptr[row] = (int32_t)rowbase;
  const uint32_t mass_desc = 0xC0000000u | (uint32_t)row;
  if (a.fixed[row]) {
    if (lane == 0) {
      a.colidx[rowbase] = (int32_t)row;
      a.useg[rowbase] = (int32_t)srcbase;
      if (a.desc) a.desc[srcbase] = mass_desc;
      if (a.fdesc) a.fdesc[srcbase] = mass_desc;
    }
    return;
  }
  int32_t* ht = keys[w];
  int32_t* hc = cnt[w];
  for (int t = lane; t < kSymHT; t += 32) {
    ht[t] = -1;
    hc[t] = 0;
  }
  __syncwarp();
  int diag_slot = 0;
  if (lane == 0) {
    bool fresh;
    diag_slot = set_insert(ht, (int32_t)row, fresh);
    hc[diag_slot] = 1;
  }
  diag_slot = __shfl_sync(0xffffffffu, diag_slot, 0);
  __syncwarp();
  const int32_t j0 = a.gseg[row], j1 = a.gseg[row + 1];
  // ---- pass 1: the set of columns and the number of sources per column -----------------------------
  int nu = lane == 0 ? 1 : 0;
  for (int32_t j = j0; j < j1; j += 8) {
    const Candidate k = make_candidate(a, row, j + (lane >> 2), j1, lane & 3);
    if (k.keep) {
      bool fresh;
      const int slot = set_insert(ht, k.col, fresh);
      atomicAdd(&hc[slot], 1);
      nu += fresh ? 1 : 0;
    }
    if (__reduce_add_sync(0xffffffffu, nu) > kSymMaxU) return;   // flagged by row_count_kernel; rebuilt by the sort path
  }
  __syncwarp();
  // ---- compact the occupied slots ---------------------------------------------------------------------
  int U = 0;
  for (int g = 0; g < kSymHT; g += 32) {
    const int slot = g + lane;
    const bool occ = ht[slot] != -1;
    const unsigned m = __ballot_sync(0xffffffffu, occ);
    if (occ) {
      const int p = U + __popc(m & ((1u << lane) - 1u));
      ucol[w][p] = ht[slot];
      uslot[w][p] = (uint16_t)slot;
    }
    U += __popc(m);
  }
  __syncwarp();
  // ---- rank the columns (all distinct), publish colidx, counts by rank --------------------------------
  for (int k = lane; k < U; k += 32) {
    const int32_t mine = ucol[w][k];
    int r = 0;
    for (int m = 0; m < U; ++m) r += ucol[w][m] < mine ? 1 : 0;
    const int slot = uslot[w][k];
    rank_of[w][slot] = (uint16_t)r;
    cur[w][r] = hc[slot];
    a.colidx[rowbase + r] = mine;
  }
  __syncwarp();
  // ---- counts -> run starts (exclusive scan over the ranks, 32 at a time) ------------------------------
  int carry = 0;
  for (int g = 0; g < U; g += 32) {
    const int r = g + lane;
    const int c = r < U ? cur[w][r] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (r < U) {
      const int start = carry + inc - c;
      cur[w][r] = start;
      a.useg[rowbase + r] = (int32_t)(srcbase + start);
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncwarp();
  // ---- pass 2: place every source at its run's cursor, in list order ----------------------------------
  if (lane == 0) {
    const int r = rank_of[w][diag_slot];
    const int p = cur[w][r];
    if (a.desc) a.desc[srcbase + p] = mass_desc;
    if (a.fdesc) a.fdesc[srcbase + p] = mass_desc;
    cur[w][r] = p + 1;
  }
  __syncwarp();
  for (int32_t j = j0; j < j1; j += 8) {
    const Candidate k = make_candidate(a, row, j + (lane >> 2), j1, lane & 3);
    const unsigned r = k.keep ? (unsigned)rank_of[w][set_find(ht, k.col)] : (0x10000u | (unsigned)lane);
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    int p = 0;
    if (k.keep) p = cur[w][r] + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
    if (k.keep && (peers & ((1u << lane) - 1u)) == 0u) cur[w][r] += __popc(peers);   // the group's first lane
    __syncwarp();
    if (k.keep) {
      if (a.desc) a.desc[srcbase + p] = k.desc;
      if (a.fdesc) a.fdesc[srcbase + p] = k.fdesc;
    }
  }
}

}  // namespace b200ipc

using namespace b200ipc;

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

// The row-wise symbolic phase.  Expects h->fam, h->fixed, h->gseg and h->gslot_b (incidence runs) in
// place.  Returns 0 with *overflow = true when some row is too long for it (nothing usable was built).
int symbolic_by_rows(b200ipc_assembly* h, bool want_desc, bool want_fdesc, bool* overflow, cudaStream_t st) {
  const int64_t nverts = h->nverts;
  const FamDesc& fd = h->fam;
  int64_t offdiag = 0;   // sub-block slots off the diagonal: bound on the blocks beyond the N diagonal ones
  for (int f = 0; f < fd.nfam; ++f) offdiag += fd.nb[f] * fd.s[f] * (fd.s[f] - 1);
  const int64_t max_blocks = nverts + offdiag, max_sources = h->nslots;
  CK(h->row_counts.reserve(nverts + 1));
  CK(h->row_base.reserve(nverts + 1));
  CK(h->rowptr.reserve(nverts + 1));
  CK(h->colidx.reserve(max_blocks));
  CK(h->useg.reserve(max_blocks + 1));
  if (want_desc) CK(h->desc.reserve(max_sources));
  if (want_fdesc) CK(h->fdesc.reserve(max_sources));
  CK(h->scalars.reserve(4));
  CK(cudaMemsetAsync(h->scalars.ptr, 0, 4 * sizeof(int64_t), st));

  SymArgs a;
  a.fd = fd;
  a.nverts = nverts;
  a.fixed = h->fixed.ptr;
  a.gseg = h->gseg.ptr;
  a.gperm = h->gslot_b.ptr;
  a.counts = h->row_counts.ptr;
  a.base = h->row_base.ptr;
  a.rowptr = h->rowptr.ptr;
  a.colidx = h->colidx.ptr;
  a.useg = h->useg.ptr;
  a.desc = want_desc ? h->desc.ptr : nullptr;
  a.fdesc = want_fdesc ? h->fdesc.ptr : nullptr;
  a.scalars = h->scalars.ptr;

  row_count_kernel<<<(unsigned)((nverts + 1 + kCountWarps - 1) / kCountWarps), 32 * kCountWarps, 0, st>>>(a);
  RC(post_launch());
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, h->row_counts.ptr, h->row_base.ptr, (int)(nverts + 1), st));
  CK(h->temp.reserve(tb));
  CK(cub::DeviceScan::ExclusiveSum(h->temp.ptr, tb, h->row_counts.ptr, h->row_base.ptr, (int)(nverts + 1), st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  row_emit_kernel<<<(unsigned)((nverts + 1 + kEmitWarps - 1) / kEmitWarps), 32 * kEmitWarps, 0, st>>>(a);
  RC(post_launch());
  int64_t host[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(host, h->scalars.ptr, sizeof(host), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *overflow = host[2] != 0;
  if (*overflow) return 0;
  h->nnzb = host[0];
  h->nvalid = host[1];
  h->max_row = host[3];
  h->have_desc = want_desc;
  h->have_fdesc = want_fdesc;
  return 0;
}

}  // namespace b200ipc
