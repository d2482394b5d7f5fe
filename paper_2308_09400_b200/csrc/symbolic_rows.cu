// Row-wise symbolic assembly: the pattern and the source runs of the BSR matrix built per block-row
// from the vertex-incidence runs, without a global sort of the 16 n_c (row, col) slots.
//
// The sort-based phase (assembly.cu) keys every sub-block slot by row*N+col and radix-sorts all of
// them: five passes over 16.5 M 64-bit keys for 1 M contacts, 1.26 ms, four times the numeric phase.
// But the slots of row i are exactly the sub-blocks (a, c) of the blocks incident to vertex i with
// v[a] = i, and the incidence runs -- (block, local vertex) pairs per vertex in list order -- already
// exist for the gradient scatter (one 17-bit sort of 4 n_c keys).  So:
//
//   emit   one warp per row walks the row's incidences, eight per trip (lane = 4 jj + c handles sub-block
//          c of incidence jj; the loads of the next two trips are in flight), and drops the column ids into
//          a per-warp hash set in shared memory, counting the sources of each.  It then ranks the distinct
//          columns (rank = number of smaller ones, U^2 / 32 compares per lane, U ~ 17; a column that is a
//          Dirichlet vertex is dropped here, once per column instead of once per source), turns the counts
//          into run starts and walks the incidences once more: a source's position inside its run is the
//          run's cursor plus the number of earlier lanes of the trip with the same column
//          (__match_any_sync), so every run lists its sources in list order, the mass slot first -- the
//          order the sort-based phase produces, hence bitwise the same matrices.  Everything a row
//          produces goes to the row's own SLAB, [4 gseg[i] + i, 4 gseg[i+1] + i + 1): the number of its
//          sub-block slots bounds both its sources and its columns, so no count pass and no scan precede
//          the writes.  Both 32-bit source descriptor tables of the numeric kernels are written in place
//          (slab-spaced: a run is [useg[u], uend[u])).
//   scan   one exclusive sum over the row lengths -> rowptr.
//   pack   colidx and the run bounds move from the slabs to their compact places.
//
// Rows are tried with a 128-slot set first (<= 64 distinct columns: every row of a cloth scene; 15 KB of
// shared memory per CTA); a row that does not fit is redone by a second launch with 512 slots, and a row
// with more than 256 distinct columns raises a flag: the caller then rebuilds the pattern with the
// sort-based phase.  No atomics on global data except that flag, a max and an integer sum: deterministic.
#include <cub/cub.cuh>

#include "launch.cuh"
#include "../../include/b200ipc.h"

#include "assembly.cuh"

namespace b200ipc {

constexpr int kSymHT = 512;      // hash slots per warp (power of two), large rows
constexpr int kSymMaxU = 256;    // distinct columns per row this path handles
constexpr int kSmallHT = 128;    // rows with at most kSmallMaxU distinct columns (all of a cloth scene's)
constexpr int kSmallMaxU = 64;

struct SymArgs {
  FamDesc fd;
  uint32_t voff[kMaxFam + 1];         // fd.vert_off as 32-bit, 0xffffffff beyond the last family
  int64_t nverts;
  const uint8_t* fixed;
  const int32_t* gseg;                // (N+1) incidence runs per vertex
  const uint32_t* gperm;              // gradient slots b*s+a (family offset included), sorted by vertex
  int32_t* rowlen;                    // (N+1): kept columns per row, -1 = redo with the large set; entry N = 0
  int32_t* slab_col;                  // slab-spaced: columns, run starts, run ends
  int32_t* slab_beg;
  int32_t* slab_end;
  uint32_t* desc;                     // slab-spaced; may be null (families that do not fit the 32-bit descriptors)
  uint32_t* fdesc;                    // may be null
  int64_t* scalars;                   // [1] sources kept, [2] overflow flag, [3] longest row
};

// One decoded incidence (block b of family f, local vertex la; r = b s + la) as seen by lane (jj, c).
struct Incidence {
  uint32_t f, s, r, la;
  bool valid;     // the incidence exists and c < s
};

__device__ __forceinline__ uint32_t load_slot(const SymArgs& a, int32_t j, int32_t j1) { return j < j1 ? a.gperm[j] : 0xffffffffu; }

// 32-bit arithmetic throughout: the slot count is below 2^31, and s is 2, 3 or 4 (shift / multiply-high
// instead of a division).
__device__ __forceinline__ Incidence decode(const SymArgs& a, uint32_t q, int c) {
  Incidence k;
  k.f = k.r = k.la = 0;
  k.s = 0;
  k.valid = false;
  if (q != 0xffffffffu) {
    uint32_t f = 0;
#pragma unroll
    for (int t = 1; t < kMaxFam; ++t) f += q >= a.voff[t] ? 1u : 0u;
    const uint32_t s = (uint32_t)a.fd.s[f];
    const uint32_t r = q - a.voff[f];
    const uint32_t b = s == 4u ? r >> 2 : (s == 2u ? r >> 1 : __umulhi(r, 0xAAAAAAABu) >> 1);
    k.f = f;
    k.s = s;
    k.r = r;
    k.la = r - b * s;
    k.valid = (uint32_t)c < s;
  }
  return k;
}

__device__ __forceinline__ int32_t load_col(const SymArgs& a, const Incidence& k, int c) {
  return k.valid ? (int32_t)a.fd.vids[k.f][(int64_t)k.r - k.la + c] : -1;
}

// The per-warp column set: open addressing over `size` slots (a power of two, 32 - log2 size = shift).
__device__ __forceinline__ int hash_home(int32_t col, int shift) { return (int)(((uint32_t)col * 2654435761u) >> shift); }

// insert into the warp's set; returns the slot, fresh = this call created it
__device__ __forceinline__ int set_insert(int32_t* keys, int shift, int mask, int32_t col, bool& fresh) {
  int h = hash_home(col, shift);
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
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ int set_find(const int32_t* keys, int shift, int mask, int32_t col) {
  int h = hash_home(col, shift);
  while (keys[h] != col) h = (h + 1) & mask;
  return h;
}

// Walk the incidences of a row, eight per trip, with the loads of the next trips in flight: the slot of trip
// t+2 and the column of trip t+1 are requested before trip t is processed (the three loads of a trip --
// slot, column, and whatever `body` gathers -- are a dependent chain; un-pipelined the kernels sat on it).
template <typename BODY>
__device__ __forceinline__ void for_each_candidate(const SymArgs& a, int32_t j0, int32_t j1, int lane, BODY body) {
  const int jj = lane >> 2, c = lane & 3;
  Incidence cur = decode(a, load_slot(a, j0 + jj, j1), c);
  int32_t col = load_col(a, cur, c);
  uint32_t qn = load_slot(a, j0 + 8 + jj, j1);
  for (int32_t j = j0; j < j1; j += 8) {
    const Incidence nxt = decode(a, qn, c);
    const int32_t coln = load_col(a, nxt, c);
    qn = load_slot(a, j + 16 + jj, j1);
    if (!body(cur, col, c)) return;
    cur = nxt;
    col = coln;
  }
}

constexpr uint16_t kDropped = 0xffff;

// One row, by one warp, with a set of HT slots (<= MAXU distinct columns).  Returns false when the row does not
// fit (nothing was written).
template <int HT, int MAXU>
__device__ __forceinline__ bool emit_row(const SymArgs& a, int64_t row, int lane, int32_t* ht, int32_t* hc,
                                         uint16_t* rank_of, int32_t* ucol, uint16_t* uslot, int32_t* cur) {
  const int32_t j0 = a.gseg[row], j1 = a.gseg[row + 1];
  const int64_t slab = 4ll * j0 + row;
  const uint32_t mass_desc = 0xC0000000u | (uint32_t)row;
  if (a.fixed[row]) {   // Dirichlet row: the unit diagonal, one (mass) source
    if (lane == 0) {
      a.rowlen[row] = 1;
      a.slab_col[slab] = (int32_t)row;
      a.slab_beg[slab] = (int32_t)slab;
      a.slab_end[slab] = (int32_t)slab + 1;
      if (a.desc) a.desc[slab] = mass_desc;
      if (a.fdesc) a.fdesc[slab] = mass_desc;
      atomicAdd(reinterpret_cast<unsigned long long*>(a.scalars + 1), 1ull);
    }
    return true;
  }
  // at most 4 deg + 1 distinct columns: a smaller set for short rows
  int size = 32;
  while (size < HT && size < 2 * (4 * (j1 - j0) + 1)) size <<= 1;
  const int mask = size - 1, shift = 32 - (31 - __clz(size));
  for (int t = lane; t < size; t += 32) {
    ht[t] = -1;
    hc[t] = 0;
  }
  __syncwarp();
  int diag_slot = 0, nu = 0;
  if (lane == 0) {
    bool fresh;
    diag_slot = set_insert(ht, shift, mask, (int32_t)row, fresh);   // the diagonal block always exists; its first source is the mass slot
    hc[diag_slot] = 1;
    nu = 1;
  }
  diag_slot = __shfl_sync(0xffffffffu, diag_slot, 0);
  __syncwarp();
  // ---- pass 1: the set of columns and the number of sources per column -----------------------------
  bool over = false;
  for_each_candidate(a, j0, j1, lane, [&](const Incidence&, int32_t col, int) {
    if (col >= 0) {
      bool fresh;
      atomicAdd(&hc[set_insert(ht, shift, mask, col, fresh)], 1);
      nu += fresh ? 1 : 0;
    }
    if (__reduce_add_sync(0xffffffffu, nu) > MAXU) {   // the set never fills: at most 32 new columns per trip
      over = true;
      return false;
    }
    return true;
  });
  if (over) return false;
  __syncwarp();
  // ---- compact the kept columns; dropped ones (Dirichlet vertices other than the row) are marked ---------
  int U = 0;
  for (int g = 0; g < size; g += 32) {
    const int slot = g + lane;
    const int32_t col = ht[slot];
    bool keep = false;
    if (col >= 0) {
      keep = col == (int32_t)row || !a.fixed[col];
      if (!keep) rank_of[slot] = kDropped;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int p = U + __popc(m & ((1u << lane) - 1u));
      ucol[p] = col;
      uslot[p] = (uint16_t)slot;
    }
    U += __popc(m);
  }
  __syncwarp();
  // ---- rank the columns (all distinct), publish them, counts by rank ------------------------------------
  for (int k = lane; k < U; k += 32) {
    const int32_t mine = ucol[k];
    int r = 0;
    for (int m = 0; m < U; ++m) r += ucol[m] < mine ? 1 : 0;
    const int slot = uslot[k];
    rank_of[slot] = (uint16_t)r;
    cur[r] = hc[slot];
    a.slab_col[slab + r] = mine;
  }
  __syncwarp();
  // ---- counts -> run bounds (exclusive scan over the ranks, 32 at a time) -------------------------------
  int carry = 0;
  for (int g = 0; g < U; g += 32) {
    const int r = g + lane;
    const int c = r < U ? cur[r] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (r < U) {
      const int start = carry + inc - c;
      cur[r] = start;
      a.slab_beg[slab + r] = (int32_t)(slab + start);
      a.slab_end[slab + r] = (int32_t)(slab + start + c);
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    a.rowlen[row] = U;
    atomicAdd(reinterpret_cast<unsigned long long*>(a.scalars + 1), (unsigned long long)carry);
    atomicMax(reinterpret_cast<unsigned long long*>(a.scalars + 3), (unsigned long long)U);
  }
  __syncwarp();
  // ---- pass 2: place every source at its run's cursor, in list order ----------------------------------
  if (lane == 0) {
    const int r = rank_of[diag_slot];
    const int p = cur[r];
    if (a.desc) a.desc[slab + p] = mass_desc;
    if (a.fdesc) a.fdesc[slab + p] = mass_desc;
    cur[r] = p + 1;
  }
  __syncwarp();
  const unsigned below = (1u << lane) - 1u;
  for_each_candidate(a, j0, j1, lane, [&](const Incidence& k, int32_t col, int c) {
    unsigned r = kDropped;
    if (col >= 0) r = rank_of[set_find(ht, shift, mask, col)];
    const bool keep = r != kDropped;
    const unsigned peers = __match_any_sync(0xffffffffu, keep ? r : (0x10000u | (unsigned)lane));
    int p = 0;
    if (keep) p = cur[r] + __popc(peers & below);
    __syncwarp();
    if (keep && (peers & below) == 0u) cur[r] += __popc(peers);   // the group's first lane
    __syncwarp();
    if (keep) {
      const uint32_t za = 3u * k.r;                      // element index of z_a = 3 (b s + a)
      // row-major ((b D + 3a) D + 3c) / 3, D = 3s; sub-block-major 9 (b s^2 + a s + c) / 3
      if (a.desc) a.desc[slab + p] = (k.f << 30) | (za * k.s + (uint32_t)(a.fd.cmul[k.f] * c));
      if (a.fdesc) a.fdesc[slab + p] = (k.f << 30) | ((uint32_t)(c - (int)k.la + 3) << 27) | za;
    }
    return true;
  });
  return true;
}

#define B200IPC_ROW_SMEM(HT, MAXU, WARPS)                                              \
  __shared__ int32_t keys[WARPS][HT];      /* column of each occupied slot, -1 = empty */ \
  __shared__ int32_t cnt[WARPS][HT];       /* sources per slot */                        \
  __shared__ uint16_t rank_of[WARPS][HT];  /* rank of the slot's column among the kept columns */ \
  __shared__ int32_t ucol[WARPS][MAXU];    /* the row's distinct kept columns (unordered) */ \
  __shared__ uint16_t uslot[WARPS][MAXU];  /* their slots */                             \
  __shared__ int32_t cur[WARPS][MAXU];     /* per rank: source count -> run start -> write cursor */

// first try: every row, small set
__global__ void __launch_bounds__(256) row_emit_small_kernel(const __grid_constant__ SymArgs a) {
  B200IPC_ROW_SMEM(kSmallHT, kSmallMaxU, 8)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + w;
  if (row > a.nverts) return;
  if (row == a.nverts) {
    if (lane == 0) a.rowlen[row] = 0;
    return;
  }
  if (!emit_row<kSmallHT, kSmallMaxU>(a, row, lane, keys[w], cnt[w], rank_of[w], ucol[w], uslot[w], cur[w]))
    if (lane == 0) a.rowlen[row] = -1;
}

// second try: a persistent grid scans the row lengths 32 at a time and redoes the rows marked -1 with the large
// set (none in a cloth scene: the launch then costs a 300 KB read)
__global__ void __launch_bounds__(128) row_emit_large_kernel(const __grid_constant__ SymArgs a) {
  B200IPC_ROW_SMEM(kSymHT, kSymMaxU, 4)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * 4;
  for (int64_t r0 = 32 * ((int64_t)blockIdx.x * 4 + w); r0 < a.nverts; r0 += 32 * warps) {
    const int64_t mine = r0 + lane;
    unsigned todo = __ballot_sync(0xffffffffu, mine < a.nverts && a.rowlen[mine] < 0);
    while (todo) {
      const int64_t row = r0 + (__ffs(todo) - 1);
      todo &= todo - 1;
      if (!emit_row<kSymHT, kSymMaxU>(a, row, lane, keys[w], cnt[w], rank_of[w], ucol[w], uslot[w], cur[w])) {
        if (lane == 0) {
          a.scalars[2] = 1;      // the caller rebuilds this pattern with the sort-based phase
          a.rowlen[row] = 1;
        }
      }
      __syncwarp();
    }
  }
}

// slab -> compact: one warp per row
__global__ void __launch_bounds__(256) row_pack_kernel(int64_t nverts, const int32_t* __restrict__ gseg,
                                                       const int32_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ slab_col,
                                                       const int32_t* __restrict__ slab_beg,
                                                       const int32_t* __restrict__ slab_end,
                                                       int32_t* __restrict__ colidx, int32_t* __restrict__ useg,
                                                       int32_t* __restrict__ uend) {
  const int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nverts) return;
  const int32_t r0 = rowptr[row], len = rowptr[row + 1] - r0;
  const int64_t slab = 4ll * gseg[row] + row;
  for (int k = lane; k < len; k += 32) {
    colidx[r0 + k] = slab_col[slab + k];
    useg[r0 + k] = slab_beg[slab + k];
    uend[r0 + k] = slab_end[slab + k];
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
  const int64_t nslab = 4 * h->ngslots + nverts;   // slab space: every row's sub-block slots padded to 4 per incidence
  if (nslab >= (1ll << 31)) {
    *overflow = true;   // 32-bit run bounds: leave it to the sort path (which has its own limit)
    return 0;
  }
  CK(h->row_len.reserve(nverts + 1));
  CK(h->rowptr.reserve(nverts + 1));
  CK(h->slab_col.reserve(nslab)); CK(h->slab_beg.reserve(nslab)); CK(h->slab_end.reserve(nslab));
  if (want_desc) CK(h->desc.reserve(nslab));
  if (want_fdesc) CK(h->fdesc.reserve(nslab));
  CK(h->scalars.reserve(4));
  CK(cudaMemsetAsync(h->scalars.ptr, 0, 4 * sizeof(int64_t), st));

  SymArgs a;
  a.fd = fd;
  for (int f = 0; f <= kMaxFam; ++f) a.voff[f] = f < fd.nfam ? (uint32_t)fd.vert_off[f] : 0xffffffffu;
  a.nverts = nverts;
  a.fixed = h->fixed.ptr;
  a.gseg = h->gseg.ptr;
  a.gperm = h->gslot_b.ptr;
  a.rowlen = h->row_len.ptr;
  a.slab_col = h->slab_col.ptr;
  a.slab_beg = h->slab_beg.ptr;
  a.slab_end = h->slab_end.ptr;
  a.desc = want_desc ? h->desc.ptr : nullptr;
  a.fdesc = want_fdesc ? h->fdesc.ptr : nullptr;
  a.scalars = h->scalars.ptr;

  row_emit_small_kernel<<<(unsigned)((nverts + 1 + 7) / 8), 256, 0, st>>>(a);
  RC(post_launch());
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  row_emit_large_kernel<<<(unsigned)(2 * sms), 128, 0, st>>>(a);
  RC(post_launch());
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, h->row_len.ptr, h->rowptr.ptr, (int)(nverts + 1), st));
  CK(h->temp.reserve(tb));
  CK(cub::DeviceScan::ExclusiveSum(h->temp.ptr, tb, h->row_len.ptr, h->rowptr.ptr, (int)(nverts + 1), st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  // one synchronisation: the block count sizes colidx and the run bounds
  int64_t host[4] = {0, 0, 0, 0};
  int32_t nnzb32 = 0;
  CK(cudaMemcpyAsync(host, h->scalars.ptr, sizeof(host), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nnzb32, h->rowptr.ptr + nverts, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *overflow = host[2] != 0;
  if (*overflow) return 0;
  h->nnzb = nnzb32;
  h->nvalid = host[1];
  h->max_row = host[3];
  CK(h->colidx.reserve(h->nnzb)); CK(h->useg.reserve(h->nnzb + 1)); CK(h->uend.reserve(h->nnzb + 1));
  row_pack_kernel<<<(unsigned)((32 * nverts + 255) / 256), 256, 0, st>>>(nverts, h->gseg.ptr, h->rowptr.ptr, h->slab_col.ptr,
                                                                      h->slab_beg.ptr, h->slab_end.ptr, h->colidx.ptr,
                                                                      h->useg.ptr, h->uend.ptr);
  RC(post_launch());
  h->have_desc = want_desc;
  h->have_fdesc = want_fdesc;
  return 0;
}

}  // namespace b200ipc
