// Broad phase of find_contact_pairs (proximity.py:232-248, :275-319) on the device: the candidate
// point-triangle and edge-edge queries the narrow phase (narrow.cu) classifies.
//
// The reference tests every (surface vertex, triangle) and every (edge, edge) pair for AABB overlap --
// O(n^2) boolean matrices.  Here both joins run on a uniform grid:
//   1. the boxes of the "B" elements (triangle AABB; edge AABB inflated by d_hat/2) are built once and
//      each is filed under ONE cell, the cell of its lower corner (counting sort on dense grids, one radix
//      sort of n keys otherwise; no multi-cell binning, so no pair can be found twice); the largest box
//      extent per axis is reduced on the device alongside; boxes much larger than a cell get a coarse
//      grid of their own (two size classes);
//   2. every "A" box (vertex box [p - d_hat, p + d_hat]; inflated edge AABB) probes the cells that can
//      hold the lower corner of an overlapping B box, [A.lo - max extent, A.hi], finds each cell
//      column's run (dense cell table, or binary search on large grids), and -- eight lanes per A box
//      walking the runs laid end to end -- keeps a pair when
//        - the boxes overlap (the reference's own predicate lo_a <= hi_b && lo_b <= hi_a on the same
//          fp64 box corners, so the candidate SET equals the reference's),
//        - the reference's incidence filters pass (vertex not a corner of the triangle, :286;
//          edge index i < j and no shared endpoint, :311-317);
//      and appends (A, B) as global vertex ids to a staging list in ONE pass: hits are buffered in
//      registers and flushed with one atomic per warp; when the list is too small the pass only counts,
//      the list is regrown with head-room and the pass repeated (first query of a scene, or a contact set
//      that grew by more than the head-room).
// The candidate SET is deterministic, its order is not -- and does not matter: the narrow phase sorts by
// a total order over (kind, vertices, origin query), the CCD filter takes a minimum.
// The same join with swept boxes (both ends of a step, margin 1e-3 d_hat) is sweep_candidates
// (proximity.py:388-421), the candidate set of the CCD step filter (accd.cu).
#include <cmath>
#include <cub/cub.cuh>

#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

#ifndef B200IPC_BROAD_THREADS
#define B200IPC_BROAD_THREADS 256
#endif
constexpr int kBT = B200IPC_BROAD_THREADS;

template <typename T>
struct BroadBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    const size_t want = n + n / 4 + 64;  // head-room: contact sets drift from step to step
    cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

struct Grid {
  double ox, oy, oz;  // origin
  double inv;         // 1 / cell
  int mx, my, mz;     // largest cell index per axis (coordinates beyond are clamped: cells merge, still exact)
  int sy, sx;         // key = cx << sx | cy << sy | cz: as few key bits as the grid needs (fewer sort passes)
};

struct __align__(16) Box {
  double lx, ly, lz, hx, hy, hz;
};

__device__ __forceinline__ int cell_of(double x, double o, double inv, int maxc) {
  const double c = floor((x - o) * inv);
  return c < 0.0 ? 0 : (c > (double)maxc ? maxc : (int)c);
}
__device__ __forceinline__ uint64_t cell_key(const Grid& g, int cx, int cy, int cz) {
  return ((uint64_t)cx << g.sx) | ((uint64_t)cy << g.sy) | (uint64_t)cz;
}
__device__ __forceinline__ void ld3(const double* p, int v, double& x, double& y, double& z) {
  x = p[3ll * v];
  y = p[3ll * v + 1];
  z = p[3ll * v + 2];
}

// Box of element i.  KIND 0: surface vertex, 1: triangle, 2: edge.  The box covers the element at
// `pos` and -- when `dir` is given -- at pos + dir (the swept box of sweep_candidates,
// proximity.py:393-401, :409-412), grown by `m` on every side.  Static detection uses dir = NULL and
// m = d_hat / 0 / d_hat/2 (proximity.py:278-281, :305-307): min(p, p) - m = p - m and x - 0.0 = x, so
// the corners are bit-identical to the reference's.
struct Boxes {
  const double* pos;
  const double* dir;   // NULL: static
  double m[3];         // margin per KIND
};

__device__ __forceinline__ void grow(Box& b, const Boxes& in, int v, bool first) {
  double x, y, z;
  ld3(in.pos, v, x, y, z);
  if (first) {
    b.lx = b.hx = x; b.ly = b.hy = y; b.lz = b.hz = z;
  } else {
    b.lx = fmin(b.lx, x); b.ly = fmin(b.ly, y); b.lz = fmin(b.lz, z);
    b.hx = fmax(b.hx, x); b.hy = fmax(b.hy, y); b.hz = fmax(b.hz, z);
  }
}

template <int KIND>
__device__ __forceinline__ Box make_box(const Boxes& in, const int32_t* __restrict__ elems, int64_t i) {
  constexpr int NV = KIND == 0 ? 1 : (KIND == 1 ? 3 : 2);
  int v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = elems[NV * i + k];
  Box b;
#pragma unroll
  for (int k = 0; k < NV; ++k) grow(b, in, v[k], k == 0);
  if (in.dir) {  // end-of-step positions pos + dir: min / max over both poses (the order of the
                 // reference's nested minimum() calls does not matter: min and max are exact)
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double x, y, z, dx, dy, dz;
      ld3(in.pos, v[k], x, y, z);
      ld3(in.dir, v[k], dx, dy, dz);
      x = x + dx; y = y + dy; z = z + dz;
      b.lx = fmin(b.lx, x); b.ly = fmin(b.ly, y); b.lz = fmin(b.lz, z);
      b.hx = fmax(b.hx, x); b.hy = fmax(b.hy, y); b.hz = fmax(b.hz, z);
    }
  }
  const double m = in.m[KIND];
  b.lx -= m; b.ly -= m; b.lz -= m;
  b.hx += m; b.hy += m; b.hz += m;
  return b;
}

struct Span {
  int x0, y0, z0, x1, y1, z1;
  __device__ __forceinline__ int64_t count() const { return (int64_t)(x1 - x0 + 1) * (y1 - y0 + 1) * (z1 - z0 + 1); }
};
__device__ __forceinline__ Span span_of(const Box& b, const Grid& g) {
  Span s;
  s.x0 = cell_of(b.lx, g.ox, g.inv, g.mx); s.y0 = cell_of(b.ly, g.oy, g.inv, g.my); s.z0 = cell_of(b.lz, g.oz, g.inv, g.mz);
  s.x1 = cell_of(b.hx, g.ox, g.inv, g.mx); s.y1 = cell_of(b.hy, g.oy, g.inv, g.my); s.z1 = cell_of(b.hz, g.oz, g.inv, g.mz);
  return s;
}

// Boxes of all elements of one kind, once per query: the join then tests 48 contiguous bytes per
// candidate instead of rebuilding the box from two or three gathered vertices.
template <int KIND>
__global__ void __launch_bounds__(kBT) make_boxes_kernel(const Boxes in, const int32_t* __restrict__ elems, int64_t n,
                                                         Box* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kBT + threadIdx.x;
  if (i < n) out[i] = make_box<KIND>(in, elems, i);
}

// Home cell (cell of the lower corner) of every B box of one SIZE CLASS -- largest extent in (lo_thr, hi_thr] -- and
// the class's largest extent per axis (ordered-bits atomicMax: extents are non-negative doubles).  A box of another
// class gets the key `sentinel` (one past the largest cell key: it sorts behind every cell and no probe reaches it).
__global__ void __launch_bounds__(kBT) home_cell_kernel(const Box* __restrict__ box, int64_t n, Grid g, double lo_thr,
                                                        double hi_thr, uint64_t sentinel, uint64_t* __restrict__ keys,
                                                        uint32_t* __restrict__ ids, unsigned long long* __restrict__ ext,
                                                        int32_t* __restrict__ count /* per cell, or null */) {
  const int64_t i = (int64_t)blockIdx.x * kBT + threadIdx.x;
  double ex = 0.0, ey = 0.0, ez = 0.0;
  if (i < n) {
    const Box b = box[i];
    ex = b.hx - b.lx; ey = b.hy - b.ly; ez = b.hz - b.lz;
    const double big = fmax(ex, fmax(ey, ez));
    const bool member = big > lo_thr && big <= hi_thr;
    keys[i] = member ? cell_key(g, cell_of(b.lx, g.ox, g.inv, g.mx), cell_of(b.ly, g.oy, g.inv, g.my), cell_of(b.lz, g.oz, g.inv, g.mz))
                     : sentinel;
    if (count) {
      if (member) atomicAdd(count + keys[i], 1);
    } else {
      ids[i] = (uint32_t)i;
    }
    if (!member) ex = ey = ez = 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ex = fmax(ex, __shfl_xor_sync(0xffffffffu, ex, o));
    ey = fmax(ey, __shfl_xor_sync(0xffffffffu, ey, o));
    ez = fmax(ez, __shfl_xor_sync(0xffffffffu, ez, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(ext, (unsigned long long)__double_as_longlong(ex));
    atomicMax(ext + 1, (unsigned long long)__double_as_longlong(ey));
    atomicMax(ext + 2, (unsigned long long)__double_as_longlong(ez));
  }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* __restrict__ a, int64_t n, uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

struct JoinArgs {
  Boxes in;
  const int32_t* a_elems;   // surf_verts (VT) or edges (EE)
  const int32_t* b_elems;   // tris (VT) or edges (EE)
  int64_t na, nbins;        // A boxes; B boxes (one sorted (home cell, box) entry each)
  Grid g;
  const uint64_t* keys;     // sorted
  const uint32_t* ids;
  const Box* bbox;          // boxes of the B elements
  const double* ext;        // largest B extent per axis (device, 3)
  const int32_t* rev;       // dense grid: rev[c] = first entry of cell c (ids grouped by cell), or null (sorted keys)
  int64_t ncell;            // 2^key_bits
  unsigned long long* total;  // pairs found (device counter)
  int4* out;                // staging list of (pairs, 4) global vertex ids
  unsigned long long cap;   // its capacity: pairs beyond it are counted, not stored
};

constexpr int kHold = 4;

template <bool EE>
__device__ __forceinline__ int4 pair_row(const JoinArgs& a, int av0, int av1, int64_t j) {
  if (EE) return make_int4(av0, av1, a.b_elems[2 * j], a.b_elems[2 * j + 1]);
  return make_int4(av0, a.b_elems[3 * j], a.b_elems[3 * j + 1], a.b_elems[3 * j + 2]);
}

// The join.  EE = false: A = vertex boxes, B = triangles.  EE = true: A = B = inflated edge boxes.
// EIGHT lanes per A box.  (Round 1's form, one thread per (box, 3 x 3 probe slot) walking its own cell column, left
// lanes idle whenever a box spans fewer than 3 x 3 columns and whenever the columns of a warp's slots hold different
// numbers of boxes -- ncu, cloth stack: 13 of 32 lanes active on average -- and paid a binary search per slot plus a
// key test per visit.)  The group first finds, one lane per column, the sorted-bin range [t0, t1) of every column
// (cx, cy, z0..z1) of the span -- two reads of the dense cell table when the grid has at most 2^21 cells, two
// binary searches otherwise -- lays the ranges end to end (prefix sum over the group, table in shared memory) and
// then walks the FLATTENED list with stride 8: every lane has a candidate until the list runs out, and the lanes
// read consecutive (id) entries.  The reference's own overlap predicate on the same fp64 corners decides, so the
// pairs are the reference's; the list order is arbitrary, which no consumer depends on (it is a set).  A lane keeps
// up to kHold hit ids in registers; the warp reserves room for all of them with one atomicAdd when its lanes have
// finished (a lane whose registers fill up mid-walk flushes with the other lanes in the same state).
#ifndef B200IPC_JOIN_GROUP
#define B200IPC_JOIN_GROUP 8
#endif
constexpr int kJoinGroup = B200IPC_JOIN_GROUP;   // lanes per A box (8 / 16 / 32 measured: see DESIGN 4.4)

template <bool EE>
__global__ void __launch_bounds__(kBT) join_kernel(const __grid_constant__ JoinArgs a) {
  __shared__ int32_t tab_t0[kBT / kJoinGroup][kJoinGroup];     // first bin entry of the column
  __shared__ int32_t tab_end[kBT / kJoinGroup][kJoinGroup];    // end of the column in the flattened list
  const int lane = threadIdx.x & 31;
  const int gl = lane & (kJoinGroup - 1);
  const int grp = threadIdx.x / kJoinGroup;
  const unsigned gmask = kJoinGroup == 32 ? 0xffffffffu : (((1u << kJoinGroup) - 1u) << (lane & ~(kJoinGroup - 1)));
  const int64_t i = ((int64_t)blockIdx.x * kBT + threadIdx.x) / kJoinGroup;
  const bool live = i < a.na;
  int32_t n = 0;
  int h0 = 0, h1 = 0, h2 = 0, h3 = 0;
  int av0 = -1, av1 = -1;
  if (live) {   // uniform over the group
    const Box A = EE ? a.bbox[i] : make_box<0>(a.in, a.a_elems, i);
    constexpr double kWiden = 1.000000001;
    Span s;
    s.x0 = cell_of(A.lx - kWiden * a.ext[0], a.g.ox, a.g.inv, a.g.mx); s.x1 = cell_of(A.hx, a.g.ox, a.g.inv, a.g.mx);
    s.y0 = cell_of(A.ly - kWiden * a.ext[1], a.g.oy, a.g.inv, a.g.my); s.y1 = cell_of(A.hy, a.g.oy, a.g.inv, a.g.my);
    s.z0 = cell_of(A.lz - kWiden * a.ext[2], a.g.oz, a.g.inv, a.g.mz); s.z1 = cell_of(A.hz, a.g.oz, a.g.inv, a.g.mz);
    if (EE) {
      av0 = a.a_elems[2 * i];
      av1 = a.a_elems[2 * i + 1];
    } else {
      av0 = a.a_elems[i];
    }
    const int ncy = s.y1 - s.y0 + 1;
    const int ncol = (s.x1 - s.x0 + 1) * ncy;
    for (int c0 = 0; c0 < ncol; c0 += kJoinGroup) {   // a group's worth of columns at a time (a cloth box spans at most nine)
      const int c = c0 + gl;
      int32_t t0 = 0, len = 0;
      if (c < ncol) {
        const int cx = s.x0 + c / ncy, cy = s.y0 + c % ncy;
        // cells (cx, cy, z0..z1) are consecutive keys
        const uint64_t k0 = cell_key(a.g, cx, cy, s.z0), k1 = cell_key(a.g, cx, cy, s.z1);
        if (a.rev) {   // dense grid: two reads of the cell-start table
          t0 = a.rev[k0];
          len = a.rev[k1 + 1] - t0;
        } else {
          // the run's end is close to its start (runs are short, most columns of a sparse grid are empty):
          // gallop from t0 instead of a second full search
          const int64_t b = lower_bound_u64(a.keys, a.nbins, k0);
          int64_t lo = b, step = 1;
          while (lo + step <= a.nbins && a.keys[lo + step - 1] <= k1) {
            lo += step;
            step <<= 1;
          }
          int64_t hi = lo + step - 1 < a.nbins ? lo + step - 1 : a.nbins;   // keys[lo - 1] <= k1 (or lo == b), keys[hi] > k1 (or hi == nbins)
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (a.keys[mid] <= k1) lo = mid + 1;
            else hi = mid;
          }
          t0 = (int32_t)b;
          len = (int32_t)(lo - b);
        }
      }
      int32_t incl = len;
#pragma unroll
      for (int o = 1; o < kJoinGroup; o <<= 1) {
        const int32_t v = __shfl_up_sync(gmask, incl, o, kJoinGroup);
        if (gl >= o) incl += v;
      }
      const int32_t total = __shfl_sync(gmask, incl, kJoinGroup - 1, kJoinGroup);
      __syncwarp(gmask);                 // the previous batch's readers are done with the table
      tab_t0[grp][gl] = t0;
      tab_end[grp][gl] = incl;
      __syncwarp(gmask);
      int col = 0;
      int32_t cend = tab_end[grp][0], cbeg = 0, ct0 = tab_t0[grp][0];
      for (int32_t f = gl; f < total; f += kJoinGroup) {
        while (f >= cend) {              // this lane's cursor moves on to the column that holds f
          ++col;
          cbeg = cend;
          cend = tab_end[grp][col];
          ct0 = tab_t0[grp][col];
        }
        const int64_t j = a.ids[ct0 + (f - cbeg)];
        if (EE && j <= i) continue;  // each unordered pair once, lower edge index first (:310)
        const Box B = a.bbox[j];
        if (!(A.lx <= B.hx && B.lx <= A.hx && A.ly <= B.hy && B.ly <= A.hy && A.lz <= B.hz && B.lz <= A.hz)) continue;
        if (EE) {
          const int b0 = a.b_elems[2 * j], b1 = a.b_elems[2 * j + 1];
          if (av0 == b0 || av0 == b1 || av1 == b0 || av1 == b1) continue;
        } else {
          const int t0v = a.b_elems[3 * j], t1v = a.b_elems[3 * j + 1], t2v = a.b_elems[3 * j + 2];
          if (av0 == t0v || av0 == t1v || av0 == t2v) continue;
        }
        if (n == kHold) {  // registers full: flush with whichever lanes are here too
          const unsigned m = __activemask();
          const int lead = __ffs(m) - 1, rank = __popc(m & ((1u << lane) - 1));
          unsigned long long base = 0;
          if (lane == lead) base = atomicAdd(a.total, (unsigned long long)kHold * __popc(m));
          base = __shfl_sync(m, base, lead) + (unsigned long long)kHold * rank;
          if (base + kHold <= a.cap) {
            a.out[base] = pair_row<EE>(a, av0, av1, h0);
            a.out[base + 1] = pair_row<EE>(a, av0, av1, h1);
            a.out[base + 2] = pair_row<EE>(a, av0, av1, h2);
            a.out[base + 3] = pair_row<EE>(a, av0, av1, h3);
          }
          n = 0;
        }
        if (n == 0) h0 = (int)j;
        else if (n == 1) h1 = (int)j;
        else if (n == 2) h2 = (int)j;
        else h3 = (int)j;
        ++n;
      }
    }
  }
  __syncwarp();
  // the whole warp is here: exclusive prefix of the held counts, one reservation per warp
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int warp_total = __shfl_sync(0xffffffffu, incl, 31);
  if (warp_total == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(a.total, (unsigned long long)warp_total);
  base = __shfl_sync(0xffffffffu, base, 0) + (unsigned long long)(incl - n);
  if (base + n <= a.cap) {
    if (n > 0) a.out[base] = pair_row<EE>(a, av0, av1, h0);
    if (n > 1) a.out[base + 1] = pair_row<EE>(a, av0, av1, h1);
    if (n > 2) a.out[base + 2] = pair_row<EE>(a, av0, av1, h2);
    if (n > 3) a.out[base + 3] = pair_row<EE>(a, av0, av1, h3);
  }
}

}  // namespace b200ipc

// One sorted bin list: the B boxes of one kind (triangles / edges) and one size class on their own grid.
struct BinSet {
  b200ipc::BroadBuf<uint64_t> keys;
  b200ipc::BroadBuf<uint32_t> ids;
  b200ipc::BroadBuf<int32_t> rev;   // dense grids (<= 2^21 cells): rev[c] = first entry of cell c, rev[ncell] = members
  b200ipc::Grid grid{};
  int key_bits = 63;
  bool dense = false;
};

struct b200ipc_broad {
  b200ipc::BroadBuf<int4> stage_vt, stage_ee;            // candidate lists of the last query
  b200ipc::BroadBuf<unsigned long long> counters;        // [0] point-triangle, [1] edge-edge pairs found
  b200ipc::BroadBuf<uint64_t> keys_a;                    // unsorted keys (scratch)
  b200ipc::BroadBuf<uint32_t> ids_a;
  b200ipc::BroadBuf<int32_t> count;                      // per-cell member counts (dense grids; scratch)
  BinSet bins[2][2];                                     // [triangles, edges][small boxes, large boxes]
  b200ipc::BroadBuf<uint8_t> temp;
  b200ipc::BroadBuf<b200ipc::Box> box_t, box_e;
  b200ipc::BroadBuf<double> ext;   // [(kind * 2 + class) * 3 ..]: largest box extent per axis of every bin list
  // state between count and fill
  bool counted = false;
  int64_t nverts = 0, n_sv = 0, n_tri = 0, n_edge = 0, n_vt = 0, n_ee = 0;
  b200ipc::Boxes in{};
  const int32_t *surf_verts = nullptr, *tris = nullptr, *edges = nullptr;
  int32_t cells[3] = {1 << 21, 1 << 21, 1 << 21};   // b200ipc_broad_set_grid_cells
  double coarse_cell = 0.0;                          // b200ipc_broad_set_coarse_cell: 0 = one size class
};

using namespace b200ipc;

#define CK(expr)                            \
  do {                                      \
    cudaError_t _e = (expr);                \
    if (_e != cudaSuccess) return -(int)_e; \
  } while (0)
#define RC(expr)       \
  do {                 \
    int _r = (expr);   \
    if (_r) return _r; \
  } while (0)

static inline unsigned bblocks(int64_t n) { return (unsigned)((n + kBT - 1) / kBT); }

// Dense grids (at most 2^kDenseBits cells) are binned by COUNTING instead of sorting: home_cell_kernel counts the
// members of every cell while it writes their keys, one exclusive sum turns the counts into cell starts
// (start[c] = first entry of cell c, start[ncell] = members), and the scatter kernel drops every member's id into its
// cell with the count as a down-counter.  The order inside a cell is arbitrary -- the join's output is a set -- and
// the join reads a column's run as start[k0] .. start[k1 + 1]: no sort, no searches (a radix sort of the 19-bit
// keys of the cloth stack plus the table passes took 76 us per bin list, this takes ~30).
constexpr int kDenseBits = 21;
namespace b200ipc {
__global__ void __launch_bounds__(kBT) scatter_ids_kernel(int64_t n, uint64_t sentinel, const uint64_t* __restrict__ keys,
                                                          const int32_t* __restrict__ start, int32_t* __restrict__ count,
                                                          uint32_t* __restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * kBT + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = keys[i];
  if (key == sentinel) return;
  ids[start[key] + atomicSub(count + key, 1) - 1] = (uint32_t)i;
}
}  // namespace b200ipc

// Grid of `cell`-sized cells over the span the host announced in fine cells (b200ipc_broad_set_grid_cells).
static void make_grid(BinSet& b, const double* origin, double cell, const int32_t* fine_cells, double fine_cell) {
  int nbits[3], cells[3];
  for (int k = 0; k < 3; ++k) {
    const double want = ceil((double)fine_cells[k] * fine_cell / cell) + 1.0;
    cells[k] = want < 1.0 ? 1 : (want > (double)(1 << 21) ? (1 << 21) : (int)want);
    if (cell == fine_cell) cells[k] = fine_cells[k];
    nbits[k] = 1;
    while ((1 << nbits[k]) < cells[k]) ++nbits[k];
  }
  b.grid = Grid{origin[0], origin[1], origin[2], 1.0 / cell, cells[0] - 1, cells[1] - 1, cells[2] - 1, nbits[2], nbits[1] + nbits[2]};
  b.key_bits = nbits[0] + nbits[1] + nbits[2];
  b.dense = b.key_bits <= kDenseBits;
}

// File every B box of one size class under its home cell and reduce the class's largest extent per axis.  Dense
// grid: counting (cell starts in b.rev, ids grouped by cell).  Otherwise: sorted keys / ids, the other class's boxes
// behind every cell under the sentinel key.
static int bin_boxes(b200ipc_broad* h, const Box* box, int64_t n, BinSet& b, double lo_thr, double hi_thr, bool classes,
                     double* ext, cudaStream_t st) {
  CK(cudaMemsetAsync(ext, 0, 3 * sizeof(double), st));
  if (n == 0) return 0;
  const uint64_t sentinel = 1ull << b.key_bits;
  CK(h->keys_a.reserve(n)); CK(h->ids_a.reserve(n)); CK(b.ids.reserve(n));
  if (b.dense) {
    const int64_t ncell = 1ll << b.key_bits;
    CK(b.rev.reserve(ncell + 1)); CK(h->count.reserve(ncell + 1));
    CK(cudaMemsetAsync(h->count.ptr, 0, (ncell + 1) * sizeof(int32_t), st));
    home_cell_kernel<<<bblocks(n), kBT, 0, st>>>(box, n, b.grid, lo_thr, hi_thr, sentinel, h->keys_a.ptr, nullptr,
                                                 reinterpret_cast<unsigned long long*>(ext), h->count.ptr);
    RC(post_launch());
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, h->count.ptr, b.rev.ptr, (int)(ncell + 1), st));
    CK(h->temp.reserve(tb));
    CK(cub::DeviceScan::ExclusiveSum(h->temp.ptr, tb, h->count.ptr, b.rev.ptr, (int)(ncell + 1), st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    scatter_ids_kernel<<<bblocks(n), kBT, 0, st>>>(n, sentinel, h->keys_a.ptr, b.rev.ptr, h->count.ptr, b.ids.ptr);
    RC(post_launch());
    return 0;
  }
  CK(b.keys.reserve(n));
  home_cell_kernel<<<bblocks(n), kBT, 0, st>>>(box, n, b.grid, lo_thr, hi_thr, sentinel, h->keys_a.ptr, h->ids_a.ptr,
                                               reinterpret_cast<unsigned long long*>(ext), nullptr);
  RC(post_launch());
  const int end_bit = b.key_bits + (classes ? 1 : 0);   // the sentinel needs one more bit
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, h->keys_a.ptr, b.keys.ptr, h->ids_a.ptr, b.ids.ptr, (int)n, 0, end_bit, st));
  CK(h->temp.reserve(tb));
  CK(cub::DeviceRadixSort::SortPairs(h->temp.ptr, tb, h->keys_a.ptr, b.keys.ptr, h->ids_a.ptr, b.ids.ptr, (int)n, 0, end_bit, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return 0;
}

extern "C" int b200ipc_broad_create(b200ipc_broad** out) {
  if (!out) return B200IPC_EINVAL;
  *out = new (std::nothrow) b200ipc_broad();
  return *out ? 0 : B200IPC_EINVAL;
}

extern "C" int b200ipc_broad_destroy(b200ipc_broad* h) {
  if (!h) return 0;
  h->stage_vt.release(); h->stage_ee.release(); h->counters.release();
  h->keys_a.release(); h->ids_a.release(); h->count.release();
  for (int k = 0; k < 2; ++k)
    for (int c = 0; c < 2; ++c) {
      h->bins[k][c].keys.release(); h->bins[k][c].ids.release(); h->bins[k][c].rev.release();
    }
  h->temp.release(); h->box_t.release(); h->box_e.release(); h->ext.release();
  delete h;
  return 0;
}

extern "C" int b200ipc_broad_set_grid_cells(b200ipc_broad* h, int32_t nx, int32_t ny, int32_t nz) {
  if (!h) return B200IPC_EINVAL;
  const int32_t want[3] = {nx, ny, nz};
  for (int k = 0; k < 3; ++k) h->cells[k] = want[k] <= 0 ? (1 << 21) : (want[k] > (1 << 21) ? (1 << 21) : want[k]);
  return 0;
}

extern "C" int b200ipc_broad_set_coarse_cell(b200ipc_broad* h, double coarse_cell) {
  if (!h || !(coarse_cell >= 0.0)) return B200IPC_EINVAL;
  h->coarse_cell = coarse_cell;
  return 0;
}

static int broad_count(b200ipc_broad* h, int64_t nverts, const Boxes& in, int64_t n_sv, const int32_t* surf_verts,
                       int64_t n_tri, const int32_t* tris, int64_t n_edge, const int32_t* edges, double cell,
                       const double* origin, int64_t* n_vt, int64_t* n_ee, void* stream) {
  if (!h || nverts <= 0 || !in.pos || n_sv < 0 || n_tri < 0 || n_edge < 0 || !origin || !n_vt || !n_ee)
    return B200IPC_EINVAL;
  if ((n_sv && !surf_verts) || (n_tri && !tris) || (n_edge && !edges)) return B200IPC_EINVAL;
  if (!(cell > 0.0)) return B200IPC_EINVAL;
  if (n_sv >= (1ll << 27) || n_tri >= (1ll << 31) || n_edge >= (1ll << 27)) return B200IPC_EINVAL;  // (box, lane) thread ids stay below 2^31
  cudaStream_t st = (cudaStream_t)stream;
  h->counted = false;
  h->nverts = nverts; h->in = in; h->n_sv = n_sv; h->surf_verts = surf_verts; h->n_tri = n_tri; h->tris = tris;
  h->n_edge = n_edge; h->edges = edges;
  h->n_vt = h->n_ee = 0;
  CK(h->ext.reserve(12));

  // Size classes.  One class: every B box on the fine grid, as the reference's scenes of uniform resolution want.
  // Two classes (the host saw edges much longer than a cell, b200ipc_broad_set_coarse_cell): boxes of up to two
  // cells stay on the fine grid, the few large ones go to a coarse grid of their own -- the probe range of a join is
  // set by the LARGEST box of its bin list, and a handful of long collider edges would otherwise make every cloth
  // vertex probe dozens of empty columns.  Each A box is joined with both lists; a pair is found in the list its B
  // box lives in, once.
  const bool classes = h->coarse_cell > 2.0 * cell;
  const int ncls = classes ? 2 : 1;
  const double split = 2.0 * cell;
  for (int k = 0; k < 2; ++k) {
    make_grid(h->bins[k][0], origin, cell, h->cells, cell);
    if (classes) make_grid(h->bins[k][1], origin, h->coarse_cell, h->cells, cell);
  }

  // boxes and bins of both joins first, then the passes, then ONE synchronisation for both counts
  const bool do_vt = n_sv && n_tri, do_ee = n_edge > 1;
  CK(h->counters.reserve(2));
  const double inf = HUGE_VAL;
  if (do_vt) {
    CK(h->box_t.reserve(n_tri));
    make_boxes_kernel<1><<<bblocks(n_tri), kBT, 0, st>>>(in, tris, n_tri, h->box_t.ptr);
    RC(post_launch());
    for (int c = 0; c < ncls; ++c)
      RC(bin_boxes(h, h->box_t.ptr, n_tri, h->bins[0][c], c == 0 ? -1.0 : split, c == 0 && classes ? split : inf, classes,
                   h->ext.ptr + 3 * c, st));
  }
  if (do_ee) {
    CK(h->box_e.reserve(n_edge));
    make_boxes_kernel<2><<<bblocks(n_edge), kBT, 0, st>>>(in, edges, n_edge, h->box_e.ptr);
    RC(post_launch());
    for (int c = 0; c < ncls; ++c)
      RC(bin_boxes(h, h->box_e.ptr, n_edge, h->bins[1][c], c == 0 ? -1.0 : split, c == 0 && classes ? split : inf, classes,
                   h->ext.ptr + 6 + 3 * c, st));
  }
  bool run_vt = do_vt, run_ee = do_ee;
  for (int attempt = 0; attempt < 2 && (run_vt || run_ee); ++attempt) {
    if (run_vt) {
      CK(cudaMemsetAsync(h->counters.ptr, 0, sizeof(unsigned long long), st));
      for (int c = 0; c < ncls; ++c) {
        const BinSet& b = h->bins[0][c];
        JoinArgs a{in, surf_verts, tris, n_sv, n_tri, b.grid, b.keys.ptr, b.ids.ptr, h->box_t.ptr, h->ext.ptr + 3 * c,
                   b.dense ? b.rev.ptr : nullptr, 1ll << b.key_bits, h->counters.ptr, h->stage_vt.ptr,
                   (unsigned long long)h->stage_vt.cap};
        join_kernel<false><<<bblocks(n_sv * kJoinGroup), kBT, 0, st>>>(a);
        RC(post_launch());
      }
    }
    if (run_ee) {
      CK(cudaMemsetAsync(h->counters.ptr + 1, 0, sizeof(unsigned long long), st));
      for (int c = 0; c < ncls; ++c) {
        const BinSet& b = h->bins[1][c];
        JoinArgs a{in, edges, edges, n_edge, n_edge, b.grid, b.keys.ptr, b.ids.ptr, h->box_e.ptr, h->ext.ptr + 6 + 3 * c,
                   b.dense ? b.rev.ptr : nullptr, 1ll << b.key_bits, h->counters.ptr + 1, h->stage_ee.ptr,
                   (unsigned long long)h->stage_ee.cap};
        join_kernel<true><<<bblocks(n_edge * kJoinGroup), kBT, 0, st>>>(a);
        RC(post_launch());
      }
    }
    unsigned long long found[2] = {0, 0};
    CK(cudaMemcpyAsync(found, h->counters.ptr, sizeof(found), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (do_vt) h->n_vt = (int64_t)found[0];
    if (do_ee) h->n_ee = (int64_t)found[1];
    // a list that was too small has only been counted: regrow it (with head-room) and repeat that pass
    run_vt = do_vt && found[0] > h->stage_vt.cap;
    run_ee = do_ee && found[1] > h->stage_ee.cap;
    if (run_vt) CK(h->stage_vt.reserve(found[0] + found[0] / 4));
    if (run_ee) CK(h->stage_ee.reserve(found[1] + found[1] / 4));
  }
  if (run_vt || run_ee) return B200IPC_ESTATE;  // the same pass cannot find more pairs the second time
  *n_vt = h->n_vt;
  *n_ee = h->n_ee;
  h->counted = true;
  return 0;
}

extern "C" int b200ipc_broad_phase_count(b200ipc_broad* h, int64_t nverts, const double* positions, int64_t n_sv,
                                         const int32_t* surf_verts, int64_t n_tri, const int32_t* tris, int64_t n_edge,
                                         const int32_t* edges, double d_hat, double cell, const double* origin,
                                         int64_t* n_vt, int64_t* n_ee, void* stream) {
  if (!(d_hat > 0.0)) return B200IPC_EINVAL;
  const Boxes in{positions, nullptr, {d_hat, 0.0, d_hat * 0.5}};
  return broad_count(h, nverts, in, n_sv, surf_verts, n_tri, tris, n_edge, edges, cell, origin, n_vt, n_ee, stream);
}

extern "C" int b200ipc_sweep_candidates_count(b200ipc_broad* h, int64_t nverts, const double* positions,
                                              const double* directions, int64_t n_sv, const int32_t* surf_verts,
                                              int64_t n_tri, const int32_t* tris, int64_t n_edge, const int32_t* edges,
                                              double margin, double cell, const double* origin, int64_t* n_vt,
                                              int64_t* n_ee, void* stream) {
  if (!directions || !(margin >= 0.0)) return B200IPC_EINVAL;
  const Boxes in{positions, directions, {margin, margin, margin}};
  return broad_count(h, nverts, in, n_sv, surf_verts, n_tri, tris, n_edge, edges, cell, origin, n_vt, n_ee, stream);
}

extern "C" int b200ipc_broad_phase_fill(b200ipc_broad* h, int32_t* vt, int32_t* ee, void* stream) {
  if (!h || !h->counted) return B200IPC_ESTATE;
  if ((h->n_vt && !vt) || (h->n_ee && !ee)) return B200IPC_EINVAL;
  if (((uintptr_t)vt | (uintptr_t)ee) & 15) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (h->n_vt) CK(cudaMemcpyAsync(vt, h->stage_vt.ptr, (size_t)h->n_vt * sizeof(int4), cudaMemcpyDeviceToDevice, st));
  if (h->n_ee) CK(cudaMemcpyAsync(ee, h->stage_ee.ptr, (size_t)h->n_ee * sizeof(int4), cudaMemcpyDeviceToDevice, st));
  return 0;
}
