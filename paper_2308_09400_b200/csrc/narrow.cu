// Narrow phase: candidate queries -> the reference's ordered contact list (find_contact_pairs,
// proximity.py:284-358), entirely on the device.
//
//   1. one thread per query: pt/ee classification (bit-exact with kernels/_core.pyx), keep
//      d2 < d_hat*d_hat, reduce to the active branch (_PT_LOCAL/_EE_LOCAL, proximity.py:100-119),
//      promote edge pairs with c < eps_x to the parallel kinds (:331-343), eps_x from rest lengths
//      (edge_parallel_eps, :251-259);
//   2. stream compaction of the kept queries (CUB select);
//   3. the reference's order (ContactStencil.sort_key, :82-83: kind.value, verts, origin): LSD radix sort
//      by (kind, verts) packed into two 64-bit words, then the few runs of equal (kind, verts) -- one
//      stencil reached from several queries -- are ordered by origin in place;
//   4. gather into the SoA stencil table.
// The broad phase (any duplicate-free superset of the near queries, incident pairs removed) is the
// caller's job; each query yields at most one stencil, so the reference's dedupe-by-origin is the
// identity on duplicate-free input.
#include <cub/cub.cuh>

#include "geom.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kNT = 256;

// region code -> reduced kind / local selection (padded with 0) / packed sub byte
__constant__ uint8_t c_pt_kind[7] = {B200IPC_PT, B200IPC_PP, B200IPC_PP, B200IPC_PP, B200IPC_PE, B200IPC_PE, B200IPC_PE};
__constant__ uint8_t c_pt_sel[7][4] = {{0, 1, 2, 3}, {0, 1, 0, 0}, {0, 2, 0, 0}, {0, 3, 0, 0},
                                       {0, 1, 2, 0}, {0, 2, 3, 0}, {0, 3, 1, 0}};
__constant__ uint8_t c_ee_kind[9] = {B200IPC_PP, B200IPC_PP, B200IPC_PE, B200IPC_PP, B200IPC_PP,
                                     B200IPC_PE, B200IPC_PE, B200IPC_PE, B200IPC_EE};
__constant__ uint8_t c_ee_sel[9][4] = {{0, 2, 0, 0}, {0, 3, 0, 0}, {0, 2, 3, 0}, {1, 2, 0, 0}, {1, 3, 0, 0},
                                       {1, 2, 3, 0}, {2, 0, 1, 0}, {3, 0, 1, 0}, {0, 1, 2, 3}};
__constant__ uint8_t c_kind_size[7] = {4, 4, 3, 4, 2, 4, 4};

struct NarrowArgs {
  const double* positions;
  const double* rest;
  int64_t n_vt, n_ee;
  const int32_t* vt;
  const int32_t* ee;
  double d_hat_sq;
  int32_t promote;
  // per-query scratch
  uint8_t* keep;
  uint8_t* kind;
  int4* verts;
  uint8_t* sub;
  double* eps;
};

__global__ void __launch_bounds__(kNT) narrow_classify_kernel(const NarrowArgs a) {
  const int64_t q = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (q >= a.n_vt + a.n_ee) return;
  const bool is_vt = q < a.n_vt;
  const int4 id = is_vt ? reinterpret_cast<const int4*>(a.vt)[q] : reinterpret_cast<const int4*>(a.ee)[q - a.n_vt];
  const int g[4] = {id.x, id.y, id.z, id.w};
  const V3 x0 = load3(a.positions, id.x), x1 = load3(a.positions, id.y), x2 = load3(a.positions, id.z),
           x3 = load3(a.positions, id.w);
  V3 gr[4];
  double d2, w0, w1;
  int kind, sel[4];
  uint8_t sub = 0;
  double eps = 0.0;
  bool promoted = false;
  if (is_vt) {
    const int code = pt_one(x0, x1, x2, x3, d2, gr, w0, w1);
    kind = c_pt_kind[code];
#pragma unroll
    for (int k = 0; k < 4; ++k) sel[k] = c_pt_sel[code][k];
  } else {
    const int code = ee_one(x0, x1, x2, x3, d2, gr, w0, w1);
    kind = c_ee_kind[code];
#pragma unroll
    for (int k = 0; k < 4; ++k) sel[k] = c_ee_sel[code][k];
    if (d2 < a.d_hat_sq) {
      const double c = cross_sq_one(x0, x1, x2, x3, gr);
      const V3 la = load3(a.rest, id.y) - load3(a.rest, id.x);
      const V3 lb = load3(a.rest, id.w) - load3(a.rest, id.z);
      eps = 1e-3 * dot3_blas(la, la) * dot3_blas(lb, lb);
      promoted = a.promote && c < eps;
    }
  }
  const bool near = d2 < a.d_hat_sq;
  a.keep[q] = near ? 1 : 0;
  if (!near) return;
  int4 v;
  if (promoted) {
    sub = (uint8_t)(sel[0] | (sel[1] << 2) | (sel[2] << 4) | (sel[3] << 6));
    const int len = c_kind_size[kind];  // entries of sub that are meaningful (4 / 3 / 2)
    if (len < 4) sub &= (uint8_t)((1u << (2 * len)) - 1u);
    kind += 1;  // EE->EEP, PE->PEP, PP->PPP
    v = id;
  } else {
    eps = 0.0;
    const int s = c_kind_size[kind];
    v.x = g[sel[0]];
    v.y = g[sel[1]];
    v.z = s >= 3 ? g[sel[2]] : -1;
    v.w = s >= 4 ? g[sel[3]] : -1;
  }
  a.kind[q] = (uint8_t)kind;
  a.verts[q] = v;
  a.sub[q] = sub;
  a.eps[q] = eps;
}

__global__ void __launch_bounds__(kNT) iota_kernel(int64_t n, uint32_t* out) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (i < n) out[i] = (uint32_t)i;
}

struct KeyArgs {
  int64_t n;           // kept queries
  int64_t n_vt;
  int bits;            // bits per (vertex id + 1)
  const uint32_t* idx; // current order (query ids)
  const uint8_t* kind;
  const int4* verts;
  const int32_t* vt;
  const int32_t* ee;
  int word;            // 0: (o2,o3)  1: (otype,o0,o1)  2: low word of (kind,v0..v3)  3: its high word
  int lowbits;         // width of the low word (words 2 / 3)
  uint64_t* keys;
};

__global__ void __launch_bounds__(kNT) narrow_keys_kernel(const KeyArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (i >= a.n) return;
  const int64_t q = a.idx[i];
  const bool is_vt = q < a.n_vt;
  uint64_t key;
  if (a.word <= 1) {
    const int4 o = is_vt ? reinterpret_cast<const int4*>(a.vt)[q] : reinterpret_cast<const int4*>(a.ee)[q - a.n_vt];
    if (a.word == 0) key = ((uint64_t)(uint32_t)o.z << a.bits) | (uint64_t)(uint32_t)o.w;
    else key = ((uint64_t)(is_vt ? 2 : 1) << (2 * a.bits)) | ((uint64_t)(uint32_t)o.x << a.bits) | (uint64_t)(uint32_t)o.y;
  } else {
    const int4 v = a.verts[q];
    // (kind, v0, v1, v2, v3) is one 4 bits + 4 x `bits` wide number, sorted LSD in two calls: the low word takes
    // the largest multiple of 8 bits (a radix pass sorts 8) below 2 x bits, the rest of (v2, v3) rides at the bottom
    // of the high word -- 72 bits at 17 bits per vertex are then 4 + 5 passes instead of 5 + 5
    const uint64_t lo = ((uint64_t)(uint32_t)(v.z + 1) << a.bits) | (uint64_t)(uint32_t)(v.w + 1);
    if (a.word == 2) key = lo & ((1ull << a.lowbits) - 1ull);
    else key = ((((uint64_t)a.kind[q] << (2 * a.bits)) | ((uint64_t)(uint32_t)(v.x + 1) << a.bits) | (uint64_t)(uint32_t)(v.y + 1))
                << (2 * a.bits - a.lowbits)) | (lo >> a.lowbits);
  }
  a.keys[i] = key;
}

// Ties of the (kind, vertices) sort: the same stencil reached from several queries (a point-point pair
// is the closest feature of every incident edge pair, ...).  The reference orders those by origin
// (type, then the query's vertex ids); runs are a handful of entries, so the head of each run orders
// it in place by insertion -- instead of two more full radix sorts over every kept query.
struct TieArgs {
  int64_t n, n_vt;
  uint32_t* idx;       // order after the (kind, vertices) sort; runs of equal keys are reordered in place
  const uint8_t* kind;
  const int4* verts;
  const int32_t* vt;
  const int32_t* ee;
};

__device__ __forceinline__ bool same_stencil(const TieArgs& a, uint32_t p, uint32_t q) {
  const int4 u = a.verts[p], v = a.verts[q];
  return a.kind[p] == a.kind[q] && u.x == v.x && u.y == v.y && u.z == v.z && u.w == v.w;
}

__device__ __forceinline__ bool origin_less(const TieArgs& a, uint32_t p, uint32_t q) {
  const bool pv = p < a.n_vt, qv = q < a.n_vt;
  if (pv != qv) return qv;  // origin type: edge-edge (1) before vertex-triangle (2)
  const int4 u = pv ? reinterpret_cast<const int4*>(a.vt)[p] : reinterpret_cast<const int4*>(a.ee)[p - a.n_vt];
  const int4 v = qv ? reinterpret_cast<const int4*>(a.vt)[q] : reinterpret_cast<const int4*>(a.ee)[q - a.n_vt];
  if (u.x != v.x) return (uint32_t)u.x < (uint32_t)v.x;
  if (u.y != v.y) return (uint32_t)u.y < (uint32_t)v.y;
  if (u.z != v.z) return (uint32_t)u.z < (uint32_t)v.z;
  return (uint32_t)u.w < (uint32_t)v.w;
}

__global__ void __launch_bounds__(kNT) narrow_ties_kernel(const TieArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (i >= a.n || i + 1 >= a.n) return;
  const uint32_t q = a.idx[i];
  if (i > 0 && same_stencil(a, a.idx[i - 1], q)) return;   // not the head of its run
  if (!same_stencil(a, q, a.idx[i + 1])) return;           // a run of one
  int64_t e = i + 2;
  while (e < a.n && same_stencil(a, q, a.idx[e])) ++e;
  for (int64_t k = i + 1; k < e; ++k) {                    // insertion sort of idx[i, e) by origin
    const uint32_t cur = a.idx[k];
    int64_t m = k;
    while (m > i && origin_less(a, cur, a.idx[m - 1])) {
      a.idx[m] = a.idx[m - 1];
      --m;
    }
    a.idx[m] = cur;
  }
}

struct GatherArgs {
  int64_t n, n_vt;
  const uint32_t* idx;
  const uint8_t* kind_in;
  const int4* verts_in;
  const uint8_t* sub_in;
  const double* eps_in;
  const int32_t* vt;
  const int32_t* ee;
  uint8_t* kind;
  int4* verts;
  uint8_t* sub;
  double* eps;
  uint8_t* otype;
  int4* origin;
  unsigned long long* hist;  // 7 counters
};

__global__ void __launch_bounds__(kNT) narrow_gather_kernel(const GatherArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  __shared__ unsigned int sh[B200IPC_NKINDS];
  if (threadIdx.x < B200IPC_NKINDS) sh[threadIdx.x] = 0;
  __syncthreads();
  if (i < a.n) {
    const int64_t q = a.idx[i];
    const bool is_vt = q < a.n_vt;
    const uint8_t k = a.kind_in[q];
    a.kind[i] = k;
    a.verts[i] = a.verts_in[q];
    a.sub[i] = a.sub_in[q];
    a.eps[i] = a.eps_in[q];
    if (a.otype) a.otype[i] = is_vt ? 2 : 1;
    if (a.origin)
      a.origin[i] = is_vt ? reinterpret_cast<const int4*>(a.vt)[q] : reinterpret_cast<const int4*>(a.ee)[q - a.n_vt];
    atomicAdd(&sh[k], 1u);
  }
  __syncthreads();
  if (threadIdx.x < B200IPC_NKINDS && sh[threadIdx.x]) atomicAdd(&a.hist[threadIdx.x], (unsigned long long)sh[threadIdx.x]);
}

static inline unsigned nblocks(int64_t n) { return (unsigned)((n + kNT - 1) / kNT); }

template <typename T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t stream) {
    st = stream;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), (n ? n : 1) * sizeof(T), stream);
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};

}  // namespace b200ipc

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

extern "C" int b200ipc_narrow_phase(int64_t nverts, const double* positions, const double* rest_positions,
                                    int64_t n_vt, const int32_t* vt, int64_t n_ee, const int32_t* ee,
                                    double d_hat_sq, int32_t promote_parallel, uint8_t* kind, int32_t* verts,
                                    uint8_t* sub, double* eps_x, uint8_t* origin_type, int32_t* origin,
                                    int64_t* n_out, int64_t* kind_off, void* stream) {
  if (nverts <= 0 || n_vt < 0 || n_ee < 0 || !positions || !n_out || !kind_off) return B200IPC_EINVAL;
  if ((n_vt && !vt) || (n_ee && (!ee || !rest_positions))) return B200IPC_EINVAL;
  if (((uintptr_t)vt | (uintptr_t)ee | (uintptr_t)verts | (uintptr_t)origin) & 15) return B200IPC_EINVAL;
  const int64_t nq = n_vt + n_ee;
  for (int k = 0; k <= B200IPC_NKINDS; ++k) kind_off[k] = 0;
  *n_out = 0;
  if (nq == 0) return 0;
  if (nq >= (1ll << 31) || nverts >= (1ll << 30)) return B200IPC_EINVAL;
  if (!kind || !verts || !sub || !eps_x) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  CK(keep_pool_memory());

  Scratch<uint8_t> keep, kq, sq, temp;
  Scratch<int4> vq;
  Scratch<double> eq;
  Scratch<uint32_t> iota, idx_a, idx_b;
  Scratch<uint64_t> key_a, key_b;
  Scratch<unsigned long long> counters;  // [0] = n_kept, [1..7] = histogram
  CK(keep.alloc(nq, st)); CK(kq.alloc(nq, st)); CK(sq.alloc(nq, st)); CK(vq.alloc(nq, st)); CK(eq.alloc(nq, st));
  CK(iota.alloc(nq, st)); CK(idx_a.alloc(nq, st)); CK(counters.alloc(8, st));
  CK(cudaMemsetAsync(counters.p, 0, 8 * sizeof(unsigned long long), st));

  NarrowArgs na{positions, rest_positions, n_vt, n_ee, vt, ee, d_hat_sq, promote_parallel,
                keep.p, kq.p, vq.p, sq.p, eq.p};
  narrow_classify_kernel<<<nblocks(nq), kNT, 0, st>>>(na);
  RC(post_launch());
  iota_kernel<<<nblocks(nq), kNT, 0, st>>>(nq, iota.p);
  RC(post_launch());

  // compaction of kept query ids (order preserved)
  size_t tb = 0;
  int* d_nsel = reinterpret_cast<int*>(counters.p);
  CK(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, keep.p, idx_a.p, d_nsel, (int)nq, st));
  CK(temp.alloc(tb, st));
  CK(cub::DeviceSelect::Flagged(temp.p, tb, iota.p, keep.p, idx_a.p, d_nsel, (int)nq, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  int nsel = 0;
  CK(cudaMemcpyAsync(&nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaMemsetAsync(counters.p, 0, sizeof(unsigned long long), st));
  const int64_t n = nsel;
  *n_out = n;
  if (n == 0) return 0;

  // LSD sort by (kind, vertices), least significant word first; ties are ordered by origin afterwards
  int bits = 1;
  while (((int64_t)1 << bits) < nverts + 1) ++bits;
  CK(idx_b.alloc(n, st)); CK(key_a.alloc(n, st)); CK(key_b.alloc(n, st));
  size_t ts = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, ts, key_a.p, key_b.p, idx_a.p, idx_b.p, (int)n, 0, 64, st));
  Scratch<uint8_t> temp2;
  CK(temp2.alloc(ts, st));
  uint32_t* cur = idx_a.p;
  uint32_t* nxt = idx_b.p;
  int lowbits = (2 * bits) / 8 * 8;
  if (lowbits == 0 || 4 * bits + 4 - lowbits > 64) lowbits = 2 * bits;   // the high word must fit 64 bits
  for (int word = 2; word < 4; ++word) {
    KeyArgs ka{n, n_vt, bits, cur, kq.p, vq.p, vt, ee, word, lowbits, key_a.p};
    narrow_keys_kernel<<<nblocks(n), kNT, 0, st>>>(ka);
    RC(post_launch());
    const int end_bit = word == 2 ? lowbits : 2 * bits + 4 + (2 * bits - lowbits);
    CK(cub::DeviceRadixSort::SortPairs(temp2.p, ts, key_a.p, key_b.p, cur, nxt, (int)n, 0, end_bit, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
  TieArgs ta{n, n_vt, cur, kq.p, vq.p, vt, ee};
  narrow_ties_kernel<<<nblocks(n), kNT, 0, st>>>(ta);
  RC(post_launch());

  GatherArgs ga{n, n_vt, cur, kq.p, vq.p, sq.p, eq.p, vt, ee, kind, reinterpret_cast<int4*>(verts), sub, eps_x,
                origin_type, reinterpret_cast<int4*>(origin), counters.p + 1};
  narrow_gather_kernel<<<nblocks(n), kNT, 0, st>>>(ga);
  RC(post_launch());
  unsigned long long hist[8];
  CK(cudaMemcpyAsync(hist, counters.p, sizeof(hist), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  kind_off[0] = 0;
  for (int k = 0; k < B200IPC_NKINDS; ++k) kind_off[k + 1] = kind_off[k] + (int64_t)hist[k + 1];
  return kind_off[B200IPC_NKINDS] == n ? 0 : B200IPC_ESTATE;
}
