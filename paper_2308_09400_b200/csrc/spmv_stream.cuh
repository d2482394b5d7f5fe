// Streamed BSR (3x3, fp64) row products: the matrix is pulled through shared memory by the bulk
// async-copy engine (TMA, cp.async.bulk + mbarrier) while the warps of the CTA reduce rows that
// already arrived.
//
// Why: the rows of a contact matrix are short (~17 blocks, 1.2 KB), so a warp-per-row kernel that
// loads straight from global memory has one or two dependent DRAM round trips per row and too
// few bytes in flight to fill HBM3e (measured 2.4 TB/s).  Here a persistent CTA owns chunks of R
// consecutive rows; the values and column indices of a chunk are ONE contiguous span each, fetched
// by two bulk copies issued by a single thread into a ring of kStages shared-memory stages.  The
// copy engine keeps ~130 KB per SM in flight without any register or issue-slot cost, and the row
// reductions read shared memory (30-cycle latency).
//
// Roles inside the CTA (21 warps): two consumer groups of 10 warps and one producer warp.  Group g
// reduces the chunks with sequence number = g (mod 2), so two chunks are being reduced while the next
// two are in flight.  A consumer warp reduces THREE rows per trip with nine lanes per row: lane
// (r, i, j) walks row r's blocks and accumulates entry (i, j) times x_j -- one shared-memory column
// index, one x gather, one shared-memory value and one FMA per block per lane, no index arithmetic --
// and two shuffles finish the three rows.  (One row per warp with cross-lane block partitioning costs
// 3x the instructions per block plus a 5-shuffle tail; this kernel was issue-bound that way.)
// The producer warp waits for a free stage (empty barrier), stores the chunk's row pointers (fetched
// while the previous stage drained) next to it and lane 0 issues the two bulk copies.  Everything is
// coupled through full/empty mbarriers only.  (Tried and dropped: row pointers by a third bulk copy
// with the block spans fetched 32 chunks ahead -- 2.7 us slower per product; L1 prefetch of the
// gathered x rows from the producer warp -- 3.8 us slower.)  (Prefetching the x rows a landed chunk will gather into L1 from the producer warp
// was measured slower -- 28.8 vs 25.0 us -- and was removed.)
//
// A chunk whose span does not fit a stage (pathologically long rows) is reduced straight from
// global memory by the same row code.  No atomics; fixed summation order: bitwise reproducible.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b200ipc {

#ifndef B200IPC_STREAM_GROUPS   // tuning overrides (scripts/build_variants.py)
#define B200IPC_STREAM_GROUPS 2
#endif
#ifndef B200IPC_STREAM_GROUP_WARPS
#define B200IPC_STREAM_GROUP_WARPS 10
#endif
#ifndef B200IPC_STREAM_STAGES
#define B200IPC_STREAM_STAGES 4
#endif
#ifndef B200IPC_STREAM_STAGE_BLOCKS
#define B200IPC_STREAM_STAGE_BLOCKS 660
#endif
#ifndef B200IPC_STREAM_CONTIG
#define B200IPC_STREAM_CONTIG 0
#endif
constexpr int kStreamGroups = B200IPC_STREAM_GROUPS;          // consumer groups (chunks reduced concurrently)
constexpr int kGroupWarps = B200IPC_STREAM_GROUP_WARPS;
constexpr int kConsumerWarps = kStreamGroups * kGroupWarps;
constexpr int kStreamThreads = 32 * (kConsumerWarps + 1);  // + producer warp
constexpr int kMaxChunkRows = 120;        // row pointers of a chunk live in the stage header
constexpr int kStreamStages = B200IPC_STREAM_STAGES;
constexpr int kStageBlocks = B200IPC_STREAM_STAGE_BLOCKS;         // 3x3 blocks per stage (plus alignment slack below)
// byte layout of one stage: values (16-byte aligned superset of the span), column indices, row pointers
constexpr int kStageValBytes = (kStageBlocks * 72 + 32 + 15) / 16 * 16;
constexpr int kStageColBytes = (kStageBlocks * 4 + 32 + 15) / 16 * 16;
constexpr int kStageRowBytes = (kMaxChunkRows + 4 + 3) / 4 * 16;
constexpr int kStageBytes = kStageValBytes + kStageColBytes + kStageRowBytes;
constexpr int kStreamSmemBytes = kStreamStages * kStageBytes + 16 * kStreamStages;  // + full/empty mbarriers

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// global -> shared bulk copy (1D TMA); dst, src and bytes are multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// global -> shared bulk copy with an L2 eviction-priority hint (pre-encoded createpolicy values)
constexpr uint64_t kL2EvictFirst = 0x12F0000000000000ull, kL2EvictLast = 0x14F0000000000000ull;
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

struct StreamMatrix {
  int64_t n;            // block rows
  int64_t nnzb;
  int32_t rows_per_chunk;  // <= kMaxChunkRows
  int32_t pad_;
  const int32_t* rowptr;   // 16-byte aligned
  const int32_t* colidx;   // 16-byte aligned
  const double* vals;      // 16-byte aligned
  unsigned long long* dbg; // timing builds only: per-CTA [full-wait, compute, empty-wait] clock sums
  // L2 residency across the products of a persistent solver loop: chunks of rows below pin_rows are fetched
  // with evict-last priority (they stay in the 126 MB L2 from one iteration to the next), the others with
  // evict-first (they stream through without displacing them).  0 = no hints (single products).
  int64_t pin_rows;
};

// Per-CTA streaming state; lives in registers (identical in every thread) and survives across the
// products of the persistent PCG kernel, so the ring is refilled for the NEXT product while the
// vector updates of the current iteration run.  Sequence numbers count this CTA's chunk loads,
// cyclically over its chunks: sequence q -> chunk blockIdx.x + (q mod nmine) * gridDim.x.
struct StreamState {
  uint32_t issued = 0;
  uint32_t consumed = 0;
  int32_t nmine = 0;       // chunks owned by this CTA
  int64_t first = 0;       // its first chunk (contiguous assignment)
};

struct StreamSmem {
  unsigned char* base;
  uint64_t* full;          // kStreamStages barriers, completed by the copy engine
  uint64_t* empty;         // kStreamStages barriers, kGroupWarps arrivals each
  __device__ __forceinline__ double* vals(int s) const { return reinterpret_cast<double*>(base + (size_t)s * kStageBytes); }
  __device__ __forceinline__ int32_t* cols(int s) const {
    return reinterpret_cast<int32_t*>(base + (size_t)s * kStageBytes + kStageValBytes);
  }
  // rows(s)[0] = number of rows, rows(s)[1] = first block b0 of the chunk,
  // rows(s)[2 + r] = rowptr[r0 + r] - b0 for r = 0..nrows (the last one = blocks of the chunk; a value
  // above kStageBlocks marks a chunk that was not staged)
  __device__ __forceinline__ int32_t* rows(int s) const {
    return reinterpret_cast<int32_t*>(base + (size_t)s * kStageBytes + kStageValBytes + kStageColBytes);
  }
};

__device__ __forceinline__ StreamSmem stream_smem(unsigned char* dyn) {
  StreamSmem s;
  s.base = dyn;
  s.full = reinterpret_cast<uint64_t*>(dyn + (size_t)kStreamStages * kStageBytes);
  s.empty = s.full + kStreamStages;
  return s;
}

__device__ __forceinline__ void stream_init(const StreamMatrix& m, const StreamSmem& sm, StreamState& st) {
  const int64_t nchunks = (m.n + m.rows_per_chunk - 1) / m.rows_per_chunk;
#if B200IPC_STREAM_CONTIG
  const int64_t per = (nchunks + (int64_t)gridDim.x - 1) / (int64_t)gridDim.x;
  st.first = per * (int64_t)blockIdx.x;
  const int64_t mine = min(per, nchunks - st.first);
#else
  const int64_t mine = (nchunks - (int64_t)blockIdx.x + (int64_t)gridDim.x - 1) / (int64_t)gridDim.x;
#endif
  st.nmine = mine < 0 ? 0 : (int32_t)mine;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStreamStages; ++s) {
      mbar_init(sm.full + s, 1);
      mbar_init(sm.empty + s, kGroupWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t stream_chunk_row(const StreamMatrix& m, const StreamState& st, uint32_t q) {
#if B200IPC_STREAM_CONTIG
  return (st.first + (int64_t)(q % (uint32_t)st.nmine)) * m.rows_per_chunk;
#else
  return ((int64_t)blockIdx.x + (int64_t)(q % (uint32_t)st.nmine) * (int64_t)gridDim.x) * m.rows_per_chunk;
#endif
}

// Issue the loads of sequence number q, whose chunk covers blocks [b0, b1) (one thread).  Each copy
// moves a 16-byte aligned superset of its span; only an array's very end may stick out of the
// allocation, and there the last elements are patched with plain loads instead.
__device__ __forceinline__ void stream_issue(const StreamMatrix& m, const StreamSmem& sm, uint32_t q, int64_t b0,
                                             int64_t b1, int64_t r0) {
  const int s = (int)(q % kStreamStages);
  uint64_t* bar = sm.full + s;
  if (b1 - b0 > kStageBlocks || b1 == b0) {  // oversize (or empty) chunk: reduced from global memory
    mbar_arrive(bar);
    return;
  }
  const int64_t va = (72 * b0) & ~15ll;
  int64_t ve = (72 * b1 + 15) & ~15ll;
  double* sv = sm.vals(s);
  if (ve > 72 * m.nnzb) {
    ve -= 16;
    sv[(ve - va) / 8] = m.vals[ve / 8];
  }
  const int64_t ca = (4 * b0) & ~15ll;
  int64_t ce = (4 * b1 + 15) & ~15ll;
  int32_t* sc = sm.cols(s);
  if (ce > 4 * m.nnzb) {
    ce -= 16;
    for (int64_t t = ce / 4; t < m.nnzb; ++t) sc[t - ca / 4] = m.colidx[t];
  }
  const uint32_t vbytes = (uint32_t)(ve - va), cbytes = (uint32_t)(ce - ca);
  mbar_expect_tx(bar, vbytes + cbytes);
  if (m.pin_rows > 0) {
    const uint64_t policy = r0 < m.pin_rows ? kL2EvictLast : kL2EvictFirst;
    if (vbytes) bulk_g2s_hint(sv, reinterpret_cast<const char*>(m.vals) + va, vbytes, bar, policy);
    if (cbytes) bulk_g2s_hint(sc, reinterpret_cast<const char*>(m.colidx) + ca, cbytes, bar, policy);
  } else {
    if (vbytes) bulk_g2s(sv, reinterpret_cast<const char*>(m.vals) + va, vbytes, bar);
    if (cbytes) bulk_g2s(sc, reinterpret_cast<const char*>(m.colidx) + ca, cbytes, bar);
  }
}

// Three rows per warp trip: lane = 9 r + 3 i + j (r < 3) walks the blocks of row r; v / ci point at
// the lane's row (shared or global memory), len is its length (0 for an absent row or lane >= 27).
// Returns, in lanes with j == 0, component i of row r.  x is read with plain (coherent) loads: the persistent PCG kernel rewrites it between
// products.
template <typename GATHER>
__device__ __forceinline__ double stream_trio_product(const double* __restrict__ v, const int32_t* __restrict__ ci,
                                                      int len, int minlen, int maxlen, GATHER xg) {
  // Trips of four blocks.  While all three rows of the trio still have four blocks left (warp-uniform
  // test) the body is branch- and predicate-free: four column indices, four gathers, four values, four
  // FMAs.  The ragged end runs predicated: indices clamped to the row's last block (whose x row is in
  // cache), values forced to zero, so an absent block adds v * x = 0.
  double acc = 0.0;
  int t = 0;
  for (; t + 4 <= minlen; t += 4) {
    const int c0 = ci[t], c1 = ci[t + 1], c2 = ci[t + 2], c3 = ci[t + 3];
    const double x0 = xg(c0), x1 = xg(c1), x2 = xg(c2), x3 = xg(c3);
    const double v0 = v[9 * t], v1 = v[9 * t + 9], v2 = v[9 * t + 18], v3 = v[9 * t + 27];
    acc = fma(v0, x0, acc);
    acc = fma(v1, x1, acc);
    acc = fma(v2, x2, acc);
    acc = fma(v3, x3, acc);
  }
  const int last = len > 0 ? len - 1 : 0;
  for (; t < maxlen; t += 4) {
    const int c0 = ci[min(t, last)], c1 = ci[min(t + 1, last)], c2 = ci[min(t + 2, last)], c3 = ci[min(t + 3, last)];
    const double x0 = xg(c0), x1 = xg(c1), x2 = xg(c2), x3 = xg(c3);
    const double v0 = t < len ? v[9 * t] : 0.0, v1 = t + 1 < len ? v[9 * t + 9] : 0.0;
    const double v2 = t + 2 < len ? v[9 * t + 18] : 0.0, v3 = t + 3 < len ? v[9 * t + 27] : 0.0;
    acc = fma(v0, x0, acc);
    acc = fma(v1, x1, acc);
    acc = fma(v2, x2, acc);
    acc = fma(v3, x3, acc);
  }
  const double t1 = __shfl_down_sync(0xffffffffu, acc, 1);
  const double t2 = __shfl_down_sync(0xffffffffu, acc, 2);
  return (acc + t1) + t2;
}

// One product y = A x over this CTA's chunks.  `limit` bounds the sequence numbers this CTA may ever
// issue: nmine for a single product; unbounded for the PCG loop, which keeps the ring filled across
// iterations and drains it with stream_drain() before exit.  emit(row, yi) is called by the lanes
// that own component i = (lane % 9) / 3 of `row` (lane % 3 == 0, lane < 27).  No block-wide barrier
// inside.
template <typename GATHER, typename EMIT>
__device__ __forceinline__ void stream_product(const StreamMatrix& m, const StreamSmem& sm, StreamState& st,
                                               uint32_t limit, GATHER xg, EMIT emit) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = st.consumed;
  const uint32_t end = base + (uint32_t)st.nmine;
  uint32_t issue_end = end + (uint32_t)(kStreamStages - kStreamGroups);  // into the next product
  if (issue_end > limit) issue_end = limit;
  if (st.nmine > 0) {
    if (warp == kConsumerWarps) {
      // ---- producer warp: waits for a drained stage, stores the chunk's row pointers, issues the copies;
      // the row pointers of the following chunk are in flight meanwhile
      uint32_t q = st.issued;
      int64_t r0 = 0;
      int nrows = 0;
      int32_t rp[(kMaxChunkRows + 32) / 32];  // this lane's row pointers of chunk q
      int32_t rb0 = 0, rb1 = 0;               // its block range
      auto load_rows = [&](uint32_t qq) {
        r0 = stream_chunk_row(m, st, qq);
        nrows = (int)min((int64_t)m.rows_per_chunk, m.n - r0);
#pragma unroll
        for (int k = 0; k < (kMaxChunkRows + 32) / 32; ++k) rp[k] = m.rowptr[r0 + min(lane + 32 * k, nrows)];
        rb0 = m.rowptr[r0];
        rb1 = m.rowptr[r0 + nrows];
      };
      if (q < issue_end) load_rows(q);
      for (; q < issue_end;) {
        const int s = (int)(q % kStreamStages);
#ifdef B200IPC_PCG_TIMING
        const long long t0 = clock64();
#endif
        if (q >= (uint32_t)kStreamStages) mbar_wait(sm.empty + s, ((q / kStreamStages) - 1u) & 1u);
#ifdef B200IPC_PCG_TIMING
        if (m.dbg && lane == 0) m.dbg[3 * blockIdx.x + 2] += (unsigned long long)(clock64() - t0);
#endif
        const int32_t b0 = rb0, b1 = rb1;
        int32_t* hdr = sm.rows(s);
#pragma unroll
        for (int k = 0; k < (kMaxChunkRows + 32) / 32; ++k)
          if (lane + 32 * k <= nrows) hdr[2 + lane + 32 * k] = rp[k] - b0;
        if (lane == 0) {
          hdr[0] = nrows;
          hdr[1] = b0;
        }
        __syncwarp();  // header stores happen before lane 0's releasing arrive
        if (lane == 0) stream_issue(m, sm, q, b0, b1, r0);
        ++q;
        if (q < issue_end) load_rows(q);  // in flight while the next stage drains
      }
    } else {
      // ---- consumer warps -------------------------------------------------------------------------
      const int group = warp / kGroupWarps, gw = warp - group * kGroupWarps;
      const int r = lane / 9, e = lane - 9 * r, j = e % 3;   // r == 3 for lanes 27..31: idle
      uint32_t q = base + ((uint32_t)group + kStreamGroups - base % kStreamGroups) % kStreamGroups;
      for (; q < end; q += kStreamGroups) {
        const int s = (int)(q % kStreamStages);
        const int64_t row0 = stream_chunk_row(m, st, q);
#ifdef B200IPC_PCG_TIMING
        const long long t0 = clock64();
#endif
        mbar_wait(sm.full + s, (q / kStreamStages) & 1u);
#ifdef B200IPC_PCG_TIMING
        const long long t1 = clock64();
#endif
        const int32_t* hdr = sm.rows(s);
        const int nrows = hdr[0];
        const int32_t cb0 = hdr[1];
        const bool staged = hdr[2 + nrows] <= kStageBlocks && hdr[2 + nrows] > 0;
        const double* sv = sm.vals(s) + (cb0 & 1) + e;   // 72 b0 mod 16 = 8 (b0 mod 2): alignment slack in doubles
        const int32_t* sc = sm.cols(s) + (cb0 & 3);      // 4 b0 mod 16 = 4 (b0 mod 4)
        for (int tr = 3 * gw; tr < nrows; tr += 3 * kGroupWarps) {
          const int row = tr + r;
          int o0 = 0, len = 0;
          const bool valid = r < 3 && row < nrows;
          if (valid) {
            o0 = hdr[2 + row];
            len = hdr[3 + row] - o0;
          }
          const int maxlen = __reduce_max_sync(0xffffffffu, len);
          const int minlen = __reduce_min_sync(0xffffffffu, valid ? len : 0x7fffffff);  // over the rows present
          double yi;
          if (staged) yi = stream_trio_product(sv + 9 * o0, sc + o0, len, minlen, maxlen, xg);
          else yi = stream_trio_product(m.vals + 9ll * ((int64_t)cb0 + o0) + e, m.colidx + (int64_t)cb0 + o0, len, minlen, maxlen, xg);
          if (j == 0 && valid) emit(row0 + row, e / 3, yi);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(sm.empty + s);
#ifdef B200IPC_PCG_TIMING
        if (m.dbg && warp == 0 && lane == 0) {
          m.dbg[3 * blockIdx.x] += (unsigned long long)(t1 - t0);
          m.dbg[3 * blockIdx.x + 1] += (unsigned long long)(clock64() - t1);
        }
#endif
      }
    }
    if (st.issued < issue_end) st.issued = issue_end;
    st.consumed = end;
  }
}

// Wait for every outstanding bulk copy before the CTA exits or reuses shared memory.
__device__ __forceinline__ void stream_drain(const StreamSmem& sm, StreamState& st) {
  __syncthreads();
  while (st.consumed < st.issued) {
    mbar_wait(sm.full + (st.consumed % kStreamStages), (st.consumed / kStreamStages) & 1u);
    ++st.consumed;
  }
}

}  // namespace b200ipc
