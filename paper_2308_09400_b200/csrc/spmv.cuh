// BSR (3x3 blocks, fp64) row product shared by the standalone SpMV and the PCG kernel.
//
// A group of LPR lanes owns one block row.  The row's values are one contiguous run of
// 9*len doubles; lanes stride over it element-wise, so every load instruction of the group reads
// LPR consecutive doubles (full sectors, no padding), while x is gathered through L1/L2
// (three consecutive doubles per block).  Each lane accumulates the three row components it
// meets, then the group reduces with shuffles.  No atomics, fixed order: bitwise reproducible.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b200ipc {

// Full-warp variant: lane = 9*g + 3*i + j with g < 3 owns entry (i,j) of every third block of the
// row, so the entry index, the x component and the accumulator are lane constants -- no index
// arithmetic, no selects.  27 of 32 lanes work; each trip reads three whole blocks (216 contiguous
// bytes) and two trips are in flight.  Five shuffles finish the row.
__device__ __forceinline__ void bsr_row_product_span(int32_t b0, int32_t nblk, int lane,
                                                     const int32_t* __restrict__ colidx,
                                                     const double* __restrict__ vals, const double* __restrict__ x,
                                                     double& y0, double& y1, double& y2) {
  const int g = lane / 9, e = lane - 9 * g;
  const int j = e % 3;
  const double* v = vals + 9ll * b0 + e;
  const int32_t* ci = colidx + b0;
  double acc = 0.0;
  if (g < 3) {
    int blk = g;
    for (; blk + 3 < nblk; blk += 6) {
      const int c0 = __ldg(ci + blk), c1 = __ldg(ci + blk + 3);
      const double v0 = v[9 * blk], v1 = v[9 * (blk + 3)];
      const double x0 = __ldg(x + 3ll * c0 + j), x1 = __ldg(x + 3ll * c1 + j);
      acc += v0 * x0;
      acc += v1 * x1;
    }
    if (blk < nblk) acc += v[9 * blk] * __ldg(x + 3ll * __ldg(ci + blk) + j);
  }
  const double s1 = __shfl_down_sync(0xffffffffu, acc, 9);
  const double s2 = __shfl_down_sync(0xffffffffu, acc, 18);
  const double t = (acc + s1) + s2;               // lanes 0..8: entry sums over all blocks
  const double t1 = __shfl_down_sync(0xffffffffu, t, 1);
  const double t2 = __shfl_down_sync(0xffffffffu, t, 2);
  const double u = (t + t1) + t2;                 // lanes 0, 3, 6: row components
  y0 = __shfl_sync(0xffffffffu, u, 0);
  y1 = __shfl_sync(0xffffffffu, u, 3);
  y2 = __shfl_sync(0xffffffffu, u, 6);
}

__device__ __forceinline__ void bsr_row_product_warp(int64_t row, int lane, const int32_t* __restrict__ rowptr,
                                                     const int32_t* __restrict__ colidx,
                                                     const double* __restrict__ vals, const double* __restrict__ x,
                                                     double& y0, double& y1, double& y2) {
  const int32_t b0 = rowptr[row];
  bsr_row_product_span(b0, rowptr[row + 1] - b0, lane, colidx, vals, x, y0, y1, y2);
}

__device__ __forceinline__ void spmv_touch(const void* p) {
  unsigned tmp;
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(tmp) : "l"(p));
  (void)tmp;
}

constexpr int kSpmvRowsPerWarp = 4;

// A warp owns kSpmvRowsPerWarp consecutive block rows: their values and column indices are ONE
// contiguous span, pulled towards L1 with one round of coalesced line touches before the rows are
// reduced one after the other -- one exposed DRAM/L2 latency per warp instead of one per row.
// emit(row, y0, y1, y2) is called (by all lanes) once per row.
template <typename EMIT>
__device__ __forceinline__ void bsr_rows_warp(int64_t row0, int64_t n, int lane, const int32_t* __restrict__ rowptr,
                                              const int32_t* __restrict__ colidx, const double* __restrict__ vals,
                                              const double* __restrict__ x, EMIT emit) {
  const int nr = (int)min((int64_t)kSpmvRowsPerWarp, n - row0);
  const int32_t mine = rowptr[row0 + min(lane, nr)];
  const int32_t s0 = __shfl_sync(0xffffffffu, mine, 0), s1 = __shfl_sync(0xffffffffu, mine, nr);
  const char* vb = reinterpret_cast<const char*>(vals + 9ll * s0);
  const int64_t vbytes = 72ll * (s1 - s0);
  for (int64_t t = 128ll * lane; t < vbytes; t += 128 * 32) spmv_touch(vb + t);
  if (4ll * lane * 32 < 4ll * (s1 - s0)) spmv_touch(colidx + s0 + 32 * lane);
  for (int i = 0; i < nr; ++i) {
    const int32_t b0 = __shfl_sync(0xffffffffu, mine, i), b1 = __shfl_sync(0xffffffffu, mine, i + 1);
    double y0, y1, y2;
    bsr_row_product_span(b0, b1 - b0, lane, colidx, vals, x, y0, y1, y2);
    emit(row0 + i, y0, y1, y2);
  }
}

// Returns (y0,y1,y2) of block row `row` in every lane of the group.
template <int LPR>
__device__ __forceinline__ void bsr_row_product(int64_t row, int lane, const int32_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ colidx,
                                                const double* __restrict__ vals, const double* __restrict__ x,
                                                double& y0, double& y1, double& y2) {
  if (LPR == 32) {
    bsr_row_product_warp(row, lane, rowptr, colidx, vals, x, y0, y1, y2);
    return;
  }
  const int32_t b0 = rowptr[row], b1 = rowptr[row + 1];
  const double* v = vals + 9ll * b0;
  const int nelem = 9 * (b1 - b0);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  // four elements per lane per trip: all value / column loads are issued before the dependent x
  // gathers, and those before the adds (rows are short -- latency, not bandwidth, is the enemy)
  for (int base = lane; base < nelem; base += 4 * LPR) {
    double val[4], xv[4];
    int col[4], ei[4], ej[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = base + u * LPR;
      const bool ok = q < nelem;
      const int blk = ok ? q / 9 : 0;
      const int e = ok ? q - 9 * blk : 0;
      ei[u] = ok ? e / 3 : 3;  // 3 = no row: contributes nowhere
      ej[u] = e - 3 * (e / 3);
      col[u] = __ldg(colidx + b0 + blk);
      val[u] = ok ? v[q] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = __ldg(x + 3ll * col[u] + ej[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double p = val[u] * xv[u];
      a0 += ei[u] == 0 ? p : 0.0;
      a1 += ei[u] == 1 ? p : 0.0;
      a2 += ei[u] == 2 ? p : 0.0;
    }
  }
#pragma unroll
  // only this group's lanes take part: neighbouring groups in the warp may run other trip counts
  const unsigned mask = LPR == 32 ? 0xffffffffu : (((1u << (LPR & 31)) - 1u) << ((threadIdx.x & 31) / LPR * LPR));
  for (int o = LPR / 2; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(mask, a0, o, LPR);
    a1 += __shfl_xor_sync(mask, a1, o, LPR);
    a2 += __shfl_xor_sync(mask, a2, o, LPR);
  }
  y0 = a0;
  y1 = a1;
  y2 = a2;
}

}  // namespace b200ipc
