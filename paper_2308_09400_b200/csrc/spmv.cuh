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

// Returns (y0,y1,y2) of block row `row` in every lane of the group.
template <int LPR>
__device__ __forceinline__ void bsr_row_product(int64_t row, int lane, const int32_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ colidx,
                                                const double* __restrict__ vals, const double* __restrict__ x,
                                                double& y0, double& y1, double& y2) {
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
