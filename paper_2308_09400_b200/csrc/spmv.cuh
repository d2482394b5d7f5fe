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
  // two elements per lane in flight per trip (independent loads), accumulated in element order
  for (int q = lane; q < nelem; q += 2 * LPR) {
    const int q2 = q + LPR;
    const bool two = q2 < nelem;
    const int blk = q / 9, blk2 = two ? q2 / 9 : blk;
    const int e = q - 9 * blk, e2 = two ? q2 - 9 * blk2 : 0;
    const int i = e / 3, j = e - 3 * i;
    const int i2 = e2 / 3, j2 = e2 - 3 * i2;
    const int c1 = __ldg(colidx + b0 + blk), c2 = __ldg(colidx + b0 + blk2);
    const double v1 = v[q], v2 = two ? v[q2] : 0.0;
    const double p = v1 * __ldg(x + 3ll * c1 + j);
    const double p2 = v2 * __ldg(x + 3ll * c2 + j2);
    a0 += i == 0 ? p : 0.0;
    a1 += i == 1 ? p : 0.0;
    a2 += i == 2 ? p : 0.0;
    a0 += (two && i2 == 0) ? p2 : 0.0;
    a1 += (two && i2 == 1) ? p2 : 0.0;
    a2 += (two && i2 == 2) ? p2 : 0.0;
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
