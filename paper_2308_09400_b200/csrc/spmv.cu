// Standalone BSR SpMV (the assembled twin of matvec_matrix_free, solver.py:251-262) and the
// block-Jacobi preconditioner (block_jacobi_preconditioner, solver.py:265-276).
#include <cstdlib>

#include "spmv.cuh"
#include "spmv_stream.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace b200ipc {

constexpr int kST = 256;

template <int LPR>
__global__ void __launch_bounds__(kST, 8) bsr_spmv_kernel(int64_t n, const int32_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ colidx,
                                                       const double* __restrict__ vals, const double* __restrict__ x,
                                                       double* __restrict__ y) {
  const int lane = threadIdx.x % LPR;
  if (LPR == 32) {
    const int64_t row0 = (((int64_t)blockIdx.x * kST + threadIdx.x) >> 5) * kSpmvRowsPerWarp;
    if (row0 >= n) return;
    bsr_rows_warp(row0, n, lane, rowptr, colidx, vals, x, [&](int64_t r, double y0, double y1, double y2) {
      if (lane < 3) y[3 * r + lane] = lane == 0 ? y0 : (lane == 1 ? y1 : y2);
    });
    return;
  }
  const int64_t row = ((int64_t)blockIdx.x * kST + threadIdx.x) / LPR;
  if (row >= n) return;  // whole groups exit together (kST % LPR == 0)
  double y0, y1, y2;
  bsr_row_product<LPR>(row, lane, rowptr, colidx, vals, x, y0, y1, y2);
  if (lane < 3) y[3 * row + lane] = lane == 0 ? y0 : (lane == 1 ? y1 : y2);
}

// Streamed product (spmv_stream.cuh): persistent CTAs, matrix staged through shared memory by TMA.
__global__ void __launch_bounds__(kStreamThreads, 1) bsr_spmv_stream_kernel(const __grid_constant__ StreamMatrix m,
                                                                             const double* __restrict__ x,
                                                                             double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char dyn[];
  const StreamSmem sm = stream_smem(dyn);
  StreamState st;
  stream_init(m, sm, st);
  const uint32_t limit = (uint32_t)st.nmine;
  const double* xj = x + (threadIdx.x & 31) % 3;  // lane = 9 r + 3 i + j
  stream_product(
      m, sm, st, limit, [&](int c) { return xj[3ll * c]; }, [&](int64_t r, int i, double yi) { y[3 * r + i] = yi; });
  stream_drain(sm, st);
}

int stream_rows_per_chunk(int64_t n, int64_t nnzb) {
  const double avg = n > 0 ? (double)nnzb / (double)n : 1.0;
  int r = (int)(0.72 * kStageBlocks / (avg > 1.0 ? avg : 1.0)) / 3 * 3;  // three rows per warp trip (cloth stack: 27 rows = 9 of a group's 10 warps busy; 24 / 27 / 30 rows: 35.1 / 34.1 / 35.1 us per PCG iteration)
  if (const char* env = getenv("B200IPC_SPMV_ROWS_PER_CHUNK")) r = atoi(env);
  return r < 3 ? 3 : (r > kMaxChunkRows ? kMaxChunkRows : r);
}

// Rows of the matrix to keep L2-resident across the iterations of a persistent solver loop: `budget_mb` MB of
// (values + column indices), from row 0.  B200IPC_L2_PIN_MB overrides the budget (0 = no hints).
int64_t stream_pin_rows(int64_t n, int64_t nnzb, double budget_mb) {
  if (const char* env = getenv("B200IPC_L2_PIN_MB")) budget_mb = atof(env);
  if (budget_mb <= 0.0 || n <= 0) return 0;
  const double per_row = 76.0 * (double)nnzb / (double)n;
  const double rows = budget_mb * 1e6 / per_row;
  return rows >= (double)n ? n : (rows < 1.0 ? 1 : (int64_t)rows);
}

// Inverse of the diagonal 3x3 block of every row (closed-form adjugate / determinant).
__global__ void __launch_bounds__(kST) block_jacobi_kernel(int64_t n, const int32_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ colidx,
                                                           const double* __restrict__ vals,
                                                           double* __restrict__ pinv) {
  const int64_t row = (int64_t)blockIdx.x * kST + threadIdx.x;
  if (row >= n) return;
  int32_t lo = rowptr[row], hi = rowptr[row + 1];
  while (lo < hi) {  // columns ascend within a row
    const int32_t mid = (lo + hi) >> 1;
    if (colidx[mid] < row) lo = mid + 1;
    else hi = mid;
  }
  const double* a = vals + 9ll * lo;  // the diagonal block always exists
  const double a00 = a[0], a01 = a[1], a02 = a[2], a10 = a[3], a11 = a[4], a12 = a[5], a20 = a[6], a21 = a[7],
               a22 = a[8];
  const double c00 = a11 * a22 - a12 * a21, c01 = a12 * a20 - a10 * a22, c02 = a10 * a21 - a11 * a20;
  const double det = a00 * c00 + a01 * c01 + a02 * c02;
  const double r = 1.0 / det;
  double* o = pinv + 9 * row;
  o[0] = c00 * r;
  o[1] = (a02 * a21 - a01 * a22) * r;
  o[2] = (a01 * a12 - a02 * a11) * r;
  o[3] = c01 * r;
  o[4] = (a00 * a22 - a02 * a20) * r;
  o[5] = (a02 * a10 - a00 * a12) * r;
  o[6] = c02 * r;
  o[7] = (a01 * a20 - a00 * a21) * r;
  o[8] = (a00 * a11 - a01 * a10) * r;
}

int pick_lpr(int64_t n, int64_t nnzb) {
  const double avg = n > 0 ? (double)nnzb / (double)n : 0.0;
  return avg >= 6.0 ? 32 : (avg >= 3.0 ? 16 : 8);
}

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int b200ipc_bsr_spmv(int64_t n, int64_t nnzb, const int32_t* rowptr, const int32_t* colidx,
                                const double* vals, const double* x, double* y, void* stream) {
  if (n < 0 || nnzb < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!rowptr || !colidx || !vals || !x || !y) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const char* mode = getenv("B200IPC_SPMV_MODE");
  const bool aligned = (((uintptr_t)vals | (uintptr_t)colidx | (uintptr_t)rowptr) & 15) == 0;
  if (aligned && !(mode && mode[0] == 'l')) {  // streamed (default); "legacy" keeps the direct-load kernels
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      if (cudaGetDevice(&dev) != cudaSuccess ||
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return B200IPC_ESTATE;
      cudaError_t e = cudaFuncSetAttribute(bsr_spmv_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kStreamSmemBytes);
      if (e != cudaSuccess) return -(int)e;
    }
    StreamMatrix m{n, nnzb, stream_rows_per_chunk(n, nnzb), 0, rowptr, colidx, vals, nullptr};
    const int64_t nchunks = (n + m.rows_per_chunk - 1) / m.rows_per_chunk;
    const unsigned grid = (unsigned)(nchunks < sms ? nchunks : sms);
    bsr_spmv_stream_kernel<<<grid, kStreamThreads, kStreamSmemBytes, st>>>(m, x, y);
    return post_launch();
  }
  const int lpr = pick_lpr(n, nnzb);
  const int64_t groups = lpr == 32 ? (n + kSpmvRowsPerWarp - 1) / kSpmvRowsPerWarp : n;
  const unsigned grid = (unsigned)((groups * lpr + kST - 1) / kST);
  if (lpr == 32) bsr_spmv_kernel<32><<<grid, kST, 0, st>>>(n, rowptr, colidx, vals, x, y);
  else if (lpr == 16) bsr_spmv_kernel<16><<<grid, kST, 0, st>>>(n, rowptr, colidx, vals, x, y);
  else bsr_spmv_kernel<8><<<grid, kST, 0, st>>>(n, rowptr, colidx, vals, x, y);
  return post_launch();
}

extern "C" int b200ipc_block_jacobi(int64_t n, const int32_t* rowptr, const int32_t* colidx, const double* vals,
                                    double* pinv, void* stream) {
  if (n < 0) return B200IPC_EINVAL;
  if (n == 0) return 0;
  if (!rowptr || !colidx || !vals || !pinv) return B200IPC_EINVAL;
  block_jacobi_kernel<<<(unsigned)((n + kST - 1) / kST), kST, 0, (cudaStream_t)stream>>>(n, rowptr, colidx, vals, pinv);
  return post_launch();
}
