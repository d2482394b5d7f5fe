// Block-Jacobi preconditioned CG (pcg_solve, solver.py:279-315) over the assembled BSR matrix,
// as ONE persistent cooperative kernel: the whole iteration loop runs on the device with three
// grid barriers per iteration and a device-side convergence test, so there is no launch or host
// round trip per iteration (vectors of a 100k-vertex scene are L2 resident; launch latency would
// dominate otherwise).  Dot products are reduced in two fixed-order stages (per-CTA partials, then
// every CTA sums the partials in the same order): results are bitwise reproducible and every CTA
// takes the same branch.
//
//   r = rhs (fixed -> 0); s = P r; delta = r.s; c = s
//   loop: q = A c; denom = c.q; stop if denom <= 0; alpha = delta/denom
//         d += alpha c; r -= alpha q; s = P r; delta' = r.s; c = s + (delta'/delta) c
//   until delta' <= tol*delta0 or the cap.
#include <cooperative_groups.h>
#include <cstdlib>

#include "spmv.cuh"
#include "spmv_stream.cuh"
#include "launch.cuh"
#include "../../include/b200ipc.h"

namespace cg = cooperative_groups;

namespace b200ipc {

constexpr int kPT = 256;
constexpr int kMaxParts = 4096;
// Matrix bytes kept L2-resident across iterations (evict-last), the rest streams evict-first (spmv_stream.cuh).
// Measured on the 102 MB bench matrix: 0 (no hints) 37.6, 1 MB 35.1, 20 MB 34.7, 30 MB 34.6, 50 MB 34.7, 70 MB 35.6,
// 90 MB 37.0 us per iteration -- the product is bound by its consumers, not by DRAM, so pinning more buys nothing.
constexpr double kPcgPinMb = 20.0;

struct PcgArgs {
  int64_t n;
  const int32_t* rowptr;
  const int32_t* colidx;
  const double* vals;
  const double* pinv;
  const uint8_t* fixed;
  const double* rhs;
  double* d;
  double *r, *s, *c, *q;    // workspace vectors (3n each)
  double* part;             // 2 * kMaxParts partial sums (ping-pong)
  double rel_tol;
  int32_t max_iters;
  b200ipc_pcg_result* result;  // device
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;  // valid in thread 0
}

// every CTA sums all partials in the same order -> identical value everywhere
__device__ __forceinline__ double sum_parts(const double* part, int nparts, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) v += part[i];
  const double t = block_sum(v, sh);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = t;
  __syncthreads();
  return bc;
}

__device__ __forceinline__ void apply_pinv(const double* __restrict__ p, double r0, double r1, double r2, double& s0,
                                           double& s1, double& s2) {
  s0 = p[0] * r0 + p[1] * r1 + p[2] * r2;
  s1 = p[3] * r0 + p[4] * r1 + p[5] * r2;
  s2 = p[6] * r0 + p[7] * r1 + p[8] * r2;
}

template <int LPR>
__global__ void __launch_bounds__(kPT) pcg_kernel(const PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kPT / 32];
  const int64_t tid = (int64_t)blockIdx.x * kPT + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * kPT;
  const int nparts = gridDim.x;
  double* part0 = a.part;
  double* part1 = a.part + kMaxParts;

  // ---- init: d = 0, r = rhs (fixed -> 0), s = P r, c = s, delta0 = r.s ------------------------
  double acc = 0.0;
  for (int64_t v = tid; v < a.n; v += nthreads) {
    const bool fx = a.fixed[v];
    const double r0 = fx ? 0.0 : a.rhs[3 * v], r1 = fx ? 0.0 : a.rhs[3 * v + 1], r2 = fx ? 0.0 : a.rhs[3 * v + 2];
    double s0, s1, s2;
    apply_pinv(a.pinv + 9 * v, r0, r1, r2, s0, s1, s2);
    a.d[3 * v] = a.d[3 * v + 1] = a.d[3 * v + 2] = 0.0;
    a.r[3 * v] = r0; a.r[3 * v + 1] = r1; a.r[3 * v + 2] = r2;
    a.s[3 * v] = s0; a.s[3 * v + 1] = s1; a.s[3 * v + 2] = s2;
    a.c[3 * v] = s0; a.c[3 * v + 1] = s1; a.c[3 * v + 2] = s2;
    acc += r0 * s0 + r1 * s1 + r2 * s2;
  }
  {
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part0[blockIdx.x] = t;
  }
  grid.sync();
  const double delta0 = sum_parts(part0, nparts, sh);
  double delta_new = delta0;
  int iters = 0;
  bool broke = false;

  if (delta0 > 0.0) {
    while (iters < a.max_iters && delta_new > a.rel_tol * delta0) {
      // ---- q = A c, denom = c.q ------------------------------------------------------------------
      acc = 0.0;
      const int lane = threadIdx.x % LPR;
      // one row per warp per trip: inside the persistent kernel the plain grid-stride row loop
      // measured faster (55 us/iteration) than multi-row spans with prefetch touches (88-94 us)
      for (int64_t row = tid / LPR; row < a.n; row += nthreads / LPR) {
        double y0, y1, y2;
        bsr_row_product<LPR>(row, lane, a.rowptr, a.colidx, a.vals, a.c, y0, y1, y2);
        if (lane == 0) {
          a.q[3 * row] = y0; a.q[3 * row + 1] = y1; a.q[3 * row + 2] = y2;
          acc += a.c[3 * row] * y0 + a.c[3 * row + 1] * y1 + a.c[3 * row + 2] * y2;
        }
      }
      {
        const double t = block_sum(acc, sh);
        if (threadIdx.x == 0) part1[blockIdx.x] = t;
      }
      grid.sync();
      const double denom = sum_parts(part1, nparts, sh);
      if (denom <= 0.0) {  // solver.py:305-306
        broke = true;
        break;
      }
      const double alpha = delta_new / denom;
      // ---- d += alpha c; r -= alpha q; s = P r; delta' = r.s -------------------------------------
      acc = 0.0;
      for (int64_t v = tid; v < a.n; v += nthreads) {
        double rr[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          a.d[3 * v + k] += alpha * a.c[3 * v + k];
          rr[k] = a.r[3 * v + k] - alpha * a.q[3 * v + k];
          a.r[3 * v + k] = rr[k];
        }
        double s0, s1, s2;
        apply_pinv(a.pinv + 9 * v, rr[0], rr[1], rr[2], s0, s1, s2);
        a.s[3 * v] = s0; a.s[3 * v + 1] = s1; a.s[3 * v + 2] = s2;
        acc += rr[0] * s0 + rr[1] * s1 + rr[2] * s2;
      }
      {
        const double t = block_sum(acc, sh);
        if (threadIdx.x == 0) part0[blockIdx.x] = t;
      }
      grid.sync();
      const double delta_old = delta_new;
      delta_new = sum_parts(part0, nparts, sh);
      const double beta = delta_new / delta_old;
      // ---- c = s + beta c ---------------------------------------------------------------------------
      for (int64_t i = tid; i < 3 * a.n; i += nthreads) a.c[i] = a.s[i] + beta * a.c[i];
      ++iters;
      grid.sync();
    }
  }
  (void)broke;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result->iters = iters;
    a.result->converged = (delta0 <= 0.0) || (delta_new <= a.rel_tol * delta0);
    a.result->delta0 = delta0;
    a.result->delta_new = delta_new;
  }
}

// ---- streamed variant (default) -----------------------------------------------------------------
// Same recurrence, TWO grid barriers per iteration.  The product q = A c pulls the matrix through
// shared memory with bulk async copies (spmv_stream.cuh), one CTA per SM, and the ring is refilled for
// the NEXT product as soon as a stage drains, so the first chunks of iteration k+1 arrive while the
// vector updates and barriers of iteration k run.
// The direction update c = s + beta c is folded into the product: vectors s and c live interleaved
// per component in two ping-pong buffers B[2] of (n, 3, 2) = (s_j, c_j) pairs; the product of
// iteration k+1 gathers one pair with ONE 16-byte load from B[k], forms c'_j = s_j + beta c_j in
// registers (the same two roundings as a stored update), and the lanes that finish row i store c'_i
// into B[k+1] -- so the separate update pass and its grid barrier disappear.  x is read with coherent loads (it changes every iteration).
struct PcgStreamArgs {
  int64_t n;
  const double* pinv;
  const uint8_t* fixed;
  const double* rhs;
  double* d;
  double* buf[2];           // (n, 3, 2): (s_j, c_j) pairs
  double* rbuf[2];          // residual, ping-pong (the update reads all three entries of a vertex)
  double* q;
  double* part;             // 2 * kMaxParts partial sums (ping-pong)
  double rel_tol;
  int32_t max_iters;
  b200ipc_pcg_result* result;  // device
};

__global__ void __launch_bounds__(kStreamThreads, 1) pcg_stream_kernel(const __grid_constant__ PcgStreamArgs a,
                                                                        const __grid_constant__ StreamMatrix m) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ double sh[kStreamThreads / 32];
  const StreamSmem sm = stream_smem(dyn);
  StreamState st;
  stream_init(m, sm, st);
  const uint32_t unbounded = 0xffffffffu;

  const int64_t tid = (int64_t)blockIdx.x * kStreamThreads + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * kStreamThreads;
  const int nparts = gridDim.x;
  const int j = (threadIdx.x & 31) % 3;  // x component of this lane inside the product (lane = 9 r + 3 i + j)
  double* part0 = a.part;
  double* part1 = a.part + kMaxParts;

  // ---- init: d = 0, r = rhs (fixed -> 0), s = P r, c = 0 (beta = 0 makes the first direction s) ------
  double acc = 0.0;
  for (int64_t v = tid; v < a.n; v += nthreads) {
    const bool fx = a.fixed[v];
    const double r0 = fx ? 0.0 : a.rhs[3 * v], r1 = fx ? 0.0 : a.rhs[3 * v + 1], r2 = fx ? 0.0 : a.rhs[3 * v + 2];
    double s0, s1, s2;
    apply_pinv(a.pinv + 9 * v, r0, r1, r2, s0, s1, s2);
    a.d[3 * v] = a.d[3 * v + 1] = a.d[3 * v + 2] = 0.0;
    a.rbuf[0][3 * v] = r0; a.rbuf[0][3 * v + 1] = r1; a.rbuf[0][3 * v + 2] = r2;
    double* w = a.buf[0] + 6 * v;
    w[0] = s0; w[2] = s1; w[4] = s2;
    w[1] = w[3] = w[5] = 0.0;
    acc += r0 * s0 + r1 * s1 + r2 * s2;
  }
  {
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part0[blockIdx.x] = t;
  }
  grid.sync();
  const double delta0 = sum_parts(part0, nparts, sh);
  double delta_new = delta0;
  double beta = 0.0;
  int iters = 0, cur = 0;

#ifdef B200IPC_PCG_TIMING
  unsigned long long tm[4] = {0, 0, 0, 0}, t0, t1;
#define PCG_TICK(k)                                            \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));     \
  tm[k] += t1 - t0;                                            \
  t0 = t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#else
#define PCG_TICK(k)
#endif
  if (delta0 > 0.0) {
    while (iters < a.max_iters && delta_new > a.rel_tol * delta0) {
      const double* bold = a.buf[cur];
      double* bnew = a.buf[cur ^ 1];
      // ---- c = s + beta c (on the fly); q = A c; denom = c.q -----------------------------------------
      acc = 0.0;
      const double2* wj = reinterpret_cast<const double2*>(bold) + j;
      stream_product(
          m, sm, st, unbounded,
          [&](int col) {
            const double2 w = wj[3ll * col];
            return w.x + beta * w.y;
          },
          [&](int64_t row, int i, double yi) {
            const double2 w = reinterpret_cast<const double2*>(bold)[3 * row + i];
            const double cn = w.x + beta * w.y;
            bnew[6 * row + 2 * i + 1] = cn;
            a.q[3 * row + i] = yi;
            acc += cn * yi;
          });
      {
        const double t = block_sum(acc, sh);
        if (threadIdx.x == 0) part1[blockIdx.x] = t;
      }
      PCG_TICK(0)
      grid.sync();
      const double denom = sum_parts(part1, nparts, sh);
      if (denom <= 0.0) break;  // solver.py:305-306
      const double alpha = delta_new / denom;
      PCG_TICK(1)
      // ---- d += alpha c; r -= alpha q; s = P r; delta' = r.s -------------------------------------
      // one thread per (vertex, component): every access below is coalesced (a thread per vertex would
      // read P^-1 with a 72-byte stride).  Each thread forms the vertex's three new residual entries --
      // the same expressions in all three threads, so they agree bitwise -- and keeps row k of P^-1.
      acc = 0.0;
      const double* __restrict__ rold = a.rbuf[cur];
      double* __restrict__ rnew = a.rbuf[cur ^ 1];
      const double* __restrict__ qv = a.q;
      const double* __restrict__ pinv = a.pinv;
      double* __restrict__ dvec = a.d;
      for (int64_t t = tid; t < 3 * a.n; t += nthreads) {
        const int64_t v = t / 3;
        const int k = (int)(t - 3 * v);
        const double rr0 = rold[3 * v] - alpha * qv[3 * v];
        const double rr1 = rold[3 * v + 1] - alpha * qv[3 * v + 1];
        const double rr2 = rold[3 * v + 2] - alpha * qv[3 * v + 2];
        const double* p = pinv + 9 * v + 3 * k;
        const double sk = p[0] * rr0 + p[1] * rr1 + p[2] * rr2;
        const double rk = k == 0 ? rr0 : (k == 1 ? rr1 : rr2);
        dvec[t] += alpha * bnew[6 * v + 2 * k + 1];
        bnew[6 * v + 2 * k] = sk;
        rnew[t] = rk;
        acc += rk * sk;
      }
      {
        const double t = block_sum(acc, sh);
        if (threadIdx.x == 0) part0[blockIdx.x] = t;
      }
      PCG_TICK(2)
      grid.sync();
      const double delta_old = delta_new;
      delta_new = sum_parts(part0, nparts, sh);
      beta = delta_new / delta_old;
      cur ^= 1;
      ++iters;
      PCG_TICK(3)
    }
  }
  stream_drain(sm, st);
#ifdef B200IPC_PCG_TIMING
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) a.part[1024 + 512 * k + blockIdx.x] = (double)tm[k];
#endif
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result->iters = iters;
    a.result->converged = (delta0 <= 0.0) || (delta_new <= a.rel_tol * delta0);
    a.result->delta0 = delta0;
    a.result->delta_new = delta_new;
  }
}

int pick_lpr(int64_t n, int64_t nnzb);  // spmv.cu
int stream_rows_per_chunk(int64_t n, int64_t nnzb);  // spmv.cu
int64_t stream_pin_rows(int64_t n, int64_t nnzb, double budget_mb);  // spmv.cu

}  // namespace b200ipc

using namespace b200ipc;

extern "C" int64_t b200ipc_pcg_workspace_bytes(int64_t n) {
  if (n < 0) return 0;
  return (int64_t)sizeof(double) * (7 * 3 * n + 2 * kMaxParts) + 256;  // streamed: 2 x (n,6) + 2 r + q
}

extern "C" int b200ipc_pcg(int64_t n, int64_t nnzb, const int32_t* rowptr, const int32_t* colidx, const double* vals,
                           const double* pinv, const uint8_t* fixed, const double* rhs, double* d, double rel_tol,
                           int32_t max_iters, void* workspace, int64_t workspace_bytes, b200ipc_pcg_result* result,
                           void* stream) {
  if (n <= 0 || nnzb < n || !rowptr || !colidx || !vals || !pinv || !fixed || !rhs || !d || !workspace || !result)
    return B200IPC_EINVAL;
  if (workspace_bytes < b200ipc_pcg_workspace_bytes(n) || max_iters < 0) return B200IPC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  PcgArgs a;
  a.n = n; a.rowptr = rowptr; a.colidx = colidx; a.vals = vals; a.pinv = pinv; a.fixed = fixed; a.rhs = rhs; a.d = d;
  double* w = static_cast<double*>(workspace);
  a.r = w; a.s = w + 3 * n; a.c = w + 6 * n; a.q = w + 9 * n;
  a.part = w + 12 * n;
  a.result = reinterpret_cast<b200ipc_pcg_result*>(a.part + 2 * kMaxParts);
  a.rel_tol = rel_tol; a.max_iters = max_iters;

  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return -(int)e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return -(int)e;
  const char* mode = getenv("B200IPC_SPMV_MODE");
  const bool aligned = (((uintptr_t)vals | (uintptr_t)colidx | (uintptr_t)rowptr) & 15) == 0;
  if (aligned && !(mode && mode[0] == 'l')) {
    StreamMatrix m{n, nnzb, stream_rows_per_chunk(n, nnzb), 0, rowptr, colidx, vals, nullptr, stream_pin_rows(n, nnzb, kPcgPinMb)};
#ifdef B200IPC_PCG_TIMING
    m.dbg = reinterpret_cast<unsigned long long*>(w + 21 * n + 3072);  // inside the partial-sum scratch
    cudaMemsetAsync(m.dbg, 0, 3 * 148 * 8, st);
#endif
    e = cudaFuncSetAttribute(pcg_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmemBytes);
    if (e != cudaSuccess) return -(int)e;
    const int64_t nchunks = (n + m.rows_per_chunk - 1) / m.rows_per_chunk;
    int64_t grid = nchunks < sms ? nchunks : sms;
    if (grid < 1) grid = 1;
    PcgStreamArgs sa;
    sa.n = n; sa.pinv = pinv; sa.fixed = fixed; sa.rhs = rhs; sa.d = d;
    sa.buf[0] = w; sa.buf[1] = w + 6 * n; sa.rbuf[0] = w + 12 * n; sa.rbuf[1] = w + 15 * n; sa.q = w + 18 * n;
    sa.part = w + 21 * n;
    sa.result = reinterpret_cast<b200ipc_pcg_result*>(sa.part + 2 * kMaxParts);
    sa.rel_tol = rel_tol; sa.max_iters = max_iters;
    a.result = sa.result;
    void* args[] = {(void*)&sa, (void*)&m};
    e = cudaLaunchCooperativeKernel((const void*)pcg_stream_kernel, dim3((unsigned)grid), dim3(kStreamThreads), args,
                                    kStreamSmemBytes, st);
    if (e != cudaSuccess) return -(int)e;
    int rc = post_launch();
    if (rc) return rc;
    e = cudaMemcpyAsync(result, a.result, sizeof(b200ipc_pcg_result), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return -(int)e;
    e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? 0 : -(int)e;
  }
  const int lpr = pick_lpr(n, nnzb);
  const void* fn = lpr == 32 ? (const void*)pcg_kernel<32> : (lpr == 16 ? (const void*)pcg_kernel<16> : (const void*)pcg_kernel<8>);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPT, 0);
  if (e != cudaSuccess) return -(int)e;
  if (per_sm < 1) return B200IPC_ESTATE;
  if (const char* env = getenv("B200IPC_PCG_CTAS_PER_SM")) {  // tuning knob: fewer CTAs = cheaper grid barriers
    const int want_per_sm = atoi(env);
    if (want_per_sm >= 1 && want_per_sm < per_sm) per_sm = want_per_sm;
  }
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t want = (n * lpr + kPT - 1) / kPT;  // no more CTAs than rows need
  if (grid > want) grid = want;
  if (grid > kMaxParts) grid = kMaxParts;
  if (grid < 1) grid = 1;
  void* args[] = {(void*)&a};
  e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(kPT), args, 0, st);
  if (e != cudaSuccess) return -(int)e;
  int rc = post_launch();
  if (rc) return rc;
  e = cudaMemcpyAsync(result, a.result, sizeof(b200ipc_pcg_result), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return -(int)e;
  e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? 0 : -(int)e;
}
