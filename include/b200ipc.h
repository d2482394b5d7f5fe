/*
 * b200ipc.h -- C ABI of the B200 (sm_100a) GIPC barrier hot path.
 *
 * Drop-in boundary for the reference package `tetipc` (arXiv 2308.09400).  Every
 * entry point names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/tetipc).  Plain pointers and sizes only; no torch or
 * Python types.  Unless a parameter says "host", every pointer is DEVICE memory
 * owned by the caller; the library never frees or retains caller buffers.  All
 * functions are asynchronous on `stream` (a cudaStream_t passed as void*; NULL =
 * the legacy default stream) unless stated otherwise, and return
 *     0   success
 *    <0   -(cudaError_t) of the failing runtime call / launch
 *    >0   argument error (B200IPC_EINVAL ...)
 * Per-stencil conditions are reported through `status` bytes, which the host side
 * turns into the reference's exceptions (gap.py:23-32).
 *
 * Arithmetic: fp64 throughout.  The library is compiled with -fmad=false so the
 * geometric predicates round exactly like the reference's compiled backend
 * (kernels/_core.pyx, x86-64 without FMA); the few places where the reference goes
 * through BLAS ddot on 3-vectors use an explicit fused chain.
 */
#ifndef B200IPC_H
#define B200IPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200IPC_ABI_VERSION 1

#define B200IPC_EINVAL 1   /* bad argument (null pointer, negative size, bad kind/size) */
#define B200IPC_ESTATE 2   /* handle used out of order (e.g. numeric before symbolic) */

/* Stencil kinds = rank of StencilKind.value in string order, i.e. the order of the
 * reference contact list (proximity.py:27-34, sort_key :82-83). */
enum {
  B200IPC_EE = 0, B200IPC_EEP = 1, B200IPC_PE = 2, B200IPC_PEP = 3,
  B200IPC_PP = 4, B200IPC_PPP = 5, B200IPC_PT = 6, B200IPC_NKINDS = 7
};

/* per-stencil status byte */
enum { B200IPC_ACTIVE = 0, B200IPC_INACTIVE = 1 /* d2 >= d_hat^2: skipped, solver.py:204 */,
       B200IPC_PENETRATION = 2 /* d2 <= 0: InterpenetrationError, gap.py:61 */ };

/* BarrierParams (barrier.py:24-53) + the solver's dt^2 (solver.py:192), pre-evaluated
 * on the host exactly as the reference's Python expressions evaluate them. */
typedef struct b200ipc_params {
  double d_hat;        /* params.d_hat                                              */
  double d_hat_sq;     /* d_hat*d_hat   -- gap.py:63, proximity.py:292,327          */
  double d_hat_pow2;   /* d_hat**2      -- solver.py:134,141,204 (libm pow)         */
  double scale;        /* kappa * d_hat**4 -- barrier.py:79                         */
  double eps_g;        /* d_thr_ratio**2   -- barrier.py:51-53                      */
  double dt2;          /* dt**2; multiplies grad and hess, not energy (solver.py:207) */
  int32_t use_filter;  /* proximal filter on lambda1 (barrier.py:114-120)           */
  int32_t form;        /* 0 = qlog (production), 1 = log (diagnostic)               */
} b200ipc_params;

/* ---- library ---------------------------------------------------------------- */
int b200ipc_abi_version(void);
/* Static string: build flags and target arch ("sm_100a"). */
const char* b200ipc_build_info(void);
/* Number of kernel launches issued by this library since load (all threads). */
int64_t b200ipc_launch_count(void);
/* dst[i] = src[idx[i]], rows of row_bytes bytes (a multiple of 4), all device pointers; idx (n) i64.  The row
 * compaction of the lagged friction state (friction.py:148-171 keeps the stencils with lambda_n > 0) and any other
 * place where the host mirror needs whole rows by index. */
int b200ipc_gather_rows(int64_t n, int64_t row_bytes, const void* src, const int64_t* idx, void* dst, void* stream);

/* Measured FP64 FMA throughput of the current device in TFLOP/s (2 flop per DFMA): a register-resident
 * DFMA microbenchmark, best of five launches.  The denominator of the fp64 rooflines.
 * *tflops is host memory; synchronises `stream`. */
int b200ipc_fp64_probe(double* tflops /* host */, void* stream);

/* ---- tetipc.kernels twins (kernels/__init__.py:28-31) ------------------------ */
/* pt_classify_batch (_core.pyx:46-106,153-171): p,t1,t2,t3 are (n,3) f64 row-major.
 * codes (n) i64, d2 (n), grad (n,4,3), w (n,2).  Any output pointer may be NULL. */
int b200ipc_pt_classify(int64_t n, const double* p, const double* t1, const double* t2,
                        const double* t3, int64_t* codes, double* d2, double* grad,
                        double* w, void* stream);
/* ee_classify_batch (_core.pyx:109-150,174-192). codes = 3*ra+rb, w = (s,t). */
int b200ipc_ee_classify(int64_t n, const double* a1, const double* a2, const double* b1,
                        const double* b2, int64_t* codes, double* d2, double* grad,
                        double* w, void* stream);
/* cross_sq_batch (_core.pyx:195-219): c (n), grad (n,4,3). */
int b200ipc_cross_sq(int64_t n, const double* a1, const double* a2, const double* b1,
                     const double* b2, double* c, double* grad, void* stream);
/* matvec_blocks (_core.pyx:222-247): out += scatter(H_b . gather(x)).
 * hess (nb,3s,3s) f64, vids (nb,s) i64, x/out (3N).  s in {2,3,4}.  Accumulation order is
 * not the serial block order of the reference (fp64 atomics); see DESIGN.md. */
int b200ipc_matvec_blocks(int64_t nb, int32_t s, const double* hess, const int64_t* vids,
                          const double* x, double* out, void* stream);
/* matvec_matrix_free (solver.py:251-262) = begin + matvec_blocks per family + end:
 * begin: vin = v with fixed rows zeroed, out = m * vin;  end: out[fixed] = v[fixed]. */
int b200ipc_matvec_begin(int64_t nverts, const double* masses, const uint8_t* fixed, const double* v,
                         double* vin, double* out, void* stream);
int b200ipc_matvec_end(int64_t nverts, const uint8_t* fixed, const double* v, double* out, void* stream);

/* ---- contact stencils: energy, gradient, PSD block ---------------------------- */
/* Fused twin of stencil_distance (proximity.py:183-222), parallel_measure (:225-229),
 * build_diagonal_jacobian (gap.py:56-82), barrier scalars (barrier.py:76-120),
 * build_local_quadratic (barrier.py:163-177), mollified_* (mollifier.py:55-144,191-210),
 * SimState._barrier_energy (solver.py:127-146) and the barrier loop of
 * assemble_local_quadratics (solver.py:202-209).
 *
 * The stencil table is sorted by kind (the reference list order); kind_off[k]..kind_off[k+1]
 * (host array of 8 int64) is the row range of kind k.
 *   positions (nverts,3) f64
 *   verts     (n,4) i32, -1 padded          sub (n) u8 (two bits per local index)
 *   eps_x     (n) f64 (parallel kinds)
 * Outputs (any may be NULL to skip it):
 *   energy (n)  per-stencil b(g) or e(c) b(g), g = d2/d_hat**2, not dt2-scaled; 0 if inactive
 *   status (n)  u8
 *   grad2/hess2 (n_PP,6)/(n_PP,6,6); grad3/hess3 (n_PE,9)/(n_PE,9,9);
 *   grad4/hess4 (n4,12)/(n4,12,12) with n4 = n_EE+n_EEP+n_PEP+n_PPP+n_PT, rows in that
 *   order -- the size families of group_blocks (solver.py:237-248).  Inactive rows are
 *   written as zeros.  grad/hess are dt2-scaled. */
int b200ipc_barrier_stencils(const b200ipc_params* params /* host */, int64_t nverts,
                             const double* positions, int64_t n, const int64_t* kind_off /* host[8] */,
                             const int32_t* verts, const uint8_t* sub, const double* eps_x,
                             double* energy, uint8_t* status,
                             double* grad2, double* hess2, double* grad3, double* hess3,
                             double* grad4, double* hess4, void* stream);

/* ---- per-stencil entry points kept as batched kernels ------------------------- */
/* stencil_distance (proximity.py:183-222) + parallel_measure (:225-229) +
 * build_diagonal_jacobian (gap.py:56-82) for n table rows in any order (kind is a device
 * array here).  All outputs padded to four vertex rows: d2 (n), grad_d2 (n,4,3),
 * witness (n,2), f (n), grad_f (n,4,3); parallel kinds only: c (n), grad_c (n,4,3),
 * sqrt_c (n), grad_sqrt_c (n,4,3) (rows of other kinds untouched).  status compares against
 * d_hat*d_hat like gap.py:61-64.  Any output may be NULL. */
int b200ipc_diagonal_jacobian(const b200ipc_params* params /* host */, int64_t nverts,
                              const double* positions, int64_t n, const uint8_t* kind,
                              const int32_t* verts, const uint8_t* sub,
                              double* d2, double* grad_d2, double* witness, double* f, double* grad_f,
                              double* c, double* grad_c, double* sqrt_c, double* grad_sqrt_c,
                              uint8_t* status, void* stream);
/* build_local_quadratic (barrier.py:163-177) / build_mollified_local_quadratic
 * (mollifier.py:191-210) from a given Jacobian: f (n), grad_f (n,12), and for parallel kinds
 * sqrt_c (n), grad_sqrt_c (n,12), eps_x (n).  grad (n,12), hess (n,12,12), padded, times dt2. */
int b200ipc_blocks_from_jacobian(const b200ipc_params* params /* host */, int64_t n, const uint8_t* kind,
                                 const double* f, const double* grad_f, const double* sqrt_c,
                                 const double* grad_sqrt_c, const double* eps_x,
                                 double* grad, double* hess, void* stream);
/* barrier_value/dg/d2g, lambda1, lambda23, filtered_lambda1 (barrier.py:76-120) at g (n):
 * out (n,6) = (b, b', b'', lambda1, lambda23, filtered lambda1). */
int b200ipc_barrier_scalars(const b200ipc_params* params /* host */, int64_t n, const double* g,
                            double* out, void* stream);
/* mollified_eigensystem (mollifier.py:106-144) at (g, c, eps_x) (n each): out (n,12) =
 * (lam_gamma1, lam_g1, t, p, lambda7', lambda8', q_gamma, q_f, b_gamma, b_g, e_k, e_k'). */
int b200ipc_mollified_eigensystem(const b200ipc_params* params /* host */, int64_t n, const double* g,
                                  const double* c, const double* eps_x, double* out, void* stream);

/* Same as b200ipc_barrier_stencils plus the rank-1 factors of the blocks: fac2 (n_PP,6), fac3
 * (n_PE,9), fac4 (n4,12) with hess_b = fac_b fac_b^T exactly (the dense entries are those products).
 * Pass hess* = NULL to skip the dense blocks when only the assembled matrix is needed
 * (b200ipc_assemble_numeric_factors): the step then writes 24 s instead of 72 s^2 bytes per block. */
int b200ipc_barrier_stencils_ex(const b200ipc_params* params /* host */, int64_t nverts,
                                const double* positions, int64_t n, const int64_t* kind_off /* host[8] */,
                                const int32_t* verts, const uint8_t* sub, const double* eps_x,
                                double* energy, uint8_t* status,
                                double* grad2, double* hess2, double* grad3, double* hess3,
                                double* grad4, double* hess4,
                                double* fac2, double* fac3, double* fac4, void* stream);

/* Same as b200ipc_barrier_stencils_ex with a choice of the dense blocks' DEVICE layout.  The reference's
 * LocalQuadratic.hess (solver.py:202-209) is the row-major (3s,3s) array, B200IPC_LAYOUT_DENSE; with
 * B200IPC_LAYOUT_SUBBLOCK the same numbers leave as (nb, s, s, 3, 3): element [b][a][c][i][j] = hess_b[3a+i][3c+j],
 * every 3x3 vertex-pair sub-block 72 contiguous bytes -- what the BSR assembly gathers (one line per source
 * instead of three).  An internal format between this call and b200ipc_assemble_numeric (see
 * b200ipc_assembly_set_layout); the host-facing view is a permute of it.  grad / fac / energy / status unchanged. */
#define B200IPC_LAYOUT_DENSE 0
#define B200IPC_LAYOUT_SUBBLOCK 1
int b200ipc_barrier_stencils_layout(const b200ipc_params* params /* host */, int64_t nverts,
                                    const double* positions, int64_t n, const int64_t* kind_off /* host[8] */,
                                    const int32_t* verts, const uint8_t* sub, const double* eps_x,
                                    double* energy, uint8_t* status,
                                    double* grad2, double* hess2, double* grad3, double* hess3,
                                    double* grad4, double* hess4,
                                    double* fac2, double* fac3, double* fac4, int32_t hess_layout, void* stream);

/* Sum of energy[0..n) (the scalar of SimState._barrier_energy, solver.py:127-146) and the
 * counts of status==1 / status==2, deterministic two-pass.  result: device double[1];
 * counts: device int64[2] (inactive, penetration); workspace: device scratch of at least
 * B200IPC_REDUCE_WS_BYTES. */
#define B200IPC_REDUCE_WS_BYTES 16384
int b200ipc_reduce_energy(int64_t n, const double* energy, const uint8_t* status,
                          double* result, int64_t* counts, void* workspace, void* stream);

/* ---- broad phase: scene -> candidate queries ------------------------------------ */
/* The AABB stage of find_contact_pairs (proximity.py:232-248, :275-319) as a uniform-grid join.
 * VT candidates: every (surface vertex v, triangle t) whose boxes [x_v - d_hat, x_v + d_hat] and
 * AABB(t) overlap and v is not a corner of t (:278-287).  EE candidates: every pair of edges i < j
 * whose AABBs, each inflated by d_hat/2, overlap and that share no endpoint (:305-317).  The overlap
 * predicate is the reference's own (lo_a <= hi_b && lo_b <= hi_a on the same fp64 corners), so the
 * candidate SETS equal the reference's; each pair is reported exactly once.  surf_verts (n_sv) i32,
 * tris (n_tri,3) i32, edges (n_edge,2) i32, positions (nverts,3) f64: device.  `cell` (> 0, typically
 * max(2 d_hat, median edge length)) and origin[3] (host; at or below the scene's lower corner) define
 * the grid; they affect speed only.
 * _count bins and joins once to size the outputs (*n_vt, *n_ee: host; synchronises `stream`);
 * _fill writes vt (n_vt,4) = (v, t1, t2, t3) and ee (n_ee,4) = (a1, a2, b1, b2), both 16-byte
 * aligned i32, ready for b200ipc_narrow_phase.  The input arrays must stay alive and unchanged
 * between the two calls.  One handle per scene/GPU; not thread-safe. */
typedef struct b200ipc_broad b200ipc_broad;
int b200ipc_broad_create(b200ipc_broad** out);
int b200ipc_broad_destroy(b200ipc_broad* h);
/* Optional speed hint for the next queries: the scene spans at most nx x ny x nz grid cells from `origin`
 * (<= 0: the default 2^21 per axis).  Cell keys then take ceil(log2) bits per axis and the binning sort
 * runs 3 radix passes instead of 8.  Coordinates beyond the hinted span fall into the boundary cells:
 * slower there, the candidate set is unchanged. */
int b200ipc_broad_set_grid_cells(b200ipc_broad* h, int32_t nx, int32_t ny, int32_t nz);
/* Size classes of the grid join (speed only; the candidate set is the reference's either way).  coarse_cell = 0
 * (default): every box is filed on the one grid of `cell`-sized cells.  coarse_cell > 2 cell: boxes whose largest
 * extent exceeds two cells are filed on a second grid of coarse_cell-sized cells and joined separately, so that a
 * few long collider edges do not widen the probe range of every cloth vertex (the probe range of a bin list is
 * its largest box).  The host mirror sets it from the longest edge of the scene when that is much longer than a
 * cell (cloth draped on a coarse sphere: broad phase 1.50 -> see DESIGN 4.4). */
int b200ipc_broad_set_coarse_cell(b200ipc_broad* h, double coarse_cell);
int b200ipc_broad_phase_count(b200ipc_broad* h, int64_t nverts, const double* positions,
                              int64_t n_sv, const int32_t* surf_verts, int64_t n_tri, const int32_t* tris,
                              int64_t n_edge, const int32_t* edges, double d_hat, double cell,
                              const double* origin /* host[3] */, int64_t* n_vt /* host */,
                              int64_t* n_ee /* host */, void* stream);
int b200ipc_broad_phase_fill(b200ipc_broad* h, int32_t* vt, int32_t* ee, void* stream);

/* sweep_candidates (proximity.py:388-421): the same join on SWEPT boxes -- every element's AABB over
 * its pose at `positions` and at positions + directions, grown by `margin` (the reference uses
 * 1e-3 d_hat) -- with the same incidence filters.  Sizes the outputs; b200ipc_broad_phase_fill then
 * writes vt (PAIR_PT candidates) and ee (PAIR_EE candidates). */
int b200ipc_sweep_candidates_count(b200ipc_broad* h, int64_t nverts, const double* positions,
                                   const double* directions, int64_t n_sv, const int32_t* surf_verts,
                                   int64_t n_tri, const int32_t* tris, int64_t n_edge, const int32_t* edges,
                                   double margin, double cell, const double* origin /* host[3] */,
                                   int64_t* n_vt /* host */, int64_t* n_ee /* host */, void* stream);

/* ---- additive CCD ------------------------------------------------------------------ */
/* Pair kinds of tetipc.kernels (kernels/__init__.py:21-26). */
#define B200IPC_PAIR_PT 0
#define B200IPC_PAIR_EE 1
#define B200IPC_PAIR_PE 2
#define B200IPC_PAIR_PP 3
/* accd_max_step (kernels/_core.pyx:272-325) for n pairs, one thread each: the largest step fraction
 * t in [0,1] along `directions` that keeps the pair's distance >= (1 - slack) * (current distance),
 * by conservative advancement with the reference's exits and iteration cap; bit-identical per pair.
 * ids (n,4) i32 global vertex ids (16-byte aligned; unused entries ignored): PT (p,t1,t2,t3),
 * EE (a1,a2,b1,b2), PE (p,e1,e2), PP (a,b).  pair_kind: u8 per pair, or NULL for `uniform_kind`.
 * step (n) f64; status (n) u8, may be NULL: 0 ok, 2 = current distance not positive (the reference
 * raises ValueError, :307-308; step is 0 there). */
int b200ipc_accd_max_step(int64_t n, const int32_t* ids, const uint8_t* pair_kind, int32_t uniform_kind,
                          const double* positions, const double* directions, double slack,
                          int32_t max_iter, double* step, uint8_t* status, void* stream);
/* global_ccd_filter (proximity.py:424-432) over the candidate lists of sweep_candidates: *alpha
 * (device double) = min(1, min over pairs of their ACCD bound); *n_invalid (device int64, may be
 * NULL) = pairs whose current distance is not positive (they do not enter the minimum; the
 * reference raises).  The minimum is exact and order-free, so the result is deterministic. */
int b200ipc_ccd_filter(int64_t n_vt, const int32_t* vt, int64_t n_ee, const int32_t* ee,
                       const double* positions, const double* directions, double slack, int32_t max_iter,
                       double* alpha /* device[1] */, int64_t* n_invalid /* device[1] */, void* stream);
/* The same filter over ANY superset of sweep_candidates' lists (e.g. one swept join with a margin of d_hat/2 that
 * also serves as the candidate set of every line-search detection along the step): each pair is first put to the
 * reference's own swept-box test (proximity.py:388-421) at `sweep_margin` (the reference: 1e-3 d_hat), the
 * survivors are compacted on the device and go through ACCD -- same minimum as b200ipc_ccd_filter over the
 * reference's list.  scratch: device, 16 (n_vt + n_ee) + 16 bytes, 16-byte aligned. */
int b200ipc_ccd_filter_swept(int64_t n_vt, const int32_t* vt, int64_t n_ee, const int32_t* ee,
                             const double* positions, const double* directions, double sweep_margin, double slack,
                             int32_t max_iter, void* scratch, double* alpha /* device[1] */,
                             int64_t* n_invalid /* device[1] */, void* stream);

/* ---- narrow phase: candidate queries -> ordered contact list ------------------- */
/* find_contact_pairs without its broad phase (proximity.py:284-358).  vt (n_vt,4) i32 =
 * (vertex, t1, t2, t3) and ee (n_ee,4) i32 = (a1, a2, b1, b2): any duplicate-free superset of
 * the near queries with incident / adjacent pairs already removed.  Keeps d2 < d_hat_sq
 * (= d_hat*d_hat), reduces to the active branch, promotes edge pairs with c < eps_x
 * (edge_parallel_eps from rest_positions) when promote_parallel, and sorts by the reference key
 * (kind.value, verts, origin).  Outputs have capacity n_vt+n_ee rows: kind u8, verts (.,4) i32
 * (-1 padded), sub u8, eps_x f64, origin_type u8 (1 "ee", 2 "vt"; may be NULL), origin (.,4) i32
 * (may be NULL).  *n_out and kind_off[8] are host; synchronises `stream`. */
int b200ipc_narrow_phase(int64_t nverts, const double* positions, const double* rest_positions,
                         int64_t n_vt, const int32_t* vt, int64_t n_ee, const int32_t* ee,
                         double d_hat_sq, int32_t promote_parallel,
                         uint8_t* kind, int32_t* verts, uint8_t* sub, double* eps_x,
                         uint8_t* origin_type, int32_t* origin,
                         int64_t* n_out /* host */, int64_t* kind_off /* host[8] */, void* stream);

/* ---- lagged smooth Coulomb friction (friction.py) ----------------------------------- */
/* update_friction_state (friction.py:148-171) for a whole kind-sorted stencil table: per stencil the
 * witness weights, contact normal, tangent frame (build_basis, :128-145) and lambda_n = |one side's
 * summed RAW (not dt^2-scaled) barrier gradient|.  grad2/3/4: the barrier gradient families
 * (nb,3s) in group_blocks order as written by b200ipc_barrier_stencils with dt2 = 1.  frame (n,12):
 * cn[4] = coeffs/|coeffs|, t1[3], t2[3], lambda_n, 0 -- the sliding basis is T[3v:3v+3, k] = cn_v t_k.
 * status (n) u8: 0 datum, 1 skipped (d2 <= 0 or lambda_n <= 0, as the reference skips them),
 * 3 undefined contact normal (the reference raises ValueError, :138-139).  kind_off: host[8]. */
int b200ipc_friction_state(int64_t n, const int64_t* kind_off /* host[8] */, const int32_t* verts,
                           const uint8_t* sub, const double* positions, const double* grad2,
                           const double* grad3, const double* grad4, double* frame, uint8_t* status,
                           void* stream);
/* The friction part of assemble_local_quadratics / _friction_energy (solver.py:147-152, :210-214) for a
 * kind-sorted table of friction data (rows with status 0, compacted): u = T^T (x - x_start)
 * (friction.py:174-178), energy (n, by table row, NOT dt^2-scaled) = mu lambda_n f0(|u|) (:49-52), gradient
 * families = -dt^2 friction_force (:55-61), hess families = dt^2 friction_hessian_psd (:64-82): rank-2
 * closed form w_p p p^T + w_q q q^T.  Families in group_blocks order; any output may be NULL. */
int b200ipc_friction_blocks(int64_t n, const int64_t* kind_off /* host[8] */, const int32_t* verts,
                            const double* frame, const double* x, const double* x_start, double mu,
                            double eps_v, double dt, double* energy, double* grad2, double* hess2,
                            double* grad3, double* hess3, double* grad4, double* hess4, void* stream);
/* potential / friction_force / friction_hessian_psd (friction.py:49-82) with an explicit basis
 * (n,3s,2) and tangential displacement u (n,2): potential (n), force (n,3s), hess (n,3s,3s) -- none of
 * them dt^2-scaled, like the reference functions; any output may be NULL. */
int b200ipc_friction_explicit(int64_t n, int32_t s, const double* basis, const double* u,
                              const double* lambda_n, double mu, double eps_v, double dt,
                              double* potential, double* force, double* hess, void* stream);

/* ---- stable neo-Hookean tetrahedra (elasticity.py) ----------------------------------- */
/* rest_data (elasticity.py:39-56): rest_inv (t,3,3) = inverse rest-shape matrices, vols (t) signed
 * rest volumes, from tets (t,4) i32 (16-byte aligned) and rest positions.  The dvec(F)/dx maps are
 * not stored: they are rest_inv rearranged. */
int b200ipc_elastic_rest(int64_t ntets, const int32_t* tets, const double* rest_positions,
                         double* rest_inv, double* vols, void* stream);
/* batch_grad_hess (elasticity.py:128-137): per tet the volume-scaled energy (t), gradient (t,12) and
 * 12x12 Hessian (t,12,12), the 9x9 dPsi/dF^2 projected PSD when `project` (the reference uses LAPACK
 * eigh; here the closed-form twist / flip / scaling eigensystem from a 3x3 SVD of F -- the projection
 * is unique).  grad and hess are multiplied by
 * `scale` (dt^2, solver.py:196-200), energy is not.  mu, lam: per-tet Lame parameters.  Any output
 * may be NULL. */
int b200ipc_elastic_blocks(int64_t ntets, const int32_t* tets, const double* positions,
                           const double* rest_inv, const double* vols, const double* mu, const double* lam,
                           double scale, int32_t project, double* energy, double* grad, double* hess,
                           void* stream);

/* ---- assembly into the 3x3-block sparse global matrix (BSR) -------------------- */
/* The reference's production path is matrix-free; the assembled matrix is the one its tests
 * build densely (tests/test_solver.py:71-84): A = diag(m_i I3) + sum_b scatter(H_b), fixed
 * rows/cols zeroed, unit diagonal.  Pattern := {(i,j): i,j in one block's vert_ids} U {(i,i)},
 * fixed rows reduced to the diagonal; columns ascend within a row.
 *
 * A handle owns the pattern and sort workspaces of ONE contact set (one per scene/GPU; not
 * thread-safe).  Families are the (hess, vids) pairs of group_blocks (solver.py:237-248):
 * fam_s[f] in {2,3,4}, fam_nb[f] blocks, fam_vids[f] device (nb,s) int64. */
typedef struct b200ipc_assembly b200ipc_assembly;
int b200ipc_assembly_create(b200ipc_assembly** out);
int b200ipc_assembly_destroy(b200ipc_assembly* h);
/* Numeric kernel choice.  0 (default) = automatic: per-block runs whenever the 32-bit descriptors apply
 * (<= 3 families, each below 24 GiB) -- walker 2 while runs are short (fewer than 4 sources per block on
 * average), else walker 1 -- and row-wise otherwise.  1 = per-block runs, three-group walker: one warp owns
 * eight consecutive output blocks, prefetches their source descriptors, lanes (g, e) sum entry e of every
 * third source.  2 = per-block runs, trio walker: three blocks per warp trip, nine lanes per block walk the
 * whole run.  4 = row-wise (one warp per block-row reads every dense block once as contiguous three-row
 * runs, accumulates in shared memory).  All are atomic-free and deterministic; results agree to round-off;
 * b200ipc_assemble_numeric_factors follows the same choice and is bitwise equal to the dense path of the
 * same walker.  Other values: B200IPC_EINVAL. */
int b200ipc_assembly_set_variant(b200ipc_assembly* h, int32_t variant);
/* Symbolic phase choice.  0 (default) = row-wise: one warp per block-row builds the row's column set and
 * source runs from the vertex-incidence runs (shared-memory hash set, ranks, stable placement; no global
 * sort of the 16 n_c slots), falling back to 1 when a row has more than 256 distinct columns.  1 = sort by
 * key (stable radix sort of every (row, col) slot).  Identical pattern, run order and matrices. */
int b200ipc_assembly_set_symbolic(b200ipc_assembly* h, int32_t mode);
/* Layout of the dense blocks b200ipc_assemble_numeric will be given: bit f of tiled_mask set = family f (the
 * f-th of b200ipc_assemble_symbolic) is B200IPC_LAYOUT_SUBBLOCK, clear = the reference's row-major blocks
 * (default).  The source descriptors are written by the symbolic phase, so the mask takes effect at the NEXT
 * b200ipc_assemble_symbolic.  Walkers 1 / 2 only: with a sub-block-major family the row-wise kernel (variant 4,
 * or more than three families) returns B200IPC_EINVAL.  Same sums in the same order: bitwise equal matrices. */
int b200ipc_assembly_set_layout(b200ipc_assembly* h, uint32_t tiled_mask);
/* out[4] (host) = {symbolic path that built the current pattern (1 sort, 2 row-wise), longest block row
 * (-1: not measured), nnzb, kept source slots}.  B200IPC_ESTATE before the first symbolic call. */
int b200ipc_assembly_stats(b200ipc_assembly* h, int64_t* out);
/* Build the pattern and the source runs.   fixed: device u8 (nverts).  Synchronises
 * `stream` once and returns the number of 3x3 blocks in *nnzb_out (host).  The vids buffers must stay
 * valid until the next symbolic call (the sort path builds the descriptor tables of the numeric kernels
 * from them on the first numeric call that needs them).  The row-wise numeric kernel (variant 4, or more
 * than three families) addresses a row's blocks with 16 bits: it returns B200IPC_EINVAL for a pattern
 * with a block row of 65535 or more entries; the per-block-run kernels have no such limit. */
int b200ipc_assemble_symbolic(b200ipc_assembly* h, int64_t nverts, const uint8_t* fixed, int32_t nfam,
                              const int32_t* fam_s /* host */, const int64_t* fam_nb /* host */,
                              const int64_t* const* fam_vids /* host array of device ptrs */,
                              int64_t* nnzb_out /* host */, void* stream);
/* Copy the pattern out: rowptr (nverts+1) i32, colidx (nnzb) i32, device. */
int b200ipc_assembly_pattern(b200ipc_assembly* h, int32_t* rowptr, int32_t* colidx, void* stream);
/* vals (nnzb,3,3) = segmented sum of the sub-blocks in list order; no atomics, deterministic.
 * fam_hess[f]: device (nb,3s,3s). */
int b200ipc_assemble_numeric(b200ipc_assembly* h, const double* masses,
                             const double* const* fam_hess /* host array of device ptrs */,
                             double* vals, void* stream);
/* Numeric assembly straight from the rank-1 factors of b200ipc_barrier_stencils_ex (barrier
 * families only; fam_fac[f]: device (nb,3s)); at most 3 families.  Bitwise identical to
 * b200ipc_assemble_numeric (walkers 1 / 2, same variant setting) on the dense blocks of the same factors. */
int b200ipc_assemble_numeric_factors(b200ipc_assembly* h, const double* masses,
                                     const double* const* fam_fac /* host array of device ptrs */,
                                     double* vals, void* stream);
/* SimState.gradient (solver.py:218-226): out (3 nverts) = m (x - x_tilde) + sum scatter(grad_b),
 * fixed rows 0.  fam_grad[f]: device (nb,3s). */
int b200ipc_scatter_gradient(b200ipc_assembly* h, const double* masses, const double* x,
                             const double* x_tilde, const double* const* fam_grad /* host array */,
                             double* out, void* stream);

/* ---- solver kernels over the assembled matrix ---------------------------------- */
/* y = A x (the assembled twin of matvec_matrix_free, solver.py:251-262). */
int b200ipc_bsr_spmv(int64_t nverts, int64_t nnzb, const int32_t* rowptr, const int32_t* colidx,
                     const double* vals, const double* x, double* y, void* stream);
/* block_jacobi_preconditioner (solver.py:265-276): pinv (nverts,3,3) = inverse diagonal blocks. */
int b200ipc_block_jacobi(int64_t nverts, const int32_t* rowptr, const int32_t* colidx,
                         const double* vals, double* pinv, void* stream);
typedef struct b200ipc_pcg_result {
  int32_t iters;
  int32_t converged;   /* delta_new <= rel_tol*delta0 (or delta0 <= 0) */
  double delta0;
  double delta_new;
} b200ipc_pcg_result;
int64_t b200ipc_pcg_workspace_bytes(int64_t nverts);
/* pcg_solve (solver.py:279-315) as one persistent cooperative kernel.  rhs, d: (3 nverts);
 * fixed: u8 (nverts).  Synchronises `stream`; *result is host memory. */
int b200ipc_pcg(int64_t nverts, int64_t nnzb, const int32_t* rowptr, const int32_t* colidx,
                const double* vals, const double* pinv, const uint8_t* fixed, const double* rhs,
                double* d, double rel_tol, int32_t max_iters, void* workspace, int64_t workspace_bytes,
                b200ipc_pcg_result* result /* host */, void* stream);

/* ---- multilevel additive Schwarz preconditioner -------------
 * The reference package has only block_jacobi_preconditioner (solver.py:265-276); the paper's GPU solver adds
 * the MAS preconditioner of Wu et al. 2022 and picks per simulation whichever is faster.  Same choice here:
 * b200ipc_pcg stays the parity default, b200ipc_pcg_mas is the alternative.  One handle per scene/GPU.
 *   order : Morton order of `positions` ((nverts,3) device f64; isotropic 10-bit cells over the largest
 *           extent); NULL = index order.  Domains are runs of 32 vertices in that order.
 *   setup : per level the 96x96 domain matrices (Galerkin, piecewise-constant prolongation) gathered from the
 *           assembled BSR matrix, inverted (fp64 Gauss-Jordan in shared memory), stored symmetrised in fp32.
 *           levels in {1, 2}.  Dirichlet vertices (`fixed`, u8 device, must stay valid while the handle is
 *           used) are kept out of the coarse spaces, so corrections leave them exactly at rest.  Needs
 *           b200ipc_mas_order first; call again whenever vals change.
 *   apply : z = sum_l P_l D_l^-1 P_l^T r, (3 nverts) device vectors.
 *   get_order : rank (nverts) i32 device = position of each vertex in the domain order. */
typedef struct b200ipc_mas b200ipc_mas;
int b200ipc_mas_create(b200ipc_mas** out);
int b200ipc_mas_destroy(b200ipc_mas* h);
int b200ipc_mas_order(b200ipc_mas* h, int64_t nverts, const double* positions, void* stream);
int b200ipc_mas_get_order(b200ipc_mas* h, int32_t* rank, void* stream);
int b200ipc_mas_setup(b200ipc_mas* h, int64_t nverts, int64_t nnzb, const int32_t* rowptr,
                      const int32_t* colidx, const double* vals, const uint8_t* fixed, int32_t levels,
                      void* stream);
int b200ipc_mas_apply(b200ipc_mas* h, const double* r, double* z, void* stream);
int64_t b200ipc_pcg_mas_workspace_bytes(int64_t nverts);
/* pcg_solve (solver.py:279-315) driven by the MAS operator of `h`, one persistent cooperative kernel.  The
 * loop STOPS ON THE REFERENCE'S RULE, measured with the block-Jacobi inverses `pinv`:
 * r . P_bj r <= rel_tol * (r0 . P_bj r0); result->delta0 / delta_new are those two quantities.  rowptr,
 * colidx, vals must be 16-byte aligned.  Synchronises `stream`; *result is host memory. */
int b200ipc_pcg_mas(b200ipc_mas* h, int64_t nverts, int64_t nnzb, const int32_t* rowptr,
                    const int32_t* colidx, const double* vals, const double* pinv, const uint8_t* fixed,
                    const double* rhs, double* d, double rel_tol, int32_t max_iters, void* workspace,
                    int64_t workspace_bytes, b200ipc_pcg_result* result /* host */, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200IPC_H */
