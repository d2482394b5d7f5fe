/*
 * oracle_c.c -- plain-C restatement of the reference's per-stencil barrier path.
 * TEST / BASELINE INFRASTRUCTURE ONLY: used by tests (cross-check of the NumPy oracle) and by
 * bench.py's cpu_baseline / --impl reference legs; never by the product package.
 *
 * Parity status: pinned through tests/test_oracle_c.py (bit-exact classification against the
 * frozen outputs of the reference's compiled backend, blocks against the frozen reference
 * blocks), see oracle/tetipc_oracle.py for the pinning story.
 *
 * Follows (paths under /root/reference/pkg/src/tetipc):
 *   kernels/_core.pyx:22-219   dot/cross, _pt_one, _ee_one, cross_sq       (scalar, no FMA)
 *   proximity.py:170-222       _point_edge_eval, stencil_distance           (np.dot -> fma chain)
 *   gap.py:56-82               f, grad f, sqrt c, grad sqrt c
 *   barrier.py:76-120,163-177  scalars, lambda1, filter, rank-1 block
 *   mollifier.py:55-144,191-210 mollifier, 2x2 coupled eigen system, block
 *   solver.py:127-146,202-209  energy with g = d2/d_hat**2, dt^2 scaling, inactive skip
 * One stencil per loop iteration, pthreads across stencils (the work is independent per stencil;
 * the reference itself is single-threaded).  Build: see oracle/Makefile (-O2 -ffp-contract=off).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

/* ---- tiny static-schedule parallel-for on pthreads (this image's gcc has no libgomp) ---- */
typedef void (*range_fn)(int64_t begin, int64_t end, void* ctx);
typedef struct { range_fn fn; void* ctx; int64_t begin, end; } range_job;
static int g_threads = 1;
static void* range_thread(void* arg) { range_job* j = (range_job*)arg; j->fn(j->begin, j->end, j->ctx); return 0; }
static void parallel_for(int64_t n, range_fn fn, void* ctx) {
  int nt = g_threads < 1 ? 1 : (g_threads > 256 ? 256 : g_threads);
  if ((int64_t)nt > n) nt = n > 0 ? (int)n : 1;
  if (nt == 1) { fn(0, n, ctx); return; }
  pthread_t th[256];
  range_job jobs[256];
  const int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    jobs[t].fn = fn; jobs[t].ctx = ctx;
    jobs[t].begin = t * chunk; jobs[t].end = (t + 1) * chunk < n ? (t + 1) * chunk : n;
    pthread_create(&th[t], 0, range_thread, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], 0);
}
void oracle_set_threads(int n) { g_threads = n; }
int oracle_num_threads(void) { return g_threads; }

enum { K_EE = 0, K_EEP, K_PE, K_PEP, K_PP, K_PPP, K_PT };

typedef struct {
  double d_hat, d_hat_sq, d_hat_pow2, scale, eps_g, dt2;
  int32_t use_filter, form;
} oracle_params;

typedef struct { double x, y, z; } v3;

static inline v3 vsub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static inline v3 vscale(double s, v3 a) { v3 r = {s * a.x, s * a.y, s * a.z}; return r; }
static inline double dot3(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline double dot3_blas(v3 a, v3 b) { return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x)); }
static inline v3 cross3(v3 a, v3 b) {
  v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
  return r;
}
static inline double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
static inline v3 ld(const double* p, int64_t i) { v3 r = {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; return r; }

static int pt_one(v3 p, v3 t1, v3 t2, v3 t3, double* d2, v3 g[4], double* w1o, double* w2o) {
  v3 ab = vsub(t2, t1), ac = vsub(t3, t1), ap = vsub(p, t1);
  double d1 = dot3(ab, ap), d2_ = dot3(ac, ap);
  v3 bp = vsub(p, t2);
  double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  v3 cp = vsub(p, t3);
  double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  double vc = d1 * d4 - d3 * d2_, vb = d5 * d2_ - d1 * d6, va = d3 * d6 - d5 * d4;
  double w1 = 0.0, w2 = 0.0;
  int code;
  if (d1 <= 0.0 && d2_ <= 0.0) code = 1;
  else if (d3 >= 0.0 && d4 <= d3) { code = 2; w1 = 1.0; }
  else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) { code = 4; w1 = d1 / (d1 - d3); }
  else if (d6 >= 0.0 && d5 <= d6) { code = 3; w2 = 1.0; }
  else if (vb <= 0.0 && d2_ >= 0.0 && d6 <= 0.0) { code = 6; w2 = d2_ / (d2_ - d6); }
  else if (va <= 0.0 && d4 - d3 >= 0.0 && d5 - d6 >= 0.0) {
    code = 5;
    double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    w1 = 1.0 - t; w2 = t;
  } else {
    code = 0;
    double denom = va + vb + vc;
    w1 = vb / denom; w2 = vc / denom;
  }
  double w0 = 1.0 - w1 - w2;
  v3 cl = {w0 * t1.x + w1 * t2.x + w2 * t3.x, w0 * t1.y + w1 * t2.y + w2 * t3.y, w0 * t1.z + w1 * t2.z + w2 * t3.z};
  v3 r = vsub(p, cl);
  *d2 = dot3(r, r);
  g[0] = vscale(2.0, r); g[1] = vscale(-2.0 * w0, r); g[2] = vscale(-2.0 * w1, r); g[3] = vscale(-2.0 * w2, r);
  *w1o = w1; *w2o = w2;
  return code;
}

static int ee_one(v3 a1, v3 a2, v3 b1, v3 b2, double* d2, v3 g[4], double* so, double* to) {
  v3 da = vsub(a2, a1), db = vsub(b2, b1), r = vsub(a1, b1);
  double a = dot3(da, da), e = dot3(db, db), f = dot3(db, r), b = dot3(da, db), c = dot3(da, r);
  double denom = a * e - b * b;
  double s = denom > 0.0 ? clamp01((b * f - c * e) / denom) : 0.0;
  double t = (b * s + f) / e;
  if (t < 0.0) { t = 0.0; s = clamp01(-c / a); }
  else if (t > 1.0) { t = 1.0; s = clamp01((b - c) / a); }
  int ra = s <= 0.0 ? 0 : (s >= 1.0 ? 1 : 2), rb = t <= 0.0 ? 0 : (t >= 1.0 ? 1 : 2);
  v3 rv = {(a1.x + s * da.x) - (b1.x + t * db.x), (a1.y + s * da.y) - (b1.y + t * db.y),
           (a1.z + s * da.z) - (b1.z + t * db.z)};
  *d2 = dot3(rv, rv);
  g[0] = vscale(2.0 * (1.0 - s), rv); g[1] = vscale(2.0 * s, rv);
  g[2] = vscale(-2.0 * (1.0 - t), rv); g[3] = vscale(-2.0 * t, rv);
  *so = s; *to = t;
  return 3 * ra + rb;
}

static double cross_sq_one(v3 a1, v3 a2, v3 b1, v3 b2, v3 g[4]) {
  v3 u = vsub(a2, a1), v = vsub(b2, b1), w = cross3(u, v);
  v3 gu = cross3(v, w), gv = cross3(w, u);
  g[0] = vscale(-2.0, gu); g[1] = vscale(2.0, gu); g[2] = vscale(-2.0, gv); g[3] = vscale(2.0, gv);
  return dot3(w, w);
}

static double pe_one(v3 p, v3 e1, v3 e2, v3 g[3]) {
  v3 e = vsub(e2, e1), pe = vsub(p, e1);
  double ee = dot3_blas(e, e);
  double t = clamp01(dot3_blas(pe, e) / ee);
  v3 r = vsub(pe, vscale(t, e));
  g[0] = vscale(2.0, r); g[1] = vscale(-2.0 * (1.0 - t), r); g[2] = vscale(-2.0 * t, r);
  return dot3_blas(r, r);
}

static double pp_one(v3 a, v3 b, v3 g[2]) {
  v3 r = vsub(a, b);
  g[0] = vscale(2.0, r); g[1] = vscale(-2.0, r);
  return dot3_blas(r, r);
}

static void barrier_scalars(int form, double g, double S, double* b, double* bg, double* bgg) {
  double lg = log(g), om = 1.0 - g;
  if (form == 0) {
    *b = S * (om * om) * lg * lg;
    *bg = S * (-2.0 * om * lg * lg + 2.0 * (om * om) * lg / g);
    *bgg = S * (2.0 * lg * lg - 8.0 * om * lg / g + 2.0 * (om * om) * (1.0 - lg) / (g * g));
  } else {
    *b = -S * (om * om) * lg;
    *bg = S * (2.0 * om * lg - (om * om) / g);
    *bgg = S * (-2.0 * lg + om * (3.0 * g + 1.0) / (g * g));
  }
}

static double lambda1_at(int form, double g, double S) {
  double b, bg, bgg;
  barrier_scalars(form, g, S, &b, &bg, &bgg);
  return 4.0 * g * bgg + 2.0 * bg;
}

void oracle_pt_classify(int64_t n, const double* p, const double* t1, const double* t2, const double* t3,
                        int64_t* codes, double* d2, double* grad, double* w) {
  for (int64_t i = 0; i < n; ++i) {
    v3 g[4];
    codes[i] = pt_one(ld(p, i), ld(t1, i), ld(t2, i), ld(t3, i), &d2[i], g, &w[2 * i], &w[2 * i + 1]);
    memcpy(grad + 12 * i, g, sizeof(g));
  }
}

void oracle_ee_classify(int64_t n, const double* a1, const double* a2, const double* b1, const double* b2,
                        int64_t* codes, double* d2, double* grad, double* w) {
  for (int64_t i = 0; i < n; ++i) {
    v3 g[4];
    codes[i] = ee_one(ld(a1, i), ld(a2, i), ld(b1, i), ld(b2, i), &d2[i], g, &w[2 * i], &w[2 * i + 1]);
    memcpy(grad + 12 * i, g, sizeof(g));
  }
}

/* One table row: energy, status, gradient (3s) and block (3s x 3s) written densely at grad/hess. */
static void one_stencil(const oracle_params* prm, const double* pos, int kind, const int32_t* vid, int sub,
                        double eps, double* energy, uint8_t* status, double* grad, double* hess) {
  const int s = kind == K_PP ? 2 : (kind == K_PE ? 3 : 4);
  const int D = 3 * s;
  const int par = kind == K_EEP || kind == K_PEP || kind == K_PPP;
  v3 x[4], gd[4], rows[4], gc[4];
  for (int k = 0; k < s; ++k) x[k] = ld(pos, vid[k]);
  memset(gd, 0, sizeof(gd));
  double d2, w0, w1;
  int loc[4] = {sub & 3, (sub >> 2) & 3, (sub >> 4) & 3, (sub >> 6) & 3};
  switch (kind) {
    case K_PP: d2 = pp_one(x[0], x[1], gd); break;
    case K_PE: d2 = pe_one(x[0], x[1], x[2], gd); break;
    case K_PT: pt_one(x[0], x[1], x[2], x[3], &d2, gd, &w0, &w1); break;
    case K_EE: ee_one(x[0], x[1], x[2], x[3], &d2, gd, &w0, &w1); break;
    case K_EEP:
      ee_one(x[loc[0]], x[loc[1]], x[loc[2]], x[loc[3]], &d2, rows, &w0, &w1);
      for (int k = 0; k < 4; ++k) gd[loc[k]] = rows[k];
      break;
    case K_PEP:
      d2 = pe_one(x[loc[0]], x[loc[1]], x[loc[2]], rows);
      for (int k = 0; k < 3; ++k) gd[loc[k]] = rows[k];
      break;
    default:
      d2 = pp_one(x[loc[0]], x[loc[1]], rows);
      for (int k = 0; k < 2; ++k) gd[loc[k]] = rows[k];
  }
  const int st = d2 <= 0.0 ? 2 : (d2 >= prm->d_hat_pow2 ? 1 : 0);
  if (status) *status = (uint8_t)st;
  if (st != 0) {
    if (energy) *energy = 0.0;
    if (grad) memset(grad, 0, D * sizeof(double));
    if (hess) memset(hess, 0, D * D * sizeof(double));
    return;
  }
  const double d = sqrt(d2), f = d / prm->d_hat, den = 2.0 * d * prm->d_hat, g = f * f;
  double b, bg, bgg;
  barrier_scalars(prm->form, g, prm->scale, &b, &bg, &bgg);
  double en = 0.0;
  if (energy) {
    double eb, t1_, t2_;
    barrier_scalars(prm->form, d2 / prm->d_hat_pow2, prm->scale, &eb, &t1_, &t2_);
    en = eb;
  }
  double uf[12], uc[12], w[12], gr[12], lam;
  const double* gdp = (const double*)gd;
  for (int k = 0; k < D; ++k) uf[k] = gdp[k] / den;
  if (!par) {
    double l1 = 4.0 * g * bgg + 2.0 * bg;
    if (prm->use_filter && !(g >= prm->eps_g)) l1 = lambda1_at(prm->form, prm->eps_g, prm->scale);
    lam = l1 > 0.0 ? l1 : 0.0;
    const double coef = 2.0 * f * bg;
    for (int k = 0; k < D; ++k) { w[k] = uf[k]; gr[k] = coef * uf[k]; }
  } else {
    const double c = cross_sq_one(x[0], x[1], x[2], x[3], gc);
    const double sc = sqrt(c), cc = sc * sc;
    const double* gcp = (const double*)gc;
    for (int k = 0; k < 12; ++k) uc[k] = sc > 0.0 ? gcp[k] / (2.0 * sc) : 0.0;
    double e = 1.0, de = 0.0, d2e = 0.0;
    if (cc < eps) { e = -(cc * cc) / (eps * eps) + 2.0 * cc / eps; de = -2.0 * cc / (eps * eps) + 2.0 / eps; d2e = -2.0 / (eps * eps); }
    if (energy) en = (c < eps ? -(c * c) / (eps * eps) + 2.0 * c / eps : 1.0) * en;
    const double b_gamma = de * b, b_gamma2 = d2e * b, b_g = e * bg, b_g2 = e * bgg, b_gamma_g = de * bg;
    const double lg1 = 2.0 * (b_gamma + 2.0 * cc * b_gamma2), lf1 = 2.0 * (b_g + 2.0 * g * b_g2);
    const double t = b_gamma_g * sqrt(cc) * sqrt(g);
    const double dl = lg1 - lf1;
    const double p = 0.5 * sqrt(dl * dl + 64.0 * t * t);
    const double lam8 = 0.5 * (lg1 + lf1) + p;
    double qc, qf;
    if (fabs(8.0 * t) < 1e-12 * (fabs(lg1) + fabs(lf1)) || t == 0.0) { qc = lg1 >= lf1 ? 1.0 : 0.0; qf = 1.0 - qc; }
    else { const double k2 = (dl + 2.0 * p) / (8.0 * t), nrm = sqrt(k2 * k2 + 1.0); qc = k2 / nrm; qf = 1.0 / nrm; }
    lam = lam8 > 0.0 ? lam8 : 0.0;
    const double cgc = b_gamma * 2.0 * sc, cgf = b_g * 2.0 * f;
    for (int k = 0; k < 12; ++k) { w[k] = qc * uc[k] + qf * uf[k]; gr[k] = cgc * uc[k] + cgf * uf[k]; }
  }
  if (energy) *energy = en;
  if (grad) for (int k = 0; k < D; ++k) grad[k] = prm->dt2 * gr[k];
  if (hess)
    for (int r = 0; r < D; ++r)
      for (int c = 0; c < D; ++c) hess[r * D + c] = prm->dt2 * (lam * (w[r] * w[c]));
}

typedef struct {
  const oracle_params* prm; const double* positions; int kind; int64_t off;
  const int32_t* verts; const uint8_t* sub; const double* eps_x;
  double* energy; uint8_t* status; double* gb; double* hb; int D;
} kind_ctx;

static void kind_range(int64_t begin, int64_t end, void* arg) {
  const kind_ctx* c = (const kind_ctx*)arg;
  for (int64_t j = begin; j < end; ++j) {
    const int64_t i = c->off + j;
    one_stencil(c->prm, c->positions, c->kind, c->verts + 4 * i, c->sub ? c->sub[i] : 0, c->eps_x ? c->eps_x[i] : 0.0,
                c->energy ? c->energy + i : 0, c->status ? c->status + i : 0, c->gb ? c->gb + c->D * j : 0,
                c->hb ? c->hb + c->D * c->D * j : 0);
  }
}

/* Same contract as b200ipc_barrier_stencils (include/b200ipc.h), host pointers. */
int oracle_barrier_stencils(const oracle_params* prm, const double* positions, int64_t n, const int64_t* kind_off,
                            const int32_t* verts, const uint8_t* sub, const double* eps_x, double* energy,
                            uint8_t* status, double* grad2, double* hess2, double* grad3, double* hess3,
                            double* grad4, double* hess4) {
  const int fam4[5] = {K_EE, K_EEP, K_PEP, K_PPP, K_PT};
  int64_t row4[7] = {0, 0, 0, 0, 0, 0, 0}, acc = 0;
  for (int j = 0; j < 5; ++j) { row4[fam4[j]] = acc; acc += kind_off[fam4[j] + 1] - kind_off[fam4[j]]; }
  for (int k = 0; k < 7; ++k) {
    const int64_t off = kind_off[k], cnt = kind_off[k + 1] - off;
    const int s = k == K_PP ? 2 : (k == K_PE ? 3 : 4);
    const int D = 3 * s;
    double* gb = s == 2 ? grad2 : (s == 3 ? grad3 : (grad4 ? grad4 + 12 * row4[k] : 0));
    double* hb = s == 2 ? hess2 : (s == 3 ? hess3 : (hess4 ? hess4 + 144 * row4[k] : 0));
    kind_ctx c = {prm, positions, k, off, verts, sub, eps_x, energy, status, gb, hb, D};
    parallel_for(cnt, kind_range, &c);
  }
  return 0;
}

/* matvec_blocks (kernels/_core.pyx:222-247): serial block order, like the reference. */
void oracle_matvec_blocks(int64_t nb, int32_t s, const double* hess, const int64_t* vids, const double* x, double* out) {
  const int D = 3 * s;
  double xl[12], yl[12];
  for (int64_t b = 0; b < nb; ++b) {
    for (int v = 0; v < s; ++v)
      for (int i = 0; i < 3; ++i) xl[3 * v + i] = x[3 * vids[b * s + v] + i];
    for (int r = 0; r < D; ++r) {
      double a = 0.0;
      for (int c = 0; c < D; ++c) a += hess[(b * D + r) * D + c] * xl[c];
      yl[r] = a;
    }
    for (int v = 0; v < s; ++v)
      for (int i = 0; i < 3; ++i) out[3 * vids[b * s + v] + i] += yl[3 * v + i];
  }
}
