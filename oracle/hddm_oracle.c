/*
 * hddm_oracle.c -- single-threaded C restatement of the reference's DDM hot
 * path (arXiv 1807.04180, reference `helmddm`). TEST INFRASTRUCTURE ONLY: the
 * checker for the CUDA engine, never part of the product (see hddm_oracle.h).
 *
 * Every block cites the reference file:line whose behaviour it restates
 * (paths relative to /root/reference/proj). The arithmetic is written in the
 * same operation order as the reference so that, compiled with
 * -ffp-contract=off, results agree with the reference bit for bit on the pinned
 * configurations (tests/test_oracle_vs_ref.py); tolerances are still used in
 * the tests.
 */
#define _GNU_SOURCE
#include "hddm_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef double complex cplx;

static char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* orc_last_error(void) { return g_err; }

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

/* complex / real, component-wise (libstdc++ complex<double>::operator/=(double)) */
static inline cplx cdivr(cplx z, double t) { return CMPLX(creal(z) / t, cimag(z) / t); }
/* complex * real (component-wise, as complex<double> * double) */
static inline cplx cmulr(cplx z, double t) { return CMPLX(creal(z) * t, cimag(z) * t); }
/* |z|^2 as std::norm (x*x + y*y) */
static inline double cnorm(cplx z) { return creal(z) * creal(z) + cimag(z) * cimag(z); }

/* ---------------------------------------------------------------- geometry */
/* GridSpec, proj/include/helmddm/partition.hpp:13-31 */
typedef struct {
  double x0, y0, h;
  int mx, my, n1, n2, nov, nramp;
  int ext, gnx, gny, mcx, mcy;
} grid_t;

/* SubdomainWindow + BlendWeights, partition.hpp:39-58, partition.cpp:51-83 */
typedef struct {
  int i, j, cx0, cx1, cy0, cy1;
  int wx0, wy0, nx, ny;
  int lint, rint, bint, tint;
  double *wx, *wy;
  int own[4]; /* owned global node rect, ddm.cpp:90-94 */
} sub_t;

/* beta0 quintic taper, partition.cpp:7-11 */
static double beta0(double t) {
  if (t <= 0) return 1.0;
  if (t >= 1) return 0.0;
  return 1.0 - t * t * t * (10.0 - 15.0 * t + 6.0 * t * t);
}

/* axis_weights, partition.cpp:34-47 */
static void axis_weights(double* w, int o, int n, int c0, int c1, int lo_int,
                         int hi_int, int nov) {
  for (int t = 0; t < n; ++t) {
    const int p = o + t;
    double v = 1.0;
    if (p < c0)
      v = lo_int ? beta0((double)(c0 - 1 - p) / nov) : 1.0;
    else if (p > c1)
      v = hi_int ? beta0((double)(p - c1 - 1) / nov) : 1.0;
    w[t] = v;
  }
}

/* check_spec, partition.cpp:15-28 */
static int check_spec(const grid_t* g) {
  if (!(g->h > 0)) return fail(2, "grid spacing must be positive");
  if (g->mx < 1 || g->my < 1) return fail(2, "interior cell counts must be positive");
  if (g->n1 < 1 || g->n2 < 1) return fail(2, "subdomain counts must be positive");
  if (g->mx % g->n1 || g->my % g->n2)
    return fail(2, "interior cells must divide evenly among subdomains");
  if (g->nramp < 1) return fail(2, "absorber ramp width must be positive");
  if (g->nov < 0) return fail(2, "overlap width must be nonnegative");
  const int split = g->n1 > 1 || g->n2 > 1;
  if (split && g->nov < 1) return fail(2, "overlap width must be positive when the domain is split");
  if (split && (g->mx / g->n1 < g->nov + 1 || g->my / g->n2 < g->nov + 1))
    return fail(2, "subdomain cores too small for the requested overlap");
  return 0;
}

/* ------------------------------------------------------------------ medium */
/* MediumModel / eval_wavenumber, medium.hpp:17-38, medium.cpp:8-50.
 * kind 2 (lens) is this repo's extension for BASELINE config 3:
 * both coordinates are clamped into the interior. */
typedef struct {
  int kind;
  double omega, velocity;
  int nl;
  double *ylo, *yhi, *c;
  double bx0, bx1, by0, by1, margin;
  double lamp, lxc, lyc, lw;
  double cmin, cmax;
} medium_t;

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

static double lens_c(const medium_t* m, double xc, double yc) {
  const double dx = xc - m->lxc, dy = yc - m->lyc;
  return m->velocity - m->lamp * exp(-(dx * dx + dy * dy) / m->lw);
}

static int eval_k(const medium_t* m, double x, double y, double* k) {
  if (x < m->bx0 - m->margin || x > m->bx1 + m->margin || y < m->by0 - m->margin ||
      y > m->by1 + m->margin)
    return fail(1, "eval_wavenumber: point outside the padded domain");
  const double yc = clampd(y, m->by0, m->by1);
  double c;
  if (m->kind == 0) {
    c = m->velocity;
  } else if (m->kind == 1) {
    c = m->c[m->nl - 1];
    for (int l = 0; l < m->nl; ++l)
      if (yc <= m->yhi[l]) {
        c = m->c[l];
        break;
      }
  } else {
    c = lens_c(m, clampd(x, m->bx0, m->bx1), yc);
  }
  *k = m->omega / c;
  return 0;
}

/* -------------------------------------------------------------- operator */
/* DiscreteOperator, discretize.hpp:32-70 */
typedef struct {
  int x0, y0, nx, ny;
  double h;
  cplx *a1n, *ia1h, *a2n, *ia2h;
  double* k2;
} op_t;

/* shifted_sigma, pml.cpp:7-12 */
static double shifted_sigma(double s0, double d, double dsh, double t) {
  if (t <= dsh) return 0.0;
  if (t >= dsh + d) return s0;
  const double s = (t - dsh) / d;
  return s0 * s * s;
}

/* alpha_axis, discretize.cpp:21-37 */
static cplx alpha_axis(int m, int c0, int c1, int lo_int, int hi_int,
                       const grid_t* g, double sigma0) {
  const double h2 = 0.5 * g->h;
  const double d = g->nramp * g->h;
  double sig = 0;
  const int dl = 2 * c0 - m;
  if (dl > 0) sig += shifted_sigma(sigma0, d, lo_int ? g->nov * g->h : 0.0, dl * h2);
  const int dr = m - 2 * c1;
  if (dr > 0) sig += shifted_sigma(sigma0, d, hi_int ? g->nov * g->h : 0.0, dr * h2);
  return CMPLX(1.0, sig);
}

/* build_operator, discretize.cpp:41-79 */
static int build_op(op_t* op, const grid_t* g, int x0, int y0, int nx, int ny,
                    int cx0, int cx1, int cy0, int cy1, int li, int ri, int bi,
                    int ti, const medium_t* med, double sigma0) {
  op->x0 = x0;
  op->y0 = y0;
  op->nx = nx;
  op->ny = ny;
  op->h = g->h;
  op->a1n = xcalloc(nx, sizeof(cplx));
  op->ia1h = xcalloc(nx, sizeof(cplx));
  op->a2n = xcalloc(ny, sizeof(cplx));
  op->ia2h = xcalloc(ny, sizeof(cplx));
  op->k2 = xcalloc((size_t)nx * ny, sizeof(double));
  for (int lp = 0; lp < nx; ++lp) {
    const int m = 2 * (x0 + lp);
    op->a1n[lp] = alpha_axis(m, cx0, cx1, li, ri, g, sigma0);
    if (lp + 1 < nx) op->ia1h[lp] = CMPLX(1.0, 0.0) / alpha_axis(m + 1, cx0, cx1, li, ri, g, sigma0);
  }
  for (int lq = 0; lq < ny; ++lq) {
    const int m = 2 * (y0 + lq);
    op->a2n[lq] = alpha_axis(m, cy0, cy1, bi, ti, g, sigma0);
    if (lq + 1 < ny) op->ia2h[lq] = CMPLX(1.0, 0.0) / alpha_axis(m + 1, cy0, cy1, bi, ti, g, sigma0);
  }
  const double ox = g->x0 - g->ext * g->h, oy = g->y0 - g->ext * g->h;
  for (int lq = 0; lq < ny; ++lq) {
    const double y = oy + (y0 + lq) * g->h;
    for (int lp = 0; lp < nx; ++lp) {
      double k;
      if (eval_k(med, ox + (x0 + lp) * g->h, y, &k)) return 1;
      op->k2[(size_t)lq * nx + lp] = k * k;
    }
  }
  return 0;
}

static void free_op(op_t* op) {
  free(op->a1n);
  free(op->ia1h);
  free(op->a2n);
  free(op->ia2h);
  free(op->k2);
}

/* Field accessor for the stencil: buffer u covers local nodes
 * [ox, ox+stride) x [oy, ...) of the operator's window. */
typedef struct {
  const cplx* u;
  int stride, ox, oy;
} acc_t;
static inline cplx AT(const acc_t* a, int lp, int lq) {
  return a->u[(size_t)(lq - a->oy) * a->stride + (lp - a->ox)];
}

/* DiscreteOperator::stencil, discretize.hpp:43-54 (same operation order) */
static cplx stencil(const op_t* op, const acc_t* a, int lp, int lq) {
  const double ih2 = 1.0 / (op->h * op->h);
  const cplx uc = AT(a, lp, lq);
  const cplx ex = cmulr(op->a2n[lq], ih2);
  const cplx ey = cmulr(op->a1n[lp], ih2);
  const cplx t = ex * op->ia1h[lp] * (AT(a, lp + 1, lq) - uc) -
                 ex * op->ia1h[lp - 1] * (uc - AT(a, lp - 1, lq)) +
                 ey * op->ia2h[lq] * (AT(a, lp, lq + 1) - uc) -
                 ey * op->ia2h[lq - 1] * (uc - AT(a, lp, lq - 1));
  const cplx jac = op->a1n[lp] * op->a2n[lq];
  return t / jac + cmulr(uc, op->k2[(size_t)lq * op->nx + lp]);
}

/* DiscreteOperator::apply, discretize.cpp:81-96 */
static void op_apply(const op_t* op, const cplx* u, cplx* out) {
  const int nx = op->nx, ny = op->ny;
  acc_t a = {u, nx, 0, 0};
  for (int lq = 0; lq < ny; ++lq)
    for (int lp = 0; lp < nx; ++lp) {
      const size_t i = (size_t)lq * nx + lp;
      if (lp == 0 || lq == 0 || lp == nx - 1 || lq == ny - 1)
        out[i] = u[i];
      else
        out[i] = stencil(op, &a, lp, lq);
    }
}

/* ------------------------------------------------------------ sparse/CSR */
typedef struct {
  int n;
  int *rp, *ci;
  cplx* v;
} csr_t;

/* SparseMatrix::multiply, sparse.cpp:10-16 */
static void csr_mul(const csr_t* A, const cplx* x, cplx* y) {
  for (int r = 0; r < A->n; ++r) {
    cplx s = 0;
    for (int p = A->rp[r]; p < A->rp[r + 1]; ++p) s += A->v[p] * x[A->ci[p]];
    y[r] = s;
  }
}

/* DiscreteOperator::assemble, discretize.cpp:98-160: J-scaled rows, identity
 * ring rows, couplings into ring columns dropped, columns ascending. */
static void op_assemble(const op_t* op, csr_t* A) {
  const int nx = op->nx, ny = op->ny, n = nx * ny;
  const double ih2 = 1.0 / (op->h * op->h);
  A->n = n;
  A->rp = xcalloc(n + 1, sizeof(int));
  A->ci = xcalloc((size_t)5 * n, sizeof(int));
  A->v = xcalloc((size_t)5 * n, sizeof(cplx));
  int at = 0;
  for (int lq = 0; lq < ny; ++lq)
    for (int lp = 0; lp < nx; ++lp) {
      const int row = lq * nx + lp;
      if (lp == 0 || lq == 0 || lp == nx - 1 || lq == ny - 1) {
        A->ci[at] = row;
        A->v[at++] = 1.0;
        A->rp[row + 1] = at;
        continue;
      }
      const cplx ew = cmulr(op->a2n[lq] * op->ia1h[lp - 1], ih2);
      const cplx ee = cmulr(op->a2n[lq] * op->ia1h[lp], ih2);
      const cplx es = cmulr(op->a1n[lp] * op->ia2h[lq - 1], ih2);
      const cplx en = cmulr(op->a1n[lp] * op->ia2h[lq], ih2);
      const cplx jac = op->a1n[lp] * op->a2n[lq];
      const cplx diag = -(ew + ee + es + en) + cmulr(jac, op->k2[row]);
      if (lq > 1) { A->ci[at] = row - nx; A->v[at++] = es; }
      if (lp > 1) { A->ci[at] = row - 1; A->v[at++] = ew; }
      A->ci[at] = row; A->v[at++] = diag;
      if (lp < nx - 2) { A->ci[at] = row + 1; A->v[at++] = ee; }
      if (lq < ny - 2) { A->ci[at] = row + nx; A->v[at++] = en; }
      A->rp[row + 1] = at;
    }
}

static void free_csr(csr_t* A) {
  free(A->rp);
  free(A->ci);
  free(A->v);
}

/* grid_nd_order / nd_rec, sparse.cpp:20-57 */
static void nd_rec(int x0, int y0, int w, int h, int nx, int* out, int* k) {
  if (w <= 0 || h <= 0) return;
  if (w <= 6 && h <= 6) {
    for (int q = y0; q < y0 + h; ++q)
      for (int p = x0; p < x0 + w; ++p) out[(*k)++] = q * nx + p;
    return;
  }
  if (w >= h) {
    const int mid = x0 + w / 2;
    nd_rec(x0, y0, mid - x0, h, nx, out, k);
    nd_rec(mid + 1, y0, x0 + w - mid - 1, h, nx, out, k);
    for (int q = y0; q < y0 + h; ++q) out[(*k)++] = q * nx + mid;
  } else {
    const int mid = y0 + h / 2;
    nd_rec(x0, y0, w, mid - y0, nx, out, k);
    nd_rec(x0, mid + 1, w, y0 + h - mid - 1, nx, out, k);
    for (int p = x0; p < x0 + w; ++p) out[(*k)++] = mid * nx + p;
  }
}

int orc_nd_order(int nx, int ny, int* order) {
  int k = 0;
  if (nx <= 2 || ny <= 2) {
    for (int i = 0; i < nx * ny; ++i) order[k++] = i;
    return k;
  }
  for (int p = 0; p < nx; ++p) order[k++] = p;
  for (int q = 1; q < ny - 1; ++q) {
    order[k++] = q * nx;
    order[k++] = q * nx + nx - 1;
  }
  for (int p = 0; p < nx; ++p) order[k++] = (ny - 1) * nx + p;
  nd_rec(1, 1, nx - 2, ny - 2, nx, order, &k);
  return k;
}

/* Factorization (LDL^T branch), sparse.hpp:31-65 / sparse.cpp:76-303 */
typedef struct {
  int n;
  int *perm, *pinv, *Lp, *Li;
  cplx *Lx, *D;
  csr_t A;
  cplx *work, *res, *cor;
  double probe;
  long nnz;
} fact_t;

/* Up-looking unconjugated LDL^T of P A P^T, no pivoting (sparse.cpp:110-174).
 * Row k of L is a sparse triangular solve against the rows above it; the
 * elimination tree gives its nonzero pattern in topological order. */
static int ldlt_factor(fact_t* F) {
  const csr_t* A = &F->A;
  const int n = A->n;
  /* upper triangle of P A P^T by columns (build_upper, sparse.cpp:81-108) */
  int* Bp = xcalloc(n + 1, sizeof(int));
  for (int r = 0; r < n; ++r)
    for (int p = A->rp[r]; p < A->rp[r + 1]; ++p)
      if (F->pinv[r] <= F->pinv[A->ci[p]]) ++Bp[F->pinv[A->ci[p]] + 1];
  for (int k = 0; k < n; ++k) Bp[k + 1] += Bp[k];
  int* Bi = xcalloc(Bp[n], sizeof(int));
  cplx* Bx = xcalloc(Bp[n], sizeof(cplx));
  int* nxt = xcalloc(n, sizeof(int));
  memcpy(nxt, Bp, n * sizeof(int));
  for (int r = 0; r < n; ++r)
    for (int p = A->rp[r]; p < A->rp[r + 1]; ++p) {
      const int rn = F->pinv[r], cn = F->pinv[A->ci[p]];
      if (rn <= cn) {
        Bi[nxt[cn]] = rn;
        Bx[nxt[cn]++] = A->v[p];
      }
    }
  /* symbolic: elimination tree and column counts */
  int* parent = xcalloc(n, sizeof(int));
  int* cnt = xcalloc(n, sizeof(int));
  int* flag = xcalloc(n, sizeof(int));
  for (int k = 0; k < n; ++k) {
    parent[k] = -1;
    flag[k] = k;
    for (int p = Bp[k]; p < Bp[k + 1]; ++p)
      for (int i = Bi[p]; i < k && flag[i] != k; i = parent[i]) {
        if (parent[i] == -1) parent[i] = k;
        ++cnt[i];
        flag[i] = k;
      }
  }
  F->Lp = xcalloc(n + 1, sizeof(int));
  for (int k = 0; k < n; ++k) F->Lp[k + 1] = F->Lp[k] + cnt[k];
  F->Li = xcalloc(F->Lp[n], sizeof(int));
  F->Lx = xcalloc(F->Lp[n], sizeof(cplx));
  F->D = xcalloc(n, sizeof(cplx));
  /* numeric */
  cplx* y = xcalloc(n, sizeof(cplx));
  int* pat = xcalloc(n, sizeof(int));
  int* fill = xcalloc(n, sizeof(int));
  int ok = 1;
  for (int k = 0; k < n; ++k) flag[k] = -1;
  for (int k = 0; k < n && ok; ++k) {
    int top = n;
    flag[k] = k;
    for (int p = Bp[k]; p < Bp[k + 1]; ++p) {
      int i = Bi[p];
      y[i] += Bx[p];
      int len = 0;
      for (; flag[i] != k; i = parent[i]) {
        pat[len++] = i;
        flag[i] = k;
      }
      while (len > 0) pat[--top] = pat[--len];
    }
    F->D[k] = y[k];
    y[k] = 0;
    for (; top < n; ++top) {
      const int i = pat[top];
      const cplx yi = y[i];
      y[i] = 0;
      const int end = F->Lp[i] + fill[i];
      for (int p = F->Lp[i]; p < end; ++p) y[F->Li[p]] -= F->Lx[p] * yi;
      const cplx lki = yi / F->D[i];
      F->D[k] -= lki * yi;
      F->Li[end] = k;
      F->Lx[end] = lki;
      ++fill[i];
    }
    if (F->D[k] == 0) ok = 0;
  }
  free(Bp); free(Bi); free(Bx); free(nxt); free(parent); free(cnt);
  free(flag); free(y); free(pat); free(fill);
  F->nnz = (long)F->Lp[n] + n;
  return ok ? 0 : 1;
}

static double norm2v(const cplx* v, int n) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += cnorm(v[i]);
  return sqrt(s);
}

/* solve_raw, sparse.cpp:244-266 */
static void solve_raw(const fact_t* F, const cplx* b, cplx* x) {
  const int n = F->n;
  cplx* y = F->work;
  for (int k = 0; k < n; ++k) y[k] = b[F->perm[k]];
  for (int k = 0; k < n; ++k) {
    const cplx yk = y[k];
    for (int p = F->Lp[k]; p < F->Lp[k + 1]; ++p) y[F->Li[p]] -= F->Lx[p] * yk;
  }
  for (int k = 0; k < n; ++k) y[k] /= F->D[k];
  for (int k = n - 1; k >= 0; --k) {
    cplx s = y[k];
    for (int p = F->Lp[k]; p < F->Lp[k + 1]; ++p) s -= F->Lx[p] * y[F->Li[p]];
    y[k] = s;
  }
  for (int k = 0; k < n; ++k) x[F->perm[k]] = y[k];
}

/* diagnostics (test infrastructure): corrections taken and the largest first-pass
 * relative residual since the last orc_refine_stats(reset) */
static long g_ncorr = 0;
static double g_maxrel = 0;

void orc_refine_stats(long* ncorr, double* max_first_rel, int reset) {
  if (ncorr) *ncorr = g_ncorr;
  if (max_first_rel) *max_first_rel = g_maxrel;
  if (reset) {
    g_ncorr = 0;
    g_maxrel = 0;
  }
}

/* refine, sparse.cpp:268-292 */
static double refine(const fact_t* F, const cplx* b, cplx* x) {
  const int n = F->n;
  const double bn = norm2v(b, n);
  if (bn == 0) {
    memset(x, 0, n * sizeof(cplx));
    return 0;
  }
  solve_raw(F, b, x);
  double rel = -1;
  for (int it = 0; it < 12; ++it) {
    csr_mul(&F->A, x, F->res);
    for (int i = 0; i < n; ++i) F->res[i] = b[i] - F->res[i];
    const double r = norm2v(F->res, n) / bn;
    if (rel >= 0 && r >= 0.5 * rel) {
      if (r > rel)
        for (int i = 0; i < n; ++i) x[i] -= F->cor[i];
      return r < rel ? r : rel;
    }
    if (it == 0 && r > g_maxrel) g_maxrel = r;
    rel = r;
    if (rel <= 1e-11) return rel;
    ++g_ncorr;
    solve_raw(F, F->res, F->cor);
    for (int i = 0; i < n; ++i) x[i] += F->cor[i];
  }
  return rel;
}

/* Factorization::factor, sparse.cpp:203-236 (LU fallback -> SolveError) */
static int fact_factor(fact_t* F, int nx, int ny) {
  const int n = F->A.n;
  F->n = n;
  F->perm = xcalloc(n, sizeof(int));
  F->pinv = xcalloc(n, sizeof(int));
  orc_nd_order(nx, ny, F->perm);
  for (int k = 0; k < n; ++k) F->pinv[F->perm[k]] = k;
  F->work = xcalloc(n, sizeof(cplx));
  F->res = xcalloc(n, sizeof(cplx));
  F->cor = xcalloc(n, sizeof(cplx));
  if (ldlt_factor(F)) return fail(3, "LDL^T breakdown (zero pivot); no LU fallback");
  cplx* b = xcalloc(n, sizeof(cplx));
  cplx* x = xcalloc(n, sizeof(cplx));
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double re = (double)(s >> 11) * 0x1.0p-52 - 1.0;
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double im = (double)(s >> 11) * 0x1.0p-52 - 1.0;
    b[i] = CMPLX(re, im);
  }
  F->probe = refine(F, b, x);
  free(b);
  free(x);
  if (!(F->probe <= 1e-10)) return fail(3, "LDL^T probe residual above 1e-10; no LU fallback");
  return 0;
}

static void free_fact(fact_t* F) {
  free(F->perm); free(F->pinv); free(F->Lp); free(F->Li); free(F->Lx);
  free(F->D); free(F->work); free(F->res); free(F->cor);
  free_csr(&F->A);
}

/* ------------------------------------------------------------------ engine */
struct orc_engine {
  grid_t g;
  medium_t med;
  double sigma0;
  op_t gop;
  int nsub, ncls;
  sub_t* subs;
  int* class_of;
  int* members;
  op_t* cop; /* per class */
  fact_t* cf;
  int wnx, wny, nw;
  cplx **curr, **prev1, **prev2, **rhs, **wbuf;
  char *zc, *zp1, *zp2;
  cplx* assembled;
  cplx* tmp;
  int last_active_valid;
};

static int ops_equal(const op_t* a, const op_t* b) {
  return a->nx == b->nx && a->ny == b->ny &&
         !memcmp(a->a1n, b->a1n, a->nx * sizeof(cplx)) &&
         !memcmp(a->ia1h, b->ia1h, (a->nx - 1) * sizeof(cplx)) &&
         !memcmp(a->a2n, b->a2n, a->ny * sizeof(cplx)) &&
         !memcmp(a->ia2h, b->ia2h, (a->ny - 1) * sizeof(cplx)) &&
         !memcmp(a->k2, b->k2, (size_t)a->nx * a->ny * sizeof(double));
}

void orc_destroy(orc_engine* e) {
  if (!e) return;
  for (int t = 0; t < e->nsub; ++t) {
    free(e->subs[t].wx);
    free(e->subs[t].wy);
    if (e->curr) { free(e->curr[t]); free(e->prev1[t]); free(e->prev2[t]); free(e->rhs[t]); free(e->wbuf[t]); }
  }
  for (int c = 0; c < e->ncls; ++c) {
    free_op(&e->cop[c]);
    free_fact(&e->cf[c]);
  }
  free(e->cop); free(e->cf); free(e->subs); free(e->class_of); free(e->members);
  free(e->curr); free(e->prev1); free(e->prev2); free(e->rhs); free(e->wbuf);
  free(e->zc); free(e->zp1); free(e->zp2); free(e->assembled); free(e->tmp);
  free_op(&e->gop);
  free(e->med.ylo); free(e->med.yhi); free(e->med.c);
  free(e);
}

/* DdmEngine::DdmEngine + build_classes, ddm.cpp:62-138 */
int orc_create(const orc_problem* p, orc_engine** out) {
  *out = NULL;
  orc_engine* e = xcalloc(1, sizeof *e);
  grid_t* g = &e->g;
  g->x0 = p->x0; g->y0 = p->y0; g->h = p->h;
  g->mx = p->mx; g->my = p->my; g->n1 = p->n1; g->n2 = p->n2;
  g->nov = p->n_overlap; g->nramp = p->n_ramp;
  int rc = check_spec(g);
  if (rc) { free(e); return rc; }
  g->ext = g->nov + g->nramp;
  g->gnx = g->mx + 2 * g->ext + 1;
  g->gny = g->my + 2 * g->ext + 1;
  g->mcx = g->mx / g->n1;
  g->mcy = g->my / g->n2;

  medium_t* m = &e->med;
  m->kind = p->medium_kind;
  m->omega = p->omega;
  m->velocity = p->velocity;
  m->nl = p->n_layers;
  m->ylo = xcalloc(m->nl, sizeof(double));
  m->yhi = xcalloc(m->nl, sizeof(double));
  m->c = xcalloc(m->nl, sizeof(double));
  for (int l = 0; l < m->nl; ++l) {
    m->ylo[l] = p->layer_ylo[l];
    m->yhi[l] = p->layer_yhi[l];
    m->c[l] = p->layer_c[l];
  }
  m->bx0 = g->x0; m->bx1 = g->x0 + g->mx * g->h;
  m->by0 = g->y0; m->by1 = g->y0 + g->my * g->h;
  m->margin = (g->ext + 1) * g->h; /* ddm.cpp:66-67 */
  m->lamp = p->lens_amp; m->lxc = p->lens_xc; m->lyc = p->lens_yc; m->lw = p->lens_w;
  /* c_min / c_max, medium.cpp:8-20; lens: extremes over clamped lattice nodes */
  if (m->kind == 0) {
    m->cmin = m->cmax = m->velocity;
  } else if (m->kind == 1) {
    if (m->nl < 1) { orc_destroy(e); return fail(2, "layered medium needs layers"); }
    m->cmin = m->cmax = m->c[0];
    for (int l = 0; l < m->nl; ++l) {
      if (m->c[l] < m->cmin) m->cmin = m->c[l];
      if (m->c[l] > m->cmax) m->cmax = m->c[l];
    }
  } else {
    const double ox = g->x0 - g->ext * g->h, oy = g->y0 - g->ext * g->h;
    m->cmin = INFINITY;
    m->cmax = -INFINITY;
    for (int q = 0; q < g->gny; ++q)
      for (int pp = 0; pp < g->gnx; ++pp) {
        const double c = lens_c(m, clampd(ox + pp * g->h, m->bx0, m->bx1),
                                clampd(oy + q * g->h, m->by0, m->by1));
        if (c < m->cmin) m->cmin = c;
        if (c > m->cmax) m->cmax = c;
      }
  }
  const double kmin = m->omega / m->cmax;
  e->sigma0 = p->sigma0 > 0 ? p->sigma0
                            : 3.0 * p->c_sigma / (kmin * (g->nramp * g->h)); /* pml.cpp:14-16 */
  /* global operator with global_layout (discretize.cpp:11-14) */
  if (build_op(&e->gop, g, 0, 0, g->gnx, g->gny, g->ext, g->ext + g->mx, g->ext,
               g->ext + g->my, 0, 0, 0, 0, m, e->sigma0)) {
    orc_destroy(e);
    return 1;
  }
  /* partition */
  e->nsub = g->n1 * g->n2;
  e->subs = xcalloc(e->nsub, sizeof(sub_t));
  for (int j = 0; j < g->n2; ++j)
    for (int i = 0; i < g->n1; ++i) {
      sub_t* s = &e->subs[j * g->n1 + i];
      s->i = i; s->j = j;
      s->cx0 = g->ext + i * g->mcx; s->cx1 = s->cx0 + g->mcx;
      s->cy0 = g->ext + j * g->mcy; s->cy1 = s->cy0 + g->mcy;
      s->wx0 = s->cx0 - g->ext; s->wy0 = s->cy0 - g->ext;
      s->nx = g->mcx + 2 * g->ext + 1; s->ny = g->mcy + 2 * g->ext + 1;
      s->lint = i > 0; s->rint = i < g->n1 - 1;
      s->bint = j > 0; s->tint = j < g->n2 - 1;
      s->wx = xcalloc(s->nx, sizeof(double));
      s->wy = xcalloc(s->ny, sizeof(double));
      axis_weights(s->wx, s->wx0, s->nx, s->cx0, s->cx1, s->lint, s->rint, g->nov);
      axis_weights(s->wy, s->wy0, s->ny, s->cy0, s->cy1, s->bint, s->tint, g->nov);
      s->own[0] = i == 0 ? 0 : g->ext + i * g->mcx + 1;
      s->own[1] = i == g->n1 - 1 ? g->gnx - 1 : g->ext + (i + 1) * g->mcx;
      s->own[2] = j == 0 ? 0 : g->ext + j * g->mcy + 1;
      s->own[3] = j == g->n2 - 1 ? g->gny - 1 : g->ext + (j + 1) * g->mcy;
    }
  e->wnx = e->subs[0].nx;
  e->wny = e->subs[0].ny;
  e->nw = e->wnx * e->wny;
  /* classes: bitwise-identical coefficient arrays share a factorization */
  e->class_of = xcalloc(e->nsub, sizeof(int));
  e->members = xcalloc(e->nsub, sizeof(int));
  e->cop = xcalloc(e->nsub, sizeof(op_t));
  e->cf = xcalloc(e->nsub, sizeof(fact_t));
  for (int t = 0; t < e->nsub; ++t) {
    const sub_t* s = &e->subs[t];
    op_t op;
    if (build_op(&op, g, s->wx0, s->wy0, s->nx, s->ny, s->cx0, s->cx1, s->cy0,
                 s->cy1, s->lint, s->rint, s->bint, s->tint, m, e->sigma0)) {
      free_op(&op);
      orc_destroy(e);
      return 1;
    }
    int cls = -1;
    for (int c = 0; c < e->ncls && cls < 0; ++c)
      if (ops_equal(&e->cop[c], &op)) cls = c;
    if (cls < 0) {
      cls = e->ncls++;
      e->cop[cls] = op;
    } else {
      free_op(&op);
    }
    e->class_of[t] = cls;
    ++e->members[cls];
  }
  const double t0 = now_ms();
  for (int c = 0; c < e->ncls; ++c) {
    op_assemble(&e->cop[c], &e->cf[c].A);
    rc = fact_factor(&e->cf[c], e->cop[c].nx, e->cop[c].ny);
    if (rc) {
      /* keep remaining classes freeable */
      for (int c2 = c + 1; c2 < e->ncls; ++c2) op_assemble(&e->cop[c2], &e->cf[c2].A);
      orc_destroy(e);
      return rc;
    }
  }
  (void)t0;
  e->curr = xcalloc(e->nsub, sizeof(cplx*));
  e->prev1 = xcalloc(e->nsub, sizeof(cplx*));
  e->prev2 = xcalloc(e->nsub, sizeof(cplx*));
  e->rhs = xcalloc(e->nsub, sizeof(cplx*));
  e->wbuf = xcalloc(e->nsub, sizeof(cplx*));
  for (int t = 0; t < e->nsub; ++t) {
    e->curr[t] = xcalloc(e->nw, sizeof(cplx));
    e->prev1[t] = xcalloc(e->nw, sizeof(cplx));
    e->prev2[t] = xcalloc(e->nw, sizeof(cplx));
    e->rhs[t] = xcalloc(e->nw, sizeof(cplx));
    e->wbuf[t] = xcalloc((size_t)(e->wnx + 2) * (e->wny + 2), sizeof(cplx));
  }
  e->zc = xcalloc(e->nsub, 1);
  e->zp1 = xcalloc(e->nsub, 1);
  e->zp2 = xcalloc(e->nsub, 1);
  e->assembled = xcalloc((size_t)g->gnx * g->gny, sizeof(cplx));
  e->tmp = xcalloc((size_t)g->gnx * g->gny, sizeof(cplx));
  *out = e;
  return 0;
}

long orc_n_global(const orc_engine* e) { return (long)e->g.gnx * e->g.gny; }
double orc_sigma0(const orc_engine* e) { return e->sigma0; }
int orc_num_classes(const orc_engine* e) { return e->ncls; }
int orc_class_of(const orc_engine* e, int t) { return t >= 0 && t < e->nsub ? e->class_of[t] : -1; }
int orc_window_dims(const orc_engine* e, int* nx, int* ny) {
  *nx = e->wnx;
  *ny = e->wny;
  return 0;
}

int orc_class_info(const orc_engine* e, int c, int* members, long* nnz,
                   double* probe, int* is_ldlt) {
  if (c < 0 || c >= e->ncls) return 1;
  *members = e->members[c];
  *nnz = e->cf[c].nnz;
  *probe = e->cf[c].probe;
  *is_ldlt = 1;
  return 0;
}

int orc_class_solve(const orc_engine* e, int c, const double* b, double* x,
                    double* relres) {
  if (c < 0 || c >= e->ncls) return 1;
  const double r = refine(&e->cf[c], (const cplx*)b, (cplx*)x);
  if (relres) *relres = r;
  return 0;
}

int orc_apply_global(const orc_engine* e, const double* u, double* out) {
  op_apply(&e->gop, (const cplx*)u, (cplx*)out);
  return 0;
}

/* transfer_patch, transfer.cpp:7-62 */
static void transfer_patch(int d, const sub_t* t, int nov, int* bx) {
  const int ix0 = t->wx0 + 1, ix1 = t->wx0 + t->nx - 2;
  const int iy0 = t->wy0 + 1, iy1 = t->wy0 + t->ny - 2;
  int p0 = ix0, p1 = ix1, q0 = iy0, q1 = iy1;
  const int fromL = d == 1 || d == 5 || d == 7; /* Right, DownRight, UpRight */
  const int fromR = d == 0 || d == 4 || d == 6; /* Left, DownLeft, UpLeft */
  const int fromB = d == 3 || d == 6 || d == 7; /* Up, UpLeft, UpRight */
  const int fromT = d == 2 || d == 4 || d == 5; /* Down, DownLeft, DownRight */
  if (fromL) { p0 = t->cx0 + 1; p1 = t->cx0 + 1 + nov; }
  if (fromR) { p0 = t->cx1 - 1 - nov; p1 = t->cx1 - 1; }
  if (fromB) { q0 = t->cy0 + 1; q1 = t->cy0 + 1 + nov; }
  if (fromT) { q0 = t->cy1 - 1 - nov; q1 = t->cy1 - 1; }
  bx[0] = p0 > ix0 ? p0 : ix0;
  bx[1] = p1 < ix1 ? p1 : ix1;
  bx[2] = q0 > iy0 ? q0 : iy0;
  bx[3] = q1 < iy1 ? q1 : iy1;
}

/* transfer_beta, partition.cpp:131-152 */
static double transfer_beta(int d, const sub_t* t, int nov, int p, int q) {
  const double fl = beta0((double)(p - t->cx0 - 1) / nov);
  const double fr = beta0((double)(t->cx1 - 1 - p) / nov);
  const double fb = beta0((double)(q - t->cy0 - 1) / nov);
  const double fa = beta0((double)(t->cy1 - 1 - q) / nov);
  switch (d) {
    case 0: return fr;
    case 1: return fl;
    case 2: return fa;
    case 3: return fb;
    case 4: return fr * fa;
    case 5: return fl * fa;
    case 6: return fr * fb;
    case 7: return fl * fb;
  }
  return 0.0;
}

/* add_transfer, transfer.cpp:64-88: acc -= L_t(beta_d v) on the patch, v read
 * as zero outside the source window. */
static void add_transfer(int d, const op_t* op, const sub_t* t, int nov,
                         const sub_t* src, const cplx* v, cplx* acc, cplx* w) {
  int b[4];
  transfer_patch(d, t, nov, b);
  if (b[1] < b[0] || b[3] < b[2]) return;
  const int wx0 = b[0] - 1, wy0 = b[2] - 1;
  const int wnx = b[1] - b[0] + 3, wny = b[3] - b[2] + 3;
  for (int q = wy0; q < wy0 + wny; ++q)
    for (int p = wx0; p < wx0 + wnx; ++p) {
      cplx vv = 0;
      if (p >= src->wx0 && p < src->wx0 + src->nx && q >= src->wy0 && q < src->wy0 + src->ny)
        vv = v[(size_t)(q - src->wy0) * src->nx + (p - src->wx0)];
      w[(size_t)(q - wy0) * wnx + (p - wx0)] =
          vv != 0 ? cmulr(vv, transfer_beta(d, t, nov, p, q)) : 0;
    }
  acc_t a = {w, wnx, wx0 - t->wx0, wy0 - t->wy0};
  for (int q = b[2]; q <= b[3]; ++q)
    for (int p = b[0]; p <= b[1]; ++p)
      acc[(size_t)(q - t->wy0) * t->nx + (p - t->wx0)] -=
          stencil(op, &a, p - t->wx0, q - t->wy0);
}

/* kGatherOrder / source_offset, partition.hpp:74-76, partition.cpp:99-111 */
static const int kDI[8] = {+1, -1, 0, 0, +1, -1, +1, -1};
static const int kDJ[8] = {0, 0, +1, -1, +1, +1, -1, -1};

/* accumulate_weighted, ddm.cpp:216-235 */
static void accumulate(orc_engine* e, int t) {
  const sub_t* s = &e->subs[t];
  const int nov = e->g.nov, gnx = e->g.gnx;
  const int x0 = s->lint ? s->cx0 - nov : s->wx0;
  const int x1 = s->rint ? s->cx1 + nov : s->wx0 + s->nx - 1;
  const int y0 = s->bint ? s->cy0 - nov : s->wy0;
  const int y1 = s->tint ? s->cy1 + nov : s->wy0 + s->ny - 1;
  const cplx* u = e->curr[t];
  for (int q = y0; q <= y1; ++q) {
    const double wy = s->wy[q - s->wy0];
    if (wy == 0) continue;
    for (int p = x0; p <= x1; ++p) {
      const double w = s->wx[p - s->wx0] * wy;
      if (w != 0)
        e->assembled[(size_t)q * gnx + p] +=
            cmulr(u[(size_t)(q - s->wy0) * s->nx + (p - s->wx0)], w);
    }
  }
}

/* DdmEngine::sweep, ddm.cpp:174-214 */
static void sweep(orc_engine* e, int step, const cplx* f, orc_stats* st) {
  const grid_t* g = &e->g;
  for (int t = 0; t < e->nsub; ++t) {
    const sub_t* s = &e->subs[t];
    cplx* rhs = e->rhs[t];
    memset(rhs, 0, e->nw * sizeof(cplx));
    int any = 0;
    if (step == 1 && f) { /* restrict_owned, ddm.cpp:159-172 */
      for (int q = s->own[2]; q <= s->own[3]; ++q)
        for (int p = s->own[0]; p <= s->own[1]; ++p) {
          const cplx val = f[(size_t)q * g->gnx + p];
          if (val != 0) {
            rhs[(size_t)(q - s->wy0) * s->nx + (p - s->wx0)] = val;
            any = 1;
          }
        }
    }
    const op_t* op = &e->cop[e->class_of[t]];
    for (int d = 0; d < 8; ++d) {
      const int si = s->i + kDI[d], sj = s->j + kDJ[d];
      if (si < 0 || si >= g->n1 || sj < 0 || sj >= g->n2) continue;
      const int src = sj * g->n1 + si;
      const int corner = d >= 4;
      if ((corner ? e->zp2 : e->zp1)[src]) continue;
      add_transfer(d, op, s, g->nov, &e->subs[src],
                   corner ? e->prev2[src] : e->prev1[src], rhs, e->wbuf[t]);
      any = 1;
    }
    if (!any) {
      e->zc[t] = 1;
      continue;
    }
    e->zc[t] = 0;
    /* scale_rhs in place, discretize.cpp:162-172 */
    for (int lq = 0; lq < s->ny; ++lq)
      for (int lp = 0; lp < s->nx; ++lp) {
        const size_t i = (size_t)lq * s->nx + lp;
        if (lp == 0 || lq == 0 || lp == s->nx - 1 || lq == s->ny - 1)
          rhs[i] = 0;
        else
          rhs[i] = (op->a1n[lp] * op->a2n[lq]) * rhs[i];
      }
    refine(&e->cf[e->class_of[t]], rhs, e->curr[t]);
  }
  for (int t = 0; t < e->nsub; ++t) {
    if (e->zc[t]) ++st->skipped; else ++st->solves;
  }
  for (int t = 0; t < e->nsub; ++t)
    if (!e->zc[t]) accumulate(e, t);
  /* rotate prev2 <- prev1 <- curr (ddm.cpp:210-213) */
  cplx** tp = e->prev2; e->prev2 = e->prev1; e->prev1 = tp;
  tp = e->prev1; e->prev1 = e->curr; e->curr = tp;
  char* tz = e->zp2; e->zp2 = e->zp1; e->zp1 = tz;
  tz = e->zp1; e->zp1 = e->zc; e->zc = tz;
  e->last_active_valid = 1;
}

/* reset_state, ddm.cpp:152-157 */
static void reset_state(orc_engine* e) {
  memset(e->zc, 1, e->nsub);
  memset(e->zp1, 1, e->nsub);
  memset(e->zp2, 1, e->nsub);
  memset(e->assembled, 0, (size_t)e->g.gnx * e->g.gny * sizeof(cplx));
  e->last_active_valid = 0;
}

/* residual_norm, ddm.cpp:237-242 */
static double residual_norm(orc_engine* e, const cplx* f) {
  op_apply(&e->gop, e->assembled, e->tmp);
  const size_t n = (size_t)e->g.gnx * e->g.gny;
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += cnorm(f[i] - e->tmp[i]);
  return sqrt(s);
}

/* solve_iterative, ddm.cpp:244-278 */
int orc_solve_iterative(orc_engine* e, const double* fd, double tol,
                        int max_steps, int check_every, double* out,
                        orc_stats* st, int* hist_step, double* hist_rel,
                        int hist_cap, int* hist_len) {
  const cplx* f = (const cplx*)fd;
  const size_t n = (size_t)e->g.gnx * e->g.gny;
  if (check_every < 1) check_every = 1;
  memset(st, 0, sizeof *st);
  st->relres = -1;
  reset_state(e);
  double b2 = 0;
  for (size_t i = 0; i < n; ++i) b2 += cnorm(f[i]);
  const double bnorm = sqrt(b2);
  int nh = 0;
  if (bnorm == 0) {
    st->converged = 1;
    st->relres = 0;
    memset(out, 0, n * sizeof(cplx));
    if (hist_len) *hist_len = 0;
    return 0;
  }
  for (int s = 1; s <= max_steps; ++s) {
    const double t0 = now_ms();
    sweep(e, s, f, st);
    st->steps = s;
    if (s % check_every == 0 || s == max_steps) {
      const double rel = residual_norm(e, f) / bnorm;
      if (nh < hist_cap) {
        hist_step[nh] = s;
        hist_rel[nh] = rel;
      }
      ++nh;
      st->sweep_ms += now_ms() - t0;
      st->relres = rel;
      if (rel <= tol) {
        st->converged = 1;
        break;
      }
    } else {
      st->sweep_ms += now_ms() - t0;
    }
  }
  if (hist_len) *hist_len = nh;
  memcpy(out, e->assembled, n * sizeof(cplx));
  return 0;
}

/* precondition, ddm.cpp:280-287 (stats accumulate across calls) */
int orc_precondition(orc_engine* e, const double* r, double* z, int k,
                     orc_stats* st) {
  reset_state(e);
  const double t0 = now_ms();
  for (int s = 1; s <= k; ++s) sweep(e, s, (const cplx*)r, st);
  st->sweep_ms += now_ms() - t0;
  memcpy(z, e->assembled, (size_t)e->g.gnx * e->g.gny * sizeof(cplx));
  return 0;
}

int orc_tap_subdomain(const orc_engine* e, int t, double* rhs, double* u,
                      int* active) {
  if (t < 0 || t >= e->nsub || !e->last_active_valid) return 1;
  /* after the rotation the latest solution sits in prev1, its flag in zp1 */
  memcpy(rhs, e->rhs[t], e->nw * sizeof(cplx));
  memcpy(u, e->prev1[t], e->nw * sizeof(cplx));
  *active = !e->zp1[t];
  return 0;
}

/* --------------------------------------------------------------- fgmres */
static double vnrm2(const cplx* v, size_t n) {
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += cnorm(v[i]);
  return sqrt(s);
}
static cplx vdot(const cplx* a, const cplx* b, size_t n) {
  cplx s = 0;
  for (size_t i = 0; i < n; ++i) s += conj(a[i]) * b[i];
  return s;
}

/* fgmres, krylov.cpp:24-133, over caller operators A and M (ctx-bound); the
 * 2-D engine wires A = apply_global and M = precondition(K) (cli.cpp:217-222),
 * the 3-D extension (hddm_oracle3.c) its own pair. zs (optional) receives each
 * preconditioner output. */
typedef void (*orc_op_fn)(void* ctx, const cplx* in, cplx* out);
static int fgmres_core(size_t n, orc_op_fn Aop, orc_op_fn Mop, void* ctx,
                       const double* bd, double* xd, double tol, int max_iters,
                       int restart, orc_fgmres_out* res, double* hist, int hist_cap,
                       double* zs, int zs_cap) {
  const cplx* b = (const cplx*)bd;
  cplx* x = (cplx*)xd;
  const double tstart = now_ms();
  memset(res, 0, sizeof *res);
  res->relres = res->true_relres = -1;
  memset(x, 0, n * sizeof(cplx));
  const double bnorm = vnrm2(b, n);
  if (bnorm == 0) {
    res->converged = 1;
    res->relres = res->true_relres = 0;
    return 0;
  }
  int mcap = restart > 0 ? restart : max_iters;
  if (mcap < 1) mcap = 1;
  cplx* r = xcalloc(n, sizeof(cplx));
  memcpy(r, b, n * sizeof(cplx));
  cplx** V = xcalloc(mcap + 1, sizeof(cplx*));
  cplx** Z = xcalloc(mcap, sizeof(cplx*));
  for (int i = 0; i <= mcap; ++i) V[i] = xcalloc(n, sizeof(cplx));
  for (int i = 0; i < mcap; ++i) Z[i] = xcalloc(n, sizeof(cplx));
  cplx* H = xcalloc((size_t)mcap * (mcap + 1), sizeof(cplx)); /* H[j*(mcap+1)+i] */
  cplx* g = xcalloc(mcap + 1, sizeof(cplx));
  cplx* sn = xcalloc(mcap, sizeof(cplx));
  double* cs = xcalloc(mcap, sizeof(double));
  cplx* y = xcalloc(mcap, sizeof(cplx));
  int total = 0, stop = 0, nz = 0;
  while (!stop && total < max_iters) {
    const int m = restart > 0 ? (restart < max_iters - total ? restart : max_iters - total)
                              : max_iters - total;
    const double rnorm = vnrm2(r, n);
    if (rnorm == 0) {
      res->converged = 1;
      break;
    }
    for (int i = 0; i <= m; ++i) g[i] = 0;
    memset(H, 0, (size_t)mcap * (mcap + 1) * sizeof(cplx));
    for (size_t t = 0; t < n; ++t) V[0][t] = cdivr(r[t], rnorm);
    g[0] = rnorm;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      Mop(ctx, V[j], Z[j]);
      if (zs && nz < zs_cap) memcpy(zs + 2 * n * (size_t)nz, Z[j], n * sizeof(cplx));
      ++nz;
      cplx* w = V[j + 1];
      Aop(ctx, Z[j], w);
      cplx* Hj = H + (size_t)j * (mcap + 1);
      for (int i = 0; i <= j; ++i) {
        const cplx hij = vdot(V[i], w, n);
        Hj[i] = hij;
        for (size_t t = 0; t < n; ++t) w[t] -= hij * V[i][t];
      }
      const double hlast = vnrm2(w, n);
      Hj[j + 1] = hlast;
      for (int i = 0; i < j; ++i) {
        const cplx a = Hj[i], c = Hj[i + 1];
        Hj[i] = cmulr(a, cs[i]) + sn[i] * c;
        Hj[i + 1] = -conj(sn[i]) * a + cmulr(c, cs[i]);
      }
      const cplx a = Hj[j], c = Hj[j + 1];
      const double tt = sqrt(cnorm(a) + cnorm(c));
      if (tt == 0) {
        stop = 1;
        break;
      }
      if (a == 0) {
        cs[j] = 0;
        sn[j] = cdivr(conj(c), cabs(c));
      } else {
        cs[j] = cabs(a) / tt;
        sn[j] = cdivr(cdivr(a, cabs(a)) * conj(c), tt);
      }
      Hj[j] = cmulr(a, cs[j]) + sn[j] * c;
      Hj[j + 1] = 0;
      g[j + 1] = -conj(sn[j]) * g[j];
      g[j] = cmulr(g[j], cs[j]);
      ++total;
      k = j + 1;
      res->relres = cabs(g[j + 1]) / bnorm;
      if (total - 1 < hist_cap) hist[total - 1] = res->relres;
      if (res->relres <= tol) {
        res->converged = 1;
        stop = 1;
        break;
      }
      if (hlast == 0) {
        stop = 1;
        break;
      }
      for (size_t t = 0; t < n; ++t) w[t] = cdivr(w[t], hlast);
    }
    if (k > 0) {
      for (int i = k - 1; i >= 0; --i) {
        cplx s = g[i];
        for (int l = i + 1; l < k; ++l) s -= H[(size_t)l * (mcap + 1) + i] * y[l];
        y[i] = s / H[(size_t)i * (mcap + 1) + i];
      }
      for (int l = 0; l < k; ++l)
        for (size_t t = 0; t < n; ++t) x[t] += y[l] * Z[l][t];
    }
    if (!stop) {
      Aop(ctx, x, r);
      for (size_t t = 0; t < n; ++t) r[t] = b[t] - r[t];
    }
  }
  res->iters = total;
  Aop(ctx, x, r);
  double s = 0;
  for (size_t t = 0; t < n; ++t) s += cnorm(b[t] - r[t]);
  res->true_relres = sqrt(s) / bnorm;
  res->wall_ms = now_ms() - tstart;
  for (int i = 0; i <= mcap; ++i) free(V[i]);
  for (int i = 0; i < mcap; ++i) free(Z[i]);
  free(V); free(Z); free(H); free(g); free(sn); free(cs); free(y); free(r);
  return 0;
}

typedef struct {
  orc_engine* e;
  int K;
  orc_stats* pst;
} fgm2_ctx;
static void fgm2_A(void* c, const cplx* in, cplx* out) {
  op_apply(&((fgm2_ctx*)c)->e->gop, in, out);
}
static void fgm2_M(void* c, const cplx* in, cplx* out) {
  fgm2_ctx* x = (fgm2_ctx*)c;
  orc_precondition(x->e, (const double*)in, (double*)out, x->K, x->pst);
}

int orc_fgmres(orc_engine* e, const double* bd, double* xd, double tol,
               int max_iters, int restart, int K, orc_fgmres_out* res,
               double* hist, int hist_cap, double* zs, int zs_cap,
               orc_stats* pst) {
  memset(pst, 0, sizeof *pst);
  fgm2_ctx c = {e, K, pst};
  return fgmres_core((size_t)e->g.gnx * e->g.gny, fgm2_A, fgm2_M, &c, bd, xd, tol,
                     max_iters, restart, res, hist, hist_cap, zs, zs_cap);
}

/* the 3-D extension (BASELINE config 5; no reference exists) */
#include "hddm_oracle3.c"
