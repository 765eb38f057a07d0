/*
 * hddm_oracle3.c -- the 3-D extension of the restatement (BASELINE config 5).
 * TEST INFRASTRUCTURE ONLY (see hddm_oracle.h); compiled as part of
 * hddm_oracle.c (included at its end, sharing its static helpers).
 *
 * PARITY UNPINNED: the reference has no 3-D code
 * says the 2-D algorithm "can be straightforwardly generalized" with 3^3-1 = 26
 * transfer directions and N1+N2+N3 steps. This file is that generalization,
 * written as the 2-D restatement with one more axis, and it is the
 * specification the GPU engine's 3-D path (paper_1807_04180_b200/csrc/*3d*)
 * is checked against:
 *
 *  * GridSpec / windows / blend weights: every per-axis rule of
 *    partition.cpp:15-83 applied to x, y and z; weight = (wx * wy) * wz.
 *  * Operator: L u = J^-1 div(A grad u) + k^2 u, A = diag(a2a3/a1, a1a3/a2,
 *    a1a2/a3), J = a1 a2 a3 (discretize.hpp:32-54 with a third stretch);
 *    alpha_axis per axis (discretize.cpp:21-37). The J-scaled assembled matrix
 *    has off-diagonals (a_j a_k) * inv_a_half * h^-2 and diagonal
 *    -(w + e + s + n + b + t) + k^2 J: symmetric bit for bit, as in 2-D.
 *  * Elimination order: the window's boundary shell first (identity rows, in
 *    natural order), then nested dissection of the interior box: the longest
 *    axis is cut at its middle plane (ties x, then y, then z), halves first,
 *    the plane last; boxes of at most 3 nodes per side are leaves in natural
 *    order (sparse.cpp:20-57 with planes for lines).
 *  * Factor / solve / refine: the 2-D restatement's up-looking LDL^T,
 *    solve_raw and refine (sparse.cpp:110-292) unchanged.
 *  * Transfers: direction = source offset (ox, oy, oz) in {-1,0,1}^3 \ 0. Per
 *    axis with o = +1 the patch is [c1-1-nov, c1-1] and the taper
 *    beta0((c1-1-p)/nov), with o = -1 [c0+1, c0+1+nov] and beta0((p-c0-1)/nov)
 *    (transfer.cpp:7-62, partition.cpp:131-152); taper = bx, *= by, *= bz over
 *    the axes that move. Faces read the source's step s-1 solution, edges
 *    s-2, vertices s-3 (four rotating buffers, ddm.cpp:210-213 with one more).
 *    Gather order: the 6 faces (+x,-x,+y,-y,+z,-z), the 12 edges (xy, xz, yz
 *    planes, each in the order (+,+),(-,+),(+,-),(-,-)), the 8 vertices
 *    ((+,+,+),(-,+,+),(+,-,+),(-,-,+),(+,+,-),(-,+,-),(+,-,-),(-,-,-))
 *    -- kGatherOrder's pattern (partition.hpp:74-76) per plane.
 *  * restrict_owned / accumulate / residual / solve_iterative / precondition /
 *    fgmres: ddm.cpp:159-287 and krylov.cpp:24-133 with the third axis.
 *  * Medium: constant velocity (config 5 is constant-medium).
 */

/* ---------------------------------------------------------------- geometry */
typedef struct {
  double x0, y0, z0, h;
  int m[3], n[3], nov, nramp;
  int ext, gn[3], mc[3];
} grid3_t;

typedef struct {
  int ix[3];      /* subdomain index per axis */
  int c0[3], c1[3];
  int w0[3], nn[3];
  int lo[3], hi[3];  /* interior-facing sides */
  double* w[3];
  int own0[3], own1[3];
} sub3_t;

static int check_spec3(const grid3_t* g) {
  if (!(g->h > 0)) return fail(2, "grid spacing must be positive");
  for (int a = 0; a < 3; ++a)
    if (g->m[a] < 1) return fail(2, "interior cell counts must be positive");
  for (int a = 0; a < 3; ++a)
    if (g->n[a] < 1) return fail(2, "subdomain counts must be positive");
  for (int a = 0; a < 3; ++a)
    if (g->m[a] % g->n[a]) return fail(2, "interior cells must divide evenly among subdomains");
  if (g->nramp < 1) return fail(2, "absorber ramp width must be positive");
  if (g->nov < 0) return fail(2, "overlap width must be nonnegative");
  const int split = g->n[0] > 1 || g->n[1] > 1 || g->n[2] > 1;
  if (split && g->nov < 1) return fail(2, "overlap width must be positive when the domain is split");
  for (int a = 0; a < 3; ++a)
    if (split && g->m[a] / g->n[a] < g->nov + 1)
      return fail(2, "subdomain cores too small for the requested overlap");
  return 0;
}

/* -------------------------------------------------------------- operator */
typedef struct {
  int o[3], nn[3];
  double h;
  cplx *an[3], *iah[3];
  double* k2;
} op3_t;

static cplx alpha_axis3(int m, int c0, int c1, int lo, int hi, const grid3_t* g, double sigma0) {
  const double h2 = 0.5 * g->h;
  const double d = g->nramp * g->h;
  double sig = 0;
  const int dl = 2 * c0 - m;
  if (dl > 0) sig += shifted_sigma(sigma0, d, lo ? g->nov * g->h : 0.0, dl * h2);
  const int dr = m - 2 * c1;
  if (dr > 0) sig += shifted_sigma(sigma0, d, hi ? g->nov * g->h : 0.0, dr * h2);
  return CMPLX(1.0, sig);
}

static void build_op3(op3_t* op, const grid3_t* g, const int* o, const int* nn, const int* c0,
                      const int* c1, const int* lo, const int* hi, double k2c, double sigma0) {
  op->h = g->h;
  for (int a = 0; a < 3; ++a) {
    op->o[a] = o[a];
    op->nn[a] = nn[a];
    op->an[a] = xcalloc(nn[a], sizeof(cplx));
    op->iah[a] = xcalloc(nn[a], sizeof(cplx));
    for (int l = 0; l < nn[a]; ++l) {
      const int m = 2 * (o[a] + l);
      op->an[a][l] = alpha_axis3(m, c0[a], c1[a], lo[a], hi[a], g, sigma0);
      if (l + 1 < nn[a]) op->iah[a][l] = CMPLX(1.0, 0.0) / alpha_axis3(m + 1, c0[a], c1[a], lo[a], hi[a], g, sigma0);
    }
  }
  const size_t n = (size_t)nn[0] * nn[1] * nn[2];
  op->k2 = xcalloc(n, sizeof(double));
  for (size_t i = 0; i < n; ++i) op->k2[i] = k2c;
}

static void free_op3(op3_t* op) {
  for (int a = 0; a < 3; ++a) {
    free(op->an[a]);
    free(op->iah[a]);
  }
  free(op->k2);
}

static int ops3_equal(const op3_t* a, const op3_t* b) {
  for (int x = 0; x < 3; ++x)
    if (a->nn[x] != b->nn[x] || memcmp(a->an[x], b->an[x], a->nn[x] * sizeof(cplx)) ||
        memcmp(a->iah[x], b->iah[x], (a->nn[x] - 1) * sizeof(cplx)))
      return 0;
  return !memcmp(a->k2, b->k2, (size_t)a->nn[0] * a->nn[1] * a->nn[2] * sizeof(double));
}

/* field accessor over a box [o, o+len) of window-local nodes */
typedef struct {
  const cplx* u;
  int o[3], len[3];
} acc3_t;
static inline cplx AT3(const acc3_t* a, int p, int q, int r) {
  return a->u[((size_t)(r - a->o[2]) * a->len[1] + (q - a->o[1])) * a->len[0] + (p - a->o[0])];
}

/* the L-form 7-point stencil at an interior node (discretize.hpp:43-54, + z) */
static cplx stencil3(const op3_t* op, const acc3_t* a, int p, int q, int r) {
  const double ih2 = 1.0 / (op->h * op->h);
  const cplx* a1 = op->an[0];
  const cplx* a2 = op->an[1];
  const cplx* a3 = op->an[2];
  const cplx uc = AT3(a, p, q, r);
  const cplx ex = cmulr(a2[q] * a3[r], ih2);
  const cplx ey = cmulr(a1[p] * a3[r], ih2);
  const cplx ez = cmulr(a1[p] * a2[q], ih2);
  const cplx t = ex * op->iah[0][p] * (AT3(a, p + 1, q, r) - uc) -
                 ex * op->iah[0][p - 1] * (uc - AT3(a, p - 1, q, r)) +
                 ey * op->iah[1][q] * (AT3(a, p, q + 1, r) - uc) -
                 ey * op->iah[1][q - 1] * (uc - AT3(a, p, q - 1, r)) +
                 ez * op->iah[2][r] * (AT3(a, p, q, r + 1) - uc) -
                 ez * op->iah[2][r - 1] * (uc - AT3(a, p, q, r - 1));
  const cplx jac = a1[p] * a2[q] * a3[r];
  return t / jac + cmulr(uc, op->k2[((size_t)r * op->nn[1] + q) * op->nn[0] + p]);
}

static int on_shell3(const int* nn, int p, int q, int r) {
  return p == 0 || q == 0 || r == 0 || p == nn[0] - 1 || q == nn[1] - 1 || r == nn[2] - 1;
}

static void op3_apply(const op3_t* op, const cplx* u, cplx* out) {
  const int* nn = op->nn;
  acc3_t a = {u, {0, 0, 0}, {nn[0], nn[1], nn[2]}};
  for (int r = 0; r < nn[2]; ++r)
    for (int q = 0; q < nn[1]; ++q)
      for (int p = 0; p < nn[0]; ++p) {
        const size_t i = ((size_t)r * nn[1] + q) * nn[0] + p;
        out[i] = on_shell3(nn, p, q, r) ? u[i] : stencil3(op, &a, p, q, r);
      }
}

/* J-scaled assembled matrix, columns ascending (discretize.cpp:98-160, + z) */
static void op3_assemble(const op3_t* op, csr_t* A) {
  const int nx = op->nn[0], ny = op->nn[1], nz = op->nn[2];
  const int n = nx * ny * nz, sxy = nx * ny;
  const double ih2 = 1.0 / (op->h * op->h);
  const cplx* a1 = op->an[0];
  const cplx* a2 = op->an[1];
  const cplx* a3 = op->an[2];
  A->n = n;
  A->rp = xcalloc(n + 1, sizeof(int));
  A->ci = xcalloc((size_t)7 * n, sizeof(int));
  A->v = xcalloc((size_t)7 * n, sizeof(cplx));
  int at = 0;
  for (int r = 0; r < nz; ++r)
    for (int q = 0; q < ny; ++q)
      for (int p = 0; p < nx; ++p) {
        const int row = (r * ny + q) * nx + p;
        if (on_shell3(op->nn, p, q, r)) {
          A->ci[at] = row;
          A->v[at++] = 1.0;
          A->rp[row + 1] = at;
          continue;
        }
        const cplx yz = a2[q] * a3[r], xz = a1[p] * a3[r], xy = a1[p] * a2[q];
        const cplx cw = cmulr(yz * op->iah[0][p - 1], ih2);
        const cplx ce = cmulr(yz * op->iah[0][p], ih2);
        const cplx cs = cmulr(xz * op->iah[1][q - 1], ih2);
        const cplx cn = cmulr(xz * op->iah[1][q], ih2);
        const cplx cb = cmulr(xy * op->iah[2][r - 1], ih2);
        const cplx ct = cmulr(xy * op->iah[2][r], ih2);
        const cplx jac = a1[p] * a2[q] * a3[r];
        const cplx diag = -(cw + ce + cs + cn + cb + ct) + cmulr(jac, op->k2[row]);
        if (r > 1) { A->ci[at] = row - sxy; A->v[at++] = cb; }
        if (q > 1) { A->ci[at] = row - nx; A->v[at++] = cs; }
        if (p > 1) { A->ci[at] = row - 1; A->v[at++] = cw; }
        A->ci[at] = row; A->v[at++] = diag;
        if (p < nx - 2) { A->ci[at] = row + 1; A->v[at++] = ce; }
        if (q < ny - 2) { A->ci[at] = row + nx; A->v[at++] = cn; }
        if (r < nz - 2) { A->ci[at] = row + sxy; A->v[at++] = ct; }
        A->rp[row + 1] = at;
      }
}

/* ------------------------------------------------------- 3-D ND ordering */
#define ORC3_LEAF 3
static void nd3_rec(int x0, int y0, int z0, int w, int h, int d, int nx, int ny, int* out, int* k) {
  if (w <= 0 || h <= 0 || d <= 0) return;
  if (w <= ORC3_LEAF && h <= ORC3_LEAF && d <= ORC3_LEAF) {
    for (int r = z0; r < z0 + d; ++r)
      for (int q = y0; q < y0 + h; ++q)
        for (int p = x0; p < x0 + w; ++p) out[(*k)++] = (r * ny + q) * nx + p;
    return;
  }
  if (w >= h && w >= d) {
    const int mid = x0 + w / 2;
    nd3_rec(x0, y0, z0, mid - x0, h, d, nx, ny, out, k);
    nd3_rec(mid + 1, y0, z0, x0 + w - mid - 1, h, d, nx, ny, out, k);
    for (int r = z0; r < z0 + d; ++r)
      for (int q = y0; q < y0 + h; ++q) out[(*k)++] = (r * ny + q) * nx + mid;
  } else if (h >= d) {
    const int mid = y0 + h / 2;
    nd3_rec(x0, y0, z0, w, mid - y0, d, nx, ny, out, k);
    nd3_rec(x0, mid + 1, z0, w, y0 + h - mid - 1, d, nx, ny, out, k);
    for (int r = z0; r < z0 + d; ++r)
      for (int p = x0; p < x0 + w; ++p) out[(*k)++] = (r * ny + mid) * nx + p;
  } else {
    const int mid = z0 + d / 2;
    nd3_rec(x0, y0, z0, w, h, mid - z0, nx, ny, out, k);
    nd3_rec(x0, y0, mid + 1, w, h, z0 + d - mid - 1, nx, ny, out, k);
    for (int q = y0; q < y0 + h; ++q)
      for (int p = x0; p < x0 + w; ++p) out[(*k)++] = (mid * ny + q) * nx + p;
  }
}

int orc3_nd_order(int nx, int ny, int nz, int* order) {
  int k = 0;
  const int nn[3] = {nx, ny, nz};
  if (nx <= 2 || ny <= 2 || nz <= 2) {
    for (int i = 0; i < nx * ny * nz; ++i) order[k++] = i;
    return k;
  }
  for (int r = 0; r < nz; ++r)
    for (int q = 0; q < ny; ++q)
      for (int p = 0; p < nx; ++p)
        if (on_shell3(nn, p, q, r)) order[k++] = (r * ny + q) * nx + p;
  nd3_rec(1, 1, 1, nx - 2, ny - 2, nz - 2, nx, ny, order, &k);
  return k;
}

static int fact3_factor(fact_t* F, int nx, int ny, int nz) {
  const int n = F->A.n;
  F->n = n;
  F->perm = xcalloc(n, sizeof(int));
  F->pinv = xcalloc(n, sizeof(int));
  orc3_nd_order(nx, ny, nz, F->perm);
  for (int k = 0; k < n; ++k) F->pinv[F->perm[k]] = k;
  F->work = xcalloc(n, sizeof(cplx));
  F->res = xcalloc(n, sizeof(cplx));
  F->cor = xcalloc(n, sizeof(cplx));
  if (ldlt_factor(F)) return fail(3, "LDL^T breakdown (zero pivot); no LU fallback");
  /* the probe of sparse.cpp:218-227 */
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

/* ------------------------------------------------------------------ engine */
struct orc3_engine {
  grid3_t g;
  double omega, velocity, sigma0;
  op3_t gop;
  int nsub, ncls;
  sub3_t* subs;
  int* class_of;
  int* members;
  op3_t* cop;
  fact_t* cf;
  int nn[3], nw;
  cplx **curr, **prev[3], **rhs, *wbuf;
  char *zc, *zp[3];
  cplx *assembled, *tmp;
  int last_valid;
};

void orc3_destroy(orc3_engine* e) {
  if (!e) return;
  for (int t = 0; t < e->nsub; ++t) {
    for (int a = 0; a < 3; ++a) free(e->subs[t].w[a]);
    if (e->curr) {
      free(e->curr[t]);
      for (int k = 0; k < 3; ++k) free(e->prev[k][t]);
      free(e->rhs[t]);
    }
  }
  for (int c = 0; c < e->ncls; ++c) {
    free_op3(&e->cop[c]);
    free_fact(&e->cf[c]);
  }
  free(e->cop); free(e->cf); free(e->subs); free(e->class_of); free(e->members);
  free(e->curr);
  for (int k = 0; k < 3; ++k) { free(e->prev[k]); free(e->zp[k]); }
  free(e->rhs); free(e->wbuf); free(e->zc); free(e->assembled); free(e->tmp);
  free_op3(&e->gop);
  free(e);
}

int orc3_create(const orc3_problem* p, orc3_engine** out) {
  *out = NULL;
  orc3_engine* e = xcalloc(1, sizeof *e);
  grid3_t* g = &e->g;
  g->x0 = p->x0; g->y0 = p->y0; g->z0 = p->z0; g->h = p->h;
  g->m[0] = p->mx; g->m[1] = p->my; g->m[2] = p->mz;
  g->n[0] = p->n1; g->n[1] = p->n2; g->n[2] = p->n3;
  g->nov = p->n_overlap; g->nramp = p->n_ramp;
  int rc = check_spec3(g);
  if (rc) { free(e); return rc; }
  if (!(p->velocity > 0) || !(p->omega > 0)) { free(e); return fail(2, "velocity and omega must be positive"); }
  g->ext = g->nov + g->nramp;
  for (int a = 0; a < 3; ++a) {
    g->gn[a] = g->m[a] + 2 * g->ext + 1;
    g->mc[a] = g->m[a] / g->n[a];
  }
  e->omega = p->omega;
  e->velocity = p->velocity;
  const double kmin = p->omega / p->velocity;
  e->sigma0 = p->sigma0 > 0 ? p->sigma0 : 3.0 * p->c_sigma / (kmin * (g->nramp * g->h));
  const double k2c = kmin * kmin;
  {
    const int o[3] = {0, 0, 0};
    const int c0[3] = {g->ext, g->ext, g->ext};
    const int c1[3] = {g->ext + g->m[0], g->ext + g->m[1], g->ext + g->m[2]};
    const int z[3] = {0, 0, 0};
    build_op3(&e->gop, g, o, g->gn, c0, c1, z, z, k2c, e->sigma0);
  }
  e->nsub = g->n[0] * g->n[1] * g->n[2];
  e->subs = xcalloc(e->nsub, sizeof(sub3_t));
  for (int t = 0; t < e->nsub; ++t) {
    sub3_t* s = &e->subs[t];
    s->ix[0] = t % g->n[0];
    s->ix[1] = (t / g->n[0]) % g->n[1];
    s->ix[2] = t / (g->n[0] * g->n[1]);
    for (int a = 0; a < 3; ++a) {
      const int i = s->ix[a];
      s->c0[a] = g->ext + i * g->mc[a];
      s->c1[a] = s->c0[a] + g->mc[a];
      s->w0[a] = s->c0[a] - g->ext;
      s->nn[a] = g->mc[a] + 2 * g->ext + 1;
      s->lo[a] = i > 0;
      s->hi[a] = i < g->n[a] - 1;
      s->w[a] = xcalloc(s->nn[a], sizeof(double));
      axis_weights(s->w[a], s->w0[a], s->nn[a], s->c0[a], s->c1[a], s->lo[a], s->hi[a], g->nov);
      s->own0[a] = i == 0 ? 0 : g->ext + i * g->mc[a] + 1;
      s->own1[a] = i == g->n[a] - 1 ? g->gn[a] - 1 : g->ext + (i + 1) * g->mc[a];
    }
  }
  for (int a = 0; a < 3; ++a) e->nn[a] = e->subs[0].nn[a];
  e->nw = e->nn[0] * e->nn[1] * e->nn[2];
  e->class_of = xcalloc(e->nsub, sizeof(int));
  e->members = xcalloc(e->nsub, sizeof(int));
  e->cop = xcalloc(e->nsub, sizeof(op3_t));
  e->cf = xcalloc(e->nsub, sizeof(fact_t));
  for (int t = 0; t < e->nsub; ++t) {
    const sub3_t* s = &e->subs[t];
    op3_t op;
    build_op3(&op, g, s->w0, s->nn, s->c0, s->c1, s->lo, s->hi, k2c, e->sigma0);
    int cls = -1;
    for (int c = 0; c < e->ncls && cls < 0; ++c)
      if (ops3_equal(&e->cop[c], &op)) cls = c;
    if (cls < 0) {
      cls = e->ncls++;
      e->cop[cls] = op;
    } else {
      free_op3(&op);
    }
    e->class_of[t] = cls;
    ++e->members[cls];
  }
  for (int c = 0; c < e->ncls; ++c) op3_assemble(&e->cop[c], &e->cf[c].A);
  for (int c = 0; c < e->ncls; ++c) {
    rc = fact3_factor(&e->cf[c], e->nn[0], e->nn[1], e->nn[2]);
    if (rc) {
      orc3_destroy(e);
      return rc;
    }
  }
  e->curr = xcalloc(e->nsub, sizeof(cplx*));
  for (int k = 0; k < 3; ++k) {
    e->prev[k] = xcalloc(e->nsub, sizeof(cplx*));
    e->zp[k] = xcalloc(e->nsub, 1);
  }
  e->rhs = xcalloc(e->nsub, sizeof(cplx*));
  for (int t = 0; t < e->nsub; ++t) {
    e->curr[t] = xcalloc(e->nw, sizeof(cplx));
    for (int k = 0; k < 3; ++k) e->prev[k][t] = xcalloc(e->nw, sizeof(cplx));
    e->rhs[t] = xcalloc(e->nw, sizeof(cplx));
  }
  e->wbuf = xcalloc((size_t)(e->nn[0] + 2) * (e->nn[1] + 2) * (e->nn[2] + 2), sizeof(cplx));
  e->zc = xcalloc(e->nsub, 1);
  const size_t ng = (size_t)g->gn[0] * g->gn[1] * g->gn[2];
  e->assembled = xcalloc(ng, sizeof(cplx));
  e->tmp = xcalloc(ng, sizeof(cplx));
  *out = e;
  return 0;
}

long orc3_n_global(const orc3_engine* e) { return (long)e->g.gn[0] * e->g.gn[1] * e->g.gn[2]; }
double orc3_sigma0(const orc3_engine* e) { return e->sigma0; }
int orc3_num_classes(const orc3_engine* e) { return e->ncls; }
int orc3_class_of(const orc3_engine* e, int t) { return t >= 0 && t < e->nsub ? e->class_of[t] : -1; }
int orc3_window_dims(const orc3_engine* e, int* nn) {
  for (int a = 0; a < 3; ++a) nn[a] = e->nn[a];
  return 0;
}
int orc3_class_info(const orc3_engine* e, int c, int* members, long* nnz, double* probe) {
  if (c < 0 || c >= e->ncls) return 1;
  *members = e->members[c];
  *nnz = e->cf[c].nnz;
  *probe = e->cf[c].probe;
  return 0;
}
int orc3_class_solve(const orc3_engine* e, int c, const double* b, double* x, double* relres) {
  if (c < 0 || c >= e->ncls) return 1;
  const double r = refine(&e->cf[c], (const cplx*)b, (cplx*)x);
  if (relres) *relres = r;
  return 0;
}
int orc3_apply_global(const orc3_engine* e, const double* u, double* out) {
  op3_apply(&e->gop, (const cplx*)u, (cplx*)out);
  return 0;
}
/* the class's assembled matrix times x (window-local natural order) */
int orc3_class_matvec(const orc3_engine* e, int c, const double* x, double* y) {
  if (c < 0 || c >= e->ncls) return 1;
  csr_mul(&e->cf[c].A, (const cplx*)x, (cplx*)y);
  return 0;
}

/* gather order: 6 faces, 12 edges, 8 vertices (header comment) */
static const int kO3[26][3] = {
    {+1, 0, 0}, {-1, 0, 0}, {0, +1, 0}, {0, -1, 0}, {0, 0, +1}, {0, 0, -1},
    {+1, +1, 0}, {-1, +1, 0}, {+1, -1, 0}, {-1, -1, 0},
    {+1, 0, +1}, {-1, 0, +1}, {+1, 0, -1}, {-1, 0, -1},
    {0, +1, +1}, {0, -1, +1}, {0, +1, -1}, {0, -1, -1},
    {+1, +1, +1}, {-1, +1, +1}, {+1, -1, +1}, {-1, -1, +1},
    {+1, +1, -1}, {-1, +1, -1}, {+1, -1, -1}, {-1, -1, -1}};

int orc3_direction(int d, int* o) {
  if (d < 0 || d >= 26) return 1;
  for (int a = 0; a < 3; ++a) o[a] = kO3[d][a];
  return 0;
}

/* patch box (global nodes, inclusive) of direction d on target t */
static void transfer_patch3(const int* o, const sub3_t* t, int nov, int* lo, int* hi) {
  for (int a = 0; a < 3; ++a) {
    const int i0 = t->w0[a] + 1, i1 = t->w0[a] + t->nn[a] - 2;
    int p0 = i0, p1 = i1;
    if (o[a] > 0) { p0 = t->c1[a] - 1 - nov; p1 = t->c1[a] - 1; }
    if (o[a] < 0) { p0 = t->c0[a] + 1; p1 = t->c0[a] + 1 + nov; }
    lo[a] = p0 > i0 ? p0 : i0;
    hi[a] = p1 < i1 ? p1 : i1;
  }
}

static double transfer_beta3(const int* o, const sub3_t* t, int nov, const int* P) {
  double b = 1.0;
  int first = 1;
  for (int a = 0; a < 3; ++a) {
    if (!o[a]) continue;
    const double v = o[a] > 0 ? beta0((double)(t->c1[a] - 1 - P[a]) / nov)
                              : beta0((double)(P[a] - t->c0[a] - 1) / nov);
    b = first ? v : b * v;
    first = 0;
  }
  return b;
}

static void add_transfer3(const int* o, const op3_t* op, const sub3_t* t, int nov,
                          const sub3_t* src, const cplx* v, cplx* acc, cplx* w) {
  int lo[3], hi[3];
  transfer_patch3(o, t, nov, lo, hi);
  for (int a = 0; a < 3; ++a)
    if (hi[a] < lo[a]) return;
  int wo[3], wl[3];
  for (int a = 0; a < 3; ++a) {
    wo[a] = lo[a] - 1;
    wl[a] = hi[a] - lo[a] + 3;
  }
  for (int r = 0; r < wl[2]; ++r)
    for (int q = 0; q < wl[1]; ++q)
      for (int p = 0; p < wl[0]; ++p) {
        const int P[3] = {wo[0] + p, wo[1] + q, wo[2] + r};
        int in = 1;
        for (int a = 0; a < 3; ++a) in &= P[a] >= src->w0[a] && P[a] < src->w0[a] + src->nn[a];
        cplx vv = 0;
        if (in)
          vv = v[((size_t)(P[2] - src->w0[2]) * src->nn[1] + (P[1] - src->w0[1])) * src->nn[0] +
                 (P[0] - src->w0[0])];
        w[((size_t)r * wl[1] + q) * wl[0] + p] = vv != 0 ? cmulr(vv, transfer_beta3(o, t, nov, P)) : 0;
      }
  acc3_t a = {w, {wo[0] - t->w0[0], wo[1] - t->w0[1], wo[2] - t->w0[2]}, {wl[0], wl[1], wl[2]}};
  for (int r = lo[2]; r <= hi[2]; ++r)
    for (int q = lo[1]; q <= hi[1]; ++q)
      for (int p = lo[0]; p <= hi[0]; ++p) {
        const int lp = p - t->w0[0], lq = q - t->w0[1], lr = r - t->w0[2];
        acc[((size_t)lr * t->nn[1] + lq) * t->nn[0] + lp] -= stencil3(op, &a, lp, lq, lr);
      }
}

static void accumulate3(orc3_engine* e, int t) {
  const sub3_t* s = &e->subs[t];
  const int nov = e->g.nov;
  const int* gn = e->g.gn;
  int x0[3], x1[3];
  for (int a = 0; a < 3; ++a) {
    x0[a] = s->lo[a] ? s->c0[a] - nov : s->w0[a];
    x1[a] = s->hi[a] ? s->c1[a] + nov : s->w0[a] + s->nn[a] - 1;
  }
  const cplx* u = e->curr[t];
  for (int r = x0[2]; r <= x1[2]; ++r) {
    const double wz = s->w[2][r - s->w0[2]];
    if (wz == 0) continue;
    for (int q = x0[1]; q <= x1[1]; ++q) {
      const double wy = s->w[1][q - s->w0[1]];
      if (wy == 0) continue;
      for (int p = x0[0]; p <= x1[0]; ++p) {
        const double w = s->w[0][p - s->w0[0]] * wy * wz;
        if (w != 0)
          e->assembled[((size_t)r * gn[1] + q) * gn[0] + p] +=
              cmulr(u[((size_t)(r - s->w0[2]) * s->nn[1] + (q - s->w0[1])) * s->nn[0] + (p - s->w0[0])], w);
      }
    }
  }
}

static void sweep3(orc3_engine* e, int step, const cplx* f, orc_stats* st) {
  const grid3_t* g = &e->g;
  const int* gn = g->gn;
  for (int t = 0; t < e->nsub; ++t) {
    const sub3_t* s = &e->subs[t];
    cplx* rhs = e->rhs[t];
    memset(rhs, 0, e->nw * sizeof(cplx));
    int any = 0;
    if (step == 1 && f) {
      for (int r = s->own0[2]; r <= s->own1[2]; ++r)
        for (int q = s->own0[1]; q <= s->own1[1]; ++q)
          for (int p = s->own0[0]; p <= s->own1[0]; ++p) {
            const cplx val = f[((size_t)r * gn[1] + q) * gn[0] + p];
            if (val != 0) {
              rhs[((size_t)(r - s->w0[2]) * s->nn[1] + (q - s->w0[1])) * s->nn[0] + (p - s->w0[0])] = val;
              any = 1;
            }
          }
    }
    const op3_t* op = &e->cop[e->class_of[t]];
    for (int d = 0; d < 26; ++d) {
      const int* o = kO3[d];
      int si[3], okk = 1;
      for (int a = 0; a < 3; ++a) {
        si[a] = s->ix[a] + o[a];
        okk &= si[a] >= 0 && si[a] < g->n[a];
      }
      if (!okk) continue;
      const int src = (si[2] * g->n[1] + si[1]) * g->n[0] + si[0];
      const int lag = (o[0] != 0) + (o[1] != 0) + (o[2] != 0);  /* 1 face, 2 edge, 3 vertex */
      if (e->zp[lag - 1][src]) continue;
      add_transfer3(o, op, s, g->nov, &e->subs[src], e->prev[lag - 1][src], rhs, e->wbuf);
      any = 1;
    }
    if (!any) {
      e->zc[t] = 1;
      continue;
    }
    e->zc[t] = 0;
    for (int r = 0; r < s->nn[2]; ++r)
      for (int q = 0; q < s->nn[1]; ++q)
        for (int p = 0; p < s->nn[0]; ++p) {
          const size_t i = ((size_t)r * s->nn[1] + q) * s->nn[0] + p;
          if (on_shell3(s->nn, p, q, r))
            rhs[i] = 0;
          else
            rhs[i] = (op->an[0][p] * op->an[1][q] * op->an[2][r]) * rhs[i];
        }
    refine(&e->cf[e->class_of[t]], rhs, e->curr[t]);
  }
  for (int t = 0; t < e->nsub; ++t) {
    if (e->zc[t]) ++st->skipped; else ++st->solves;
  }
  for (int t = 0; t < e->nsub; ++t)
    if (!e->zc[t]) accumulate3(e, t);
  /* rotate prev3 <- prev2 <- prev1 <- curr */
  cplx** tp = e->prev[2];
  e->prev[2] = e->prev[1];
  e->prev[1] = e->prev[0];
  e->prev[0] = e->curr;
  e->curr = tp;
  char* tz = e->zp[2];
  e->zp[2] = e->zp[1];
  e->zp[1] = e->zp[0];
  e->zp[0] = e->zc;
  e->zc = tz;
  e->last_valid = 1;
}

static void reset_state3(orc3_engine* e) {
  memset(e->zc, 1, e->nsub);
  for (int k = 0; k < 3; ++k) memset(e->zp[k], 1, e->nsub);
  memset(e->assembled, 0, (size_t)orc3_n_global(e) * sizeof(cplx));
  e->last_valid = 0;
}

static double residual_norm3(orc3_engine* e, const cplx* f) {
  op3_apply(&e->gop, e->assembled, e->tmp);
  const size_t n = (size_t)orc3_n_global(e);
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += cnorm(f[i] - e->tmp[i]);
  return sqrt(s);
}

int orc3_solve_iterative(orc3_engine* e, const double* fd, double tol, int max_steps,
                         int check_every, double* out, orc_stats* st, int* hist_step,
                         double* hist_rel, int hist_cap, int* hist_len) {
  const cplx* f = (const cplx*)fd;
  const size_t n = (size_t)orc3_n_global(e);
  if (check_every < 1) check_every = 1;
  memset(st, 0, sizeof *st);
  st->relres = -1;
  reset_state3(e);
  const double bnorm = vnrm2(f, n);
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
    sweep3(e, s, f, st);
    st->steps = s;
    if (s % check_every == 0 || s == max_steps) {
      const double rel = residual_norm3(e, f) / bnorm;
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

int orc3_precondition(orc3_engine* e, const double* r, double* z, int k, orc_stats* st) {
  reset_state3(e);
  const double t0 = now_ms();
  for (int s = 1; s <= k; ++s) sweep3(e, s, (const cplx*)r, st);
  st->sweep_ms += now_ms() - t0;
  memcpy(z, e->assembled, (size_t)orc3_n_global(e) * sizeof(cplx));
  return 0;
}

int orc3_tap_subdomain(const orc3_engine* e, int t, double* rhs, double* u, int* active) {
  if (t < 0 || t >= e->nsub || !e->last_valid) return 1;
  memcpy(rhs, e->rhs[t], e->nw * sizeof(cplx));
  memcpy(u, e->prev[0][t], e->nw * sizeof(cplx));
  *active = !e->zp[0][t];
  return 0;
}

typedef struct {
  orc3_engine* e;
  int K;
  orc_stats* pst;
} fgm3_ctx;
static void fgm3_A(void* c, const cplx* in, cplx* out) { op3_apply(&((fgm3_ctx*)c)->e->gop, in, out); }
static void fgm3_M(void* c, const cplx* in, cplx* out) {
  fgm3_ctx* x = (fgm3_ctx*)c;
  orc3_precondition(x->e, (const double*)in, (double*)out, x->K, x->pst);
}

int orc3_fgmres(orc3_engine* e, const double* b, double* x, double tol, int max_iters,
                int restart, int K, orc_fgmres_out* res, double* hist, int hist_cap,
                double* zs, int zs_cap, orc_stats* pst) {
  memset(pst, 0, sizeof *pst);
  fgm3_ctx c = {e, K, pst};
  return fgmres_core((size_t)orc3_n_global(e), fgm3_A, fgm3_M, &c, b, x, tol, max_iters,
                     restart, res, hist, hist_cap, zs, zs_cap);
}
