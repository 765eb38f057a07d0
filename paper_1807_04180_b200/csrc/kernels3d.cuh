// Device tables and launchers of the 3-D path (BASELINE config 5).
#pragma once

#include "dev.cuh"

namespace hddm3 {

using hddm::cplx;

// one supernode (engine3d.h Sn3) as the kernels see it
struct DSn3 {
  int c0, n, r, parent;
  int ch0, ch1, pad0, pad1;
  long long linv_off, pan_off, upd_off, cmap_off, rows_off, front_off, ext_off;
  int aent0, aent1;
};

// a piece of a supernode's work: rows / columns [a, b), with the supernode's
// offsets carried along (one load per task)
struct Task3 {
  int s, a, b, pad;
  int c0, n, r, pad2;
  long long linv, pan, upd, cmap, rows, pad3;
};

// ------------------------------------------------------------ factorization
struct Fac3Args {
  const DSn3* sn;
  cplx* fronts;          // workspace of the class batch
  long long fw;          // complex words per class in the workspace
  const int* aent_i;
  const int* aent_j;
  const cplx* aval;      // per class: the assembled entries of aent (class-major)
  long long naent;
  const int* ext;
  cplx* vals;            // factor values, per class stride nvals
  cplx* valsT;           // the same blocks transposed (row-major) for the backward sweep
  long long nvals;
  int cls0;              // first class of the batch
};
constexpr int kNB = 32;  // panel width of the blocked partial LDL^T

void f3_scatter(const Fac3Args& F, const int* lv, int nlv, int nb, cudaStream_t st);
void f3_extadd(const Fac3Args& F, const int* lv, int nlv, int nb, int slot, int maxr, cudaStream_t st);
void f3_dfac(const Fac3Args& F, const int* lv, int nlv, int nb, int k0, cudaStream_t st);
void f3_trsm(const Fac3Args& F, const int* lv, int nlv, int nb, int k0, int maxrows, cudaStream_t st);
void f3_update(const Fac3Args& F, const int* lv, int nlv, int nb, int k0, long long maxtiles,
               cudaStream_t st);
void f3_extract(const Fac3Args& F, const int* lv, int nlv, int nb, long long maxent, cudaStream_t st);

// ------------------------------------------------------------------ solve
// RHS t (a subdomain, or a class's representative for probes) lives at
// B + t * nw (factor order); its forward/backward update vector at U + t * nupd.
struct Solve3Args {
  const DSn3* sn;
  const cplx* vals;   // forward layout: inverse blocks and panels column major
  const cplx* valsT;  // backward layout: the same blocks row major
  long long nvals;
  const int* rows_all;
  const int* cmap0;
  const int* cmap1;
  const cplx* B;
  cplx* X;
  cplx* Y;
  cplx* U;
  long long nw, nupd;
  int nshell;
  const int* cls_ptr;
  const int* cls_mem;
  const int* flag;  // RHS t takes part iff (flag[t] != 0) == flag_on
  int flag_on;
  int mg;           // right-hand sides per member group: 1 or kMG
};
constexpr int kMG = 4;  // right-hand sides per CTA pass (member group)

// fdiag / fpanel: the first nbig tasks are CTA tasks (8 warps split the columns of
// 32 rows), the rest warp tasks (8 per CTA: supernodes with few columns)
void s3_ring(const Solve3Args& A, int ncls, int ngroups, cudaStream_t st);
void s3_fasm(const Solve3Args& A, const Task3* t, int nt, int ncls, int ngroups, cudaStream_t st);
void s3_fdiag(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ngroups, cudaStream_t st);
void s3_fpanel(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ngroups, cudaStream_t st);
void s3_bgather(const Solve3Args& A, const Task3* t, int nt, int ncls, int ngroups, cudaStream_t st);
// leaves (no children, <= 32 nodes), a warp per leaf; nt a multiple of 8
void s3_fleaf(const Solve3Args& A, const Task3* t, int nt, int ncls, int ngroups, cudaStream_t st);
void s3_bleaf(const Solve3Args& A, const Task3* t, int nt, int ncls, int ngroups, cudaStream_t st);
void s3_bpanel(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ngroups, cudaStream_t st);
void s3_bdiag(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ngroups, cudaStream_t st);

// ------------------------------------------------------------------ DDM step
struct Sub3Dev {
  int ix[3], w0[3];
  int c0[3], c1[3];
  int lo[3], hi[3];
  int own0[3], own1[3];
  int cls, pad;
};

struct Step3Args {
  int n[3], nsub, nov, nn[3], gn[3], nw, nshell;
  double ih2, k2;
  const Sub3Dev* sub;
  const cplx* cop;   // per class: an[0..2], iah[0..2] (each nn[a] long), stride cop_stride
  int cop_stride;
  const double* wts; // per subdomain: wx, wy, wz (nn[0] + nn[1] + nn[2])
  const int* perm;
  const int* pinv;
  const cplx* f;     // global field (restrict_owned at step 1)
  int* fany;
  int* zc;           // flags of this step
  const int* zp[3];  // flags of steps s-1, s-2, s-3
  cplx* B;
  cplx* Ucur;
  const cplx* Up[3];
  cplx* asmb;
  const int* cov;    // per axis a, global coordinate P: two covering subdomain indices (or -1)
  int step;
  long long* counts; // solves, skipped
  // transfer tables (window-local, identical for every window): the nodes of the union
  // of the 26 patches, per node its (direction, 7 source positions, 7 tapers) entries
  int npatch;
  const int* pnode;      // window node
  const int* pent;       // npatch + 1: entry range per node
  const int* edir;       // per entry: direction (gather order)
  const int* esrc;       // per entry: 7 source-window factor positions (-1: outside)
  const double* ebeta;   // per entry: 7 tapers
};

void d3_fany(const Step3Args& A, cudaStream_t st);
void d3_flags(const Step3Args& A, cudaStream_t st);
void d3_rhs(const Step3Args& A, cudaStream_t st);  // base (all nodes) + transfers (patch nodes)
void d3_accumulate(const Step3Args& A, cudaStream_t st);

struct Glob3Args {
  int gn[3];
  double ih2, k2;
  const cplx* ga;  // an[0..2], iah[0..2] of the global box
};
void d3_apply_global(const Glob3Args& G, const cplx* u, cplx* out, const cplx* f, double* part,
                     cudaStream_t st);
void d3_apply_global_ind(const Glob3Args& G, cplx* const* U, int du, cplx* const* O, int dout,
                         const int* jp, cudaStream_t st);

// residual check and refinement (refine, proj/src/sparse.cpp:268-292)
struct Chk3Args {
  int nn[3], nw, nsub, nchunk;
  double ih2, k2;
  const Sub3Dev* sub;
  const cplx* cop;
  int cop_stride;
  const int* perm;
  const int* pinv;
  const cplx* B;
  cplx* X;
  cplx* R;        // residual out (prep) or nullptr
  cplx* C;        // correction
  const int* flag;  // t checked iff (flag[t] != 0) == flag_on
  int flag_on;
  double* part;   // nsub x nchunk x 2 partial sums
  double* rel_cur;
  double* rel_prev;
  int* need;
  int* ncorr;
  int* undo;
  int* any;
  double* max_rel;
  int* corr_count;
  unsigned long long cond;  // WHILE handle (0: none)
};
void c3_partials(const Chk3Args& C, int write_resid, cudaStream_t st);
void c3_first(const Chk3Args& C, cudaStream_t st);   // after the first solve
void c3_apply(const Chk3Args& C, cudaStream_t st);   // X += C for need
void c3_decide(const Chk3Args& C, cudaStream_t st);  // stagnation rule, undo flags, loop condition
void c3_undo(const Chk3Args& C, cudaStream_t st);

}  // namespace hddm3
