/*
 * hddm_oracle.h -- CPU restatement of the reference DDM hot path, in C.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the CUDA engine is compared
 * against; it is never linked into, called by, or used as a fallback for the
 * product library (paper_1807_04180_b200/). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity is PINNED: tests/test_oracle_vs_ref.py runs this restatement and the
 * unmodified reference (oracle/_ref/libhelmddm_ref.so, built from
 * /root/reference/proj/src by oracle/Makefile) on identical inputs, and the
 * committed fixtures under tests/golden/ (tests/golden/make_golden.py) carry the
 * reference's outputs to machines without /root/reference.
 *
 * Complex arrays are interleaved (re, im) doubles; global fields are row-major,
 * x fastest, over the dilated global window (proj/include/helmddm/types.hpp:37-56).
 */
#ifndef HDDM_ORACLE_H
#define HDDM_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double x0, y0, h;
  int mx, my, n1, n2, n_overlap, n_ramp;
  double omega;
  int medium_kind; /* 0 constant, 1 layered, 2 gaussian lens */
  double velocity; /* constant c, or lens background c0 */
  int n_layers;
  const double* layer_ylo;
  const double* layer_yhi;
  const double* layer_c;
  double c_sigma, sigma0;
  int threads; /* ignored: the restatement is single-threaded */
  /* lens: c = velocity - lens_amp * exp(-((x-xc)^2 + (y-yc)^2) / lens_w) */
  double lens_amp, lens_xc, lens_yc, lens_w;
} orc_problem;

typedef struct {
  int steps;
  long solves, skipped;
  double relres;
  int converged;
  double factor_ms, sweep_ms;
} orc_stats;

typedef struct {
  int iters;
  int converged;
  double relres, true_relres;
  double wall_ms;
} orc_fgmres_out;

typedef struct orc_engine orc_engine;

const char* orc_last_error(void);
int orc_create(const orc_problem* p, orc_engine** out);
void orc_destroy(orc_engine* e);
long orc_n_global(const orc_engine* e);
double orc_sigma0(const orc_engine* e);
int orc_num_classes(const orc_engine* e);
int orc_class_info(const orc_engine* e, int c, int* members, long* nnz,
                   double* probe, int* is_ldlt);
int orc_class_of(const orc_engine* e, int t);
int orc_apply_global(const orc_engine* e, const double* u, double* out);
int orc_solve_iterative(orc_engine* e, const double* f, double tol,
                        int max_steps, int check_every, double* out,
                        orc_stats* st, int* hist_step, double* hist_rel,
                        int hist_cap, int* hist_len);
int orc_precondition(orc_engine* e, const double* r, double* z, int k,
                     orc_stats* st);
int orc_fgmres(orc_engine* e, const double* b, double* x, double tol,
               int max_iters, int restart, int K, orc_fgmres_out* res,
               double* hist, int hist_cap, double* zs, int zs_cap,
               orc_stats* pst);
/* Debug/parity taps: after precondition(f, K=s) the scaled right-hand side
 * and solution of subdomain t at step s (window-local natural order). */
int orc_tap_subdomain(const orc_engine* e, int t, double* rhs, double* u,
                      int* active);
/* Solve with class c's factorization (solve_raw + refine semantics). */
int orc_class_solve(const orc_engine* e, int c, const double* b, double* x,
                    double* relres);
/* Window operator coefficient arrays of class c (for kernel unit tests). */
int orc_window_dims(const orc_engine* e, int* nx, int* ny);
int orc_nd_order(int nx, int ny, int* order);

/* diagnostics: refinement corrections and largest first-pass relative residual since the
 * last reset (test infrastructure) */
void orc_refine_stats(long* ncorr, double* max_first_rel, int reset);


/* ---- 3-D extension (BASELINE config 5; hddm_oracle3.c). PARITY UNPINNED: the
 * reference has no 3-D code; this is the generalization PAPER.md:829 describes,
 * written out in hddm_oracle3.c's header, and the specification the GPU engine's
 * 3-D path is checked against. Global fields are x fastest, then y, then z. */
typedef struct {
  double x0, y0, z0, h;
  int mx, my, mz, n1, n2, n3, n_overlap, n_ramp;
  double omega, velocity; /* constant medium */
  double c_sigma, sigma0;
} orc3_problem;

typedef struct orc3_engine orc3_engine;
int orc3_create(const orc3_problem* p, orc3_engine** out);
void orc3_destroy(orc3_engine* e);
long orc3_n_global(const orc3_engine* e);
double orc3_sigma0(const orc3_engine* e);
int orc3_num_classes(const orc3_engine* e);
int orc3_class_of(const orc3_engine* e, int t);
int orc3_window_dims(const orc3_engine* e, int* nn);
int orc3_class_info(const orc3_engine* e, int c, int* members, long* nnz, double* probe);
int orc3_class_solve(const orc3_engine* e, int c, const double* b, double* x, double* relres);
int orc3_class_matvec(const orc3_engine* e, int c, const double* x, double* y);
int orc3_apply_global(const orc3_engine* e, const double* u, double* out);
int orc3_solve_iterative(orc3_engine* e, const double* f, double tol, int max_steps,
                         int check_every, double* out, orc_stats* st, int* hist_step,
                         double* hist_rel, int hist_cap, int* hist_len);
int orc3_precondition(orc3_engine* e, const double* r, double* z, int k, orc_stats* st);
int orc3_fgmres(orc3_engine* e, const double* b, double* x, double tol, int max_iters,
                int restart, int K, orc_fgmres_out* res, double* hist, int hist_cap,
                double* zs, int zs_cap, orc_stats* pst);
int orc3_tap_subdomain(const orc3_engine* e, int t, double* rhs, double* u, int* active);
int orc3_nd_order(int nx, int ny, int nz, int* order);
int orc3_direction(int d, int* o);

#ifdef __cplusplus
}
#endif
#endif
