/*
 * hddm3.h -- C-ABI of the engine's 3-D path (BASELINE config 5), in libhddm.so.
 *
 * The reference has no 3-D code; PAPER.md:829 describes the
 * generalization (26 transfer directions, N1+N2+N3 steps). The 3-D entry points
 * mirror the 2-D ones in hddm.h one for one -- same names with hddm3_, same
 * argument meaning, memkind, return codes (0 ok, 2 ConfigError, 3 SolveError,
 * 1 other) and error behaviour -- so a caller of DdmEngine's 2-D surface finds
 * the same surface in 3-D. The math is the restatement oracle/hddm_oracle3.c
 * (its header spells it out); global fields are x fastest, then y, then z.
 *
 * There is NO CPU fallback: without a usable CUDA device hddm3_create fails.
 */
#ifndef HDDM3_H
#define HDDM3_H

#include "hddm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* DdmConfig in 3-D: GridSpec with a z axis (partition.hpp:13-31 per axis) and a
 * constant medium (medium.hpp:17-29, kind Constant). */
typedef struct hddm3_problem_s {
  double x0, y0, z0, h;
  int mx, my, mz, n1, n2, n3, n_overlap, n_ramp;
  double omega, velocity;
  double c_sigma, sigma0;
  int device;
} hddm3_problem;

typedef struct hddm3_engine hddm3_engine;

const char* hddm3_last_error(const hddm3_engine* e);

/* DdmEngine::DdmEngine -- host setup, symbolic analysis, batched multifrontal
 * LDL^T of every class on the GPU, probe solve (> 1e-10: SolveError). */
int hddm3_create(const hddm3_problem* p, hddm3_engine** out);
void hddm3_destroy(hddm3_engine* e);

long hddm3_n_global(const hddm3_engine* e);
double hddm3_sigma0(const hddm3_engine* e);
double hddm3_factor_ms(const hddm3_engine* e);
int hddm3_num_subdomains(const hddm3_engine* e);
int hddm3_num_classes(const hddm3_engine* e);
int hddm3_class_of(const hddm3_engine* e, int t);
/* members, factor_nonzeros (nnz(L) + n, as the restatement counts it), probe relres */
int hddm3_class_info(const hddm3_engine* e, int c, int* members, long* nnz, double* probe_relres);
int hddm3_window_dims(const hddm3_engine* e, int* nn3);

int hddm3_apply_global(hddm3_engine* e, const double* u, double* out, int memkind);
int hddm3_solve_iterative(hddm3_engine* e, const double* f, double tol, int max_steps,
                          int check_every, double* out, int memkind, hddm_stats* stats,
                          int* hist_step, double* hist_rel, double* hist_ms, int hist_cap,
                          int* hist_len);
int hddm3_precondition(hddm3_engine* e, const double* r, double* z, int ksteps, int memkind,
                       hddm_stats* stats);
int hddm3_fgmres(hddm3_engine* e, const double* b, double* x, double tol, int max_iters,
                 int restart, int ksteps, int memkind, hddm_fgmres_result* res, double* hist,
                 int hist_cap, hddm_stats* pstats);

/* ---- parity / measurement taps ---- */
int hddm3_fgmres_z(hddm3_engine* e, int j, double* out, int memkind);
/* after the last sweep: subdomain t's scaled RHS and solution (window-local
 * natural order) and its active flag */
int hddm3_tap_subdomain(hddm3_engine* e, int t, double* rhs, double* u, int* active);
/* solve with class c's factors (window-local natural order, host memory) */
int hddm3_class_solve(hddm3_engine* e, int c, const double* b, double* x, double* relres);
/* host-only symbolic analysis of an nx*ny*nz window (no GPU): nnz(L)+n, stored
 * dense-supernode entries (D + packed inverse diagonal blocks + panels), supernodes,
 * tree height, and the front workspace (complex words) of one class */
int hddm3_symbolic_stats(int nx, int ny, int nz, long* nnz_ref, long* stored, int* nsuper,
                         int* height, long* front_words);
int hddm3_nd_order(int nx, int ny, int nz, int* order);
int hddm3_footprint(const hddm3_engine* e, long* stored_per_class, long* ref_nnz_per_class,
                    long* device_bytes);
/* device time of one batched solve (all classes, all members active) on the
 * right-hand sides of the last sweep, averaged over reps graph launches */
int hddm3_time_solve(hddm3_engine* e, int reps, double* ms_per_solve);
int hddm3_solve_launches(const hddm3_engine* e);
int hddm3_refine_stats(const hddm3_engine* e, double* max_local_relres, int* corrections);
int hddm3_set_timing(hddm3_engine* e, int enable);
int hddm3_stage_times(hddm3_engine* e, double* ms, long long* count, int cap, int* n);
long long hddm3_launch_count(const hddm3_engine* e);
void* hddm3_stream(const hddm3_engine* e);

#ifdef __cplusplus
}
#endif
#endif
