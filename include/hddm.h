/*
 * hddm.h -- C-ABI of the B200-native DDM engine (libhddm.so).
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json
 * (north_star): the reference's C++ entry points in proj/include/helmddm/ are
 * re-expressed as plain C functions over plain pointers and sizes. A header-only
 * C++ shim (include/helmddm_b200/ddm.hpp) rebuilds the reference's class
 * surface on top of these functions; INTEGRATION.md shows the bindings.
 *
 * Each entry point names the reference interface it replaces. Complex arrays
 * are interleaved (re, im) doubles (std::complex<double> layout,
 * proj/include/helmddm/types.hpp:10); global fields are row-major with x fastest
 * over the dilated global window (types.hpp:37-56), n_global() entries.
 *
 * memkind: HDDM_HOST -> caller pointers are host memory (the engine copies
 * through pinned staging and synchronises before returning);
 * HDDM_DEVICE -> pointers are device memory on the engine's device, work is
 * ordered on the engine's stream and the call still synchronises before
 * returning (statistics are host values).
 *
 * Return codes mirror the reference CLI (proj/src/cli.cpp:453-469):
 * 0 ok, 2 configuration error (ConfigError), 3 solve error (SolveError),
 * 1 any other error (CUDA failure, std::domain_error, ...).
 * There is NO CPU fallback: without a usable CUDA device hddm_create fails.
 */
#ifndef HDDM_H
#define HDDM_H

#ifdef __cplusplus
extern "C" {
#endif

#define HDDM_HOST 0
#define HDDM_DEVICE 1

#define HDDM_OK 0
#define HDDM_ERR_OTHER 1
#define HDDM_ERR_CONFIG 2
#define HDDM_ERR_SOLVE 3

#define HDDM_MEDIUM_CONSTANT 0
#define HDDM_MEDIUM_LAYERED 1
#define HDDM_MEDIUM_LENS 2

/* DdmConfig (proj/include/helmddm/ddm.hpp:15-22) flattened: GridSpec
 * (partition.hpp:13-31) + MediumModel (medium.hpp:17-29) + c_sigma/sigma0.
 * medium_kind LENS is this repo's extension (BASELINE config 3):
 * c(x,y) = velocity - lens_amp * exp(-((x-lens_xc)^2 + (y-lens_yc)^2) / lens_w)
 * with (x, y) clamped into the interior box. */
typedef struct hddm_problem_s {
  double x0, y0, h;
  int mx, my, n1, n2, n_overlap, n_ramp;
  double omega;
  int medium_kind;
  double velocity;
  int n_layers;
  const double* layer_ylo;
  const double* layer_yhi;
  const double* layer_c;
  double c_sigma, sigma0;
  int threads; /* accepted for DdmConfig parity; unused (the GPU replaces WorkerPool) */
  double lens_amp, lens_xc, lens_yc, lens_w;
  int device; /* CUDA device ordinal */
  /* MediumModel::interior and ::margin (medium.hpp:23-24) when has_box != 0; else
   * the grid's interior box and (n_ext + 1) h, as make_setup sets them
   * (config.cpp:175-223). The margin is raised to (n_ext + 1) h (ddm.cpp:66-67). */
  int has_box;
  double box_x0, box_x1, box_y0, box_y1, margin;
} hddm_problem;

/* DdmStats (ddm.hpp:30-39) without the history vector (returned separately). */
typedef struct {
  int steps;
  long solves, skipped;
  double relres;
  int converged;
  double factor_ms, sweep_ms;
} hddm_stats;

/* FgmresResult (krylov.hpp:18-25) without the vectors. */
typedef struct {
  int iters;
  int converged;
  double relres, true_relres;
  double wall_ms;
} hddm_fgmres_result;

typedef struct hddm_engine hddm_engine;

/* Last error message of the calling thread (create failures) or of engine e. */
const char* hddm_last_error(const hddm_engine* e);

/* DdmEngine::DdmEngine(const DdmConfig&)  -- ddm.hpp:55, ddm.cpp:62-101.
 * Host setup (partition, coefficients, classes, symbolic analysis), then the
 * batched numeric LDL^T of every class on the GPU and its probe solve
 * (sparse.cpp:203-236). A probe residual above 1e-10 is a SolveError (3):
 * there is no LU fallback. */
int hddm_create(const hddm_problem* p, hddm_engine** out);
void hddm_destroy(hddm_engine* e);

/* Accessors -- ddm.hpp:57-63 */
long hddm_n_global(const hddm_engine* e);
double hddm_sigma0(const hddm_engine* e);
double hddm_factor_ms(const hddm_engine* e);
int hddm_num_subdomains(const hddm_engine* e);
int hddm_num_classes(const hddm_engine* e);
/* OpClassInfo (ddm.hpp:41-46): members, factor_nonzeros() as the reference
 * counts it (nnz(L)+n), probe_relres, backend ("ldlt" -> 1). */
int hddm_class_info(const hddm_engine* e, int c, int* members, long* nnz,
                    double* probe_relres, int* is_ldlt);
int hddm_class_of(const hddm_engine* e, int t);

/* DdmEngine::apply_global(const Complex* u, Complex* out) -- ddm.hpp:66 */
int hddm_apply_global(hddm_engine* e, const double* u, double* out, int memkind);

/* DdmEngine::solve_iterative(f, tol, max_steps, stats, check_every) --
 * ddm.hpp:72-74, ddm.cpp:244-278. out receives the assembled global field.
 * hist_* (may be NULL) receive the evaluated (step, relres, wall_ms). */
int hddm_solve_iterative(hddm_engine* e, const double* f, double tol,
                         int max_steps, int check_every, double* out,
                         int memkind, hddm_stats* stats, int* hist_step,
                         double* hist_rel, double* hist_ms, int hist_cap,
                         int* hist_len);

/* DdmEngine::precondition(r, z, ksteps, stats) -- ddm.hpp:78, ddm.cpp:280-287.
 * Solve counts and sweep time ACCUMULATE into *stats (as the reference). */
int hddm_precondition(hddm_engine* e, const double* r, double* z, int ksteps,
                      int memkind, hddm_stats* stats);

/* fgmres(n, A=apply_global, M=precondition(K), b, x, opt) -- krylov.hpp:31-33
 * wired as proj/src/cli.cpp:210-228; restart 0 = no restart. Device-resident:
 * V, Z, H, Givens state never leave HBM. hist (may be NULL) receives the
 * recursive relres per iteration; pstats accumulates preconditioner stats. */
int hddm_fgmres(hddm_engine* e, const double* b, double* x, double tol,
                int max_iters, int restart, int ksteps, int memkind,
                hddm_fgmres_result* res, double* hist, int hist_cap,
                hddm_stats* pstats);

/* ---- sharded runs (not part of the reference surface) ----
 * One engine per rank solves its block of subdomains: hddm_set_owned marks them
 * (NULL: all). precondition(r, K) then runs as begin, K x (hddm_step, halo exchange),
 * end: after step s each rank packs the solution and zero flag of its subdomains a
 * neighbouring rank's transfers read (window-local factor order, n_w complex each),
 * sends them, and unpacks what it receives; end returns this rank's assembled field,
 * which the ranks sum (ddm.cpp:280-287 distributed; paper_1807_04180_b200/shard.py). */
int hddm_set_owned(hddm_engine* e, const int* owned);
int hddm_precondition_begin(hddm_engine* e, const double* r, int memkind);
int hddm_step(hddm_engine* e, int s);
int hddm_halo_pack(hddm_engine* e, int s, const int* ts, int nts, double* buf, int* flags);
int hddm_halo_unpack(hddm_engine* e, int s, const int* ts, int nts, const double* buf,
                     const int* flags);
int hddm_precondition_end(hddm_engine* e, double* z, int memkind, hddm_stats* stats);
/* FGMRES over the sharded preconditioner: with a hook set, hddm_fgmres runs its restart
 * cycles host-driven and calls fn(user, 1, s) after every DDM step s (the caller
 * exchanges halos there) and fn(user, 2, K) after the K steps of each preconditioner
 * application (the caller sums the ranks' assembled fields, hddm_assembled read /
 * write = 0 / 1). Every rank runs the same Krylov recurrence on identical vectors. */
typedef void (*hddm_step_hook)(void* user, int stage, int s);
int hddm_set_step_hook(hddm_engine* e, hddm_step_hook fn, void* user);
int hddm_assembled(hddm_engine* e, double* buf, int write);

/* ---- parity / measurement taps (not part of the reference surface) ---- */

/* Z_j = M(V_j) of the last FGMRES restart cycle of hddm_fgmres (j < the cycle's
 * usable columns), n_global() complex -- the preconditioned vectors the reference's
 * fgmres keeps (krylov.cpp:59-63), for per-iteration parity. */
int hddm_fgmres_z(hddm_engine* e, int j, double* out, int memkind);

/* After the last sweep: subdomain t's scaled right-hand side and solution in
 * window-local natural order (n_w complex each) and its active flag. */
int hddm_tap_subdomain(hddm_engine* e, int t, double* rhs, double* u,
                       int* active);
/* Solve A_c x = b with class c's factors (window-local natural order,
 * host memory); relres = ||b - A x|| / ||b|| as refine() reports it. */
int hddm_class_solve(hddm_engine* e, int c, const double* b, double* x,
                     double* relres);
/* Window node counts and the reference elimination order (perm[pos] = node). */
int hddm_window_dims(const hddm_engine* e, int* nx, int* ny);
int hddm_nd_order(int nx, int ny, int* order);
/* Factor entries one class's forward sweep reads: the full sweep (= nnz(L)) and
 * the sweep of steps >= 2, whose right-hand sides are nonzero only on the
 * transfer patches (subtrees without patch nodes are skipped; SURVEY 8(d) counts
 * only the blocks read). Measurement accessor. */
int hddm_fwd_entries(const hddm_engine* e, long long* full, long long* sparse_rhs);

/* Host-only symbolic analysis of an nx-by-ny window (no GPU needed):
 * the reference's factor_nonzeros() (nnz(L)+n, sparse.cpp:238-240), the
 * strictly-lower entries the engine stores, supernode count, tree height. */
int hddm_symbolic_stats(int nx, int ny, long* nnz_ref, long* stored, int* nsuper,
                        int* height);
/* Symbolic/footprint figures: stored factor values per class, the
 * reference's nnz(L)+n per class, total device bytes held by the engine. */
int hddm_footprint(const hddm_engine* e, long* stored_per_class,
                   long* ref_nnz_per_class, long* device_bytes);
/* Per-stage device timing (CUDA events on the engine stream, resolved
 * lazily, so the timed region is not synchronised): enable/reset, then read
 * the accumulated milliseconds and event-pair counts per stage
 * (hddm_stage_name(i)). hddm_launch_count: kernels this engine launched since
 * the last hddm_set_timing. */
int hddm_set_timing(hddm_engine* e, int enable);
int hddm_stage_times(hddm_engine* e, double* ms, long long* count, int cap, int* n);
const char* hddm_stage_name(int i);
long long hddm_launch_count(const hddm_engine* e);
/* Device time of one batched solve stage (forward + backward sweeps of every
 * class for all subdomains, steady state: all active), averaged over reps
 * CUDA-graph launches on the engine stream; uses the right-hand sides of the
 * last sweep. hddm_solve_launches: kernels in that stage. */
int hddm_time_solve(hddm_engine* e, int reps, double* ms_per_solve);
/* Tuning aid: lane shape (E element lanes) of forward level `level` of the
 * steady-state plan; which = 0/1 pulls of singleton / member tiles, 2/3 inverse
 * rows; E = 0 restores the heuristic. Drops the cached step graphs. Process-wide. */
int hddm_tune_fwd_shape(hddm_engine* e, int which, int level, int E);
int hddm_solve_launches(const hddm_engine* e);
/* Device time of one launch of a step stage kernel on the state of the last sweep
 * (>= 3 steps): which = 0 the 8-direction source transfer (k_rhs_transfer),
 * 1 the per-subdomain residual check (k_check), 2 the blend-accumulate (into scratch).
 * CUDA events on the engine stream, averaged over reps launches. */
int hddm_time_kernel(hddm_engine* e, int which, int reps, double* ms_per_launch);
/* Refinement diagnostics of the last call: the largest local-solve residual
 * ||b - A x||/||b|| seen (refine's first pass, sparse.cpp:268-292) and how many
 * local solves exceeded the reference's 1e-11 correction threshold. */
int hddm_refine_stats(const hddm_engine* e, double* max_local_relres, int* corrections);
/* The solver in use (descriptive). */
const char* hddm_solver_desc(const hddm_engine* e);
/* CUDA stream (cudaStream_t) the engine orders its work on. */
void* hddm_stream(const hddm_engine* e);

#ifdef __cplusplus
}
#endif
#endif
