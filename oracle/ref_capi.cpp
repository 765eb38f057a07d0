// C entry points over the UNMODIFIED reference library (helmddm, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Test and
// baseline infrastructure only: tests/ use it to pin the C restatement
// (oracle/hddm_oracle.c) and the CUDA engine, bench.py --impl reference times
// it as the reference CPU arm. Nothing in the product links it.
//
// The functions mirror the reference's public API:
//   DdmEngine(cfg)                    proj/include/helmddm/ddm.hpp:55
//   DdmEngine::apply_global           ddm.hpp:66
//   DdmEngine::solve_iterative        ddm.hpp:72-74
//   DdmEngine::precondition           ddm.hpp:78
//   DdmEngine::class_info             ddm.hpp:63
//   fgmres                            proj/include/helmddm/krylov.hpp:31-33
//   run_cli, parse_config_text,       proj/include/helmddm/cli.hpp,
//   make_setup, the artifact writers  config.hpp, io.hpp (CLI parity)
// and the error -> exit-code mapping of proj/src/cli.cpp:453-469.
#include <chrono>
#include <complex>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "helmddm/cli.hpp"
#include "helmddm/config.hpp"
#include "helmddm/ddm.hpp"
#include "helmddm/io.hpp"
#include "helmddm/krylov.hpp"
#include "helmddm/oracle.hpp"

using namespace helmddm;

extern "C" {

struct ref_problem {
  double x0, y0, h;
  int mx, my, n1, n2, n_overlap, n_ramp;
  double omega;
  int medium_kind;  // 0 constant, 1 layered
  double velocity;
  int n_layers;
  const double* layer_ylo;
  const double* layer_yhi;
  const double* layer_c;
  double c_sigma, sigma0;
  int threads;
};

struct ref_stats {
  int steps;
  long solves, skipped;
  double relres;
  int converged;
  double factor_ms, sweep_ms;
};

struct ref_fgmres_out {
  int iters;
  int converged;
  double relres, true_relres;
  double wall_ms;
};
}

namespace {

thread_local std::string g_err;

int map_error() {
  try {
    throw;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const SolveError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

DdmConfig make_cfg(const ref_problem* p) {
  DdmConfig cfg;
  GridSpec& g = cfg.grid;
  g.x0 = p->x0;
  g.y0 = p->y0;
  g.h = p->h;
  g.mx = p->mx;
  g.my = p->my;
  g.n1 = p->n1;
  g.n2 = p->n2;
  g.n_overlap = p->n_overlap;
  g.n_ramp = p->n_ramp;
  MediumModel& m = cfg.medium;
  m.kind = p->medium_kind == 1 ? MediumKind::Layered : MediumKind::Constant;
  m.omega = p->omega;
  m.velocity = p->velocity;
  for (int i = 0; i < p->n_layers; ++i)
    m.layers.push_back({p->layer_ylo[i], p->layer_yhi[i], p->layer_c[i]});
  m.interior = g.interior_box();
  m.margin = (g.n_ext() + 1) * g.h;
  cfg.c_sigma = p->c_sigma;
  cfg.sigma0 = p->sigma0;
  cfg.threads = p->threads;
  return cfg;
}

void fill_stats(const DdmStats& s, double factor_ms, ref_stats* o) {
  if (!o) return;
  o->steps = s.steps;
  o->solves = s.solves;
  o->skipped = s.skipped;
  o->relres = s.relres;
  o->converged = s.converged ? 1 : 0;
  o->factor_ms = factor_ms;
  o->sweep_ms = s.sweep_ms;
}

const Complex* cx(const double* p) { return reinterpret_cast<const Complex*>(p); }
Complex* cx(double* p) { return reinterpret_cast<Complex*>(p); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_create(const ref_problem* p, void** out) {
  try {
    *out = new DdmEngine(make_cfg(p));
    return 0;
  } catch (...) {
    *out = nullptr;
    return map_error();
  }
}

void ref_destroy(void* e) { delete static_cast<DdmEngine*>(e); }

long ref_n_global(void* e) { return long(static_cast<DdmEngine*>(e)->n_global()); }
double ref_sigma0(void* e) { return static_cast<DdmEngine*>(e)->sigma0(); }
double ref_factor_ms(void* e) { return static_cast<DdmEngine*>(e)->factor_ms(); }
int ref_num_classes(void* e) {
  return int(static_cast<DdmEngine*>(e)->class_info().size());
}

int ref_class_info(void* e, int c, int* members, long* nnz, double* probe,
                   int* is_ldlt) {
  const auto ci = static_cast<DdmEngine*>(e)->class_info();
  if (c < 0 || c >= int(ci.size())) return 1;
  *members = ci[c].members;
  *nnz = long(ci[c].factor_nnz);
  *probe = ci[c].probe_relres;
  *is_ldlt = std::strcmp(ci[c].backend, "ldlt") == 0 ? 1 : 0;
  return 0;
}

int ref_apply_global(void* e, const double* u, double* out) {
  try {
    static_cast<DdmEngine*>(e)->apply_global(cx(u), cx(out));
    return 0;
  } catch (...) {
    return map_error();
  }
}

// Runs solve_iterative; hist_* receive (step, relres) of evaluated steps.
int ref_solve_iterative(void* e, const double* f, double tol, int max_steps,
                        int check_every, double* out, ref_stats* st,
                        int* hist_step, double* hist_rel, int hist_cap,
                        int* hist_len) {
  try {
    auto* eng = static_cast<DdmEngine*>(e);
    const size_t n = eng->n_global();
    std::vector<Complex> fv(cx(f), cx(f) + n);
    DdmStats s;
    const FieldGrid u = eng->solve_iterative(fv, tol, max_steps, s, check_every);
    std::memcpy(out, u.v.data(), n * sizeof(Complex));
    fill_stats(s, eng->factor_ms(), st);
    int k = 0;
    for (const auto& r : s.history) {
      if (k < hist_cap) {
        hist_step[k] = r.step;
        hist_rel[k] = r.relres;
      }
      ++k;
    }
    if (hist_len) *hist_len = k;
    return 0;
  } catch (...) {
    return map_error();
  }
}

int ref_precondition(void* e, const double* r, double* z, int k, ref_stats* st) {
  try {
    auto* eng = static_cast<DdmEngine*>(e);
    DdmStats s;
    eng->precondition(cx(r), cx(z), k, s);
    fill_stats(s, eng->factor_ms(), st);
    return 0;
  } catch (...) {
    return map_error();
  }
}

// fgmres with A = apply_global, M = precondition(K) exactly as
// proj/src/cli.cpp:217-222 wires them. Optionally records each Z_j
// (preconditioner output) into zs (zs_cap vectors of n_global complex).
int ref_fgmres(void* e, const double* b, double* x, double tol, int max_iters,
               int restart, int K, ref_fgmres_out* res, double* hist,
               int hist_cap, double* zs, int zs_cap, ref_stats* pst) {
  try {
    auto* eng = static_cast<DdmEngine*>(e);
    const size_t n = eng->n_global();
    DdmStats ps;
    int zcount = 0;
    LinearOp A = [eng](const Complex* u, Complex* y) { eng->apply_global(u, y); };
    LinearOp M = [&](const Complex* r, Complex* z) {
      eng->precondition(r, z, K, ps);
      if (zs && zcount < zs_cap)
        std::memcpy(zs + 2 * n * size_t(zcount), z, n * sizeof(Complex));
      ++zcount;
    };
    FgmresOptions o;
    o.tol = tol;
    o.max_iters = max_iters;
    o.restart = restart;
    std::vector<Complex> bv(cx(b), cx(b) + n), xv;
    const auto t0 = std::chrono::steady_clock::now();
    const FgmresResult r = fgmres(n, A, M, bv, xv, o);
    const double ms = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0)
                          .count();
    std::memcpy(x, xv.data(), n * sizeof(Complex));
    res->iters = r.iters;
    res->converged = r.converged ? 1 : 0;
    res->relres = r.relres;
    res->true_relres = r.true_relres;
    res->wall_ms = ms;
    for (int i = 0; i < int(r.history.size()) && i < hist_cap; ++i)
      hist[i] = r.history[i];
    fill_stats(ps, eng->factor_ms(), pst);
    return 0;
  } catch (...) {
    return map_error();
  }
}

// One-shot global LDL^T solve (proj/src/oracle.cpp:202-225).
int ref_direct_solve(const ref_problem* p, const double* f, double* out) {
  try {
    DdmConfig cfg = make_cfg(p);
    const size_t n = size_t(cfg.grid.nodes_x()) * cfg.grid.nodes_y();
    std::vector<Complex> fv(cx(f), cx(f) + n);
    const FieldGrid u =
        direct_solve_global(cfg.grid, cfg.medium, cfg.c_sigma, fv, cfg.sigma0);
    std::memcpy(out, u.v.data(), n * sizeof(Complex));
    return 0;
  } catch (...) {
    return map_error();
  }
}

// ---------------------------------------------------------------- CLI parity
// The reference command line in-process (proj/src/cli.cpp:453).
int ref_run_cli(int argc, char** argv) { return run_cli(argc, argv); }

struct ref_setup_out {
  int mx, my, n1, n2, n_overlap, n_ramp;
  double h, x0, y0, omega;
  int medium_kind;  // 0 constant, 1 layered
  double velocity;
  int n_layers;
  double layer_ylo[64], layer_yhi[64], layer_c[64];
  int source_kind;  // 0 gaussian, 1 point
  double source_x, source_y, k_source;
  double c_sigma, sigma0;
  int mode;         // 0 ddm, 1 fgmres, 2 direct
  double tol, krylov_tol;
  int max_steps, check_every, precond_k, krylov_max_iter, krylov_restart, threads;
};

// parse_config_text + make_setup (config.cpp:155-228); overrides are
// newline-separated key=value pairs. Returns the CLI exit code of a failure.
int ref_setup(const char* text, const char* overrides, ref_setup_out* o, char* err, int errlen) {
  try {
    std::vector<std::string> ov;
    std::string all = overrides ? overrides : "";
    size_t a = 0;
    while (a < all.size()) {
      size_t b = all.find('\n', a);
      if (b == std::string::npos) b = all.size();
      if (b > a) ov.push_back(all.substr(a, b - a));
      a = b + 1;
    }
    const RunConfig c = parse_config_text(text, ov);
    const ProblemSetup st = make_setup(c);
    o->mx = st.grid.mx;
    o->my = st.grid.my;
    o->n1 = st.grid.n1;
    o->n2 = st.grid.n2;
    o->n_overlap = st.grid.n_overlap;
    o->n_ramp = st.grid.n_ramp;
    o->h = st.grid.h;
    o->x0 = st.grid.x0;
    o->y0 = st.grid.y0;
    o->omega = st.medium.omega;
    o->medium_kind = st.medium.kind == MediumKind::Constant ? 0 : 1;
    o->velocity = st.medium.velocity;
    o->n_layers = int(std::min<size_t>(64, st.medium.layers.size()));
    for (int i = 0; i < o->n_layers; ++i) {
      o->layer_ylo[i] = st.medium.layers[i].y_lo;
      o->layer_yhi[i] = st.medium.layers[i].y_hi;
      o->layer_c[i] = st.medium.layers[i].velocity;
    }
    o->source_kind = st.source.kind == SourceKind::PointDelta ? 1 : 0;
    o->source_x = st.source.x;
    o->source_y = st.source.y;
    o->k_source = st.k_source;
    o->c_sigma = c.c_sigma;
    o->sigma0 = c.sigma0;
    o->mode = c.mode == "ddm" ? 0 : c.mode == "fgmres" ? 1 : 2;
    o->tol = c.tol;
    o->krylov_tol = c.krylov_tol;
    o->max_steps = c.max_steps;
    o->check_every = c.check_every;
    o->precond_k = c.precond_k;
    o->krylov_max_iter = c.krylov_max_iter;
    o->krylov_restart = c.krylov_restart;
    o->threads = c.threads;
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen > 0) std::snprintf(err, size_t(errlen), "%s", e.what());
    return map_error();
  }
}

// sample_source on the global window of the setup above (medium.cpp:52-73).
int ref_sample_source(const char* text, double* out) {
  try {
    const RunConfig c = parse_config_text(text, {});
    const ProblemSetup st = make_setup(c);
    const FieldGrid f =
        sample_source(st.source, st.grid.lattice(), st.grid.global_window(), st.k_source);
    std::memcpy(out, f.v.data(), f.v.size() * sizeof(Complex));
    return 0;
  } catch (...) {
    return map_error();
  }
}

}  // extern "C"
