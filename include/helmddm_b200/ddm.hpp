// Header-only C++ shim: the reference's DdmEngine / fgmres surface
// (proj/include/helmddm/ddm.hpp:15-109, krylov.hpp:9-33) rebuilt over the C-ABI
// of libhddm.so (include/hddm.h), so reference-side callers (cli.cpp:170-261,
// the test suites) switch engines by changing the include and namespace.
// Errors are rethrown as ConfigError / SolveError like the reference
// (types.hpp:58-66).
#pragma once

#include <complex>
#include <stdexcept>
#include <string>
#include <vector>

#include "hddm.h"

namespace helmddm_b200 {

using Complex = std::complex<double>;

struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct SolveError : std::runtime_error {
  explicit SolveError(const std::string& m) : std::runtime_error(m) {}
};

// GridSpec (partition.hpp:13-31)
struct GridSpec {
  double x0 = 0, y0 = 0, h = 0;
  int mx = 0, my = 0, n1 = 1, n2 = 1, n_overlap = 10, n_ramp = 20;
  int n_ext() const { return n_overlap + n_ramp; }
  int nodes_x() const { return mx + 2 * n_ext() + 1; }
  int nodes_y() const { return my + 2 * n_ext() + 1; }
};

enum class MediumKind { Constant = 0, Layered = 1, Lens = 2 };
struct Layer {
  double y_lo = 0, y_hi = 0, velocity = 1;
};
// MediumModel (medium.hpp:17-29) + lens extension
struct MediumModel {
  MediumKind kind = MediumKind::Constant;
  double omega = 0, velocity = 1;
  std::vector<Layer> layers;
  double lens_amp = 0, lens_xc = 0, lens_yc = 0, lens_w = 1;
};

// DdmConfig (ddm.hpp:15-22)
struct DdmConfig {
  GridSpec grid;
  MediumModel medium;
  double c_sigma = 25.0;
  double sigma0 = 0;
  bool force_lu = false;  // accepted; the GPU path has only the LDL^T backend
  int threads = 1;        // accepted; the GPU replaces the WorkerPool
  int device = 0;
};

struct StepRecord {
  int step = 0;
  double relres = 0, wall_ms = 0;
};
struct DdmStats {
  int steps = 0;
  long solves = 0, skipped = 0;
  double relres = -1;
  bool converged = false;
  double factor_ms = 0, sweep_ms = 0;
  std::vector<StepRecord> history;
};
struct OpClassInfo {
  int members = 0;
  const char* backend = "";
  size_t factor_nnz = 0;
  double probe_relres = 0;
};
struct FgmresOptions {
  double tol = 1e-6;
  int max_iters = 200;
  int restart = 0;
};
struct FgmresResult {
  int iters = 0;
  bool converged = false;
  double relres = -1, true_relres = -1;
  std::vector<double> history;
};

namespace detail {
inline void check(int rc, const hddm_engine* e) {
  if (rc == HDDM_OK) return;
  const std::string m = hddm_last_error(e);
  if (rc == HDDM_ERR_CONFIG) throw ConfigError(m);
  if (rc == HDDM_ERR_SOLVE) throw SolveError(m);
  throw std::runtime_error(m);
}
inline const double* dp(const Complex* p) { return reinterpret_cast<const double*>(p); }
inline double* dp(Complex* p) { return reinterpret_cast<double*>(p); }
}  // namespace detail

// DdmEngine (ddm.hpp:53-109) on one B200
class DdmEngine {
 public:
  explicit DdmEngine(const DdmConfig& cfg) : cfg_(cfg) {
    std::vector<double> lo, hi, c;
    for (const Layer& l : cfg.medium.layers) {
      lo.push_back(l.y_lo);
      hi.push_back(l.y_hi);
      c.push_back(l.velocity);
    }
    hddm_problem p{};
    p.x0 = cfg.grid.x0;
    p.y0 = cfg.grid.y0;
    p.h = cfg.grid.h;
    p.mx = cfg.grid.mx;
    p.my = cfg.grid.my;
    p.n1 = cfg.grid.n1;
    p.n2 = cfg.grid.n2;
    p.n_overlap = cfg.grid.n_overlap;
    p.n_ramp = cfg.grid.n_ramp;
    p.omega = cfg.medium.omega;
    p.medium_kind = int(cfg.medium.kind);
    p.velocity = cfg.medium.velocity;
    p.n_layers = int(lo.size());
    p.layer_ylo = lo.data();
    p.layer_yhi = hi.data();
    p.layer_c = c.data();
    p.c_sigma = cfg.c_sigma;
    p.sigma0 = cfg.sigma0;
    p.threads = cfg.threads;
    p.lens_amp = cfg.medium.lens_amp;
    p.lens_xc = cfg.medium.lens_xc;
    p.lens_yc = cfg.medium.lens_yc;
    p.lens_w = cfg.medium.lens_w;
    p.device = cfg.device;
    detail::check(hddm_create(&p, &e_), nullptr);
  }
  ~DdmEngine() { hddm_destroy(e_); }
  DdmEngine(const DdmEngine&) = delete;
  DdmEngine& operator=(const DdmEngine&) = delete;

  const GridSpec& grid() const { return cfg_.grid; }
  double sigma0() const { return hddm_sigma0(e_); }
  size_t n_global() const { return size_t(hddm_n_global(e_)); }
  double factor_ms() const { return hddm_factor_ms(e_); }
  std::vector<OpClassInfo> class_info() const {
    std::vector<OpClassInfo> out;
    for (int c = 0; c < hddm_num_classes(e_); ++c) {
      int m = 0, ld = 0;
      long nnz = 0;
      double pr = 0;
      detail::check(hddm_class_info(e_, c, &m, &nnz, &pr, &ld), e_);
      out.push_back({m, ld ? "ldlt" : "lu", size_t(nnz), pr});
    }
    return out;
  }

  void apply_global(const Complex* u, Complex* out) const {
    detail::check(hddm_apply_global(e_, detail::dp(u), detail::dp(out), HDDM_HOST), e_);
  }

  std::vector<Complex> solve_iterative(const std::vector<Complex>& f, double tol, int max_steps,
                                       DdmStats& stats, int check_every = 1) {
    if (f.size() != n_global()) throw SolveError("source vector size mismatch");
    std::vector<Complex> out(n_global());
    std::vector<int> hs(size_t(max_steps) + 1);
    std::vector<double> hr(hs.size()), hm(hs.size());
    hddm_stats st{};
    int hl = 0;
    detail::check(hddm_solve_iterative(e_, detail::dp(f.data()), tol, max_steps, check_every,
                                       detail::dp(out.data()), HDDM_HOST, &st, hs.data(),
                                       hr.data(), hm.data(), int(hs.size()), &hl),
                  e_);
    stats.steps = st.steps;
    stats.solves = st.solves;
    stats.skipped = st.skipped;
    stats.relres = st.relres;
    stats.converged = st.converged != 0;
    stats.factor_ms = st.factor_ms;
    stats.sweep_ms = st.sweep_ms;
    stats.history.clear();
    for (int i = 0; i < hl && i < int(hs.size()); ++i) stats.history.push_back({hs[i], hr[i], hm[i]});
    return out;
  }

  void precondition(const Complex* r, Complex* z, int ksteps, DdmStats& stats) {
    hddm_stats st{};
    st.solves = stats.solves;
    st.skipped = stats.skipped;
    st.sweep_ms = stats.sweep_ms;
    detail::check(hddm_precondition(e_, detail::dp(r), detail::dp(z), ksteps, HDDM_HOST, &st), e_);
    stats.solves = st.solves;
    stats.skipped = st.skipped;
    stats.sweep_ms = st.sweep_ms;
  }

  // fgmres(n, A=apply_global, M=precondition(K), b, x, opt), device-resident
  FgmresResult fgmres(const std::vector<Complex>& b, std::vector<Complex>& x,
                      const FgmresOptions& opt, int ksteps, DdmStats& pstats) {
    x.assign(n_global(), Complex(0));
    hddm_fgmres_result r{};
    std::vector<double> hist(size_t(std::max(opt.max_iters, 1)));
    hddm_stats st{};
    st.solves = pstats.solves;
    st.skipped = pstats.skipped;
    st.sweep_ms = pstats.sweep_ms;
    detail::check(hddm_fgmres(e_, detail::dp(b.data()), detail::dp(x.data()), opt.tol,
                              opt.max_iters, opt.restart, ksteps, HDDM_HOST, &r, hist.data(),
                              int(hist.size()), &st),
                  e_);
    pstats.solves = st.solves;
    pstats.skipped = st.skipped;
    pstats.sweep_ms = st.sweep_ms;
    FgmresResult out;
    out.iters = r.iters;
    out.converged = r.converged != 0;
    out.relres = r.relres;
    out.true_relres = r.true_relres;
    out.history.assign(hist.begin(), hist.begin() + r.iters);
    return out;
  }

 private:
  DdmConfig cfg_;
  hddm_engine* e_ = nullptr;
};

}  // namespace helmddm_b200
