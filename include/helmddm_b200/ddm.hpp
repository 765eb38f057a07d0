// Header-only C++ shim: the reference's DdmEngine / fgmres surface
// (proj/include/helmddm/ddm.hpp:15-109, krylov.hpp:9-33) rebuilt over the C-ABI
// of libhddm.so (include/hddm.h), so reference-side callers (cli.cpp:170-261,
// the test suites) switch engines by changing the include and namespace.
// Errors are rethrown as ConfigError / SolveError like the reference
// (types.hpp:58-66).
#pragma once

#include <chrono>
#include <cmath>
#include <complex>
#include <functional>
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
  std::vector<double> iter_ms;  // host FGMRES only (the device one times the whole solve)
};

// LinearOp (krylov.hpp:9): y = Op(x) on n complex values
using LinearOp = std::function<void(const Complex*, Complex*)>;

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

// fgmres(n, A, M, b, x, opt) over caller-supplied operators (krylov.hpp:31-33,
// krylov.cpp:24-133), restated host-side: right-preconditioned flexible GMRES from
// x = 0, modified Gram-Schmidt, complex Givens rotations, the recursive residual
// per iteration, cyclic restart with the residual recomputed, stop on tol / a
// dead column / an invariant subspace, true residual of the returned x. The
// production path is DdmEngine::fgmres (device-resident, A = apply_global,
// M = precondition); this form keeps host-lambda callers and lets the caller's
// FGMRES drive the GPU preconditioner. M may be empty.
inline FgmresResult fgmres(size_t n, const LinearOp& A, const LinearOp& M,
                           const std::vector<Complex>& b, std::vector<Complex>& x,
                           const FgmresOptions& opt) {
  using clock = std::chrono::steady_clock;
  auto norm = [n](const std::vector<Complex>& v) {
    double s = 0;
    for (size_t t = 0; t < n; ++t) s += std::norm(v[t]);
    return std::sqrt(s);
  };
  FgmresResult res;
  x.assign(n, Complex(0));
  const double bnorm = norm(b);
  if (bnorm == 0) {
    res.converged = true;
    res.relres = res.true_relres = 0;
    return res;
  }
  std::vector<Complex> r(b.begin(), b.begin() + long(n));
  int total = 0;
  bool stop = false;
  while (!stop && total < opt.max_iters) {
    const int m = opt.restart > 0 ? std::min(opt.restart, opt.max_iters - total) : opt.max_iters - total;
    const double rnorm = norm(r);
    if (rnorm == 0) {
      res.converged = true;
      break;
    }
    std::vector<std::vector<Complex>> V(1, r), Z;
    for (Complex& c : V[0]) c /= rnorm;
    // column j of the (rotated) Hessenberg matrix: H[j][0..j+1]
    std::vector<std::vector<Complex>> H;
    std::vector<Complex> g(static_cast<size_t>(m) + 1, Complex(0));
    std::vector<Complex> sn(static_cast<size_t>(m));
    std::vector<double> cs(static_cast<size_t>(m));
    g[0] = rnorm;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      const auto t0 = clock::now();
      Z.emplace_back(n);
      if (M)
        M(V[size_t(j)].data(), Z.back().data());
      else
        Z.back() = V[size_t(j)];
      std::vector<Complex> w(n);
      A(Z.back().data(), w.data());
      H.emplace_back(size_t(j) + 2, Complex(0));
      std::vector<Complex>& h = H.back();
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
        Complex d = 0;
        const std::vector<Complex>& vi = V[size_t(i)];
        for (size_t t = 0; t < n; ++t) d += std::conj(vi[t]) * w[t];
        h[size_t(i)] = d;
        for (size_t t = 0; t < n; ++t) w[t] -= d * vi[t];
      }
      const double hlast = norm(w);
      h[size_t(j) + 1] = hlast;
      for (int i = 0; i < j; ++i) {  // earlier rotations on the new column
        const Complex a = h[size_t(i)], c = h[size_t(i) + 1];
        h[size_t(i)] = cs[size_t(i)] * a + sn[size_t(i)] * c;
        h[size_t(i) + 1] = -std::conj(sn[size_t(i)]) * a + cs[size_t(i)] * c;
      }
      const Complex a = h[size_t(j)], c = h[size_t(j) + 1];
      const double tn = std::sqrt(std::norm(a) + std::norm(c));
      if (tn == 0) {  // dead column: dropped, stop
        H.pop_back();
        Z.pop_back();
        stop = true;
        break;
      }
      if (a == Complex(0)) {
        cs[size_t(j)] = 0;
        sn[size_t(j)] = std::conj(c) / std::abs(c);
      } else {
        cs[size_t(j)] = std::abs(a) / tn;
        sn[size_t(j)] = (a / std::abs(a)) * std::conj(c) / tn;
      }
      h[size_t(j)] = cs[size_t(j)] * a + sn[size_t(j)] * c;
      h[size_t(j) + 1] = 0;
      g[size_t(j) + 1] = -std::conj(sn[size_t(j)]) * g[size_t(j)];
      g[size_t(j)] = cs[size_t(j)] * g[size_t(j)];
      ++total;
      k = j + 1;
      res.relres = std::abs(g[size_t(j) + 1]) / bnorm;
      res.history.push_back(res.relres);
      res.iter_ms.push_back(std::chrono::duration<double, std::milli>(clock::now() - t0).count());
      if (res.relres <= opt.tol) {
        res.converged = true;
        stop = true;
        break;
      }
      if (hlast == 0) {  // invariant subspace
        stop = true;
        break;
      }
      for (Complex& cv : w) cv /= hlast;
      V.push_back(std::move(w));
    }
    if (k > 0) {  // back substitution on the rotated triangle, x += Z y
      std::vector<Complex> y(static_cast<size_t>(k));
      for (int i = k - 1; i >= 0; --i) {
        Complex s = g[size_t(i)];
        for (int l = i + 1; l < k; ++l) s -= H[size_t(l)][size_t(i)] * y[size_t(l)];
        y[size_t(i)] = s / H[size_t(i)][size_t(i)];
      }
      for (int l = 0; l < k; ++l)
        for (size_t t = 0; t < n; ++t) x[t] += y[size_t(l)] * Z[size_t(l)][t];
    }
    if (!stop) {  // restart from the explicit residual
      A(x.data(), r.data());
      for (size_t t = 0; t < n; ++t) r[t] = b[t] - r[t];
    }
  }
  res.iters = total;
  std::vector<Complex> ax(n);
  A(x.data(), ax.data());
  double s = 0;
  for (size_t t = 0; t < n; ++t) s += std::norm(b[t] - ax[t]);
  res.true_relres = std::sqrt(s) / bnorm;
  return res;
}

}  // namespace helmddm_b200
