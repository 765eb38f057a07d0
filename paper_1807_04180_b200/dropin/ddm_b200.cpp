// DdmEngine of the drop-in header (include/helmddm_b200/dropin/helmddm/ddm.hpp)
// over the C-ABI of libhddm.so. Replaces the reference's src/ddm.cpp; every
// member keeps the reference's semantics (ddm.cpp:55-287):
//   * the partition, sigma0 and the global operator come from the reference's own
//     build_partition / default_sigma0 / build_operator (so partition(), grid(),
//     global_op() and the ConfigError messages are the reference's);
//   * the DDM itself -- factorization, sweeps, residuals -- runs on the GPU;
//   * C return codes are rethrown as ConfigError / SolveError (types.hpp:58-63).
#include <algorithm>
#include <string>

#include "hddm.h"
#include "helmddm/ddm.hpp"
#include "helmddm/pml.hpp"

namespace helmddm {

namespace {

void check(int rc, const hddm_engine* e) {
  if (rc == HDDM_OK) return;
  const std::string m = hddm_last_error(e);
  if (rc == HDDM_ERR_CONFIG) throw ConfigError(m);
  if (rc == HDDM_ERR_SOLVE) throw SolveError(m);
  throw std::runtime_error(m);
}

const double* dp(const Complex* p) { return reinterpret_cast<const double*>(p); }
double* dp(Complex* p) { return reinterpret_cast<double*>(p); }

}  // namespace

DdmEngine::DdmEngine(const DdmConfig& cfg) : cfg_(cfg), part_(build_partition(cfg.grid)) {
  const GridSpec& g = part_.g;
  cfg_.medium.margin = std::max(cfg_.medium.margin, (g.n_ext() + 1) * g.h);  // ddm.cpp:66-67
  sigma0_ = cfg_.sigma0 > 0 ? cfg_.sigma0
                            : default_sigma0(cfg_.c_sigma, cfg_.medium.k_min(), g.n_ramp * g.h);
  gop_ = build_operator(g, g.global_window(), global_layout(g), cfg_.medium, sigma0_);
  std::vector<double> lo, hi, c;
  for (const Layer& l : cfg_.medium.layers) {
    lo.push_back(l.y_lo);
    hi.push_back(l.y_hi);
    c.push_back(l.velocity);
  }
  hddm_problem p{};
  p.x0 = g.x0;
  p.y0 = g.y0;
  p.h = g.h;
  p.mx = g.mx;
  p.my = g.my;
  p.n1 = g.n1;
  p.n2 = g.n2;
  p.n_overlap = g.n_overlap;
  p.n_ramp = g.n_ramp;
  p.omega = cfg_.medium.omega;
  p.medium_kind = cfg_.medium.kind == MediumKind::Layered ? HDDM_MEDIUM_LAYERED : HDDM_MEDIUM_CONSTANT;
  p.velocity = cfg_.medium.velocity;
  p.n_layers = int(lo.size());
  p.layer_ylo = lo.data();
  p.layer_yhi = hi.data();
  p.layer_c = c.data();
  p.c_sigma = cfg_.c_sigma;
  p.sigma0 = sigma0_;
  p.threads = cfg_.threads;
  p.has_box = 1;  // the medium's interior box and margin, as the caller set them
  p.box_x0 = cfg_.medium.interior.x0;
  p.box_x1 = cfg_.medium.interior.x1;
  p.box_y0 = cfg_.medium.interior.y0;
  p.box_y1 = cfg_.medium.interior.y1;
  p.margin = cfg_.medium.margin;
  p.device = 0;
  check(hddm_create(&p, &eng_), nullptr);
  factor_ms_ = hddm_factor_ms(eng_);
}

DdmEngine::~DdmEngine() { hddm_destroy(eng_); }

std::vector<OpClassInfo> DdmEngine::class_info() const {
  std::vector<OpClassInfo> out;
  for (int c = 0; c < hddm_num_classes(eng_); ++c) {
    int members = 0, ldlt = 0;
    long nnz = 0;
    double probe = 0;
    check(hddm_class_info(eng_, c, &members, &nnz, &probe, &ldlt), eng_);
    OpClassInfo ci;
    ci.members = members;
    ci.backend = ldlt ? "ldlt" : "lu";
    ci.factor_nnz = size_t(nnz);
    ci.probe_relres = probe;
    out.push_back(ci);
  }
  return out;
}

void DdmEngine::apply_global(const Complex* u, Complex* out) const {
  check(hddm_apply_global(eng_, dp(u), dp(out), HDDM_HOST), eng_);
}

FieldGrid DdmEngine::solve_iterative(const std::vector<Complex>& f, double tol, int max_steps,
                                     DdmStats& stats, int check_every) {
  if (f.size() != n_global()) throw SolveError("source vector size mismatch");  // ddm.cpp:247
  FieldGrid u(part_.g.global_window(), part_.g.h);
  const int cap = std::max(max_steps, 1) + 1;
  std::vector<int> hs(cap);
  std::vector<double> hr(cap), hm(cap);
  int nh = 0;
  hddm_stats st{};
  check(hddm_solve_iterative(eng_, dp(f.data()), tol, max_steps, check_every, dp(u.v.data()), HDDM_HOST,
                             &st, hs.data(), hr.data(), hm.data(), cap, &nh),
        eng_);
  // accumulate as the reference does (ddm.cpp:254-277): counts, sweep time and the
  // evaluated steps add up across calls; steps / relres / converged are updated
  stats.solves += st.solves;
  stats.skipped += st.skipped;
  stats.sweep_ms += st.sweep_ms;
  if (st.steps > 0) stats.steps = st.steps;
  if (nh > 0 || st.converged) stats.relres = st.relres;
  if (st.converged) stats.converged = true;
  for (int i = 0; i < std::min(nh, cap); ++i) stats.history.push_back({hs[i], hr[i], hm[i]});
  return u;
}

void DdmEngine::precondition(const Complex* r, Complex* z, int ksteps, DdmStats& stats) {
  hddm_stats st{};  // the engine accumulates counts into it; merged below (ddm.cpp:285)
  check(hddm_precondition(eng_, dp(r), dp(z), ksteps, HDDM_HOST, &st), eng_);
  stats.solves += st.solves;
  stats.skipped += st.skipped;
  stats.sweep_ms += st.sweep_ms;
  stats.factor_ms = factor_ms_;
}

}  // namespace helmddm
