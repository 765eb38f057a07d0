// Drop-in check of the C++ shim: the reference's test_ddm.cpp scenarios
// (make_cfg, proj/tests/test_ddm.cpp:15-30) written against helmddm_b200.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "helmddm_b200/ddm.hpp"

using namespace helmddm_b200;

static DdmConfig make_cfg(int mx, int n1, int n2, double freq, int n_ov, int n_ramp) {
  DdmConfig cfg;
  cfg.grid.h = 1.0 / mx;
  cfg.grid.mx = cfg.grid.my = mx;
  cfg.grid.n1 = n1;
  cfg.grid.n2 = n2;
  cfg.grid.n_overlap = n_ov;
  cfg.grid.n_ramp = n_ramp;
  cfg.medium.omega = 2 * M_PI * freq;
  return cfg;
}

#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                           \
    }                                                         \
  } while (0)

int main() {
  DdmEngine eng(make_cfg(40, 2, 2, 4.0, 4, 8));
  const size_t n = eng.n_global();
  std::vector<Complex> f(n, Complex(0));
  f[n / 2 + 7] = Complex(1600.0, 0.0);
  DdmStats st;
  const std::vector<Complex> u = eng.solve_iterative(f, 1e-8, 25, st);
  CHECK(st.converged && st.relres <= 1e-8 && st.history.back().step == st.steps);
  // 2x2 split converges within a few sweeps (test_ddm.cpp:133-149)
  CHECK(st.steps <= 10);
  for (const OpClassInfo& c : eng.class_info()) CHECK(c.probe_relres <= 1e-10);
  // power-of-two scaling is exact (test_ddm.cpp:232-242)
  std::vector<Complex> z1(n), z2(n), f2(n);
  for (size_t i = 0; i < n; ++i) f2[i] = 2.0 * f[i];
  DdmStats ps;
  eng.precondition(f.data(), z1.data(), 3, ps);
  eng.precondition(f2.data(), z2.data(), 3, ps);
  for (size_t i = 0; i < n; ++i) CHECK(z2[i] == 2.0 * z1[i]);
  // FGMRES preconditioned by the DDM
  std::vector<Complex> x;
  FgmresOptions o;
  o.tol = 1e-8;
  o.max_iters = 40;
  o.restart = 30;
  DdmStats fs;
  const FgmresResult r = eng.fgmres(f, x, o, 2, fs);
  CHECK(r.converged && r.true_relres <= 1e-7);
  // the reference API with host lambdas: fgmres(n, A, M, b, x, opt) driving the
  // GPU operators (krylov.hpp:31-33) agrees with the device-resident FGMRES
  LinearOp A = [&eng](const Complex* u, Complex* out) { eng.apply_global(u, out); };
  DdmStats hs;
  LinearOp M = [&eng, &hs](const Complex* v, Complex* z) { eng.precondition(v, z, 2, hs); };
  std::vector<Complex> xh;
  const FgmresResult rh = fgmres(n, A, M, f, xh, o);
  CHECK(rh.converged && rh.iters == r.iters && rh.true_relres <= 1e-7);
  double num = 0, den = 0;
  for (size_t i = 0; i < n; ++i) {
    num += std::norm(xh[i] - x[i]);
    den += std::norm(x[i]);
  }
  CHECK(std::sqrt(num / den) <= 1e-8);
  // configuration errors surface as ConfigError (partition.cpp:15-28)
  bool threw = false;
  try {
    DdmEngine bad(make_cfg(41, 2, 2, 4.0, 4, 8));
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("shim ok: %d sweeps, relres %.3e, fgmres %d iters\n", st.steps, st.relres, r.iters);
  return 0;
}
