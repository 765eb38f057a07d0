// The shim's host fgmres(n, A, M, b, x, opt) (LinearOp callbacks) on a small
// dense complex system, CPU only: converges to the Gaussian-elimination solution,
// with and without restart and with a variable preconditioner.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "helmddm_b200/ddm.hpp"

using namespace helmddm_b200;

#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                           \
    }                                                         \
  } while (0)

int main() {
  const int n = 30;
  std::vector<Complex> A(size_t(n) * n), b(n);
  unsigned long long s = 12345;
  auto rnd = [&s] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return double(s >> 11) * 0x1.0p-53 - 0.5;
  };
  for (int i = 0; i < n; ++i) {
    b[i] = Complex(rnd(), rnd());
    for (int j = 0; j < n; ++j) A[size_t(i) * n + j] = Complex(rnd(), rnd()) * 0.3 + (i == j ? 4.0 : 0.0);
  }
  // reference solution by Gaussian elimination with partial pivoting
  std::vector<Complex> G = A, xs = b;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(G[size_t(i) * n + k]) > std::abs(G[size_t(p) * n + k])) p = i;
    for (int j = 0; j < n; ++j) std::swap(G[size_t(k) * n + j], G[size_t(p) * n + j]);
    std::swap(xs[k], xs[p]);
    for (int i = k + 1; i < n; ++i) {
      const Complex f = G[size_t(i) * n + k] / G[size_t(k) * n + k];
      for (int j = k; j < n; ++j) G[size_t(i) * n + j] -= f * G[size_t(k) * n + j];
      xs[i] -= f * xs[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) xs[i] -= G[size_t(i) * n + j] * xs[j];
    xs[i] /= G[size_t(i) * n + i];
  }
  LinearOp Aop = [&](const Complex* v, Complex* y) {
    for (int i = 0; i < n; ++i) {
      Complex acc = 0;
      for (int j = 0; j < n; ++j) acc += A[size_t(i) * n + j] * v[j];
      y[i] = acc;
    }
  };
  int calls = 0;
  LinearOp Mvar = [&](const Complex* v, Complex* z) {  // Jacobi on odd calls, identity else
    ++calls;
    for (int i = 0; i < n; ++i) z[i] = (calls % 2) ? v[i] / A[size_t(i) * n + i] : v[i];
  };
  for (int restart : {0, 7}) {
    FgmresOptions o;
    o.tol = 1e-12;
    o.max_iters = 200;
    o.restart = restart;
    std::vector<Complex> x;
    const FgmresResult r = fgmres(n, Aop, restart ? Mvar : LinearOp(), b, x, o);
    CHECK(r.converged && r.true_relres <= 1e-11 && int(r.history.size()) == r.iters);
    double e = 0, d = 0;
    for (int i = 0; i < n; ++i) {
      e += std::norm(x[i] - xs[i]);
      d += std::norm(xs[i]);
    }
    CHECK(std::sqrt(e / d) <= 1e-10);
  }
  std::vector<Complex> x0;
  const FgmresResult r0 = fgmres(n, Aop, LinearOp(), std::vector<Complex>(n), x0, FgmresOptions());
  CHECK(r0.converged && r0.iters == 0 && x0.size() == size_t(n));
  std::printf("host fgmres ok\n");
  return 0;
}
