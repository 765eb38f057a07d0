// Host setup: grid, partition, medium, PML coefficient arrays and operator
// classes -- the part of DdmEngine's constructor that stays on the host
// (proj/src/ddm.cpp:62-128). Formulas follow SURVEY.md Appendix A; each block
// cites the reference lines it reproduces. Nothing here touches the GPU.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <string>

#include "hddm_internal.h"

namespace hddm {

namespace {

using cd = std::complex<double>;

// beta0, proj/src/partition.cpp:7-11
double beta0(double t) {
  if (t <= 0) return 1.0;
  if (t >= 1) return 0.0;
  return 1.0 - t * t * t * (10.0 - 15.0 * t + 6.0 * t * t);
}

// axis_weights, partition.cpp:34-47
void axis_weights(std::vector<double>& w, int o, int n, int c0, int c1, bool lo,
                  bool hi, int nov) {
  w.assign(n, 1.0);
  for (int t = 0; t < n; ++t) {
    const int p = o + t;
    double v = 1.0;
    if (p < c0)
      v = lo ? beta0(double(c0 - 1 - p) / nov) : 1.0;
    else if (p > c1)
      v = hi ? beta0(double(p - c1 - 1) / nov) : 1.0;
    w[t] = v;
  }
}

// shifted_sigma, pml.cpp:7-12
double shifted_sigma(double s0, double d, double dsh, double t) {
  if (t <= dsh) return 0.0;
  if (t >= dsh + d) return s0;
  const double s = (t - dsh) / d;
  return s0 * s * s;
}

// alpha_axis, discretize.cpp:21-37
cd alpha_axis(int m, int c0, int c1, bool lo, bool hi, const Setup& S) {
  const double h2 = 0.5 * S.h;
  const double d = S.nramp * S.h;
  double sig = 0;
  const int dl = 2 * c0 - m;
  if (dl > 0) sig += shifted_sigma(S.sigma0, d, lo ? S.nov * S.h : 0.0, dl * h2);
  const int dr = m - 2 * c1;
  if (dr > 0) sig += shifted_sigma(S.sigma0, d, hi ? S.nov * S.h : 0.0, dr * h2);
  return cd(1.0, sig);
}

void put(std::vector<double>& v, int i, cd z) {
  v[2 * i] = z.real();
  v[2 * i + 1] = z.imag();
}

// build_operator's 1-D arrays, discretize.cpp:41-70
void axis_arrays(const Setup& S, int x0, int nx, int c0, int c1, bool lo, bool hi,
                 std::vector<double>& an, std::vector<double>& iah) {
  an.assign(2 * size_t(nx), 0.0);
  iah.assign(2 * size_t(nx), 0.0);
  for (int lp = 0; lp < nx; ++lp) {
    const int m = 2 * (x0 + lp);
    put(an, lp, alpha_axis(m, c0, c1, lo, hi, S));
    if (lp + 1 < nx) put(iah, lp, 1.0 / alpha_axis(m + 1, c0, c1, lo, hi, S));
  }
}

double lens_c(const Medium& m, double xc, double yc) {
  const double dx = xc - m.lxc, dy = yc - m.lyc;
  return m.velocity - m.lamp * std::exp(-(dx * dx + dy * dy) / m.lw);
}

// eval_wavenumber, medium.cpp:31-50 (+ lens extension, both axes clamped)
bool eval_k(const Medium& m, double x, double y, double& k) {
  if (x < m.bx0 - m.margin || x > m.bx1 + m.margin || y < m.by0 - m.margin ||
      y > m.by1 + m.margin)
    return false;
  const double yc = std::clamp(y, m.by0, m.by1);
  double c;
  if (m.kind == 0) {
    c = m.velocity;
  } else if (m.kind == 1) {
    c = m.c.back();
    for (size_t l = 0; l < m.c.size(); ++l)
      if (yc <= m.yhi[l]) {
        c = m.c[l];
        break;
      }
  } else {
    c = lens_c(m, std::clamp(x, m.bx0, m.bx1), yc);
  }
  k = m.omega / c;
  return true;
}

}  // namespace

int build_setup(const hddm_problem& p, Setup& S, std::string& msg) {
  S = Setup();
  S.x0 = p.x0;
  S.y0 = p.y0;
  S.h = p.h;
  S.mx = p.mx;
  S.my = p.my;
  S.n1 = p.n1;
  S.n2 = p.n2;
  S.nov = p.n_overlap;
  S.nramp = p.n_ramp;
  S.c_sigma = p.c_sigma;
  // check_spec, partition.cpp:15-28
  auto cfg_err = [&](const char* m) {
    msg = m;
    return HDDM_ERR_CONFIG;
  };
  if (!(S.h > 0)) return cfg_err("grid spacing must be positive");
  if (S.mx < 1 || S.my < 1) return cfg_err("interior cell counts must be positive");
  if (S.n1 < 1 || S.n2 < 1) return cfg_err("subdomain counts must be positive");
  if (S.mx % S.n1 || S.my % S.n2)
    return cfg_err("interior cells must divide evenly among subdomains");
  if (S.nramp < 1) return cfg_err("absorber ramp width must be positive");
  if (S.nov < 0) return cfg_err("overlap width must be nonnegative");
  const bool split = S.n1 > 1 || S.n2 > 1;
  if (split && S.nov < 1) return cfg_err("overlap width must be positive when the domain is split");
  if (split && (S.mx / S.n1 < S.nov + 1 || S.my / S.n2 < S.nov + 1))
    return cfg_err("subdomain cores too small for the requested overlap");
  S.ext = S.nov + S.nramp;
  S.gnx = S.mx + 2 * S.ext + 1;
  S.gny = S.my + 2 * S.ext + 1;
  S.mcx = S.mx / S.n1;
  S.mcy = S.my / S.n2;

  Medium& m = S.med;
  m.kind = p.medium_kind;
  m.omega = p.omega;
  m.velocity = p.velocity;
  for (int l = 0; l < p.n_layers; ++l) {
    m.ylo.push_back(p.layer_ylo[l]);
    m.yhi.push_back(p.layer_yhi[l]);
    m.c.push_back(p.layer_c[l]);
  }
  m.bx0 = S.x0;
  m.bx1 = S.x0 + S.mx * S.h;
  m.by0 = S.y0;
  m.by1 = S.y0 + S.my * S.h;
  m.margin = (S.ext + 1) * S.h;  // ddm.cpp:66-67
  if (p.has_box) {  // the caller's MediumModel::interior / margin (medium.hpp:23-24)
    m.bx0 = p.box_x0;
    m.bx1 = p.box_x1;
    m.by0 = p.box_y0;
    m.by1 = p.box_y1;
    m.margin = std::max(p.margin, m.margin);
  }
  m.lamp = p.lens_amp;
  m.lxc = p.lens_xc;
  m.lyc = p.lens_yc;
  m.lw = p.lens_w;
  const double ox = S.x0 - S.ext * S.h, oy = S.y0 - S.ext * S.h;
  if (m.kind == 0) {
    m.cmin = m.cmax = m.velocity;
  } else if (m.kind == 1) {
    if (m.c.empty()) return cfg_err("layered medium needs at least one layer");
    m.cmin = *std::min_element(m.c.begin(), m.c.end());
    m.cmax = *std::max_element(m.c.begin(), m.c.end());
  } else if (m.kind == 2) {
    m.cmin = INFINITY;
    m.cmax = -INFINITY;
    for (int q = 0; q < S.gny; ++q)
      for (int pp = 0; pp < S.gnx; ++pp) {
        const double c = lens_c(m, std::clamp(ox + pp * S.h, m.bx0, m.bx1),
                                std::clamp(oy + q * S.h, m.by0, m.by1));
        m.cmin = std::min(m.cmin, c);
        m.cmax = std::max(m.cmax, c);
      }
  } else {
    return cfg_err("unknown medium kind");
  }
  // sigma0 = default_sigma0(c_sigma, k_min, n_ramp h), ddm.cpp:68-71, pml.cpp:14-16
  const double kmin = m.omega / m.cmax;
  S.sigma0 = p.sigma0 > 0 ? p.sigma0 : 3.0 * p.c_sigma / (kmin * (S.nramp * S.h));

  // global operator (global_layout, discretize.cpp:11-14) and nodal k^2
  axis_arrays(S, 0, S.gnx, S.ext, S.ext + S.mx, false, false, S.gop.a1n, S.gop.ia1h);
  axis_arrays(S, 0, S.gny, S.ext, S.ext + S.my, false, false, S.gop.a2n, S.gop.ia2h);
  S.k2.assign(size_t(S.gnx) * S.gny, 0.0);
  for (int q = 0; q < S.gny; ++q) {
    const double y = oy + q * S.h;
    for (int pp = 0; pp < S.gnx; ++pp) {
      double k;
      if (!eval_k(m, ox + pp * S.h, y, k)) {
        msg = "eval_wavenumber: point outside the padded domain";
        return HDDM_ERR_OTHER;
      }
      S.k2[size_t(q) * S.gnx + pp] = k * k;
    }
  }

  // partition, partition.cpp:51-83; owned rects ddm.cpp:90-94
  const int nsub = S.n1 * S.n2;
  S.subs.resize(nsub);
  S.subop.resize(nsub);
  for (int j = 0; j < S.n2; ++j)
    for (int i = 0; i < S.n1; ++i) {
      Sub& s = S.subs[j * S.n1 + i];
      s.i = i;
      s.j = j;
      s.cx0 = S.ext + i * S.mcx;
      s.cx1 = s.cx0 + S.mcx;
      s.cy0 = S.ext + j * S.mcy;
      s.cy1 = s.cy0 + S.mcy;
      s.wx0 = s.cx0 - S.ext;
      s.wy0 = s.cy0 - S.ext;
      s.nx = S.mcx + 2 * S.ext + 1;
      s.ny = S.mcy + 2 * S.ext + 1;
      s.lint = i > 0;
      s.rint = i < S.n1 - 1;
      s.bint = j > 0;
      s.tint = j < S.n2 - 1;
      axis_weights(s.wx, s.wx0, s.nx, s.cx0, s.cx1, s.lint, s.rint, S.nov);
      axis_weights(s.wy, s.wy0, s.ny, s.cy0, s.cy1, s.bint, s.tint, S.nov);
      s.own[0] = i == 0 ? 0 : S.ext + i * S.mcx + 1;
      s.own[1] = i == S.n1 - 1 ? S.gnx - 1 : S.ext + (i + 1) * S.mcx;
      s.own[2] = j == 0 ? 0 : S.ext + j * S.mcy + 1;
      s.own[3] = j == S.n2 - 1 ? S.gny - 1 : S.ext + (j + 1) * S.mcy;
      WinOp& w = S.subop[j * S.n1 + i];
      axis_arrays(S, s.wx0, s.nx, s.cx0, s.cx1, s.lint, s.rint, w.a1n, w.ia1h);
      axis_arrays(S, s.wy0, s.ny, s.cy0, s.cy1, s.bint, s.tint, w.a2n, w.ia2h);
    }

  // classes: bitwise-identical coefficient arrays (op_equal, ddm.cpp:37-50,
  // 103-128). Window k^2 is a sub-block of the global k^2 (same lattice nodes).
  const int wnx = S.subs[0].nx, wny = S.subs[0].ny;
  auto same = [&](int a, int b) {
    const WinOp &A = S.subop[a], &B = S.subop[b];
    if (std::memcmp(A.a1n.data(), B.a1n.data(), A.a1n.size() * 8) ||
        std::memcmp(A.ia1h.data(), B.ia1h.data(), A.ia1h.size() * 8) ||
        std::memcmp(A.a2n.data(), B.a2n.data(), A.a2n.size() * 8) ||
        std::memcmp(A.ia2h.data(), B.ia2h.data(), A.ia2h.size() * 8))
      return false;
    const Sub &sa = S.subs[a], &sb = S.subs[b];
    for (int q = 0; q < wny; ++q)
      if (std::memcmp(&S.k2[size_t(sa.wy0 + q) * S.gnx + sa.wx0],
                      &S.k2[size_t(sb.wy0 + q) * S.gnx + sb.wx0], size_t(wnx) * 8))
        return false;
    return true;
  };
  S.ncls = 0;
  for (int t = 0; t < nsub; ++t) {
    int cls = -1;
    for (int c = 0; c < S.ncls && cls < 0; ++c)
      if (same(S.cls_rep[c], t)) cls = c;
    if (cls < 0) {
      cls = S.ncls++;
      S.cls_rep.push_back(t);
    }
    S.subs[t].cls = cls;
  }
  S.cls_ptr.assign(S.ncls + 1, 0);
  for (int t = 0; t < nsub; ++t) ++S.cls_ptr[S.subs[t].cls + 1];
  for (int c = 0; c < S.ncls; ++c) S.cls_ptr[c + 1] += S.cls_ptr[c];
  S.cls_members.assign(nsub, 0);
  std::vector<int> fill(S.cls_ptr.begin(), S.cls_ptr.end() - 1);
  for (int t = 0; t < nsub; ++t) S.cls_members[fill[S.subs[t].cls]++] = t;
  return 0;
}

}  // namespace hddm
