// Host setup and symbolic analysis of the 3-D path (BASELINE config 5).
//
// Geometry and coefficients: every per-axis rule of the 2-D setup
// (proj/src/partition.cpp:15-83, discretize.cpp:21-79, pml.cpp:7-16) applied to
// x, y and z, as the restatement oracle/hddm_oracle3.c writes it out (the
// reference has no 3-D code). Classes: bitwise-identical coefficient arrays
// share one factorization (ddm.cpp:19-50).
//
// Symbolic: shell-first plane-separator nested dissection (hddm_oracle3.c's
// order, sparse.cpp:20-57 with planes for lines), one supernode per nd call,
// dense supernode row structures, the exact nnz(L) of the restatement's
// up-looking factor, and the front / update / scatter maps of the GPU's
// multifrontal factorization and dense supernodal solves.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <stdexcept>

#include "engine3d.h"

namespace hddm3 {

namespace {

constexpr int kLeaf = 3;  // boxes of at most 3 nodes per side are leaves (ORC3_LEAF)

double beta0(double t) {
  if (t <= 0) return 1.0;
  if (t >= 1) return 0.0;
  return 1.0 - t * t * t * (10.0 - 15.0 * t + 6.0 * t * t);
}

double shifted_sigma(double s0, double d, double dsh, double t) {
  if (t <= dsh) return 0.0;
  if (t >= dsh + d) return s0;
  const double s = (t - dsh) / d;
  return s0 * s * s;
}

using cd = std::complex<double>;

cd alpha_axis(int m, int c0, int c1, bool lo, bool hi, const Setup3& S) {
  const double h2 = 0.5 * S.h;
  const double d = S.nramp * S.h;
  double sig = 0;
  const int dl = 2 * c0 - m;
  if (dl > 0) sig += shifted_sigma(S.sigma0, d, lo ? S.nov * S.h : 0.0, dl * h2);
  const int dr = m - 2 * c1;
  if (dr > 0) sig += shifted_sigma(S.sigma0, d, hi ? S.nov * S.h : 0.0, dr * h2);
  return cd(1.0, sig);
}

void build_op(Op3& op, const Setup3& S, const int* o, const int* nn, const int* c0, const int* c1,
              const int* lo, const int* hi) {
  for (int a = 0; a < 3; ++a) {
    op.an[a].assign(2 * size_t(nn[a]), 0.0);
    op.iah[a].assign(2 * size_t(nn[a]), 0.0);
    for (int l = 0; l < nn[a]; ++l) {
      const int m = 2 * (o[a] + l);
      const cd v = alpha_axis(m, c0[a], c1[a], lo[a], hi[a], S);
      op.an[a][2 * l] = v.real();
      op.an[a][2 * l + 1] = v.imag();
      if (l + 1 < nn[a]) {
        const cd iv = cd(1.0, 0.0) / alpha_axis(m + 1, c0[a], c1[a], lo[a], hi[a], S);
        op.iah[a][2 * l] = iv.real();
        op.iah[a][2 * l + 1] = iv.imag();
      }
    }
  }
}

bool op_equal(const Op3& a, const Op3& b) {
  for (int x = 0; x < 3; ++x)
    if (a.an[x] != b.an[x] || a.iah[x] != b.iah[x]) return false;
  return true;  // k^2 is one constant for the whole medium
}

void axis_weights(std::vector<double>& w, int o, int n, int c0, int c1, bool lo, bool hi, int nov) {
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

}  // namespace

int build_setup3(const hddm3_problem& p, Setup3& S, std::string& msg) {
  S = Setup3();
  S.x0 = p.x0;
  S.y0 = p.y0;
  S.z0 = p.z0;
  S.h = p.h;
  const int m[3] = {p.mx, p.my, p.mz}, nd[3] = {p.n1, p.n2, p.n3};
  for (int a = 0; a < 3; ++a) {
    S.m[a] = m[a];
    S.n[a] = nd[a];
  }
  S.nov = p.n_overlap;
  S.nramp = p.n_ramp;
  // check_spec, partition.cpp:15-28 per axis
  auto cfg = [&](const char* s) {
    msg = s;
    return HDDM_ERR_CONFIG;
  };
  if (!(p.h > 0)) return cfg("grid spacing must be positive");
  for (int a = 0; a < 3; ++a)
    if (m[a] < 1) return cfg("interior cell counts must be positive");
  for (int a = 0; a < 3; ++a)
    if (nd[a] < 1) return cfg("subdomain counts must be positive");
  for (int a = 0; a < 3; ++a)
    if (m[a] % nd[a]) return cfg("interior cells must divide evenly among subdomains");
  if (p.n_ramp < 1) return cfg("absorber ramp width must be positive");
  if (p.n_overlap < 0) return cfg("overlap width must be nonnegative");
  const bool split = nd[0] > 1 || nd[1] > 1 || nd[2] > 1;
  if (split && p.n_overlap < 1) return cfg("overlap width must be positive when the domain is split");
  for (int a = 0; a < 3; ++a)
    if (split && m[a] / nd[a] < p.n_overlap + 1) return cfg("subdomain cores too small for the requested overlap");
  if (!(p.velocity > 0) || !(p.omega > 0)) return cfg("velocity and omega must be positive");
  S.ext = S.nov + S.nramp;
  for (int a = 0; a < 3; ++a) {
    S.gn[a] = m[a] + 2 * S.ext + 1;
    S.mc[a] = m[a] / nd[a];
  }
  S.omega = p.omega;
  S.velocity = p.velocity;
  const double kmin = p.omega / p.velocity;
  S.sigma0 = p.sigma0 > 0 ? p.sigma0 : 3.0 * p.c_sigma / (kmin * (S.nramp * S.h));  // pml.cpp:14-16
  S.k2 = kmin * kmin;
  {
    const int o[3] = {0, 0, 0}, z[3] = {0, 0, 0};
    const int c0[3] = {S.ext, S.ext, S.ext};
    const int c1[3] = {S.ext + m[0], S.ext + m[1], S.ext + m[2]};
    build_op(S.gop, S, o, S.gn, c0, c1, z, z);
  }
  const int nsub = nd[0] * nd[1] * nd[2];
  S.subs.resize(nsub);
  S.subop.resize(nsub);
  for (int t = 0; t < nsub; ++t) {
    Sub3& s = S.subs[t];
    s.ix[0] = t % nd[0];
    s.ix[1] = (t / nd[0]) % nd[1];
    s.ix[2] = t / (nd[0] * nd[1]);
    for (int a = 0; a < 3; ++a) {
      const int i = s.ix[a];
      s.c0[a] = S.ext + i * S.mc[a];
      s.c1[a] = s.c0[a] + S.mc[a];
      s.w0[a] = s.c0[a] - S.ext;
      s.nn[a] = S.mc[a] + 2 * S.ext + 1;
      s.lo[a] = i > 0;
      s.hi[a] = i < nd[a] - 1;
      axis_weights(s.w[a], s.w0[a], s.nn[a], s.c0[a], s.c1[a], s.lo[a], s.hi[a], S.nov);
      s.own0[a] = i == 0 ? 0 : S.ext + i * S.mc[a] + 1;
      s.own1[a] = i == nd[a] - 1 ? S.gn[a] - 1 : S.ext + (i + 1) * S.mc[a];
    }
    build_op(S.subop[t], S, s.w0, s.nn, s.c0, s.c1, s.lo, s.hi);
    int cls = -1;
    for (int c = 0; c < S.ncls && cls < 0; ++c)
      if (op_equal(S.subop[S.cls_rep[c]], S.subop[t])) cls = c;
    if (cls < 0) {
      cls = S.ncls++;
      S.cls_rep.push_back(t);
    }
    s.cls = cls;
  }
  S.cls_ptr.assign(S.ncls + 1, 0);
  for (int t = 0; t < nsub; ++t) ++S.cls_ptr[S.subs[t].cls + 1];
  for (int c = 0; c < S.ncls; ++c) S.cls_ptr[c + 1] += S.cls_ptr[c];
  S.cls_members.assign(nsub, 0);
  std::vector<int> fill(S.cls_ptr.begin(), S.cls_ptr.end() - 1);
  for (int t = 0; t < nsub; ++t) S.cls_members[fill[S.subs[t].cls]++] = t;
  return 0;
}

// --------------------------------------------------------------- symbolic
namespace {

struct Nd3 {
  int nx, ny;
  std::vector<int>& order;
  std::vector<Sn3>& sn;
  int rec(int x0, int y0, int z0, int w, int h, int d) {
    if (w <= 0 || h <= 0 || d <= 0) return -1;
    Sn3 node;
    node.box[0] = x0; node.box[1] = y0; node.box[2] = z0;
    node.box[3] = w; node.box[4] = h; node.box[5] = d;
    int a = -1, b = -1;
    std::vector<int> own;
    if (w <= kLeaf && h <= kLeaf && d <= kLeaf) {
      for (int r = z0; r < z0 + d; ++r)
        for (int q = y0; q < y0 + h; ++q)
          for (int p = x0; p < x0 + w; ++p) own.push_back((r * ny + q) * nx + p);
    } else if (w >= h && w >= d) {
      const int mid = x0 + w / 2;
      a = rec(x0, y0, z0, mid - x0, h, d);
      b = rec(mid + 1, y0, z0, x0 + w - mid - 1, h, d);
      for (int r = z0; r < z0 + d; ++r)
        for (int q = y0; q < y0 + h; ++q) own.push_back((r * ny + q) * nx + mid);
    } else if (h >= d) {
      const int mid = y0 + h / 2;
      a = rec(x0, y0, z0, w, mid - y0, d);
      b = rec(x0, mid + 1, z0, w, y0 + h - mid - 1, d);
      for (int r = z0; r < z0 + d; ++r)
        for (int p = x0; p < x0 + w; ++p) own.push_back((r * ny + mid) * nx + p);
    } else {
      const int mid = z0 + d / 2;
      a = rec(x0, y0, z0, w, h, mid - z0);
      b = rec(x0, y0, mid + 1, w, h, z0 + d - mid - 1);
      for (int q = y0; q < y0 + h; ++q)
        for (int p = x0; p < x0 + w; ++p) own.push_back((mid * ny + q) * nx + p);
    }
    node.c0 = int(order.size());
    order.insert(order.end(), own.begin(), own.end());
    node.n = int(own.size());
    for (int c : {a, b})
      if (c >= 0) node.ch[node.nch++] = c;
    sn.push_back(node);
    const int id = int(sn.size()) - 1;
    for (int k = 0; k < sn[id].nch; ++k) sn[sn[id].ch[k]].parent = id;
    return id;
  }
};

bool on_shell(const int* nn, int p, int q, int r) {
  return p == 0 || q == 0 || r == 0 || p == nn[0] - 1 || q == nn[1] - 1 || r == nn[2] - 1;
}

}  // namespace

std::vector<int> nd_order3(int nx, int ny, int nz) {
  Sym3 S;
  build_sym3(nx, ny, nz, S);
  return S.perm;
}

// The dense-supernode structure of an ND tree: heights / depths, row structures, exact nnz(L), value / update /
// front layouts, extend-add maps and the assembled-matrix scatter lists. nbr(v, k),
// k < nk, is the k-th interior neighbour of window node v or -1.
template <class Nbr>
void finish_dense(Sym3& S, Nbr nbr, int nk) {
  const int n = S.n;
  const int nsn = int(S.sn.size());
  for (int s = 0; s < nsn; ++s) {
    int hgt = 0;
    for (int k = 0; k < S.sn[s].nch; ++k) hgt = std::max(hgt, S.sn[S.sn[s].ch[k]].height + 1);
    S.sn[s].height = hgt;
    S.max_height = std::max(S.max_height, hgt);
  }
  S.sn[S.root].depth = 0;
  for (int s = nsn - 1; s >= 0; --s)
    if (S.sn[s].parent >= 0) {
      S.sn[s].depth = S.sn[S.sn[s].parent].depth + 1;
      S.max_depth = std::max(S.max_depth, S.sn[s].depth);
    }
  // dense supernode row structures (postorder: children first)
  for (int s = 0; s < nsn; ++s) {
    Sn3& a = S.sn[s];
    const int end = a.c0 + a.n;
    std::vector<int> cand;
    for (int k = 0; k < a.nch; ++k)
      for (int r : S.sn[a.ch[k]].rows)
        if (r >= end) cand.push_back(r);
    for (int i = 0; i < a.n; ++i) {
      const int v = S.perm[a.c0 + i];
      for (int k = 0; k < nk; ++k) {
        const int u = nbr(v, k);
        if (u >= 0 && S.pinv[u] >= end) cand.push_back(S.pinv[u]);
      }
    }
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    a.rows = std::move(cand);
  }
  // exact nnz(L) of the up-looking factor: elimination tree + row counts
  {
    std::vector<int> parent(n, -1), anc(n, -1), mark(n, -1);
    long nnz = 0;
    for (int k = S.nshell; k < n; ++k) {
      const int v = S.perm[k];
      for (int d = 0; d < nk; ++d) {
        const int u = nbr(v, d);
        if (u < 0) continue;
        int i = S.pinv[u];
        while (i >= 0 && i < k) {
          const int nxt = anc[i];
          anc[i] = k;
          if (nxt == -1) parent[i] = k;
          i = nxt;
        }
      }
    }
    for (int k = S.nshell; k < n; ++k) {
      mark[k] = k;
      const int v = S.perm[k];
      for (int d = 0; d < nk; ++d) {
        const int u = nbr(v, d);
        if (u < 0) continue;
        for (int i = S.pinv[u]; i >= 0 && i < k && mark[i] != k; i = parent[i]) {
          mark[i] = k;
          ++nnz;
        }
      }
    }
    S.nnz_ref = nnz + n;
  }
  // value layout, update vectors, child maps, rows
  S.linv_off.assign(nsn, 0);
  S.pan_off.assign(nsn, 0);
  S.upd_off.assign(nsn, 0);
  S.cmap_off.assign(nsn + 1, 0);
  S.rows_off.assign(nsn + 1, 0);
  long off = n;  // D first
  long upd = 0, cm = 0, ro = 0;
  S.stored_lower = 0;
  for (int s = 0; s < nsn; ++s) {
    const Sn3& a = S.sn[s];
    const long r = long(a.rows.size());
    S.linv_off[s] = off;
    off += long(a.n) * (a.n - 1) / 2;
    S.pan_off[s] = off;
    off += r * a.n;
    S.stored_lower += long(a.n) * (a.n - 1) / 2 + r * a.n;
    S.upd_off[s] = upd;
    upd += r;
    S.cmap_off[s] = cm;
    cm += a.n + r;
    S.rows_off[s] = ro;
    ro += r;
  }
  S.nvals = off;
  S.nupd = upd;
  S.cmap_off[nsn] = cm;
  S.rows_off[nsn] = ro;
  S.rows_all.reserve(ro);
  for (int s = 0; s < nsn; ++s) S.rows_all.insert(S.rows_all.end(), S.sn[s].rows.begin(), S.sn[s].rows.end());
  S.cmap0.assign(cm, -1);
  S.cmap1.assign(cm, -1);
  for (int s = 0; s < nsn; ++s) {
    const Sn3& a = S.sn[s];
    for (int k = 0; k < a.nch; ++k) {
      const int c = a.ch[k];
      const auto& cr = S.sn[c].rows;
      for (size_t i = 0; i < cr.size(); ++i) {
        const int P = cr[i];
        int f;
        if (P < a.c0 + a.n) {
          f = P - a.c0;
        } else {
          auto it = std::lower_bound(a.rows.begin(), a.rows.end(), P);
          if (it == a.rows.end() || *it != P) throw std::runtime_error("child row outside the parent front");
          f = a.n + int(it - a.rows.begin());
        }
        (k == 0 ? S.cmap0 : S.cmap1)[S.cmap_off[s] + f] = int(S.upd_off[c] + long(i));
      }
    }
  }
  // fronts (2n + r) x (n + r), extend-add maps, assembled-matrix scatter lists
  S.front_off.assign(nsn, 0);
  S.ext_off.assign(nsn + 1, 0);
  S.front_words = 0;
  for (int s = 0; s < nsn; ++s) {
    const Sn3& a = S.sn[s];
    const long r = long(a.rows.size());
    S.front_off[s] = S.front_words;
    S.front_words += (2L * a.n + r) * (a.n + r);
  }
  for (int s = 0; s < nsn; ++s) {
    S.ext_off[s] = long(S.ext.size());
    const Sn3& a = S.sn[s];
    if (a.parent < 0) continue;
    const Sn3& p = S.sn[a.parent];
    for (int P : a.rows) {
      int f;
      if (P < p.c0 + p.n) {
        f = P - p.c0;
      } else {
        auto it = std::lower_bound(p.rows.begin(), p.rows.end(), P);
        f = p.n + int(it - p.rows.begin());
      }
      S.ext.push_back(f);
    }
  }
  S.ext_off[nsn] = long(S.ext.size());
  S.aent_ptr.assign(nsn + 1, 0);
  for (int s = 0; s < nsn; ++s) {
    const Sn3& a = S.sn[s];
    S.aent_ptr[s] = int(S.aent_i.size());
    for (int j = 0; j < a.n; ++j) {
      const int v = S.perm[a.c0 + j];
      S.aent_i.push_back(j);
      S.aent_j.push_back(j);
      S.aent_node.push_back(v);
      S.aent_kind.push_back(0);
      for (int k = 0; k < nk; ++k) {
        const int u = nbr(v, k);
        if (u < 0) continue;
        const int P = S.pinv[u];
        if (P <= a.c0 + j) continue;  // upper triangle / descendants
        int f;
        if (P < a.c0 + a.n) {
          f = P - a.c0;
        } else {
          auto it = std::lower_bound(a.rows.begin(), a.rows.end(), P);
          if (it == a.rows.end() || *it != P) throw std::runtime_error("matrix entry outside the front");
          f = a.n + int(it - a.rows.begin());
        }
        S.aent_i.push_back(f);
        S.aent_j.push_back(j);
        S.aent_node.push_back(v);
        S.aent_kind.push_back(1 + k);
      }
    }
  }
  S.aent_ptr[nsn] = int(S.aent_i.size());
}


void build_sym3(int nx, int ny, int nz, Sym3& S) {
  if (nx <= 2 || ny <= 2 || nz <= 2) throw std::runtime_error("window too small for the 3-D ND solver");
  S = Sym3();
  S.nn[0] = nx;
  S.nn[1] = ny;
  S.nn[2] = nz;
  S.n = nx * ny * nz;
  const int n = S.n, sxy = nx * ny;
  for (int r = 0; r < nz; ++r)
    for (int q = 0; q < ny; ++q)
      for (int p = 0; p < nx; ++p)
        if (on_shell(S.nn, p, q, r)) S.perm.push_back((r * ny + q) * nx + p);
  S.nshell = int(S.perm.size());
  Nd3 b{nx, ny, S.perm, S.sn};
  S.root = b.rec(1, 1, 1, nx - 2, ny - 2, nz - 2);
  if (int(S.perm.size()) != n) throw std::runtime_error("3-D ND order is not a permutation");
  S.pinv.assign(n, -1);
  for (int k = 0; k < n; ++k) S.pinv[S.perm[k]] = k;
  // interior neighbours of a window node (-1: shell or outside)
  auto nbr = [&](int v, int k) -> int {
    const int p = v % nx, q = (v / nx) % ny, r = v / sxy;
    int pp = p, qq = q, rr = r;
    switch (k) {
      case 0: pp = p - 1; break;
      case 1: pp = p + 1; break;
      case 2: qq = q - 1; break;
      case 3: qq = q + 1; break;
      case 4: rr = r - 1; break;
      default: rr = r + 1; break;
    }
    if (pp < 0 || qq < 0 || rr < 0 || pp >= nx || qq >= ny || rr >= nz) return -1;
    if (on_shell(S.nn, pp, qq, rr)) return -1;
    return (rr * ny + qq) * nx + pp;
  };
  finish_dense(S, nbr, 6);
}

}  // namespace hddm3
