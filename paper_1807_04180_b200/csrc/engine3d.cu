// The engine's 3-D path (BASELINE config 5) behind include/hddm3.h: host
// setup, the batched multifrontal factorization of every class, the DDM step
// (flags, 26-direction RHS, dense supernodal solves, refine inside a WHILE graph
// node, blend-accumulate) captured as CUDA graphs, the device-resident FGMRES,
// and the C-ABI. The reference has no 3-D code: the math is the restatement
// oracle/hddm_oracle3.c, generalizing ddm.cpp / krylov.cpp / sparse.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dense_factor.h"
#include "engine3d.h"
#include "kernels.cuh"
#include "kernels3d.cuh"
#include "kernels_krylov.cuh"

using hddm::cplx;
using namespace hddm3;

namespace {

thread_local std::string g_err3;

struct SolveErr3 : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigErr3 : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK3(x)                                                                           \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                               " at " __FILE__ ":" + std::to_string(__LINE__));          \
  } while (0)

double now_ms3() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

inline cplx cmk3(double r, double i) { return make_double2(r, i); }

constexpr int kChunks = 32;    // residual-check partials per RHS
constexpr int kDiagRows = 32;  // rows per forward inverse / panel task

}  // namespace

struct hddm3_engine {
  Setup3 S;
  Sym3 Y;
  int dev = -1;
  cudaStream_t st = nullptr, st2 = nullptr;
  std::string err;
  int nsub = 0, ncls = 0, nw = 0, ngroups = 1, max_members = 1, mg = 4;
  long long ng = 0;
  double factor_ms = 0;
  std::vector<double> probe;
  size_t dev_bytes = 0;  // bytes currently allocated
  std::vector<std::pair<void*, size_t>> allocs;
  long long launches = 0;
  int last_step = 0;
  double last_max_rel = 0;
  int last_corr = 0;

  // symbolic tables
  DSn3* d_sn = nullptr;
  int *d_rows = nullptr, *d_cmap0 = nullptr, *d_cmap1 = nullptr;
  int *d_perm = nullptr, *d_pinv = nullptr;
  int *d_cls_ptr = nullptr, *d_cls_mem = nullptr;
  cplx* d_vals = nullptr;
  cplx* d_valsT = nullptr;  // backward (row-major) copy of the blocks
  struct Lvl {
    Task3* d = nullptr;
    int n = 0, nbig = 0;
  };
  std::vector<Lvl> f_asm, f_diag, f_pan, b_gat, b_pan, b_diag;
  Lvl f_leaf, b_leaf;  // fused leaf kernels (all leaves at most 32 nodes)
  // per subdomain
  Sub3Dev* d_sub = nullptr;
  cplx* d_cop = nullptr;
  int cop_stride = 0;
  double* d_wts = nullptr;
  int* d_cov = nullptr;
  // transfer tables (k3d_rhs_xfer)
  int npatch = 0;
  int *d_pnode = nullptr, *d_pent = nullptr, *d_edir = nullptr, *d_esrc = nullptr;
  double* d_ebeta = nullptr;
  void build_transfer_tables();
  cplx* d_U[4] = {};
  int* d_Z[4] = {};
  cplx *d_B = nullptr, *d_Y = nullptr, *d_UPD = nullptr, *d_R = nullptr, *d_C = nullptr;
  int *d_fany = nullptr, *d_isrep = nullptr;
  long long* d_counts = nullptr;
  double *d_part_chk = nullptr, *d_rel_cur = nullptr, *d_rel_prev = nullptr, *d_maxrel = nullptr;
  int *d_need = nullptr, *d_ncorr = nullptr, *d_undo = nullptr, *d_any = nullptr, *d_ccount = nullptr;
  // global
  cplx* d_ga = nullptr;
  cplx *d_f = nullptr, *d_asm = nullptr;
  double *d_part = nullptr, *d_scal = nullptr, *h_scal = nullptr;
  // graphs: step 1 and steps >= 2 by s mod 4
  cudaGraphExec_t step_exec[5] = {};
  int step_kernels[5] = {};
  // krylov
  int kry_m = 0;
  std::vector<cplx*> V, Z;
  cplx **d_Vptr = nullptr, **d_Zptr = nullptr;
  cplx *d_H = nullptr, *d_g = nullptr, *d_sn_g = nullptr, *d_y = nullptr;
  cplx *d_b = nullptr, *d_x = nullptr, *d_r = nullptr;
  double* d_cs = nullptr;
  hddm::KryState *d_ks = nullptr, *h_ks = nullptr;
  double* d_hist = nullptr;
  int d_hist_cap = 0, kry_k_last = 0, kry_K = -1, kry_iter_kernels = 0;
  cudaGraphExec_t kry_exec = nullptr;

  template <class T>
  T* dalloc(size_t n) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    CK3(cudaMalloc(&p, bytes));
    allocs.push_back({p, bytes});
    dev_bytes += bytes;
    return static_cast<T*>(p);
  }
  void dfree(void* p) {
    auto it = std::find_if(allocs.begin(), allocs.end(), [p](const auto& a) { return a.first == p; });
    if (it != allocs.end()) {
      dev_bytes -= it->second;
      allocs.erase(it);
    }
    cudaFree(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = dalloc<T>(v.size());
    if (!v.empty()) CK3(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    CK3(cudaStreamSynchronize(st));
    return p;
  }
  ~hddm3_engine() {
    if (dev >= 0) cudaSetDevice(dev);
    for (auto& a : allocs) cudaFree(a.first);
    if (h_scal) cudaFreeHost(h_scal);
    if (h_ks) cudaFreeHost(h_ks);
    if (kry_exec) cudaGraphExecDestroy(kry_exec);
    for (auto& g : step_exec)
      if (g) cudaGraphExecDestroy(g);
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }

  void create(const hddm3_problem& p);
  void build_plan();
  void factorize();
  void run_probe();
  Solve3Args solve_args(const cplx* B, cplx* X, const int* flag, int on);
  void enqueue_solve(const Solve3Args& A, cudaStream_t s);
  int solve_launches() const;
  Step3Args step_args(int s, const cplx* f);
  Chk3Args chk_args(const cplx* B, cplx* X, const int* flag, int on, unsigned long long cond);
  void enqueue_step_front(int s, cudaStream_t stream, unsigned long long cond);
  void enqueue_refine_body(int s, cudaStream_t stream, unsigned long long cond);
  int capture_step(int s, cudaGraph_t g);
  void build_step_graph(int v);
  void run_step(int s);
  void reset_state();
  void host_refine(const cplx* B, cplx* X, const int* flag, int on);
  double device_norm(const cplx* v);
  Glob3Args gargs() const {
    Glob3Args G;
    for (int a = 0; a < 3; ++a) G.gn[a] = S.gn[a];
    G.ih2 = 1.0 / (S.h * S.h);
    G.k2 = S.k2;
    G.ga = d_ga;
    return G;
  }
  void ensure_krylov(int m);
  hddm::KryArgs kry_args(unsigned long long cond);
  int enqueue_kry_iteration(int K, unsigned long long cond, cudaGraph_t body);
  void build_kry_graph(int K);
  void drop_graphs() {
    for (auto& g : step_exec)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    if (kry_exec) {
      cudaGraphExecDestroy(kry_exec);
      kry_exec = nullptr;
    }
  }
};

// ----------------------------------------------------------------- creation
void hddm3_engine::create(const hddm3_problem& p) {
  std::string msg;
  const int rc = build_setup3(p, S, msg);
  if (rc == HDDM_ERR_CONFIG) throw ConfigErr3(msg);
  if (rc) throw std::runtime_error(msg);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw std::runtime_error("no CUDA device available (the engine has no CPU fallback)");
  if (p.device < 0 || p.device >= ndev) throw ConfigErr3("invalid CUDA device ordinal");
  dev = p.device;
  CK3(cudaSetDevice(dev));
  CK3(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK3(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  CK3(cudaMallocHost(&h_scal, 64 * sizeof(double)));
  CK3(cudaMallocHost(&h_ks, sizeof(hddm::KryState)));
  nsub = int(S.subs.size());
  ncls = S.ncls;
  ng = (long long)S.gn[0] * S.gn[1] * S.gn[2];
  build_sym3(S.subs[0].nn[0], S.subs[0].nn[1], S.subs[0].nn[2], Y);
  nw = Y.n;
  for (int c = 0; c < ncls; ++c) max_members = std::max(max_members, S.cls_ptr[c + 1] - S.cls_ptr[c]);
  mg = max_members == 1 ? 1 : kMG;
  ngroups = (max_members + mg - 1) / mg;

  // symbolic tables
  std::vector<DSn3> sn(Y.sn.size());
  for (size_t s = 0; s < Y.sn.size(); ++s) {
    const Sn3& a = Y.sn[s];
    DSn3& d = sn[s];
    d.c0 = a.c0;
    d.n = a.n;
    d.r = int(a.rows.size());
    d.parent = a.parent;
    d.ch0 = a.nch > 0 ? a.ch[0] : -1;
    d.ch1 = a.nch > 1 ? a.ch[1] : -1;
    d.pad0 = d.pad1 = 0;
    d.linv_off = Y.linv_off[s];
    d.pan_off = Y.pan_off[s];
    d.upd_off = Y.upd_off[s];
    d.cmap_off = Y.cmap_off[s];
    d.rows_off = Y.rows_off[s];
    d.front_off = Y.front_off[s];
    d.ext_off = Y.ext_off[s];
    d.aent0 = Y.aent_ptr[s];
    d.aent1 = Y.aent_ptr[s + 1];
  }
  d_sn = upload(sn);
  d_rows = upload(Y.rows_all);
  d_cmap0 = upload(Y.cmap0);
  d_cmap1 = upload(Y.cmap1);
  d_perm = upload(Y.perm);
  d_pinv = upload(Y.pinv);
  d_cls_ptr = upload(S.cls_ptr);
  d_cls_mem = upload(S.cls_members);
  build_plan();

  // per subdomain
  std::vector<Sub3Dev> subs(nsub);
  const int* nn = S.subs[0].nn;
  cop_stride = 2 * (nn[0] + nn[1] + nn[2]);
  std::vector<cplx> cop(size_t(ncls) * cop_stride);
  std::vector<double> wts(size_t(nsub) * (nn[0] + nn[1] + nn[2]));
  for (int t = 0; t < nsub; ++t) {
    const Sub3& s = S.subs[t];
    Sub3Dev& d = subs[t];
    for (int a = 0; a < 3; ++a) {
      d.ix[a] = s.ix[a];
      d.w0[a] = s.w0[a];
      d.c0[a] = s.c0[a];
      d.c1[a] = s.c1[a];
      d.lo[a] = s.lo[a];
      d.hi[a] = s.hi[a];
      d.own0[a] = s.own0[a];
      d.own1[a] = s.own1[a];
    }
    d.cls = s.cls;
    d.pad = 0;
    double* w = &wts[size_t(t) * (nn[0] + nn[1] + nn[2])];
    for (int a = 0, o = 0; a < 3; o += nn[a], ++a) std::copy(s.w[a].begin(), s.w[a].end(), w + o);
  }
  for (int c = 0; c < ncls; ++c) {
    const Op3& op = S.subop[S.cls_rep[c]];
    cplx* o = &cop[size_t(c) * cop_stride];
    int k = 0;
    for (int a = 0; a < 3; ++a)
      for (int l = 0; l < nn[a]; ++l) o[k++] = cmk3(op.an[a][2 * l], op.an[a][2 * l + 1]);
    for (int a = 0; a < 3; ++a)
      for (int l = 0; l < nn[a]; ++l) o[k++] = cmk3(op.iah[a][2 * l], op.iah[a][2 * l + 1]);
  }
  d_sub = upload(subs);
  d_cop = upload(cop);
  d_wts = upload(wts);
  // covering subdomains per global coordinate and axis (accumulate regions)
  {
    std::vector<int> cov(2 * size_t(S.gn[0] + S.gn[1] + S.gn[2]), -1);
    for (int a = 0, base = 0; a < 3; base += S.gn[a], ++a)
      for (int i = 0; i < S.n[a]; ++i) {
        int ix[3] = {0, 0, 0};
        ix[a] = i;
        const Sub3& s = S.subs[(ix[2] * S.n[1] + ix[1]) * S.n[0] + ix[0]];
        const int x0 = s.lo[a] ? s.c0[a] - S.nov : s.w0[a];
        const int x1 = s.hi[a] ? s.c1[a] + S.nov : s.w0[a] + s.nn[a] - 1;
        for (int P = x0; P <= x1; ++P) {
          int* c = &cov[2 * size_t(base + P)];
          if (c[0] < 0)
            c[0] = i;
          else if (c[1] < 0)
            c[1] = i;
          else
            throw ConfigErr3("more than 2 overlapping subdomains per axis coordinate");
        }
      }
    d_cov = upload(cov);
  }
  build_transfer_tables();
  for (int k = 0; k < 4; ++k) {
    d_U[k] = dalloc<cplx>(size_t(nsub) * nw);
    d_Z[k] = dalloc<int>(nsub);
  }
  d_B = dalloc<cplx>(size_t(nsub) * nw);
  d_Y = dalloc<cplx>(size_t(nsub) * nw);
  d_R = dalloc<cplx>(size_t(nsub) * nw);
  d_C = dalloc<cplx>(size_t(nsub) * nw);
  d_UPD = dalloc<cplx>(size_t(nsub) * std::max<long>(1, Y.nupd));
  CK3(cudaMemsetAsync(d_U[0], 0, sizeof(cplx) * size_t(nsub) * nw, st));
  d_fany = dalloc<int>(nsub);
  d_counts = dalloc<long long>(2);
  d_part_chk = dalloc<double>(size_t(nsub) * kChunks * 2);
  d_rel_cur = dalloc<double>(nsub);
  d_rel_prev = dalloc<double>(nsub);
  d_maxrel = dalloc<double>(1);
  d_need = dalloc<int>(nsub);
  d_ncorr = dalloc<int>(nsub);
  d_undo = dalloc<int>(nsub);
  d_any = dalloc<int>(1);
  d_ccount = dalloc<int>(1);
  CK3(cudaMemsetAsync(d_undo, 0, sizeof(int) * nsub, st));
  {
    std::vector<int> rep(nsub, 0);
    for (int c = 0; c < ncls; ++c) rep[S.cls_rep[c]] = 1;
    d_isrep = upload(rep);
  }
  // global
  {
    std::vector<cplx> ga(2 * size_t(S.gn[0] + S.gn[1] + S.gn[2]));
    int k = 0;
    for (int a = 0; a < 3; ++a)
      for (int l = 0; l < S.gn[a]; ++l) ga[k++] = cmk3(S.gop.an[a][2 * l], S.gop.an[a][2 * l + 1]);
    for (int a = 0; a < 3; ++a)
      for (int l = 0; l < S.gn[a]; ++l) ga[k++] = cmk3(S.gop.iah[a][2 * l], S.gop.iah[a][2 * l + 1]);
    d_ga = upload(ga);
  }
  d_f = dalloc<cplx>(ng);
  d_asm = dalloc<cplx>(ng);
  d_part = dalloc<double>(2 * size_t(hddm::reduce_blocks()));
  d_scal = dalloc<double>(64);
  factorize();
  run_probe();
}

// Structural transfer tables (transfer_patch / transfer_beta in 3-D, hddm_oracle3.c):
// every window has the same shape and its core at the same local offset, so the union of
// the 26 patches, the directions covering each of its nodes, the source-window position
// of each of the 7 stencil points and their tapers are window-local and computed once.
// Nodes in factor order (coalesced writes of b); entries per node in gather order.
void hddm3_engine::build_transfer_tables() {
  static const int kO[26][3] = {
      {+1, 0, 0}, {-1, 0, 0}, {0, +1, 0}, {0, -1, 0}, {0, 0, +1}, {0, 0, -1},
      {+1, +1, 0}, {-1, +1, 0}, {+1, -1, 0}, {-1, -1, 0},
      {+1, 0, +1}, {-1, 0, +1}, {+1, 0, -1}, {-1, 0, -1},
      {0, +1, +1}, {0, -1, +1}, {0, +1, -1}, {0, -1, -1},
      {+1, +1, +1}, {-1, +1, +1}, {+1, -1, +1}, {-1, -1, +1},
      {+1, +1, -1}, {-1, +1, -1}, {+1, -1, -1}, {-1, -1, -1}};
  static const int kDp[7][3] = {{0, 0, 0}, {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
  const int* nn = Y.nn;
  const int nov = S.nov, c0L = S.ext;  // window-local core: [ext, ext + mc] per axis
  auto beta0h = [](double t) {
    if (t <= 0) return 1.0;
    if (t >= 1) return 0.0;
    return 1.0 - t * t * t * (10.0 - 15.0 * t + 6.0 * t * t);
  };
  std::vector<int> pnode, pent(1, 0), edir, esrc;
  std::vector<double> ebeta;
  for (int pos = 0; pos < nw; ++pos) {
    const int v = Y.perm[pos];
    const int L[3] = {v % nn[0], (v / nn[0]) % nn[1], v / (nn[0] * nn[1])};
    bool interior = true;
    for (int a = 0; a < 3; ++a) interior = interior && L[a] > 0 && L[a] < nn[a] - 1;
    if (!interior) continue;
    int cnt = 0;
    for (int d = 0; d < 26; ++d) {
      bool in = true;
      for (int a = 0; a < 3; ++a) {
        const int o = kO[d][a], e1 = S.ext + S.mc[a];  // window-local core [ext, ext + mc]
        if (o > 0) in = in && L[a] >= e1 - 1 - nov && L[a] <= e1 - 1;
        if (o < 0) in = in && L[a] >= c0L + 1 && L[a] <= c0L + 1 + nov;
      }
      if (!in) continue;
      ++cnt;
      edir.push_back(d);
      for (int k = 0; k < 7; ++k) {
        int ls[3], G[3];
        bool inside = true;
        for (int a = 0; a < 3; ++a) {
          G[a] = L[a] + kDp[k][a];                 // target-local (= global - w0_t)
          ls[a] = G[a] - kO[d][a] * S.mc[a];       // source-local
          inside = inside && ls[a] >= 0 && ls[a] < nn[a];
        }
        esrc.push_back(inside ? Y.pinv[(ls[2] * nn[1] + ls[1]) * nn[0] + ls[0]] : -1);
        double b = 1.0;
        bool first = true;
        for (int a = 0; a < 3; ++a) {
          const int o = kO[d][a], e1 = S.ext + S.mc[a];
          if (!o) continue;
          const double bv = o > 0 ? beta0h(double(e1 - 1 - G[a]) / nov) : beta0h(double(G[a] - c0L - 1) / nov);
          b = first ? bv : b * bv;
          first = false;
        }
        ebeta.push_back(b);
      }
    }
    if (cnt) {
      pnode.push_back(v);
      pent.push_back(int(edir.size()));
    }
  }
  npatch = int(pnode.size());
  if (npatch) {
    d_pnode = upload(pnode);
    d_pent = upload(pent);
    d_edir = upload(edir);
    d_esrc = upload(esrc);
    d_ebeta = upload(ebeta);
  }
}

// Task lists: forward levels by height (leaves first), backward levels by depth.
// Forward inverse / panel rows of supernodes with more than kSmallCols columns are
// CTA tasks (8 warps split the columns); the others warp tasks, 8 per CTA.
constexpr int kSmallCols = 64;
constexpr int kColsPerTask = 32;  // backward: lane = column

void hddm3_engine::build_plan() {
  const int nsn = int(Y.sn.size());
  auto task = [&](int s, int a, int b) {
    const Sn3& x = Y.sn[s];
    Task3 t = {};
    t.s = s;
    t.a = a;
    t.b = b;
    t.c0 = x.c0;
    t.n = x.n;
    t.r = int(x.rows.size());
    t.linv = Y.linv_off[s];
    t.pan = Y.pan_off[s];
    t.upd = Y.upd_off[s];
    t.cmap = Y.cmap_off[s];
    t.rows = Y.rows_off[s];
    return t;
  };
  auto up = [&](const std::vector<Task3>& v, int nbig = 0) {
    Lvl L;
    L.n = int(v.size());
    L.nbig = nbig;
    if (L.n) L.d = upload(v);
    return L;
  };
  // big tasks first, then the warp tasks padded to a multiple of 8
  auto split = [&](std::vector<Task3>& big, std::vector<Task3>& small) {
    const int nbig = int(big.size());
    while (small.size() % 8) small.push_back(Task3{});
    big.insert(big.end(), small.begin(), small.end());
    return nbig;
  };
  // leaves of at most 32 nodes: one fused warp kernel each way (k3s_fleaf / k3s_bleaf)
  bool fuse = true;
  for (int s = 0; s < nsn; ++s)
    if (Y.sn[s].nch == 0 && Y.sn[s].n > 32) fuse = false;
  if (fuse) {
    std::vector<Task3> lf;
    for (int s = 0; s < nsn; ++s)
      if (Y.sn[s].nch == 0) lf.push_back(task(s, 0, Y.sn[s].n));
    while (lf.size() % 8) lf.push_back(Task3{});
    f_leaf = up(lf);
    b_leaf = up(lf);
  }
  auto leaf = [&](int s) { return fuse && Y.sn[s].nch == 0; };
  for (int h = 0; h <= Y.max_height; ++h) {
    std::vector<Task3> a, db, ds, pb, ps;
    for (int s = 0; s < nsn; ++s) {
      const Sn3& x = Y.sn[s];
      if (x.height != h || leaf(s)) continue;
      const int r = int(x.rows.size());
      const bool big = x.n > kSmallCols;
      for (int i = 0; i < x.n; i += 256) a.push_back(task(s, i, std::min(x.n, i + 256)));
      for (int i = 0; i < x.n; i += kDiagRows) (big ? db : ds).push_back(task(s, i, std::min(x.n, i + kDiagRows)));
      for (int k = 0; k < r; k += kDiagRows) (big ? pb : ps).push_back(task(s, k, std::min(r, k + kDiagRows)));
    }
    f_asm.push_back(up(a));
    const int nbd = split(db, ds);
    f_diag.push_back(up(db, nbd));
    const int nbp = split(pb, ps);
    f_pan.push_back(up(pb, nbp));
  }
  for (int dd = 0; dd <= Y.max_depth; ++dd) {
    std::vector<Task3> g, pb, ps, db, ds;
    for (int s = 0; s < nsn; ++s) {
      const Sn3& x = Y.sn[s];
      if (x.depth != dd || leaf(s)) continue;
      const int r = int(x.rows.size());
      for (int k = 0; k < r; k += 256) g.push_back(task(s, k, std::min(r, k + 256)));
      for (int j = 0; j < x.n; j += kColsPerTask) {
        (r > kSmallCols ? pb : ps).push_back(task(s, j, std::min(x.n, j + kColsPerTask)));
        (x.n > kSmallCols ? db : ds).push_back(task(s, j, std::min(x.n, j + kColsPerTask)));
      }
    }
    b_gat.push_back(up(g));
    const int nbp = split(pb, ps);
    b_pan.push_back(up(pb, nbp));
    const int nbd = split(db, ds);
    b_diag.push_back(up(db, nbd));
  }
}

int hddm3_engine::solve_launches() const {
  int n = 1 + (f_leaf.n > 0) + (b_leaf.n > 0);
  for (size_t h = 0; h < f_asm.size(); ++h) n += (f_asm[h].n > 0) + (f_diag[h].n > 0) + (f_pan[h].n > 0);
  for (size_t d = 0; d < b_gat.size(); ++d) n += (b_gat[d].n > 0) + (b_pan[d].n > 0) + (b_diag[d].n > 0);
  return n;
}

// --------------------------------------------------------------- factorization
// Batched multifrontal LDL^T (the restatement's up-looking factor up to rounding,
// sparse.cpp:110-174): classes in batches sized to a workspace budget, fronts level
// by level (height), each level: assemble (scatter A, extend-add the children's
// contribution blocks), blocked partial factorization of the own columns with the
// identity rows E riding along, extraction of D, the inverse diagonal blocks and
// the panels.
void hddm3_engine::factorize() {
  const double t0 = now_ms3();
  const int nsn = int(Y.sn.size());
  const double ih2 = 1.0 / (S.h * S.h);
  using cd = std::complex<double>;
  const long long naent = (long long)Y.aent_i.size();
  std::vector<cplx> aval(size_t(ncls) * naent);
  const int* nn = S.subs[0].nn;
  for (int c = 0; c < ncls; ++c) {
    const Op3& op = S.subop[S.cls_rep[c]];
    auto A = [&](int a, int l) { return cd(op.an[a][2 * l], op.an[a][2 * l + 1]); };
    auto I = [&](int a, int l) { return cd(op.iah[a][2 * l], op.iah[a][2 * l + 1]); };
    for (long long e = 0; e < naent; ++e) {
      const int v = Y.aent_node[e];
      const int p = v % nn[0], q = (v / nn[0]) % nn[1], r = v / (nn[0] * nn[1]);
      const cd yz = A(1, q) * A(2, r), xz = A(0, p) * A(2, r), xy = A(0, p) * A(1, q);
      const cd cw = yz * I(0, p - 1) * ih2, ce = yz * I(0, p) * ih2;
      const cd cs = xz * I(1, q - 1) * ih2, cn = xz * I(1, q) * ih2;
      const cd cb = xy * I(2, r - 1) * ih2, ct = xy * I(2, r) * ih2;
      cd val;
      switch (Y.aent_kind[e]) {
        case 0: val = -(cw + ce + cs + cn + cb + ct) + A(0, p) * A(1, q) * A(2, r) * S.k2; break;
        case 1: val = cw; break;
        case 2: val = ce; break;
        case 3: val = cs; break;
        case 4: val = cn; break;
        case 5: val = cb; break;
        default: val = ct; break;
      }
      aval[size_t(c) * naent + e] = cmk3(val.real(), val.imag());
    }
  }
  dense_factorize(*this, Y, d_sn, ncls, aval, d_vals, d_valsT, st);
  factor_ms = now_ms3() - t0;
}

// ----------------------------------------------------------------- solves
Solve3Args hddm3_engine::solve_args(const cplx* B, cplx* X, const int* flag, int on) {
  Solve3Args A;
  A.sn = d_sn;
  A.vals = d_vals;
  A.valsT = d_valsT;
  A.nvals = Y.nvals;
  A.rows_all = d_rows;
  A.cmap0 = d_cmap0;
  A.cmap1 = d_cmap1;
  A.B = B;
  A.X = X;
  A.Y = d_Y;
  A.U = d_UPD;
  A.nw = nw;
  A.nupd = std::max<long>(1, Y.nupd);
  A.nshell = Y.nshell;
  A.cls_ptr = d_cls_ptr;
  A.cls_mem = d_cls_mem;
  A.flag = flag;
  A.flag_on = on;
  A.mg = mg;
  return A;
}

void hddm3_engine::enqueue_solve(const Solve3Args& A, cudaStream_t s) {
  s3_ring(A, ncls, ngroups, s);
  s3_fleaf(A, f_leaf.d, f_leaf.n, ncls, ngroups, s);
  for (size_t h = 0; h < f_asm.size(); ++h) {
    s3_fasm(A, f_asm[h].d, f_asm[h].n, ncls, ngroups, s);
    s3_fdiag(A, f_diag[h].d, f_diag[h].n, f_diag[h].nbig, ncls, ngroups, s);
    s3_fpanel(A, f_pan[h].d, f_pan[h].n, f_pan[h].nbig, ncls, ngroups, s);
  }
  for (size_t d = 0; d < b_gat.size(); ++d) {
    s3_bgather(A, b_gat[d].d, b_gat[d].n, ncls, ngroups, s);
    s3_bpanel(A, b_pan[d].d, b_pan[d].n, b_pan[d].nbig, ncls, ngroups, s);
    s3_bdiag(A, b_diag[d].d, b_diag[d].n, b_diag[d].nbig, ncls, ngroups, s);
  }
  s3_bleaf(A, b_leaf.d, b_leaf.n, ncls, ngroups, s);
}

Chk3Args hddm3_engine::chk_args(const cplx* B, cplx* X, const int* flag, int on, unsigned long long cond) {
  Chk3Args C;
  for (int a = 0; a < 3; ++a) C.nn[a] = Y.nn[a];
  C.nw = nw;
  C.nsub = nsub;
  C.nchunk = kChunks;
  C.ih2 = 1.0 / (S.h * S.h);
  C.k2 = S.k2;
  C.sub = d_sub;
  C.cop = d_cop;
  C.cop_stride = cop_stride;
  C.perm = d_perm;
  C.pinv = d_pinv;
  C.B = B;
  C.X = X;
  C.R = d_R;
  C.C = d_C;
  C.flag = flag;
  C.flag_on = on;
  C.part = d_part_chk;
  C.rel_cur = d_rel_cur;
  C.rel_prev = d_rel_prev;
  C.need = d_need;
  C.ncorr = d_ncorr;
  C.undo = d_undo;
  C.any = d_any;
  C.max_rel = d_maxrel;
  C.corr_count = d_ccount;
  C.cond = cond;
  return C;
}

// refine (sparse.cpp:268-292) driven from the host: probe and class-solve taps
void hddm3_engine::host_refine(const cplx* B, cplx* X, const int* flag, int on) {
  const Chk3Args C0 = chk_args(B, X, flag, on, 0);
  c3_partials(C0, 0, st);
  c3_first(C0, st);
  Chk3Args Cn = chk_args(B, X, d_need, 1, 0);
  for (int it = 0; it < 13; ++it) {
    int any = 0;
    CK3(cudaMemcpyAsync(&any, d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK3(cudaStreamSynchronize(st));
    if (!any) break;
    c3_partials(Cn, 1, st);
    enqueue_solve(solve_args(d_R, d_C, d_need, 1), st);
    c3_apply(Cn, st);
    c3_partials(Cn, 0, st);
    c3_decide(Cn, st);
    c3_undo(Cn, st);
  }
}

// the probe of Factorization::factor (sparse.cpp:203-236), every class at once
void hddm3_engine::run_probe() {
  std::vector<cplx> b(size_t(nsub) * nw, cmk3(0, 0));
  uint64_t s = 0x9E3779B97F4A7C15ull;
  std::vector<cplx> nat(nw);
  for (int i = 0; i < nw; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double re = double(s >> 11) * 0x1.0p-52 - 1.0;
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double im = double(s >> 11) * 0x1.0p-52 - 1.0;
    nat[i] = cmk3(re, im);
  }
  for (int c = 0; c < ncls; ++c) {
    const int t = S.cls_rep[c];
    for (int v = 0; v < nw; ++v) b[size_t(t) * nw + Y.pinv[v]] = nat[v];
  }
  CK3(cudaMemcpyAsync(d_B, b.data(), sizeof(cplx) * b.size(), cudaMemcpyHostToDevice, st));
  CK3(cudaMemsetAsync(d_maxrel, 0, sizeof(double), st));
  CK3(cudaMemsetAsync(d_ccount, 0, sizeof(int), st));
  enqueue_solve(solve_args(d_B, d_U[0], d_isrep, 1), st);
  host_refine(d_B, d_U[0], d_isrep, 1);
  std::vector<double> rel(nsub);
  CK3(cudaMemcpyAsync(rel.data(), d_rel_prev, sizeof(double) * nsub, cudaMemcpyDeviceToHost, st));
  CK3(cudaStreamSynchronize(st));
  probe.assign(ncls, 0);
  for (int c = 0; c < ncls; ++c) {
    probe[c] = rel[S.cls_rep[c]];
    if (!(probe[c] <= 1e-10)) {
      char m[160];
      std::snprintf(m, sizeof m, "LDL^T probe residual %.3e above 1e-10 (class %d); no LU fallback", probe[c], c);
      throw SolveErr3(m);
    }
  }
}

// ----------------------------------------------------------------- DDM step
Step3Args hddm3_engine::step_args(int s, const cplx* f) {
  Step3Args A;
  for (int a = 0; a < 3; ++a) {
    A.n[a] = S.n[a];
    A.nn[a] = Y.nn[a];
    A.gn[a] = S.gn[a];
  }
  A.nsub = nsub;
  A.nov = S.nov;
  A.nw = nw;
  A.nshell = Y.nshell;
  A.ih2 = 1.0 / (S.h * S.h);
  A.k2 = S.k2;
  A.sub = d_sub;
  A.cop = d_cop;
  A.cop_stride = cop_stride;
  A.wts = d_wts;
  A.perm = d_perm;
  A.pinv = d_pinv;
  A.f = f;
  A.fany = d_fany;
  A.zc = d_Z[s % 4];
  A.B = d_B;
  A.Ucur = d_U[s % 4];
  for (int l = 1; l <= 3; ++l) {
    A.zp[l - 1] = d_Z[(s + 4 - l) % 4];
    A.Up[l - 1] = d_U[(s + 4 - l) % 4];
  }
  A.asmb = d_asm;
  A.cov = d_cov;
  A.step = s;
  A.counts = d_counts;
  A.npatch = npatch;
  A.pnode = d_pnode;
  A.pent = d_pent;
  A.edir = d_edir;
  A.esrc = d_esrc;
  A.ebeta = d_ebeta;
  return A;
}

void hddm3_engine::reset_state() {
  for (int k = 0; k < 4; ++k) {
    std::vector<int> ones(nsub, 1);
    CK3(cudaMemcpyAsync(d_Z[k], ones.data(), sizeof(int) * nsub, cudaMemcpyHostToDevice, st));
  }
  CK3(cudaMemsetAsync(d_asm, 0, ng * sizeof(cplx), st));
  CK3(cudaStreamSynchronize(st));
  last_step = 0;
}

// sweep (ddm.cpp:174-214 in 3-D) up to the first residual check of refine
void hddm3_engine::enqueue_step_front(int s, cudaStream_t stream, unsigned long long cond) {
  const Step3Args A = step_args(s, d_f);
  d3_flags(A, stream);
  d3_rhs(A, stream);
  enqueue_solve(solve_args(d_B, A.Ucur, A.zc, 0), stream);
  const Chk3Args C = chk_args(d_B, A.Ucur, A.zc, 0, cond);
  c3_partials(C, 0, stream);
  c3_first(C, stream);
}

void hddm3_engine::enqueue_refine_body(int s, cudaStream_t stream, unsigned long long cond) {
  const Step3Args A = step_args(s, d_f);
  const Chk3Args C = chk_args(d_B, A.Ucur, d_need, 1, cond);
  c3_partials(C, 1, stream);
  enqueue_solve(solve_args(d_R, d_C, d_need, 1), stream);
  c3_apply(C, stream);
  c3_partials(C, 0, stream);
  c3_decide(C, stream);
  c3_undo(C, stream);
}

static int variant3(int s) { return s == 1 ? 0 : 1 + (s % 4); }
static int rep3(int v) { return v == 0 ? 1 : (v == 1 ? 4 : (v == 2 ? 5 : (v == 3 ? 2 : 3))); }

int hddm3_engine::capture_step(int s, cudaGraph_t g) {
  cudaGraphConditionalHandle h;
  CK3(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
  enqueue_step_front(s, st, (unsigned long long)h);
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK3(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK3(cudaGraphAddNode(&wn, g, deps, nd, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK3(cudaStreamUpdateCaptureDependencies(st, &wn, 1, cudaStreamSetCaptureDependencies));
  CK3(cudaStreamBeginCaptureToGraph(st2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  enqueue_refine_body(s, st2, (unsigned long long)h);
  cudaGraph_t bout;
  CK3(cudaStreamEndCapture(st2, &bout));
  d3_accumulate(step_args(s, d_f), st);
  return 2 + solve_launches() + 2 + 1;
}

void hddm3_engine::build_step_graph(int v) {
  cudaGraph_t g;
  CK3(cudaGraphCreate(&g, 0));
  CK3(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  step_kernels[v] = capture_step(rep3(v), g);
  cudaGraph_t gout;
  CK3(cudaStreamEndCapture(st, &gout));
  CK3(cudaGraphInstantiate(&step_exec[v], g, 0));
  CK3(cudaGraphDestroy(g));
}

void hddm3_engine::run_step(int s) {
  static const bool no_graphs = std::getenv("HDDM_NO_GRAPHS") != nullptr;
  if (no_graphs) {  // direct launches (profiling aid); refinement driven from the host
    enqueue_step_front(s, st, 0);
    const Step3Args A = step_args(s, d_f);
    const Chk3Args C = chk_args(d_B, A.Ucur, d_need, 1, 0);
    for (int it = 0; it < 13; ++it) {
      int any = 0;
      CK3(cudaMemcpyAsync(&any, d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK3(cudaStreamSynchronize(st));
      if (!any) break;
      enqueue_refine_body(s, st, 0);
      (void)C;
    }
    d3_accumulate(A, st);
    launches += 2 + solve_launches() + 3;
    last_step = s;
    return;
  }
  const int v = variant3(s);
  if (!step_exec[v]) build_step_graph(v);
  CK3(cudaGraphLaunch(step_exec[v], st));
  launches += step_kernels[v];
  last_step = s;
}

double hddm3_engine::device_norm(const cplx* v) {
  hddm::launch_nrm2_part(v, ng, d_part, st);
  hddm::launch_finish_sum(d_part, 1, d_scal, st);
  CK3(cudaMemcpyAsync(h_scal, d_scal, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK3(cudaStreamSynchronize(st));
  return std::sqrt(h_scal[0]);
}

// ----------------------------------------------------------------- krylov
void hddm3_engine::ensure_krylov(int m) {
  if (kry_m >= m) return;
  for (cplx* p : V) dfree(p);
  for (cplx* p : Z) dfree(p);
  V.clear();
  Z.clear();
  for (int i = 0; i <= m; ++i) V.push_back(dalloc<cplx>(ng));
  for (int i = 0; i < m; ++i) Z.push_back(dalloc<cplx>(ng));
  if (d_Zptr) dfree(d_Zptr);
  d_Zptr = dalloc<cplx*>(m);
  CK3(cudaMemcpyAsync(d_Zptr, Z.data(), sizeof(cplx*) * m, cudaMemcpyHostToDevice, st));
  if (d_Vptr) dfree(d_Vptr);
  d_Vptr = dalloc<cplx*>(m + 1);
  CK3(cudaMemcpyAsync(d_Vptr, V.data(), sizeof(cplx*) * (m + 1), cudaMemcpyHostToDevice, st));
  if (!d_ks) d_ks = dalloc<hddm::KryState>(1);
  if (kry_exec) {
    CK3(cudaGraphExecDestroy(kry_exec));
    kry_exec = nullptr;
  }
  for (cplx* p : {d_H, d_g, d_sn_g, d_y})
    if (p) dfree(p);
  if (d_cs) dfree(d_cs);
  d_H = dalloc<cplx>(size_t(m) * (m + 1));
  d_g = dalloc<cplx>(m + 1);
  d_sn_g = dalloc<cplx>(m);
  d_cs = dalloc<double>(m);
  d_y = dalloc<cplx>(m);
  if (!d_b) {
    d_b = dalloc<cplx>(ng);
    d_x = dalloc<cplx>(ng);
    d_r = dalloc<cplx>(ng);
  }
  kry_m = m;
  CK3(cudaStreamSynchronize(st));
}

hddm::KryArgs hddm3_engine::kry_args(unsigned long long cond) {
  hddm::KryArgs K;
  K.ks = d_ks;
  K.V = d_Vptr;
  K.Z = d_Zptr;
  K.H = d_H;
  K.ld = kry_m + 1;
  K.g = d_g;
  K.sn = d_sn_g;
  K.cs = d_cs;
  K.hist = d_hist;
  K.part = d_part;
  K.n = ng;
  K.cond = cond;
  return K;
}

__global__ void k3_fill_int(int* p, int v, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

// one Arnoldi iteration of fgmres (krylov.cpp:57-109): Z_j = M(V_j) (K steps),
// w = A Z_j, modified Gram-Schmidt, Givens, V_{j+1} = w / hlast
int hddm3_engine::enqueue_kry_iteration(int K, unsigned long long cond, cudaGraph_t body) {
  const hddm::KryArgs KA = kry_args(cond);
  int nk = 0;
  for (int k = 0; k < 4; ++k) k3_fill_int<<<(nsub + 255) / 256, 256, 0, st>>>(d_Z[k], 1, nsub);
  CK3(cudaMemsetAsync(d_asm, 0, ng * sizeof(cplx), st));
  nk += 4;
  hddm::launch_kry_load(KA, d_f, st);
  d3_fany(step_args(1, d_f), st);
  nk += 2;
  for (int s = 1; s <= K; ++s) {
    if (body)
      nk += capture_step(s, body);
    else
      run_step(s);
  }
  hddm::launch_kry_store(KA, d_asm, st);
  d3_apply_global_ind(gargs(), d_Zptr, 0, d_Vptr, 1, &d_ks->j, st);
  hddm::launch_kry_first_dot(KA, st);
  nk += 4;
  for (int i = 0; i < kry_m; ++i) hddm::launch_kry_mgs(KA, i, st);
  nk += 2 * kry_m;
  hddm::launch_kry_givens(KA, st);
  hddm::launch_kry_next(KA, st);
  nk += 3;
  return nk;
}

void hddm3_engine::build_kry_graph(int K) {
  if (kry_exec) {
    CK3(cudaGraphExecDestroy(kry_exec));
    kry_exec = nullptr;
  }
  cudaGraph_t G;
  CK3(cudaGraphCreate(&G, 0));
  cudaGraphConditionalHandle hc;
  CK3(cudaGraphConditionalHandleCreate(&hc, G, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK3(cudaGraphAddNode(&wn, G, nullptr, 0, &cp));
  cudaGraph_t B = cp.conditional.phGraph_out[0];
  CK3(cudaStreamBeginCaptureToGraph(st, B, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  kry_iter_kernels = enqueue_kry_iteration(K, (unsigned long long)hc, B);
  cudaGraph_t out;
  CK3(cudaStreamEndCapture(st, &out));
  CK3(cudaGraphInstantiate(&kry_exec, G, 0));
  CK3(cudaGraphDestroy(G));
  kry_K = K;
}

// ----------------------------------------------------------------- C-ABI
namespace {

template <class F>
int guarded3(hddm3_engine* e, F&& fn) {
  try {
    if (e) CK3(cudaSetDevice(e->dev));
    fn();
    return HDDM_OK;
  } catch (const ConfigErr3& x) {
    (e ? e->err : g_err3) = x.what();
    return HDDM_ERR_CONFIG;
  } catch (const SolveErr3& x) {
    (e ? e->err : g_err3) = x.what();
    return HDDM_ERR_SOLVE;
  } catch (const std::exception& x) {
    (e ? e->err : g_err3) = x.what();
    return HDDM_ERR_OTHER;
  }
}

const cplx* in3(hddm3_engine* e, const double* p, int memkind, cplx* stage) {
  if (memkind == HDDM_DEVICE) return reinterpret_cast<const cplx*>(p);
  CK3(cudaMemcpyAsync(stage, p, e->ng * sizeof(cplx), cudaMemcpyHostToDevice, e->st));
  return stage;
}

void out3(hddm3_engine* e, double* p, const cplx* src, int memkind) {
  CK3(cudaMemcpyAsync(p, src, e->ng * sizeof(cplx),
                      memkind == HDDM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, e->st));
  CK3(cudaStreamSynchronize(e->st));
}

void counts3(hddm3_engine* e, long long* c) {
  CK3(cudaMemcpyAsync(c, e->d_counts, 2 * sizeof(long long), cudaMemcpyDeviceToHost, e->st));
  double mr = 0;
  int cc = 0;
  CK3(cudaMemcpyAsync(&mr, e->d_maxrel, sizeof(double), cudaMemcpyDeviceToHost, e->st));
  CK3(cudaMemcpyAsync(&cc, e->d_ccount, sizeof(int), cudaMemcpyDeviceToHost, e->st));
  CK3(cudaStreamSynchronize(e->st));
  e->last_max_rel = mr;
  e->last_corr = cc;
}

void clear_stats3(hddm3_engine* e) {
  CK3(cudaMemsetAsync(e->d_counts, 0, 2 * sizeof(long long), e->st));
  CK3(cudaMemsetAsync(e->d_maxrel, 0, sizeof(double), e->st));
  CK3(cudaMemsetAsync(e->d_ccount, 0, sizeof(int), e->st));
}

}  // namespace

extern "C" {

const char* hddm3_last_error(const hddm3_engine* e) { return e ? e->err.c_str() : g_err3.c_str(); }

int hddm3_create(const hddm3_problem* p, hddm3_engine** out) {
  *out = nullptr;
  hddm3_engine* e = new hddm3_engine();
  const int rc = guarded3(nullptr, [&] { e->create(*p); });
  if (rc) {
    delete e;
    return rc;
  }
  *out = e;
  return 0;
}
void hddm3_destroy(hddm3_engine* e) { delete e; }

long hddm3_n_global(const hddm3_engine* e) { return long(e->ng); }
double hddm3_sigma0(const hddm3_engine* e) { return e->S.sigma0; }
double hddm3_factor_ms(const hddm3_engine* e) { return e->factor_ms; }
int hddm3_num_subdomains(const hddm3_engine* e) { return e->nsub; }
int hddm3_num_classes(const hddm3_engine* e) { return e->ncls; }
int hddm3_class_of(const hddm3_engine* e, int t) { return t >= 0 && t < e->nsub ? e->S.subs[t].cls : -1; }
int hddm3_class_info(const hddm3_engine* e, int c, int* members, long* nnz, double* probe_relres) {
  if (c < 0 || c >= e->ncls) return HDDM_ERR_CONFIG;
  *members = e->S.cls_ptr[c + 1] - e->S.cls_ptr[c];
  *nnz = e->Y.nnz_ref;
  *probe_relres = e->probe[c];
  return 0;
}
int hddm3_window_dims(const hddm3_engine* e, int* nn3) {
  for (int a = 0; a < 3; ++a) nn3[a] = e->Y.nn[a];
  return 0;
}

int hddm3_apply_global(hddm3_engine* e, const double* u, double* out, int memkind) {
  return guarded3(e, [&] {
    const cplx* du = in3(e, u, memkind, e->d_f);
    cplx* dst = memkind == HDDM_DEVICE ? reinterpret_cast<cplx*>(out) : e->d_asm;
    d3_apply_global(e->gargs(), du, dst, nullptr, nullptr, e->st);
    if (memkind != HDDM_DEVICE) out3(e, out, dst, memkind);
    CK3(cudaStreamSynchronize(e->st));
  });
}

int hddm3_solve_iterative(hddm3_engine* e, const double* f, double tol, int max_steps, int check_every,
                          double* out, int memkind, hddm_stats* stats, int* hist_step, double* hist_rel,
                          double* hist_ms, int hist_cap, int* hist_len) {
  return guarded3(e, [&] {
    if (check_every < 1) check_every = 1;
    hddm_stats stt{};
    stt.relres = -1;
    stt.factor_ms = e->factor_ms;
    const cplx* df = in3(e, f, memkind, e->d_f);
    if (df != e->d_f) CK3(cudaMemcpyAsync(e->d_f, df, e->ng * sizeof(cplx), cudaMemcpyDeviceToDevice, e->st));
    const double bnorm = e->device_norm(e->d_f);
    int nh = 0;
    e->reset_state();
    clear_stats3(e);
    if (bnorm == 0) {
      stt.converged = 1;
      stt.relres = 0;
    } else {
      d3_fany(e->step_args(1, e->d_f), e->st);
      for (int s = 1; s <= max_steps; ++s) {
        const double t0 = now_ms3();
        e->run_step(s);
        stt.steps = s;
        if (s % check_every == 0 || s == max_steps) {
          d3_apply_global(e->gargs(), e->d_asm, nullptr, e->d_f, e->d_part, e->st);
          hddm::launch_finish_sum(e->d_part, 1, e->d_scal, e->st);
          CK3(cudaMemcpyAsync(e->h_scal, e->d_scal, sizeof(double), cudaMemcpyDeviceToHost, e->st));
          CK3(cudaStreamSynchronize(e->st));
          const double rel = std::sqrt(e->h_scal[0]) / bnorm;
          const double ms = now_ms3() - t0;
          if (nh < hist_cap) {
            if (hist_step) hist_step[nh] = s;
            if (hist_rel) hist_rel[nh] = rel;
            if (hist_ms) hist_ms[nh] = ms;
          }
          ++nh;
          stt.sweep_ms += ms;
          stt.relres = rel;
          if (rel <= tol) {
            stt.converged = 1;
            break;
          }
        } else {
          stt.sweep_ms += now_ms3() - t0;
        }
      }
    }
    out3(e, out, e->d_asm, memkind);
    long long cnt[2];
    counts3(e, cnt);
    stt.solves = long(cnt[0]);
    stt.skipped = long(cnt[1]);
    if (hist_len) *hist_len = nh;
    if (stats) *stats = stt;
  });
}

int hddm3_precondition(hddm3_engine* e, const double* r, double* z, int ksteps, int memkind,
                       hddm_stats* stats) {
  return guarded3(e, [&] {
    const cplx* dr = in3(e, r, memkind, e->d_f);
    if (dr != e->d_f) CK3(cudaMemcpyAsync(e->d_f, dr, e->ng * sizeof(cplx), cudaMemcpyDeviceToDevice, e->st));
    const double t0 = now_ms3();
    e->reset_state();
    clear_stats3(e);
    d3_fany(e->step_args(1, e->d_f), e->st);
    e->launches += 1;
    for (int s = 1; s <= ksteps; ++s) e->run_step(s);
    out3(e, z, e->d_asm, memkind);
    long long cnt[2];
    counts3(e, cnt);
    if (stats) {
      stats->solves += long(cnt[0]);
      stats->skipped += long(cnt[1]);
      stats->sweep_ms += now_ms3() - t0;
      stats->factor_ms = e->factor_ms;
    }
  });
}

int hddm3_fgmres(hddm3_engine* e, const double* b, double* x, double tol, int max_iters, int restart,
                 int ksteps, int memkind, hddm_fgmres_result* res, double* hist, int hist_cap,
                 hddm_stats* pstats) {
  return guarded3(e, [&] {
    const double tstart = now_ms3();
    hddm_fgmres_result R{};
    R.relres = R.true_relres = -1;
    const long long n = e->ng;
    int mcap = restart > 0 ? restart : max_iters;
    if (mcap < 1) mcap = 1;
    e->ensure_krylov(mcap);
    const int ld = e->kry_m + 1;
    cudaStream_t st = e->st;
    CK3(cudaMemcpyAsync(e->d_b, b, n * sizeof(cplx),
                        memkind == HDDM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    CK3(cudaMemsetAsync(e->d_x, 0, n * sizeof(cplx), st));
    clear_stats3(e);
    const double bnorm = e->device_norm(e->d_b);
    double sweep_ms = 0;
    e->kry_k_last = 0;
    if (e->d_hist_cap < max_iters) {
      if (e->d_hist) e->dfree(e->d_hist);
      e->d_hist_cap = std::max(max_iters, 256);
      e->d_hist = e->dalloc<double>(e->d_hist_cap);
      if (e->kry_exec) {
        CK3(cudaGraphExecDestroy(e->kry_exec));
        e->kry_exec = nullptr;
      }
    }
    const Glob3Args G = e->gargs();
    if (bnorm == 0) {
      R.converged = 1;
      R.relres = R.true_relres = 0;
    } else {
      CK3(cudaMemcpyAsync(e->d_r, e->d_b, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      hddm::KryState ks{};
      ks.max_iters = max_iters;
      ks.tol = tol;
      ks.bnorm = bnorm;
      static const bool no_graphs = std::getenv("HDDM_NO_GRAPHS") != nullptr;
      while (!ks.stop && ks.total < max_iters) {
        const int m = restart > 0 ? std::min(restart, max_iters - ks.total) : max_iters - ks.total;
        const double rnorm = e->device_norm(e->d_r);
        if (rnorm == 0) {
          ks.converged = 1;
          break;
        }
        e->h_scal[8] = rnorm;
        CK3(cudaMemcpyAsync(e->d_scal + 8, e->h_scal + 8, sizeof(double), cudaMemcpyHostToDevice, st));
        hddm::launch_scale_div(e->V[0], e->d_r, e->d_scal + 8, n, st);
        hddm::launch_init_g(e->d_g, m, e->d_scal + 8, st);
        CK3(cudaMemsetAsync(e->d_H, 0, sizeof(cplx) * size_t(e->kry_m) * ld, st));
        ks.j = 0;
        ks.m = m;
        ks.k = 0;
        ks.adv = 0;
        *e->h_ks = ks;
        CK3(cudaMemcpyAsync(e->d_ks, e->h_ks, sizeof(hddm::KryState), cudaMemcpyHostToDevice, st));
        const double ts = now_ms3();
        const int before = ks.total;
        if (no_graphs) {
          for (;;) {
            e->enqueue_kry_iteration(ksteps, 0, nullptr);
            CK3(cudaMemcpyAsync(e->h_ks, e->d_ks, sizeof(hddm::KryState), cudaMemcpyDeviceToHost, st));
            CK3(cudaStreamSynchronize(st));
            if (!e->h_ks->adv) break;
          }
        } else {
          if (!e->kry_exec || e->kry_K != ksteps) e->build_kry_graph(ksteps);
          CK3(cudaGraphLaunch(e->kry_exec, st));
          CK3(cudaMemcpyAsync(e->h_ks, e->d_ks, sizeof(hddm::KryState), cudaMemcpyDeviceToHost, st));
          CK3(cudaStreamSynchronize(st));
        }
        sweep_ms += now_ms3() - ts;
        ks = *e->h_ks;
        if (e->kry_exec) e->launches += (long long)e->kry_iter_kernels * (ks.total - before + (ks.flags & 1));
        if (hist) {
          const int lo = std::min(before, hist_cap), hi = std::min(ks.total, hist_cap);
          if (hi > lo) CK3(cudaMemcpy(hist + lo, e->d_hist + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToHost));
        }
        if (ks.total > before) R.relres = ks.relres;
        const int k = ks.k;
        e->kry_k_last = k;
        if (k > 0) {
          hddm::launch_backsolve(e->d_H, ld, e->d_g, e->d_y, k, st);
          hddm::launch_update_x(e->d_x, e->d_Zptr, e->d_y, k, n, st);
        }
        if (!ks.stop) {
          d3_apply_global(G, e->d_x, e->d_r, nullptr, nullptr, st);
          hddm::launch_bsub(e->d_r, e->d_b, n, st);
        }
      }
      R.iters = ks.total;
      R.converged = ks.converged;
      d3_apply_global(G, e->d_x, nullptr, e->d_b, e->d_part, st);
      hddm::launch_finish_sum(e->d_part, 1, e->d_scal, st);
      CK3(cudaMemcpyAsync(e->h_scal, e->d_scal, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK3(cudaStreamSynchronize(st));
      R.true_relres = std::sqrt(e->h_scal[0]) / bnorm;
    }
    out3(e, x, e->d_x, memkind);
    long long cnt[2];
    counts3(e, cnt);
    R.wall_ms = now_ms3() - tstart;
    if (res) *res = R;
    if (pstats) {
      pstats->solves += long(cnt[0]);
      pstats->skipped += long(cnt[1]);
      pstats->sweep_ms += sweep_ms;
      pstats->factor_ms = e->factor_ms;
    }
  });
}

int hddm3_fgmres_z(hddm3_engine* e, int j, double* out, int memkind) {
  return guarded3(e, [&] {
    if (j < 0 || j >= e->kry_k_last) throw ConfigErr3("no such preconditioned vector Z_j (last FGMRES cycle)");
    out3(e, out, e->Z[j], memkind);
  });
}

int hddm3_tap_subdomain(hddm3_engine* e, int t, double* rhs, double* u, int* active) {
  return guarded3(e, [&] {
    if (t < 0 || t >= e->nsub || e->last_step < 1) throw ConfigErr3("no sweep to tap");
    const int s = e->last_step;
    std::vector<cplx> b(e->nw), x(e->nw);
    int z = 1;
    CK3(cudaMemcpyAsync(b.data(), e->d_B + size_t(t) * e->nw, sizeof(cplx) * e->nw, cudaMemcpyDeviceToHost, e->st));
    CK3(cudaMemcpyAsync(x.data(), e->d_U[s % 4] + size_t(t) * e->nw, sizeof(cplx) * e->nw,
                        cudaMemcpyDeviceToHost, e->st));
    CK3(cudaMemcpyAsync(&z, e->d_Z[s % 4] + t, sizeof(int), cudaMemcpyDeviceToHost, e->st));
    CK3(cudaStreamSynchronize(e->st));
    cplx* R = reinterpret_cast<cplx*>(rhs);
    cplx* U = reinterpret_cast<cplx*>(u);
    for (int v = 0; v < e->nw; ++v) {
      R[v] = b[e->Y.pinv[v]];
      U[v] = x[e->Y.pinv[v]];
    }
    *active = !z;
  });
}

int hddm3_class_solve(hddm3_engine* e, int c, const double* b, double* x, double* relres) {
  return guarded3(e, [&] {
    if (c < 0 || c >= e->ncls) throw ConfigErr3("no such class");
    const int t = e->S.cls_rep[c];
    std::vector<int> only(e->nsub, 0);
    only[t] = 1;
    int* d_only = e->upload(only);
    std::vector<cplx> bb(e->nw);
    const cplx* bn = reinterpret_cast<const cplx*>(b);
    for (int v = 0; v < e->nw; ++v) bb[e->Y.pinv[v]] = bn[v];
    cplx* dB = e->d_B + size_t(t) * e->nw;
    cplx* dX = e->d_U[0] + size_t(t) * e->nw;
    CK3(cudaMemcpyAsync(dB, bb.data(), sizeof(cplx) * e->nw, cudaMemcpyHostToDevice, e->st));
    e->enqueue_solve(e->solve_args(e->d_B, e->d_U[0], d_only, 1), e->st);
    e->host_refine(e->d_B, e->d_U[0], d_only, 1);
    std::vector<cplx> xx(e->nw);
    double rel = 0;
    CK3(cudaMemcpyAsync(xx.data(), dX, sizeof(cplx) * e->nw, cudaMemcpyDeviceToHost, e->st));
    CK3(cudaMemcpyAsync(&rel, e->d_rel_prev + t, sizeof(double), cudaMemcpyDeviceToHost, e->st));
    CK3(cudaStreamSynchronize(e->st));
    cplx* xo = reinterpret_cast<cplx*>(x);
    for (int v = 0; v < e->nw; ++v) xo[v] = xx[e->Y.pinv[v]];
    if (relres) *relres = rel;
    e->dfree(d_only);
    e->last_step = 0;  // the U buffers no longer hold a sweep
  });
}

int hddm3_symbolic_stats(int nx, int ny, int nz, long* nnz_ref, long* stored, int* nsuper, int* height,
                         long* front_words) {
  return guarded3(nullptr, [&] {
    Sym3 Y;
    build_sym3(nx, ny, nz, Y);
    if (nnz_ref) *nnz_ref = Y.nnz_ref;
    if (stored) *stored = Y.stored_lower + Y.n;
    if (nsuper) *nsuper = int(Y.sn.size());
    if (height) *height = Y.max_height;
    if (front_words) *front_words = Y.front_words;
  });
}

int hddm3_nd_order(int nx, int ny, int nz, int* order) {
  return guarded3(nullptr, [&] {
    const std::vector<int> o = nd_order3(nx, ny, nz);
    std::copy(o.begin(), o.end(), order);
  });
}

int hddm3_footprint(const hddm3_engine* e, long* stored_per_class, long* ref_nnz_per_class, long* device_bytes) {
  *stored_per_class = e->Y.stored_lower + e->Y.n;
  *ref_nnz_per_class = e->Y.nnz_ref;
  *device_bytes = long(e->dev_bytes);
  return 0;
}

int hddm3_time_solve(hddm3_engine* e, int reps, double* ms_per_solve) {
  return guarded3(e, [&] {
    std::vector<int> zero(e->nsub, 0);
    int* d_all = e->upload(zero);  // every RHS active
    cudaGraph_t g;
    CK3(cudaGraphCreate(&g, 0));
    CK3(cudaStreamBeginCaptureToGraph(e->st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    e->enqueue_solve(e->solve_args(e->d_B, e->d_C, d_all, 0), e->st);
    cudaGraph_t go;
    CK3(cudaStreamEndCapture(e->st, &go));
    cudaGraphExec_t ex;
    CK3(cudaGraphInstantiate(&ex, g, 0));
    CK3(cudaGraphLaunch(ex, e->st));
    cudaEvent_t a, b;
    CK3(cudaEventCreate(&a));
    CK3(cudaEventCreate(&b));
    CK3(cudaEventRecord(a, e->st));
    for (int i = 0; i < reps; ++i) CK3(cudaGraphLaunch(ex, e->st));
    CK3(cudaEventRecord(b, e->st));
    CK3(cudaEventSynchronize(b));
    float ms = 0;
    CK3(cudaEventElapsedTime(&ms, a, b));
    *ms_per_solve = ms / std::max(1, reps);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
    e->dfree(d_all);
  });
}

int hddm3_solve_launches(const hddm3_engine* e) { return e->solve_launches(); }
int hddm3_refine_stats(const hddm3_engine* e, double* max_local_relres, int* corrections) {
  *max_local_relres = e->last_max_rel;
  *corrections = e->last_corr;
  return 0;
}
int hddm3_set_timing(hddm3_engine* e, int enable) {
  (void)enable;
  e->launches = 0;
  return 0;
}
int hddm3_stage_times(hddm3_engine* e, double* ms, long long* count, int cap, int* n) {
  (void)e;
  (void)ms;
  (void)count;
  (void)cap;
  *n = 0;
  return 0;
}
long long hddm3_launch_count(const hddm3_engine* e) { return e->launches; }
void* hddm3_stream(const hddm3_engine* e) { return e->st; }

}  // extern "C"
