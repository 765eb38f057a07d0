// B200 DDM engine: host orchestration + the C-ABI of include/hddm.h.
//
// DdmEngine (proj/include/helmddm/ddm.hpp:53-109) re-designed for one GPU:
//   * host: setup (setup.cpp) and symbolic analysis (symbolic.cpp), once;
//   * device: batched multifrontal factorization of every class, then each DDM
//     step is  flags -> gather-sources -> batched supernodal solves ->
//     residual check -> blend-accumulate, all HBM-resident on one stream;
//   * FGMRES keeps V, Z, H, Givens and g on the device.
// There is no CPU fallback: every numeric stage is a CUDA kernel; without a
// CUDA device hddm_create fails.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hddm.h"
#include "hddm_internal.h"
#include "kernels.cuh"
#include "kernels_krylov.cuh"

using namespace hddm;

namespace {

thread_local std::string g_err;

struct SolveErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                               " at " + __FILE__ + ":" + std::to_string(__LINE__));  \
  } while (0)

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

const char* kStageNames[] = {"flags+gather", "solve", "check", "accumulate", "global_apply",
                             "krylov"};
constexpr int kStages = 6;

}  // namespace

struct hddm_engine {
  Setup S;
  Symbolic Y;
  int dev = 0;
  cudaStream_t st = nullptr;
  std::string err;
  int nsub = 0, ncls = 0, nw = 0, wnx = 0, wny = 0, max_members = 0;
  long long ng = 0;
  double factor_ms = 0;
  std::vector<double> probe;
  size_t dev_bytes = 0;  // bytes currently allocated
  std::vector<std::pair<void*, size_t>> allocs;
  int last_step = 0;
  double last_max_rel = 0;
  int last_refine_count = 0;
  bool timing = false;
  double stage_ms[kStages] = {};

  // symbolic tables
  DevSn* d_sn = nullptr;
  DevBlk* d_blk = nullptr;
  int* d_row_first = nullptr;
  long long* d_row_off = nullptr;
  long long* d_run_off = nullptr;
  int* d_seg_ptr = nullptr;
  int2* d_seg = nullptr;
  int* d_bw_ptr = nullptr;
  std::vector<int> h_bw_ptr;
  BwRow* d_bw = nullptr;
  int* d_bw_cnt = nullptr;       // per factor position: backward rows reaching the column
  std::vector<int> h_bw_cnt;
  int* d_perm = nullptr;
  int* d_pinv = nullptr;
  SolvePlan plan;
  cplx* d_vals = nullptr;
  // separators solved by substitution (their diagonal blocks L_ss, row- and
  // column-major packed, ncls x nlss each; lss_off per supernode, -1: inverse)
  cplx* d_lss = nullptr;
  cplx* d_lssc = nullptr;
  long long* d_lss_off = nullptr;
  long long nlss = 0;
  std::vector<long long> h_lss_off;
  // per subdomain
  DevSub* d_sub = nullptr;
  cplx* d_sa = nullptr;
  int sa_stride = 0;
  double* d_wx = nullptr;
  double* d_wy = nullptr;
  // per-subdomain vector layout (VMap, dev.cuh): member-interleaved per class
  long long* d_vbase = nullptr;
  int* d_vstr = nullptr;
  long long* d_cbase = nullptr;
  std::vector<long long> h_vbase;
  std::vector<int> h_vstr;
  cplx* d_U[3] = {};
  cplx* d_B = nullptr;
  cplx* d_Y = nullptr;
  int* d_Z[3] = {};
  int* d_fany = nullptr;
  int* d_owned = nullptr;  // subdomains this engine solves (sharded runs; all by default)
  // sharded runs: called after every DDM step (stage 1, s) and after the K steps of a
  // preconditioner application (stage 2, K) of the host-driven Krylov cycle
  hddm_step_hook hook = nullptr;
  void* hook_user = nullptr;
  int* d_cls_ptr = nullptr;
  int* d_cls_mem = nullptr;
  int* d_act_ptr = nullptr;
  int* d_act_list = nullptr;
  long long* d_counts = nullptr;
  double* d_part_chk = nullptr;
  int nchunk = std::getenv("HDDM_CHECK_CHUNKS") ? std::atoi(std::getenv("HDDM_CHECK_CHUNKS")) : 32;  // residual-check partials per subdomain
  double* d_rel = nullptr;
  int* d_refine = nullptr;
  double* d_maxrel = nullptr;
  // device refinement state (refine, sparse.cpp:268-292)
  cplx* d_R = nullptr;
  cplx* d_C = nullptr;
  double* d_relcur = nullptr;
  int* d_need = nullptr;
  int* d_ncorr = nullptr;
  int* d_undo = nullptr;
  int* d_any = nullptr;
  long long* d_nfix = nullptr;
  int* d_done = nullptr;  // last-block counter of k_finish_init
  // one CUDA graph per step variant (step 1; s >= 2 by s mod 3), each with a
  // conditional WHILE node running the refinement corrections on demand
  cudaStream_t st2 = nullptr;
  struct ForkSet {  // per-tile streams of a forked solve
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t fork = nullptr;
  };
  ForkSet fork_main, fork_body;
  bool per_class_streams = true;
  cudaGraphExec_t step_exec[5] = {};
  int step_kernels[5] = {};  // kernels per step graph variant when no correction runs
  // global
  cplx* d_ga = nullptr;
  double* d_k2 = nullptr;
  cplx* d_f = nullptr;
  cplx* d_asm = nullptr;
  cplx* d_tmp = nullptr;
  int* d_colcov = nullptr;
  unsigned char* d_bmask = nullptr;  // per factor position: in the transfer-patch union
  int* d_pnode = nullptr;
  int* d_pmask = nullptr;
  int* d_xfer_pos = nullptr;
  int4* d_xblk = nullptr;  // transfer block table (kernels.cuh StepArgs::xblk)
  int nxblk = 0;
  int2* d_lpq = nullptr;    // residual-check tables (per factor position)
  int4* d_nbr = nullptr;
  double* d_k2c = nullptr;  // per class: window k^2 in factor order
  cplx* d_ctab = nullptr;         // tabulated check coefficients of the member classes
  long long* d_ctab_off = nullptr;
  double* d_xfer_beta = nullptr;
  int npatch = 0;
  int* d_rowcov = nullptr;
  double* d_part = nullptr;
  double* d_scal = nullptr;  // small scalars
  double* h_scal = nullptr;  // pinned mirror
  // krylov
  int kry_m = 0;
  std::vector<cplx*> V, Z;
  cplx** d_Zptr = nullptr;
  cplx* d_H = nullptr;
  cplx* d_g = nullptr;
  cplx* d_sn_g = nullptr;
  double* d_cs = nullptr;
  cplx* d_y = nullptr;
  cplx* d_b = nullptr;
  cplx* d_x = nullptr;
  cplx* d_r = nullptr;
  cplx** d_Vptr = nullptr;
  KryState* d_ks = nullptr;
  KryState* h_ks = nullptr;  // pinned mirror
  double* d_hist = nullptr;  // recursive relres per FGMRES iteration
  int d_hist_cap = 0;
  int kry_k_last = 0;        // usable columns of the last FGMRES cycle (Z_j taps)
  cudaGraphExec_t kry_exec = nullptr;  // one restart cycle: WHILE over Arnoldi iterations
  int kry_K = -1, kry_iter_kernels = 0;
  KryArgs kry_args(unsigned long long cond);
  int enqueue_kry_iteration(int K, unsigned long long cond, cudaGraph_t body);
  void build_kry_graph(int K);
  void launch_kry_cycle(int K, int m);

  template <class T>
  T* dalloc(size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    allocs.push_back({p, std::max<size_t>(n, 1) * sizeof(T)});
    dev_bytes += std::max<size_t>(n, 1) * sizeof(T);
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
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return p;
  }

  ~hddm_engine() {
    if (dev >= 0) cudaSetDevice(dev);
    for (auto& a : allocs) cudaFree(a.first);
    for (auto& e : ev_pool) cudaEventDestroy(e);
    if (h_scal) cudaFreeHost(h_scal);
    if (h_ks) cudaFreeHost(h_ks);
    if (kry_exec) cudaGraphExecDestroy(kry_exec);
    for (auto& g : step_exec)
      if (g) cudaGraphExecDestroy(g);
    for (ForkSet* F : {&fork_main, &fork_body}) {
      for (auto& x : F->st) cudaStreamDestroy(x);
      for (auto& x : F->ev) cudaEventDestroy(x);
      if (F->fork) cudaEventDestroy(F->fork);
    }
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }

  void create(const hddm_problem& p);
  void factorize();
  void run_probe();
  StepArgs step_args(int s, const cplx* f);
  // solve of the RHS t with (flag[t] != 0) == on: B -> X (Y scratch)
  SolveArgs solve_args(const cplx* B, cplx* X, cplx* Y, const int* flag, int on);
  // the batched solve; with `check`, each tile group's residual partials are
  // queued right behind its solve (overlapping the other groups' chains)
  void enqueue_solve(const SolveArgs& A, cudaStream_t stream, const CheckArgs* check = nullptr);
  int* d_zero = nullptr;  // nsub zero flags: every RHS active
  long long fwd_entries_full = 0, fwd_entries_sparse = 0;  // factor entries per forward sweep
  VMap vmap() const {
    VMap m;
    m.base = d_vbase;
    m.str = d_vstr;
    m.cbase = d_cbase;
    m.cptr = d_cls_ptr;
    m.cmem = d_cls_mem;
    m.ncls = ncls;
    m.total = (long long)nsub * nw;
    return m;
  }
  // one subdomain's vector between device storage and a contiguous host array
  void put_vec(cplx* dv, int t, const cplx* h, cudaStream_t s) {
    CK(cudaMemcpy2DAsync(dv + h_vbase[t], sizeof(cplx) * h_vstr[t], h, sizeof(cplx), sizeof(cplx), nw,
                         cudaMemcpyHostToDevice, s));
  }
  void get_vec(const cplx* dv, int t, cplx* h, cudaStream_t s) {
    CK(cudaMemcpy2DAsync(h, sizeof(cplx), dv + h_vbase[t], sizeof(cplx) * h_vstr[t], sizeof(cplx), nw,
                         cudaMemcpyDeviceToHost, s));
  }
  CheckArgs check_args(const cplx* Bp, const cplx* X, const int* zc, const int* only, bool sparse_b = false);
  RefineArgs refine_args(const cplx* Bp, cplx* X, const int* zc, unsigned long long cond);
  void enqueue_step_front(int s, cudaStream_t stream, unsigned long long cond);
  void enqueue_refine_body(int s, cudaStream_t stream, unsigned long long cond);
  void build_step_graph(int v);
  int capture_step(int s, cudaGraph_t g);
  void run_step(int s);
  void host_refine(const cplx* Bp, cplx* X, const int* zc);
  void reset_state();
  void fill_flags(int* p, int v, int n);
  double device_norm(const cplx* v);
  // stage timing: events recorded on the engine stream, resolved lazily (no
  // host synchronisation inside the timed region)
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<int, int>>> ev_marks;  // stage, (begin, end) pool idx
  size_t ev_next = 0;
  int open_ev[kStages] = {};
  long long launches = 0;
  cudaEvent_t next_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
  void stage_begin(int k) {
    if (!timing) return;
    open_ev[k] = int(ev_next);
    CK(cudaEventRecord(next_event(), st));
  }
  void stage_end(int k) {
    if (!timing) return;
    const int b = open_ev[k];
    const int e = int(ev_next);
    CK(cudaEventRecord(next_event(), st));
    ev_marks.push_back({k, {b, e}});
  }
  void stage_resolve() {
    if (ev_marks.empty()) return;
    CK(cudaStreamSynchronize(st));
    for (auto& m : ev_marks) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev_pool[m.second.first], ev_pool[m.second.second]));
      stage_ms[m.first] += ms;
      stage_n[m.first] += 1;
    }
    ev_marks.clear();
    ev_next = 0;
  }
  long long stage_n[kStages] = {};
  void ensure_krylov(int m);
  void build_plan();
  // window nodes in the union of the 8 transfer patches (transfer.cpp:7-62;
  // identical for every window): the only nonzero RHS entries after step 1
  std::vector<int> patch_union_mask() const {
    const int ext = S.ext, nov = S.nov;
    const int cx0 = ext, cx1 = ext + S.mcx, cy0 = ext, cy1 = ext + S.mcy;
    std::vector<int> mask(size_t(wnx) * wny, 0);
    for (int d = 0; d < 8; ++d) {
      int p0 = 1, p1 = wnx - 2, q0 = 1, q1 = wny - 2;
      const bool fL = d == 1 || d == 5 || d == 7, fR = d == 0 || d == 4 || d == 6;
      const bool fB = d == 3 || d == 6 || d == 7, fT = d == 2 || d == 4 || d == 5;
      if (fL) { p0 = std::max(p0, cx0 + 1); p1 = std::min(p1, cx0 + 1 + nov); }
      if (fR) { p0 = std::max(p0, cx1 - 1 - nov); p1 = std::min(p1, cx1 - 1); }
      if (fB) { q0 = std::max(q0, cy0 + 1); q1 = std::min(q1, cy0 + 1 + nov); }
      if (fT) { q0 = std::max(q0, cy1 - 1 - nov); q1 = std::min(q1, cy1 - 1); }
      for (int q = q0; q <= q1; ++q)
        for (int pp = p0; pp <= p1; ++pp) mask[size_t(q) * wnx + pp] |= 1 << d;
    }
    return mask;
  }
  int solve_launches() { return solve_launch_count(plan, solve_args(d_B, d_U[0], d_Y, d_zero, 0)); }
};

// ----------------------------------------------------------------- creation
void hddm_engine::create(const hddm_problem& p) {
  // configuration errors first (the reference's constructor validates the
  // partition before anything else, partition.cpp:15-28)
  std::string msg;
  const int rc = build_setup(p, S, msg);
  if (rc == HDDM_ERR_CONFIG) throw ConfigErr(msg);
  if (rc) throw std::runtime_error(msg);
  int ndev = 0;
  dev = -1;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw std::runtime_error("no CUDA device available (the engine has no CPU fallback)");
  dev = p.device;
  if (dev < 0 || dev >= ndev) throw ConfigErr("invalid CUDA device ordinal");
  CK(cudaSetDevice(dev));
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  per_class_streams = std::getenv("HDDM_SINGLE_STREAM") == nullptr;
  CK(cudaMallocHost(&h_scal, 64 * sizeof(double)));
  CK(cudaMallocHost(&h_ks, sizeof(KryState)));
  nsub = S.n1 * S.n2;
  ncls = S.ncls;
  wnx = S.subs[0].nx;
  wny = S.subs[0].ny;
  nw = wnx * wny;
  ng = (long long)S.gnx * S.gny;
  for (int c = 0; c < ncls; ++c)
    max_members = std::max(max_members, S.cls_ptr[c + 1] - S.cls_ptr[c]);
  build_symbolic(wnx, wny, Y);

  // ---- symbolic tables
  std::vector<DevSn> sn(Y.sn.size());
  for (size_t s = 0; s < Y.sn.size(); ++s) {
    const SnNode& a = Y.sn[s];
    DevSn& d = sn[s];
    d.kind = a.kind;
    d.c0 = a.c0;
    d.n = a.n;
    d.nrows = int(a.rows.size());
    d.blk0 = a.blk0;
    d.nblk = a.nblk;
    d.drow0 = a.drow0;
    d.parent = a.parent;
    d.child0 = a.nch > 0 ? a.child[0] : -1;
    d.child1 = a.nch > 1 ? a.child[1] : -1;
    d.extadd0 = a.extadd0;
    d.aent0 = Y.aent0[s];
    d.aent1 = Y.aent0[s + 1];
    d.lw = a.kind == 0 ? a.w : 0;
    d.diag_off = a.diag_off;
    d.dinv_off = a.dinv_off;
    d.front_off = a.front_off;
  }
  d_sn = upload(sn);
  std::vector<DevBlk> blk(Y.blk.size());
  for (size_t b = 0; b < Y.blk.size(); ++b) {
    const Block& a = Y.blk[b];
    blk[b] = {a.src, a.dst, a.r0, a.nr, a.row0, a.front0};
  }
  d_blk = upload(blk);
  d_row_first = upload(Y.row_first);
  std::vector<long long> roff(Y.row_off.begin(), Y.row_off.end());
  d_row_off = upload(roff);
  d_perm = upload(Y.perm);
  d_pinv = upload(Y.pinv);
  // forward runs and segments; backward rows per supernode
  {
    std::vector<long long> ro(Y.run_off.begin(), Y.run_off.end());
    d_run_off = upload(ro);
    d_seg_ptr = upload(Y.seg_ptr);
    std::vector<int2> sg(Y.seg.size());
    for (size_t k = 0; k < Y.seg.size(); ++k) sg[k] = make_int2(Y.seg[k].len, Y.seg[k].zbase);
    d_seg = upload(sg);
    std::vector<int> bptr(Y.sn.size() + 1, 0);
    std::vector<BwRow> bw;
    for (size_t s = 0; s < Y.sn.size(); ++s) {
      bptr[s] = int(bw.size());
      for (int b = Y.sn[s].blk0; b < Y.sn[s].blk0 + Y.sn[s].nblk; ++b) {
        const Block& B = Y.blk[b];
        for (int r = 0; r < B.nr; ++r) {
          const int rt = B.row0 + r;
          if (Y.row_first[rt] >= Y.sn[s].n) continue;  // empty padding row
          BwRow w;
          w.off = Y.row_off[rt];
          w.first = Y.row_first[rt];
          w.dpos = Y.sn[B.dst].c0 + B.r0 + r;
          bw.push_back(w);
        }
      }
      // by first stored column: a column pass stops at the first row beyond it
      std::stable_sort(bw.begin() + bptr[s], bw.end(),
                       [](const BwRow& a, const BwRow& b) { return a.first < b.first; });
    }
    bptr[Y.sn.size()] = int(bw.size());
    d_bw_ptr = upload(bptr);
    h_bw_ptr = bptr;
    d_bw = upload(bw);
    // rows reaching each column (first <= column): a prefix of the sorted list
    h_bw_cnt.assign(Y.n, 0);
    for (size_t s = 0; s < Y.sn.size(); ++s) {
      int k = bptr[s];
      for (int j = 0; j < Y.sn[s].n; ++j) {
        while (k < bptr[s + 1] && bw[k].first <= j) ++k;
        h_bw_cnt[Y.sn[s].c0 + j] = k - bptr[s];
      }
    }
    d_bw_cnt = upload(h_bw_cnt);
  }

  // ---- per-subdomain data
  std::vector<DevSub> subs(nsub);
  sa_stride = 2 * wnx + 2 * wny;
  std::vector<cplx> sa(size_t(nsub) * sa_stride);
  std::vector<double> wx(size_t(nsub) * wnx), wy(size_t(nsub) * wny);
  for (int t = 0; t < nsub; ++t) {
    const Sub& s = S.subs[t];
    DevSub& d = subs[t];
    d.i = s.i;
    d.j = s.j;
    d.cx0 = s.cx0;
    d.cx1 = s.cx1;
    d.cy0 = s.cy0;
    d.cy1 = s.cy1;
    d.wx0 = s.wx0;
    d.wy0 = s.wy0;
    d.lint = s.lint;
    d.rint = s.rint;
    d.bint = s.bint;
    d.tint = s.tint;
    d.own0 = s.own[0];
    d.own1 = s.own[1];
    d.own2 = s.own[2];
    d.own3 = s.own[3];
    d.cls = s.cls;
    const WinOp& w = S.subop[t];
    cplx* o = &sa[size_t(t) * sa_stride];
    for (int k = 0; k < wnx; ++k) {
      o[k] = cmk(w.a1n[2 * k], w.a1n[2 * k + 1]);
      o[wnx + k] = cmk(w.ia1h[2 * k], w.ia1h[2 * k + 1]);
    }
    for (int k = 0; k < wny; ++k) {
      o[2 * wnx + k] = cmk(w.a2n[2 * k], w.a2n[2 * k + 1]);
      o[2 * wnx + wny + k] = cmk(w.ia2h[2 * k], w.ia2h[2 * k + 1]);
    }
    std::copy(s.wx.begin(), s.wx.end(), wx.begin() + size_t(t) * wnx);
    std::copy(s.wy.begin(), s.wy.end(), wy.begin() + size_t(t) * wny);
  }
  d_sub = upload(subs);
  d_sa = upload(sa);
  d_wx = upload(wx);
  d_wy = upload(wy);
  d_cls_ptr = upload(S.cls_ptr);
  d_cls_mem = upload(S.cls_members);
  {
    h_vbase.assign(nsub, 0);
    h_vstr.assign(nsub, 0);
    std::vector<long long> cb(ncls + 1);
    for (int c = 0; c <= ncls; ++c) cb[c] = (long long)S.cls_ptr[c] * nw;
    for (int c = 0; c < ncls; ++c)
      for (int k = S.cls_ptr[c]; k < S.cls_ptr[c + 1]; ++k) {
        const int t = S.cls_members[k];
        h_vbase[t] = cb[c] + (k - S.cls_ptr[c]);
        h_vstr[t] = S.cls_ptr[c + 1] - S.cls_ptr[c];
      }
    d_vbase = upload(h_vbase);
    d_vstr = upload(h_vstr);
    d_cbase = upload(cb);
  }
  build_plan();
  for (int k = 0; k < 3; ++k) {
    d_U[k] = dalloc<cplx>(size_t(nsub) * nw);
    d_Z[k] = dalloc<int>(nsub);
  }
  d_B = dalloc<cplx>(size_t(nsub) * nw);
  d_Y = dalloc<cplx>(size_t(nsub) * nw);
  CK(cudaMemsetAsync(d_B, 0, size_t(nsub) * nw * sizeof(cplx), st));
  d_fany = dalloc<int>(nsub);
  d_owned = upload(std::vector<int>(nsub, 1));
  d_zero = dalloc<int>(nsub);
  CK(cudaMemsetAsync(d_zero, 0, sizeof(int) * nsub, st));
  d_act_ptr = dalloc<int>(ncls + 1);
  d_act_list = dalloc<int>(nsub);
  d_counts = dalloc<long long>(2);
  d_part_chk = dalloc<double>(size_t(nsub) * nchunk * 2);
  d_rel = dalloc<double>(nsub);
  d_refine = dalloc<int>(1);
  d_maxrel = dalloc<double>(1);
  d_R = dalloc<cplx>(size_t(nsub) * nw);
  d_C = dalloc<cplx>(size_t(nsub) * nw);
  d_relcur = dalloc<double>(nsub);
  d_need = dalloc<int>(nsub);
  d_ncorr = dalloc<int>(nsub);
  d_undo = dalloc<int>(nsub);
  d_any = dalloc<int>(1);
  d_nfix = dalloc<long long>(1);
  d_done = dalloc<int>(1);
  CK(cudaMemsetAsync(d_done, 0, sizeof(int), st));
  CK(cudaMemsetAsync(d_nfix, 0, sizeof(long long), st));

  // ---- global data
  std::vector<cplx> ga(size_t(2) * S.gnx + 2 * S.gny);
  for (int k = 0; k < S.gnx; ++k) {
    ga[k] = cmk(S.gop.a1n[2 * k], S.gop.a1n[2 * k + 1]);
    ga[S.gnx + k] = cmk(S.gop.ia1h[2 * k], S.gop.ia1h[2 * k + 1]);
  }
  for (int k = 0; k < S.gny; ++k) {
    ga[2 * S.gnx + k] = cmk(S.gop.a2n[2 * k], S.gop.a2n[2 * k + 1]);
    ga[2 * S.gnx + S.gny + k] = cmk(S.gop.ia2h[2 * k], S.gop.ia2h[2 * k + 1]);
  }
  d_ga = upload(ga);
  d_k2 = upload(S.k2);
  d_f = dalloc<cplx>(ng);
  d_asm = dalloc<cplx>(ng);
  d_tmp = dalloc<cplx>(ng);
  // blend coverage per global column / row (accumulate region, ddm.cpp:221-224)
  {
    std::vector<int> colcov(size_t(4) * S.gnx, -1), rowcov(size_t(4) * S.gny, -1);
    for (int i = 0; i < S.n1; ++i) {
      const Sub& s = S.subs[i];
      const int x0 = s.lint ? s.cx0 - S.nov : s.wx0;
      const int x1 = s.rint ? s.cx1 + S.nov : s.wx0 + s.nx - 1;
      for (int P = x0; P <= x1; ++P) {
        int k = 0;
        while (k < 4 && colcov[4 * P + k] >= 0) ++k;
        if (k == 4) throw ConfigErr("more than 4 overlapping subdomains per column");
        colcov[4 * P + k] = i;
      }
    }
    for (int j = 0; j < S.n2; ++j) {
      const Sub& s = S.subs[size_t(j) * S.n1];
      const int y0 = s.bint ? s.cy0 - S.nov : s.wy0;
      const int y1 = s.tint ? s.cy1 + S.nov : s.wy0 + s.ny - 1;
      for (int Q = y0; Q <= y1; ++Q) {
        int k = 0;
        while (k < 4 && rowcov[4 * Q + k] >= 0) ++k;
        if (k == 4) throw ConfigErr("more than 4 overlapping subdomains per row");
        rowcov[4 * Q + k] = j;
      }
    }
    d_colcov = upload(colcov);
    d_rowcov = upload(rowcov);
  }
  // union of the transfer patches in window-local coordinates
  // (transfer_patch, transfer.cpp:7-62; identical for every window)
  {
    const std::vector<int> mask = patch_union_mask();
    std::vector<int> pn, pm;
    for (int k = 0; k < nw; ++k) {  // factor order: coalesced writes of B
      const int node = Y.perm[k];
      if (mask[node]) {
        pn.push_back(node);
        pm.push_back(mask[node]);
      }
    }
    npatch = int(pn.size());
    d_pnode = upload(pn);
    std::vector<unsigned char> bm(nw, 0);
    for (int k = 0; k < nw; ++k) bm[k] = mask[Y.perm[k]] ? 1 : 0;
    d_bmask = upload(bm);
    d_pmask = upload(pm);
    // per (patch node, direction, stencil point C E W N S): the source-window
    // position and transfer_beta (partition.cpp:131-152) -- window-local, so
    // identical for every target window
    std::vector<int> xpos(size_t(npatch) * 40, -1);
    std::vector<double> xbeta(size_t(npatch) * 40, 0.0);
    const int dIx[8] = {+1, -1, 0, 0, +1, -1, +1, -1}, dJx[8] = {0, 0, +1, -1, +1, +1, -1, -1};
    const int dp[5] = {0, 1, -1, 0, 0}, dq[5] = {0, 0, 0, 1, -1};
    const int cx0 = S.ext, cx1 = S.ext + S.mcx, cy0 = S.ext, cy1 = S.ext + S.mcy;  // window-local core
    auto beta0h = [](double t) {
      if (t <= 0) return 1.0;
      if (t >= 1) return 0.0;
      return 1.0 - t * t * t * (10.0 - 15.0 * t + 6.0 * t * t);
    };
    for (int u = 0; u < npatch; ++u) {
      const int lp = pn[u] % wnx, lq = pn[u] / wnx;
      for (int d = 0; d < 8; ++d) {
        if (!((pm[u] >> d) & 1)) continue;
        const int sp = lp - dIx[d] * S.mcx, sq = lq - dJx[d] * S.mcy;
        const bool fromL = d == 1 || d == 5 || d == 7, fromR = d == 0 || d == 4 || d == 6;
        const bool fromB = d == 3 || d == 6 || d == 7, fromT = d == 2 || d == 4 || d == 5;
        for (int k = 0; k < 5; ++k) {
          const int xp = sp + dp[k], xq = sq + dq[k];
          const size_t e = (size_t(u) * 8 + d) * 5 + k;
          if (xp >= 0 && xq >= 0 && xp < wnx && xq < wny) xpos[e] = Y.pinv[xq * wnx + xp];
          const int p = lp + dp[k], q = lq + dq[k];
          double b = 1.0;
          if (fromL) b = beta0h(double(p - cx0 - 1) / S.nov);
          if (fromR) b = beta0h(double(cx1 - 1 - p) / S.nov);
          if (fromB) b *= beta0h(double(q - cy0 - 1) / S.nov);
          if (fromT) b *= beta0h(double(cy1 - 1 - q) / S.nov);
          xbeta[e] = b;
        }
      }
    }
    d_xfer_pos = upload(xpos);
    d_xfer_beta = upload(xbeta);
    // transfer blocks: member slabs of <= 32 per class, 256 / M patch nodes per block
    std::vector<int4> xb;
    for (int c = 0; c < ncls; ++c) {
      const int m = S.cls_ptr[c + 1] - S.cls_ptr[c];
      const int nslab = (m + 31) / 32;
      for (int sl = 0; sl < nslab; ++sl) {
        const int k0 = int((long long)m * sl / nslab), k1 = int((long long)m * (sl + 1) / nslab);
        const int M = k1 - k0, per = 256 / M;
        for (int u0 = 0; u0 < npatch; u0 += per) xb.push_back(make_int4(c, k0, M, u0));
      }
    }
    nxblk = int(xb.size());
    d_xblk = upload(xb);
  }
  // residual check tables (the J-scaled window stencil, discretize.cpp:98-160):
  // window coordinates and neighbour positions per factor position, k^2 per class
  {
    std::vector<int2> lpq(nw);
    std::vector<int4> nb(nw);
    for (int pos = 0; pos < nw; ++pos) {
      const int node = Y.perm[pos];
      const int lp = node % wnx, lq = node / wnx;
      const bool ring = lp == 0 || lq == 0 || lp == wnx - 1 || lq == wny - 1;
      lpq[pos] = make_int2(ring ? -1 : lp, lq);
      nb[pos] = make_int4(!ring && lq > 1 ? Y.pinv[node - wnx] : -1, !ring && lp > 1 ? Y.pinv[node - 1] : -1,
                          !ring && lp < wnx - 2 ? Y.pinv[node + 1] : -1,
                          !ring && lq < wny - 2 ? Y.pinv[node + wnx] : -1);
    }
    d_lpq = upload(lpq);
    d_nbr = upload(nb);
    std::vector<double> k2c(size_t(ncls) * nw, 0.0);
    for (int c = 0; c < ncls; ++c) {
      const Sub& sb = S.subs[S.cls_rep[c]];
      for (int pos = 0; pos < nw; ++pos) {
        const int node = Y.perm[pos];
        const int lp = node % wnx, lq = node / wnx;
        k2c[size_t(c) * nw + pos] = S.k2[size_t(sb.wy0 + lq) * S.gnx + sb.wx0 + lp];
      }
    }
    d_k2c = upload(k2c);
    // row coefficients tabulated for classes with >= HDDM_CTAB_MIN members (80 B per
    // position and class; the members re-read them instead of re-forming them)
    static const int ctab_min = std::getenv("HDDM_CTAB_MIN") ? std::atoi(std::getenv("HDDM_CTAB_MIN")) : 4;
    std::vector<long long> off(ncls, -1);
    long long tot = 0;
    for (int c = 0; c < ncls; ++c)
      if (S.cls_ptr[c + 1] - S.cls_ptr[c] >= ctab_min) {
        off[c] = tot;
        tot += (long long)nw * 5;
      }
    if (tot > 0) {
      d_ctab = dalloc<cplx>(size_t(tot));
      d_ctab_off = upload(off);
      const CheckArgs C = check_args(nullptr, nullptr, nullptr, nullptr);
      for (int c = 0; c < ncls; ++c)
        if (off[c] >= 0) launch_build_ctab(C, c, d_ctab + off[c], st);
    }
  }
  d_part = dalloc<double>(2 * size_t(reduce_blocks()));
  d_scal = dalloc<double>(64);

  factorize();
  run_probe();
}

// Solve plan: the ND tree level by level. Forward: leaves, then separator rows
// by height; backward: separator columns by depth, then leaf columns, then the
// leaves' band back-substitution.
void hddm_engine::build_plan() {
  const int nsn = int(Y.sn.size());
  std::vector<int2> leaves, leafcols;
  for (int s = 0; s < nsn; ++s)
    if (Y.sn[s].kind == 0) {
      leaves.push_back(make_int2(s, 0));
      for (int j = 0; j < Y.sn[s].n; ++j) leafcols.push_back(make_int2(s, j));
    }
  // Separators of SUBST_MIN..SUBST_MAX nodes are solved by substitution with L_ss
  // itself; the larger and smaller ones by their explicit inverse (HDDM_SUBST_MIN /
  // HDDM_SUBST_MAX; 0 / 0 switches substitution off)
  {
    const int smin = std::getenv("HDDM_SUBST_MIN") ? std::atoi(std::getenv("HDDM_SUBST_MIN")) : 24;
    // k_sep_trsv keeps 32 * kTrsvR = 64 rows per warp in registers
    const int smax = std::min(64, std::getenv("HDDM_SUBST_MAX") ? std::atoi(std::getenv("HDDM_SUBST_MAX")) : 64);
    std::vector<long long> off(Y.sn.size(), -1);
    nlss = 0;
    for (size_t s = 0; s < Y.sn.size(); ++s)
      if (Y.sn[s].kind == 1 && Y.sn[s].n >= smin && Y.sn[s].n <= smax && smax > 0) {
        off[s] = nlss;
        nlss += (long long)Y.sn[s].n * (Y.sn[s].n - 1) / 2;
      }
    h_lss_off = off;
    d_lss_off = upload(off);
  }
  auto level = [&](const std::vector<int2>& v) {
    SolveLevel L;
    L.nitem = int(v.size());
    L.d_items = upload(v);
    // the level's separators (items (s, 0)) for the substitution kernels
    std::vector<int2> sp;
    bool all = true;  // the substitution kernels replace a level's inverse kernel entirely
    for (const int2& it : v)
      if (it.y == 0 && Y.sn[it.x].kind == 1) {
        if (h_lss_off[it.x] >= 0)
          sp.push_back(it);
        else
          all = false;
      }
    if (!all) sp.clear();
    L.nsep = int(sp.size());
    for (const int2& it : sp) L.nmax_sep = std::max(L.nmax_sep, Y.sn[it.x].n);
    if (L.nsep) L.d_seps = upload(sp);
    return L;
  };
  // leaves: w x h boxes in natural order; with the 5-point fill their band rows
  // start at i-1 (first grid row) / i-w and are stored back to back from
  // diag_off -- the leaf kernels stream them without row tables
  for (const SnNode& nd : Y.sn)
    if (nd.kind == 0) {
      long off = nd.diag_off;
      for (int i = 0; i < nd.n; ++i) {
        const int first = i < nd.w ? (i > 0 ? i - 1 : 0) : i - nd.w;
        if (Y.row_first[nd.drow0 + i] != first || Y.row_off[nd.drow0 + i] != off || i - first > 6)
          throw std::runtime_error("leaf band profile differs from the w x h natural-order box");
        off += i - first;
      }
    }
  // member tiles (up to 32 members of one class), grouped by member count M:
  // a group shares every launch (optionally capped at HDDM_GROUP_TILES tiles)
  std::vector<int> Rs;  // distinct columns-per-CTA of the backward split kernels
  {
    std::map<int, std::vector<TileRec>> byM;
    for (int c = 0; c < ncls; ++c) {
      const int m = S.cls_ptr[c + 1] - S.cls_ptr[c];
      // ceil(m / tile_max) tiles of near-equal size: a 36-member class (config 2) runs as
      // 12 + 12 + 12 (0.935 -> 0.834 ms per solve), not 32 + 4; config 4 keeps its 14s
      static const int tile_max =
          std::max(1, std::min(32, std::getenv("HDDM_TILE_MAX") ? std::atoi(std::getenv("HDDM_TILE_MAX")) : 16));
      const int nt = (m + tile_max - 1) / tile_max;
      for (int ti = 0, k0 = 0; ti < nt; ++ti) {
        const int M = m / nt + (ti < m % nt ? 1 : 0);
        TileRec T = {};
        T.cb = (long long)S.cls_ptr[c] * nw + k0;
        T.c = c;
        T.m = m;
        for (int k = 0; k < 32; ++k) T.t[k] = S.cls_members[S.cls_ptr[c] + k0 + std::min(k, M - 1)];
        byM[M].push_back(T);
        k0 += M;
      }
    }
    // 4 tiles per group measured best at config 4 (more, shorter launch chains
    // overlap better; 1 per group is launch-bound)
    const char* cap_env = std::getenv("HDDM_GROUP_TILES");
    const int cap1 = cap_env ? std::max(1, std::atoi(cap_env)) : 4;
    const char* capm_env = std::getenv("HDDM_GROUP_TILES_M");  // groups of multi-member tiles
    const int capm = capm_env ? std::max(1, std::atoi(capm_env)) : cap1;
    for (auto& kv : byM) {
      const int M = kv.first;
      const int cap = M > 1 ? capm : cap1;
      if (std::find(Rs.begin(), Rs.end(), 32 / M) == Rs.end()) Rs.push_back(32 / M);
      for (size_t a = 0; a < kv.second.size(); a += cap) {
        const size_t b = std::min(kv.second.size(), a + size_t(cap));
        std::vector<TileRec> part(kv.second.begin() + a, kv.second.begin() + b);
        TileArg G;
        G.rec = upload(part);
        G.ntile = int(part.size());
        G.M = M;
        G.E = 1;
        G.R = 32 / M;
        tile_mags(G);
        for (auto& t : part) {
          plan.tiles.push_back(t);
          plan.tile_group.push_back(int(plan.groups.size()));
        }
        // sub-tiles of 2 members (M even) for the levels with long rows: more
        // lanes per row and more warps, the factor entries re-read per sub-tile
        TileArg Sg = G;
        const int Ms = (M % 2 == 0 && M > 2) ? 2 : 0;
        if (Ms) {
          std::vector<TileRec> sub;
          for (const TileRec& t : part)
            for (int k0 = 0; k0 < M; k0 += Ms) {
              TileRec r = t;
              r.cb = t.cb + k0;
              for (int k = 0; k < 32; ++k) r.t[k] = t.t[std::min(k0 + k, M - 1)];
              sub.push_back(r);
            }
          Sg.rec = upload(sub);
          Sg.ntile = int(sub.size());
          Sg.M = Ms;
          Sg.R = 32 / Ms;
        } else {
          Sg.ntile = 0;
        }
        plan.sub.push_back(Sg);
        plan.groups.push_back(G);
      }
    }
  }
  static const int stage_cw = std::getenv("HDDM_STAGE_CW") ? std::atoi(std::getenv("HDDM_STAGE_CW")) : 32;
  auto chunks4 = [&](SolveLevel& L, const std::vector<int>& sns) {
    std::vector<int4> ch;
    int cw = 0;
    L.one_chunk = !sns.empty();
    for (int s : sns) L.one_chunk = L.one_chunk && Y.sn[s].n <= stage_cw;
    for (int s : sns)
      for (int j = 0; j < Y.sn[s].n; j += stage_cw) {
        const int j1 = std::min(Y.sn[s].n, j + stage_cw);
        ch.push_back(make_int4(s, j, j1, h_bw_cnt[Y.sn[s].c0 + j1 - 1]));
        cw = std::max(cw, j1 - j);
      }
    L.nchunk4 = int(ch.size());
    L.d_chunks4 = upload(ch);
    L.cw_max = cw;
  };
  plan.staged = std::getenv("HDDM_NO_STAGE") == nullptr;
  if (const char* v = std::getenv("HDDM_SUB_RUN")) plan.sub_run = std::atol(v);
  if (const char* v = std::getenv("HDDM_SUB_BWD")) plan.sub_bwd_ctas = std::atoi(v);
  // programmatic dependent launch of the level chains: measured faster only when every
  // class is a singleton (config 3: 1.909 -> 1.828 ms per step); with member tiles the
  // early-resident successors take the slots the other chains' kernels need (config 4:
  // 1.666 -> 1.769 for all chains, 1.845 for the singleton chains alone; config 2: 0.80 -> 1.02)
  plan.pdl = std::getenv("HDDM_PDL") ? std::atoi(std::getenv("HDDM_PDL")) : (max_members == 1 ? 1 : 0);
  plan.fwd_leaf = level(leaves);
  plan.bwd_leaf = level(leaves);
  plan.bwd_leafcol = level(leafcols);
  {
    std::vector<int> ls;
    for (const int2& l : leaves) ls.push_back(l.x);
    chunks4(plan.bwd_leafcol, ls);
  }
  std::vector<SegRec> fseg;  // forward run segments of every level's rows
  // member-tile tensor-core pulls: 8-row blocks of each separator, the union of their
  // run segments by source supernode (kernels.cuh MmaSeg)
  std::vector<int> snof(Y.n, -1);
  for (int s = 0; s < nsn; ++s)
    for (int i = 0; i < Y.sn[s].n; ++i) snof[Y.sn[s].c0 + i] = s;
  auto mma_tables = [&](SolveLevel& L, const std::vector<int2>& items, const std::vector<int4>& rec,
                        const std::vector<SegRec>& segs) {
    std::vector<int4> blks;
    std::vector<MmaSeg> ms;
    double padded = 0, stored = 0;
    size_t k = 0;
    while (k < items.size()) {
      size_t e = k;
      while (e < items.size() && items[e].x == items[k].x && e - k < 8) ++e;
      std::map<int, std::pair<int, int>> uni;
      for (size_t r = k; r < e; ++r)
        for (int q = rec[r].y; q < rec[r].y + rec[r].z; ++q) {
          const SegRec& g = segs[q];
          const int src = snof[g.zb];
          auto it = uni.find(src);
          if (it == uni.end())
            uni[src] = {g.zb, g.zb + g.len};
          else
            it->second = {std::min(it->second.first, g.zb), std::max(it->second.second, g.zb + g.len)};
        }
      blks.push_back(make_int4(int(k), int(e - k), int(ms.size()), int(uni.size())));
      for (const auto& kv : uni) padded += double(kv.second.second - kv.second.first) * double(e - k);
      for (size_t r = k; r < e; ++r)
        for (int q = rec[r].y; q < rec[r].y + rec[r].z; ++q) stored += segs[q].len;
      for (const auto& kv : uni) {
        MmaSeg S = {};
        S.zmin = kv.second.first;
        S.ulen = kv.second.second - kv.second.first;
        for (size_t r = k; r < e; ++r)
          for (int q = rec[r].y; q < rec[r].y + rec[r].z; ++q) {
            const SegRec& g = segs[q];
            if (snof[g.zb] != kv.first) continue;
            S.lo[r - k] = g.zb;
            S.hi[r - k] = g.zb + g.len;
            S.vb[r - k] = g.off - g.zb;
          }
        ms.push_back(S);
      }
      k = e;
    }
    L.nmblk = int(blks.size());
    L.mma_fill = stored > 0 ? padded / stored : 0;
    if (L.nmblk) {
      L.d_mblk = upload(blks);
      L.d_mseg = upload(ms);
    }
  };
  for (int h = 1; h <= Y.max_height; ++h) {
    std::vector<int2> v;
    for (int s = 0; s < nsn; ++s)
      if (Y.sn[s].kind == 1 && Y.sn[s].height == h)
        for (int i = 0; i < Y.sn[s].n; ++i) v.push_back(make_int2(s, i));
    if (v.empty()) continue;
    SolveLevel L = level(v);
    std::vector<int4> rec(v.size());
    long tot = 0, dtot = 0;
    for (size_t k = 0; k < v.size(); ++k) {
      const int pos = Y.sn[v[k].x].c0 + v[k].y;
      const int sbeg = int(fseg.size());
      long long off = Y.run_off[pos];
      for (int e = Y.seg_ptr[pos]; e < Y.seg_ptr[pos + 1]; ++e) {
        fseg.push_back(SegRec{off, Y.seg[e].len, Y.seg[e].zbase});
        off += Y.seg[e].len;
      }
      rec[k] = make_int4(pos, sbeg, int(fseg.size()) - sbeg, 0);
      tot += Y.run_off[pos + 1] - Y.run_off[pos];
      dtot += v[k].y;
    }
    L.d_rec = upload(rec);
    L.avg_run = tot / long(v.size());
    L.avg_diag = dtot / long(v.size());
    mma_tables(L, v, rec, fseg);
    plan.fwd.push_back(L);
  }
  std::vector<SegRec> fseg_sp;
  std::vector<int> sn_of(Y.n, -1);  // supernode of each factor position (ring: -1)
  for (int s = 0; s < nsn; ++s)
    for (int i = 0; i < Y.sn[s].n; ++i) sn_of[Y.sn[s].c0 + i] = s;
  // forward plan for steps >= 2: only the nonzero RHS entries are the transfer
  // patches, so supernodes whose subtree holds no patch node produce z = 0
  // exactly (X is cleared first) and are skipped
  if (std::getenv("HDDM_NO_SPARSE_RHS") == nullptr) {
    const std::vector<int> mask = patch_union_mask();
    std::vector<char> act(nsn, 0);
    for (int s = 0; s < nsn; ++s) {  // postorder: children before parents
      const SnNode& a = Y.sn[s];
      char any = 0;
      for (int i = 0; i < a.n && !any; ++i) any = mask[Y.perm[a.c0 + i]] != 0;
      for (int c = 0; c < a.nch; ++c) any |= act[a.child[c]];
      act[s] = any;
    }
    std::vector<int2> lv;
    for (const int2& l : leaves)
      if (act[l.x]) lv.push_back(l);
    plan.fwd_leaf_sp = level(lv);
    for (const SolveLevel& L : plan.fwd) {
      // the level's rows, filtered to active separators (same order)
      std::vector<int2> v(L.nitem);
      CK(cudaMemcpy(v.data(), L.d_items, sizeof(int2) * L.nitem, cudaMemcpyDeviceToHost));
      std::vector<int2> keep;
      for (const int2& it : v)
        if (act[it.x]) keep.push_back(it);
      SolveLevel F;
      if (!keep.empty()) {
        F = level(keep);
        std::vector<int4> rec(keep.size());
        long tot = 0, dtot = 0;
        for (size_t k = 0; k < keep.size(); ++k) {
          const int pos = Y.sn[keep[k].x].c0 + keep[k].y;
          // only segments from active sources: the others multiply z = 0
          const int sbeg = int(fseg_sp.size());
          long long off = Y.run_off[pos];
          for (int e = Y.seg_ptr[pos]; e < Y.seg_ptr[pos + 1]; ++e) {
            if (act[sn_of[Y.seg[e].zbase]]) {
              fseg_sp.push_back(SegRec{off, Y.seg[e].len, Y.seg[e].zbase});
              tot += Y.seg[e].len;
            }
            off += Y.seg[e].len;
          }
          rec[k] = make_int4(pos, sbeg, int(fseg_sp.size()) - sbeg, 0);
          dtot += keep[k].y;
        }
        F.d_rec = upload(rec);
        F.avg_run = tot / long(keep.size());
        F.avg_diag = dtot / long(keep.size());
        mma_tables(F, keep, rec, fseg_sp);
      }
      plan.fwd_sp.push_back(F);
    }
    plan.d_fseg_sp = upload(fseg_sp);
    plan.d_sn_live = upload(std::vector<unsigned char>(act.begin(), act.end()));
    plan.has_sparse = true;
    fwd_entries_full = 0;
    fwd_entries_sparse = 0;
    for (int s = 0; s < nsn; ++s) {
      const SnNode& a = Y.sn[s];
      long long w = 0;
      if (a.kind == 1) {
        for (int i = 0; i < a.n; ++i) w += Y.run_off[a.c0 + i + 1] - Y.run_off[a.c0 + i];
        w += (long long)a.n * (a.n - 1) / 2;
      } else {
        for (int i = 0; i < a.n; ++i) w += i - Y.row_first[a.drow0 + i];
      }
      fwd_entries_full += w;
      if (act[s]) {  // runs of active rows count only their live segments (below)
        if (a.kind == 1)
          fwd_entries_sparse += (long long)a.n * (a.n - 1) / 2;
        else
          fwd_entries_sparse += w;
      }
    }
    for (const SegRec& r : fseg_sp) fwd_entries_sparse += r.len;
  }
  plan.d_fseg = upload(fseg);
  const char* env_sr = std::getenv("HDDM_SPLIT_ROWS");
  const char* env_sd = std::getenv("HDDM_SPLIT_DIAG");
  for (int d = 0; d <= Y.max_depth; ++d) {
    std::vector<int2> v;
    std::vector<int> sns;
    long rows = 0, nmax = 0;
    for (int s = 0; s < nsn; ++s)
      if (Y.sn[s].kind == 1 && Y.sn[s].depth == d) {
        sns.push_back(s);
        for (int i = 0; i < Y.sn[s].n; ++i) v.push_back(make_int2(s, i));
        rows += h_bw_ptr[s + 1] - h_bw_ptr[s];
        nmax = std::max<long>(nmax, Y.sn[s].n);
      }
    if (v.empty()) continue;
    SolveLevel L = level(v);
    chunks4(L, sns);
    {  // member-tile tensor-core kernels: blocks of up to 8 columns of one separator
      std::vector<int4> blks;
      long dsum = 0;
      for (size_t k = 0; k < v.size();) {
        size_t e = k;
        while (e < v.size() && v[e].x == v[k].x && e - k < 8) ++e;
        blks.push_back(make_int4(int(k), int(e - k), 0, 0));
        k = e;
      }
      for (const int2& it : v) dsum += Y.sn[it.x].n - 1 - it.y;
      L.avg_diag = dsum / long(v.size());
      L.nmblk = int(blks.size());
      L.d_mblk = upload(blks);
    }
    static const long split_rows_min = std::getenv("HDDM_SPLIT_ROWS_MIN") ? std::atol(std::getenv("HDDM_SPLIT_ROWS_MIN")) : 64;
    static const long split_diag_min = std::getenv("HDDM_SPLIT_DIAG_MIN") ? std::atol(std::getenv("HDDM_SPLIT_DIAG_MIN")) : 12;
    L.split_rows = rows > split_rows_min * long(sns.size());  // long row lists
    L.split_diag = nmax > split_diag_min;
    if (env_sr) L.split_rows = std::atoi(env_sr) != 0;
    if (env_sd) L.split_diag = std::atoi(env_sd) != 0;
    if (L.split_rows || L.split_diag)
      for (int Rg : Rs) {
        std::vector<int2> g;
        for (int s : sns)
          for (int i = 0; i < Y.sn[s].n; i += Rg) g.push_back(make_int2(s, i));
        L.groups[Rg] = std::make_pair(int(g.size()), upload(g));
      }
    plan.bwd.push_back(L);
  }
}

// ----------------------------------------------------------------- factorization
void hddm_engine::factorize() {
  const auto t0 = now_ms();
  const int naent = int(Y.aent_i.size());
  // matrix entries per class in front coordinates (assemble, discretize.cpp:131-158)
  std::vector<cplx> aval(size_t(ncls) * naent);
  const double ih2 = 1.0 / (S.h * S.h);
  using cd = std::complex<double>;
  for (int c = 0; c < ncls; ++c) {
    const int t = S.cls_rep[c];
    const Sub& sb = S.subs[t];
    const WinOp& w = S.subop[t];
    auto C = [](const std::vector<double>& v, int k) { return cd(v[2 * k], v[2 * k + 1]); };
    for (int e = 0; e < naent; ++e) {
      const int v = Y.aent_node[e];
      const int lp = v % wnx, lq = v / wnx;
      const cd ew = C(w.a2n, lq) * C(w.ia1h, lp - 1) * ih2;
      const cd ee = C(w.a2n, lq) * C(w.ia1h, lp) * ih2;
      const cd es = C(w.a1n, lp) * C(w.ia2h, lq - 1) * ih2;
      const cd en = C(w.a1n, lp) * C(w.ia2h, lq) * ih2;
      cd val;
      switch (Y.aent_kind[e]) {
        case 0: {
          const double k2 = S.k2[size_t(sb.wy0 + lq) * S.gnx + sb.wx0 + lp];
          val = -(ew + ee + es + en) + k2 * (C(w.a1n, lp) * C(w.a2n, lq));
          break;
        }
        case 1: val = ew; break;
        case 2: val = ee; break;
        case 3: val = es; break;
        default: val = en; break;
      }
      aval[size_t(c) * naent + e] = cmk(val.real(), val.imag());
    }
  }
  cplx* d_aval = upload(aval);
  std::vector<int> aent_i = Y.aent_i, aent_j = Y.aent_j;
  int* d_ai = upload(aent_i);
  int* d_aj = upload(aent_j);
  int* d_ext = upload(Y.extadd);
  d_vals = dalloc<cplx>(size_t(ncls) * Y.nvals);
  int fmax = 0;
  for (const SnNode& a : Y.sn) fmax = std::max(fmax, a.n + int(a.rows.size()));
  if (size_t(2) * sizeof(cplx) * fmax > factor_smem_limit())
    throw ConfigErr("a frontal matrix of " + std::to_string(fmax) +
                    " rows exceeds the factorization kernel's shared scratch");
  if (nlss > 0) {
    d_lss = dalloc<cplx>(size_t(ncls) * nlss);
    d_lssc = dalloc<cplx>(size_t(ncls) * nlss);
  }
  CK(cudaMemsetAsync(d_vals, 0, size_t(ncls) * Y.nvals * sizeof(cplx), st));
  int* d_status = dalloc<int>(ncls);
  CK(cudaMemsetAsync(d_status, 0, sizeof(int) * ncls, st));
  // class batches bounded by ~8 GB of front workspace
  const size_t per = size_t(Y.front_words) * sizeof(cplx);
  const int batch = std::max(1, int(std::min<size_t>(ncls, (size_t(8) << 30) / per)));
  cplx* d_front = dalloc<cplx>(size_t(batch) * Y.front_words);
  // nodes by height
  std::vector<std::vector<int>> lev(Y.max_height + 1);
  for (size_t s = 0; s < Y.sn.size(); ++s) lev[Y.sn[s].height].push_back(int(s));
  std::vector<int*> d_lev;
  for (auto& l : lev) d_lev.push_back(upload(l));
  for (int c0 = 0; c0 < ncls; c0 += batch) {
    const int nb = std::min(batch, ncls - c0);
    FactorArgs A;
    A.sn = d_sn;
    A.blk = d_blk;
    A.row_first = d_row_first;
    A.row_off = d_row_off;
    A.extadd = d_ext;
    A.aent_i = d_ai;
    A.aent_j = d_aj;
    A.aval = d_aval + size_t(c0) * naent;
    A.naent = naent;
    A.front = d_front;
    A.front_words = Y.front_words;
    A.vals = d_vals + size_t(c0) * Y.nvals;
    A.nvals = Y.nvals;
    A.lss = d_lss ? d_lss + size_t(c0) * nlss : nullptr;
    A.lssc = d_lssc ? d_lssc + size_t(c0) * nlss : nullptr;
    A.lss_off = d_lss_off;
    A.nlss = nlss;
    A.status = d_status + c0;
    for (size_t h = 0; h < lev.size(); ++h)
      if (!lev[h].empty()) launch_factor_level(A, d_lev[h], int(lev[h].size()), nb, fmax, st);
    CK(cudaGetLastError());
  }
  std::vector<int> status(ncls);
  CK(cudaMemcpyAsync(status.data(), d_status, sizeof(int) * ncls, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c = 0; c < ncls; ++c)
    if (status[c]) throw SolveErr("LDL^T breakdown (zero pivot); no LU fallback on the GPU path");
  for (int* p : d_lev) dfree(p);
  dfree(d_front);
  dfree(d_aval);
  dfree(d_ai);
  dfree(d_aj);
  dfree(d_ext);
  dfree(d_status);
  factor_ms = now_ms() - t0;
}

SolveArgs hddm_engine::solve_args(const cplx* Bp, cplx* X, cplx* Yp, const int* flag, int on) {
  SolveArgs A;
  A.sn = d_sn;
  A.blk = d_blk;
  A.row_first = d_row_first;
  A.row_off = d_row_off;
  A.run_off = d_run_off;
  A.seg_ptr = d_seg_ptr;
  A.seg = d_seg;
  A.bw_ptr = d_bw_ptr;
  A.bw = d_bw;
  A.bw_cnt = d_bw_cnt;
  A.vals = d_vals;
  A.nvals = Y.nvals;
  A.lss = d_lss;
  A.lssc = d_lssc;
  A.lss_off = d_lss_off;
  A.nlss = nlss;
  A.flag = flag;
  A.flag_on = on;
  A.sparse_rhs = 0;
  A.sn_live = nullptr;
  A.B = Bp;
  A.X = X;
  A.Y = Yp;
  A.vm = vmap();
  A.nw = nw;
  A.nring = Y.nring;
  return A;
}

// probe solve per class (Factorization::factor, sparse.cpp:215-235)
void hddm_engine::run_probe() {
  std::vector<cplx> bnat(nw);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  auto next = [&s] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return double(s >> 11) * 0x1.0p-52 - 1.0;
  };
  for (int i = 0; i < nw; ++i) {
    const double re = next();
    bnat[i] = cmk(re, next());
  }
  std::vector<cplx> bfo(nw);
  for (int k = 0; k < nw; ++k) bfo[k] = bnat[Y.perm[k]];
  std::vector<int> zc(nsub, 1), aptr(ncls + 1), alist(ncls);
  for (int c = 0; c < ncls; ++c) {
    const int t = S.cls_rep[c];
    zc[t] = 0;
    aptr[c] = c;
    alist[c] = t;
    put_vec(d_B, t, bfo.data(), st);
  }
  aptr[ncls] = ncls;
  CK(cudaMemcpyAsync(d_Z[0], zc.data(), sizeof(int) * nsub, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_act_ptr, aptr.data(), sizeof(int) * (ncls + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_act_list, alist.data(), sizeof(int) * ncls, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  enqueue_solve(solve_args(d_B, d_U[0], d_Y, d_Z[0], 0), st);
  CK(cudaMemsetAsync(d_refine, 0, sizeof(int), st));
  CK(cudaMemsetAsync(d_maxrel, 0, sizeof(double), st));
  host_refine(d_B, d_U[0], d_Z[0]);
  CK(cudaGetLastError());
  std::vector<double> rel(nsub);
  CK(cudaMemcpyAsync(rel.data(), d_relcur, sizeof(double) * nsub, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  probe.assign(ncls, 0);
  for (int c = 0; c < ncls; ++c) {
    probe[c] = rel[S.cls_rep[c]];
    if (!(probe[c] <= 1e-10))
      throw SolveErr("LDL^T probe residual above 1e-10 (class " + std::to_string(c) +
                     "); no LU fallback on the GPU path");
  }
}

// ----------------------------------------------------------------- DDM step
StepArgs hddm_engine::step_args(int s, const cplx* f) {
  StepArgs A;
  A.n1 = S.n1;
  A.n2 = S.n2;
  A.nsub = nsub;
  A.nov = S.nov;
  A.gnx = S.gnx;
  A.gny = S.gny;
  A.wnx = wnx;
  A.wny = wny;
  A.nw = nw;
  A.nring = Y.nring;
  A.mcx = S.mcx;
  A.mcy = S.mcy;
  A.npatch = npatch;
  A.pnode = d_pnode;
  A.pmask = d_pmask;
  A.xfer_pos = d_xfer_pos;
  A.xfer_beta = d_xfer_beta;
  A.xblk = d_xblk;
  A.nxblk = nxblk;
  A.k2c = d_k2c;
  A.ih2 = 1.0 / (S.h * S.h);
  A.sub = d_sub;
  A.sa = d_sa;
  A.sa_stride = sa_stride;
  A.wx = d_wx;
  A.wy = d_wy;
  A.k2 = d_k2;
  A.perm = d_perm;
  A.pinv = d_pinv;
  A.f = f;
  A.fany = d_fany;
  A.zc = d_Z[s % 3];
  A.zp1 = d_Z[(s + 2) % 3];
  A.zp2 = d_Z[(s + 1) % 3];
  A.vm = vmap();
  A.B = d_B;
  A.Ucur = d_U[s % 3];
  A.Up1 = d_U[(s + 2) % 3];
  A.Up2 = d_U[(s + 1) % 3];
  A.asmb = d_asm;
  A.colcov = d_colcov;
  A.rowcov = d_rowcov;
  A.step = s;
  A.cls_ptr = d_cls_ptr;
  A.cls_mem = d_cls_mem;
  A.act_ptr = d_act_ptr;
  A.act_list = d_act_list;
  A.counts = d_counts;
  A.owned = d_owned;
  return A;
}

__global__ void k_fill_int(int* p, int v, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

void hddm_engine::fill_flags(int* p, int v, int n) {
  k_fill_int<<<(n + 255) / 256, 256, 0, st>>>(p, v, n);
}

// reset_state, ddm.cpp:152-157
void hddm_engine::reset_state() {
  for (int k = 0; k < 3; ++k) fill_flags(d_Z[k], 1, nsub);
  CK(cudaMemsetAsync(d_asm, 0, ng * sizeof(cplx), st));
  last_step = 0;
}

CheckArgs hddm_engine::check_args(const cplx* Bp, const cplx* X, const int* zc,
                                  const int* only, bool sparse_b) {
  CheckArgs C;
  C.bmask = sparse_b ? d_bmask : nullptr;
  C.nw = nw;
  C.wnx = wnx;
  C.wny = wny;
  C.gnx = S.gnx;
  C.nring = Y.nring;
  C.ih2 = 1.0 / (S.h * S.h);
  C.sub = d_sub;
  C.sa = d_sa;
  C.sa_stride = sa_stride;
  C.k2 = d_k2;
  C.perm = d_perm;
  C.pinv = d_pinv;
  C.zc = zc;
  C.only = only;
  C.lpq = d_lpq;
  C.nbr = d_nbr;
  C.k2c = d_k2c;
  C.ctab = d_ctab;
  C.ctab_off = d_ctab_off;
  C.nsub = nsub;
  C.vm = vmap();
  C.B = Bp;
  C.X = X;
  C.part = d_part_chk;
  C.nchunk = nchunk;
  C.rel = d_rel;
  C.refine_flag = d_refine;
  C.max_rel = d_maxrel;
  return C;
}

RefineArgs hddm_engine::refine_args(const cplx* Bp, cplx* X, const int* zc,
                                    unsigned long long cond) {
  RefineArgs R;
  R.nsub = nsub;
  R.ncls = ncls;
  R.nw = nw;
  R.wnx = wnx;
  R.wny = wny;
  R.gnx = S.gnx;
  R.nchunk = nchunk;
  R.ih2 = 1.0 / (S.h * S.h);
  R.sub = d_sub;
  R.sa = d_sa;
  R.sa_stride = sa_stride;
  R.k2 = d_k2;
  R.perm = d_perm;
  R.pinv = d_pinv;
  R.zc = zc;
  R.lpq = d_lpq;
  R.nbr = d_nbr;
  R.k2c = d_k2c;
  R.vm = vmap();
  R.B = Bp;
  R.X = X;
  R.R = d_R;
  R.C = d_C;
  R.part = d_part_chk;
  R.rel_cur = d_relcur;
  R.need = d_need;
  R.ncorr = d_ncorr;
  R.undo = d_undo;
  R.any = d_any;
  R.nfix = d_nfix;
  R.cls_ptr = d_cls_ptr;
  R.cls_mem = d_cls_mem;
  R.act_ptr = d_act_ptr;
  R.act_list = d_act_list;
  R.cond = cond;
  return R;
}

// One DDM iteration, DdmEngine::sweep (ddm.cpp:174-214), up to the first
// refine pass: flags -> RHS assembly -> batched solves -> residual check.
void hddm_engine::enqueue_step_front(int s, cudaStream_t stream, unsigned long long cond) {
  const StepArgs A = step_args(s, d_f);
  // HDDM_STEP_SKIP (profiling aid, results invalid): 1 flags, 2 gather, 4 check, 8 accumulate
  static const int sskip = profiling_env("HDDM_STEP_SKIP") ? std::atoi(profiling_env("HDDM_STEP_SKIP")) : 0;
  if (!(sskip & 1)) launch_flags(A, ncls, stream);
  if (!(sskip & 2)) launch_gather(A, stream);
  static const bool no_solve = profiling_env("HDDM_STEP_NOSOLVE") != nullptr;  // profiling aid
  SolveArgs SA = solve_args(d_B, A.Ucur, d_Y, A.zc, 0);
  if (s >= 2 && plan.has_sparse) {  // RHS nonzero only on the transfer patches
    // skipped subtrees read as z = 0 in the backward (zval), so X need not be
    // cleared (HDDM_CLEAR_X: clear it anyway, A/B timing aid)
    static const bool clear_x = std::getenv("HDDM_CLEAR_X") != nullptr;
    if (clear_x) CK(cudaMemsetAsync(A.Ucur, 0, size_t(nsub) * nw * sizeof(cplx), stream));
    SA.sparse_rhs = 1;
  }
  // steps >= 2: B is exactly zero off the transfer patches (cleared at step 2, only the
  // patches rewritten since), so the check reads B there only
  const CheckArgs C = check_args(d_B, A.Ucur, A.zc, nullptr, s >= 2);
  if (no_solve) {
    if (!(sskip & 4)) launch_check(C, stream);
  } else if (sskip & 4) {
    enqueue_solve(SA, stream, nullptr);
  } else {
    // each group's check runs behind its own solve; the statistics after the join
    enqueue_solve(SA, stream, &C);
    launch_finish_init(C, refine_args(d_B, A.Ucur, A.zc, cond), d_done, stream);
  }
}

// The batched solve on `stream`. On the engine stream, every class runs its
// level chain on its own forked stream (classes overlap; a class's vectors stay
// L2-resident between its consecutive levels), joined afterwards.
void hddm_engine::enqueue_solve(const SolveArgs& SA, cudaStream_t stream, const CheckArgs* check) {
  const int nt = int(plan.groups.size());
  if (!per_class_streams || nt == 1 || (stream != st && stream != st2)) {
    for (int g = 0; g < nt; ++g) launch_solve_group(SA, plan, g, stream);
    if (check)
      for (int g = 0; g < nt; ++g) launch_check_tiles(*check, plan.groups[g], stream);
    return;
  }
  // one stream set per origin stream: st (step front) and st2 (the refinement
  // body, captured while st's capture is open)
  ForkSet& F = stream == st ? fork_main : fork_body;
  if (F.st.empty()) {
    F.st.resize(nt);
    F.ev.resize(nt);
    for (int g = 0; g < nt; ++g) {
      CK(cudaStreamCreateWithFlags(&F.st[g], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&F.ev[g], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&F.fork, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(F.fork, stream));
  for (int g = 0; g < nt; ++g) {
    CK(cudaStreamWaitEvent(F.st[g], F.fork, 0));
    launch_solve_group(SA, plan, g, F.st[g]);
    if (check) launch_check_tiles(*check, plan.groups[g], F.st[g]);
    CK(cudaEventRecord(F.ev[g], F.st[g]));
  }
  for (int g = 0; g < nt; ++g) CK(cudaStreamWaitEvent(stream, F.ev[g], 0));
}

// One correction pass of refine for every RHS still above 1e-11.
void hddm_engine::enqueue_refine_body(int s, cudaStream_t stream, unsigned long long cond) {
  const StepArgs A = step_args(s, d_f);
  const RefineArgs R = refine_args(d_B, A.Ucur, A.zc, cond);
  launch_refine_prep(R, stream);
  enqueue_solve(solve_args(d_R, d_C, d_Y, d_need, 1), stream);
  launch_refine_apply(R, stream);
  launch_check_partials(check_args(d_B, A.Ucur, A.zc, d_need, s >= 2), stream);
  launch_refine_decide(R, stream);
  launch_refine_undo(R, stream);
}

// step graph variants: 0 = step 1, 4 = step 2 (clears B), 1..3 = steps >= 3 by
// s mod 3 (the rotation of the U / zero-flag buffers)
static int variant_of(int s) { return s == 1 ? 0 : (s == 2 ? 4 : 1 + (s % 3)); }
static int rep_step(int v) { return v == 0 ? 1 : (v == 1 ? 3 : (v == 2 ? 4 : (v == 3 ? 5 : 2))); }

// One DDM step (flags, RHS, solve + first residual check, the refinement WHILE node,
// accumulate) captured onto st, which must be capturing into graph g. Returns the
// number of kernels the step launches when no correction pass runs.
int hddm_engine::capture_step(int s, cudaGraph_t g) {
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
  enqueue_step_front(s, st, (unsigned long long)h);
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, g, deps, nd, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(st, &wn, 1, cudaStreamSetCaptureDependencies));
  CK(cudaStreamBeginCaptureToGraph(st2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  enqueue_refine_body(s, st2, (unsigned long long)h);
  cudaGraph_t bout;
  CK(cudaStreamEndCapture(st2, &bout));
  launch_accumulate(step_args(s, d_f), st);
  // flags, RHS (base + transfer at step 1; after it B is cleared by a memset),
  // the solve, check + finish/refine-init, accumulate
  return 1 + (s == 1 ? 2 : 1) + solve_launches() + 2 + 1;
}

void hddm_engine::build_step_graph(int v) {
  const int s = rep_step(v);
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  CK(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  step_kernels[v] = capture_step(s, g);
  cudaGraph_t gout;
  CK(cudaStreamEndCapture(st, &gout));
  CK(cudaGraphInstantiate(&step_exec[v], g, 0));
  CK(cudaGraphDestroy(g));
}

void hddm_engine::run_step(int s) {
  if (!step_exec[0] && !std::getenv("HDDM_NO_GRAPHS"))
    for (int v = 0; v < 5; ++v) build_step_graph(v);  // all variants up front
  static const bool no_graphs = std::getenv("HDDM_NO_GRAPHS") != nullptr;
  if (no_graphs) {
    // direct launches (profiling aid): same kernels, refinement driven from the host
    enqueue_step_front(s, st, 0);
    const StepArgs A = step_args(s, d_f);
    for (int it = 0; it < 13; ++it) {
      int any = 0;
      CK(cudaMemcpyAsync(&any, d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (!any) break;
      enqueue_refine_body(s, st, 0);
    }
    launch_accumulate(A, st);
    launches += 1 + (s == 1 ? 2 : 1) + solve_launches() + 2 + 1;
    last_step = s;
    return;
  }
  const int v = variant_of(s);
  if (!step_exec[v]) build_step_graph(v);
  CK(cudaGraphLaunch(step_exec[v], st));
  launches += step_kernels[v];
  last_step = s;
}

// Host-driven refinement (setup-time probe and class-solve taps).
void hddm_engine::host_refine(const cplx* Bp, cplx* X, const int* zc) {
  const RefineArgs R = refine_args(Bp, X, zc, 0);
  launch_check_init(check_args(Bp, X, zc, nullptr), R, d_done, st);
  for (int it = 0; it < 13; ++it) {
    int any = 0;
    CK(cudaMemcpyAsync(&any, d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!any) break;
    launch_refine_prep(R, st);
    enqueue_solve(solve_args(d_R, d_C, d_Y, d_need, 1), st);
    launch_refine_apply(R, st);
    launch_check_partials(check_args(Bp, X, zc, d_need), st);
    launch_refine_decide(R, st);
    launch_refine_undo(R, st);
  }
}

double hddm_engine::device_norm(const cplx* v) {
  launch_nrm2_part(v, ng, d_part, st);
  launch_finish_sum(d_part, 1, d_scal, st);
  CK(cudaMemcpyAsync(h_scal, d_scal, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return std::sqrt(h_scal[0]);
}

void hddm_engine::ensure_krylov(int m) {
  if (kry_m >= m) return;
  for (cplx* p : V) dfree(p);
  for (cplx* p : Z) dfree(p);
  V.clear();
  Z.clear();
  for (int i = 0; i <= m; ++i) V.push_back(dalloc<cplx>(ng));
  for (int i = 0; i < m; ++i) Z.push_back(dalloc<cplx>(ng));
  if (d_Zptr) dfree(d_Zptr);
  d_Zptr = dalloc<cplx*>(m);
  CK(cudaMemcpyAsync(d_Zptr, Z.data(), sizeof(cplx*) * m, cudaMemcpyHostToDevice, st));
  if (d_Vptr) dfree(d_Vptr);
  d_Vptr = dalloc<cplx*>(m + 1);
  CK(cudaMemcpyAsync(d_Vptr, V.data(), sizeof(cplx*) * (m + 1), cudaMemcpyHostToDevice, st));
  if (!d_ks) d_ks = dalloc<KryState>(1);
  if (kry_exec) {  // the cycle graph holds the old buffers
    CK(cudaGraphExecDestroy(kry_exec));
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
  CK(cudaStreamSynchronize(st));
}

KryArgs hddm_engine::kry_args(unsigned long long cond) {
  KryArgs K;
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

// One Arnoldi iteration of fgmres (krylov.cpp:57-109) with the column index j on the
// device: Z_j = M(V_j) (K DDM steps), w = A Z_j, modified Gram-Schmidt (unrolled to
// the cycle length; steps beyond j exit at once), Givens, V_{j+1} = w / hlast.
// body != null: captured into that graph (step graphs inline); else launched
// directly (HDDM_NO_GRAPHS profiling path). Returns the kernels one iteration runs.
int hddm_engine::enqueue_kry_iteration(int K, unsigned long long cond, cudaGraph_t body) {
  const KryArgs KA = kry_args(cond);
  int nk = 0;
  reset_state();
  nk += 3;
  launch_kry_load(KA, d_f, st);
  launch_fany(step_args(1, d_f), st);
  nk += 2;
  for (int s = 1; s <= K; ++s) {
    if (body) {
      nk += capture_step(s, body);
    } else {
      run_step(s);
      if (hook) hook(hook_user, 1, s);  // halo exchange of a sharded run
    }
  }
  if (!body && hook) hook(hook_user, 2, K);  // sum of the ranks' assembled fields
  launch_kry_store(KA, d_asm, st);
  GlobalArgs G{S.gnx, S.gny, 1.0 / (S.h * S.h), d_ga, d_k2};
  launch_apply_global_ind(G, d_Zptr, 0, d_Vptr, 1, &d_ks->j, st);
  launch_kry_first_dot(KA, st);
  nk += 4;
  for (int i = 0; i < kry_m; ++i) launch_kry_mgs(KA, i, st);
  nk += 2 * kry_m;
  launch_kry_givens(KA, st);
  launch_kry_next(KA, st);
  nk += 3;
  return nk;
}

void hddm_engine::build_kry_graph(int K) {
  if (kry_exec) {
    CK(cudaGraphExecDestroy(kry_exec));
    kry_exec = nullptr;
  }
  cudaGraph_t G;
  CK(cudaGraphCreate(&G, 0));
  cudaGraphConditionalHandle hc;
  CK(cudaGraphConditionalHandleCreate(&hc, G, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, G, nullptr, 0, &cp));
  cudaGraph_t B = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(st, B, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  kry_iter_kernels = enqueue_kry_iteration(K, (unsigned long long)hc, B);
  cudaGraph_t out;
  CK(cudaStreamEndCapture(st, &out));
  CK(cudaGraphInstantiate(&kry_exec, G, 0));
  CK(cudaGraphDestroy(G));
  kry_K = K;
}

// The Arnoldi iterations of one restart cycle (state in d_ks, set by the caller).
void hddm_engine::launch_kry_cycle(int K, int m) {
  (void)m;
  static const bool no_graphs = std::getenv("HDDM_NO_GRAPHS") != nullptr;
  if (no_graphs || hook) {  // host-driven (profiling, sharded runs): one sync per iteration
    for (;;) {
      enqueue_kry_iteration(K, 0, nullptr);
      CK(cudaMemcpyAsync(h_ks, d_ks, sizeof(KryState), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      launches += 6 + 2 * kry_m;
      if (!h_ks->adv) break;
    }
    return;
  }
  if (!kry_exec || kry_K != K) build_kry_graph(K);
  CK(cudaGraphLaunch(kry_exec, st));
}

// ----------------------------------------------------------------- C-ABI
namespace {

template <class F>
int guarded(hddm_engine* e, F&& fn) {
  try {
    if (e) CK(cudaSetDevice(e->dev));
    fn();
    return HDDM_OK;
  } catch (const ConfigErr& x) {
    (e ? e->err : g_err) = x.what();
    return HDDM_ERR_CONFIG;
  } catch (const SolveErr& x) {
    (e ? e->err : g_err) = x.what();
    return HDDM_ERR_SOLVE;
  } catch (const std::exception& x) {
    (e ? e->err : g_err) = x.what();
    return HDDM_ERR_OTHER;
  }
}

const cplx* in_ptr(hddm_engine* e, const double* p, int memkind, cplx* stage) {
  if (memkind == HDDM_DEVICE) return reinterpret_cast<const cplx*>(p);
  CK(cudaMemcpyAsync(stage, p, e->ng * sizeof(cplx), cudaMemcpyHostToDevice, e->st));
  return stage;
}

void out_copy(hddm_engine* e, double* p, const cplx* src, int memkind) {
  if (memkind == HDDM_DEVICE) {
    if (reinterpret_cast<const cplx*>(p) != src)
      CK(cudaMemcpyAsync(p, src, e->ng * sizeof(cplx), cudaMemcpyDeviceToDevice, e->st));
  } else {
    CK(cudaMemcpyAsync(p, src, e->ng * sizeof(cplx), cudaMemcpyDeviceToHost, e->st));
  }
}

void read_counts(hddm_engine* e, long long* c) {
  CK(cudaMemcpyAsync(c, e->d_counts, 2 * sizeof(long long), cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
}

void check_refine(hddm_engine* e) {
  int flag = 0;
  double mx = 0;
  CK(cudaMemcpyAsync(&flag, e->d_refine, sizeof(int), cudaMemcpyDeviceToHost, e->st));
  CK(cudaMemcpyAsync(&mx, e->d_maxrel, sizeof(double), cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  e->last_max_rel = mx;
  e->last_refine_count = flag;  // solves whose first pass exceeded 1e-11 (corrected on device)
}

}  // namespace

extern "C" {

const char* hddm_last_error(const hddm_engine* e) { return e ? e->err.c_str() : g_err.c_str(); }

int hddm_create(const hddm_problem* p, hddm_engine** out) {
  *out = nullptr;
  auto e = std::make_unique<hddm_engine>();
  const int rc = guarded(nullptr, [&] { e->create(*p); });
  if (rc == HDDM_OK) *out = e.release();
  return rc;
}

void hddm_destroy(hddm_engine* e) { delete e; }

long hddm_n_global(const hddm_engine* e) { return long(e->ng); }
double hddm_sigma0(const hddm_engine* e) { return e->S.sigma0; }
double hddm_factor_ms(const hddm_engine* e) { return e->factor_ms; }
int hddm_num_subdomains(const hddm_engine* e) { return e->nsub; }
int hddm_num_classes(const hddm_engine* e) { return e->ncls; }
int hddm_class_of(const hddm_engine* e, int t) {
  return t >= 0 && t < e->nsub ? e->S.subs[t].cls : -1;
}

int hddm_class_info(const hddm_engine* e, int c, int* members, long* nnz, double* probe,
                    int* is_ldlt) {
  if (c < 0 || c >= e->ncls) return HDDM_ERR_CONFIG;
  *members = e->S.cls_ptr[c + 1] - e->S.cls_ptr[c];
  *nnz = long(e->Y.nnz_ref);
  *probe = e->probe[c];
  *is_ldlt = 1;
  return HDDM_OK;
}

int hddm_window_dims(const hddm_engine* e, int* nx, int* ny) {
  *nx = e->wnx;
  *ny = e->wny;
  return HDDM_OK;
}

int hddm_nd_order(int nx, int ny, int* order) {
  const std::vector<int> o = nd_order(nx, ny);
  std::copy(o.begin(), o.end(), order);
  return HDDM_OK;
}

int hddm_symbolic_stats(int nx, int ny, long* nnz_ref, long* stored, int* nsuper,
                        int* height) {
  return guarded(nullptr, [&] {
    Symbolic S;
    build_symbolic(nx, ny, S);
    *nnz_ref = long(S.nnz_ref);
    *stored = long(S.nnz_stored);
    *nsuper = int(S.sn.size());
    *height = S.max_height;
  });
}

int hddm_footprint(const hddm_engine* e, long* stored, long* ref_nnz, long* device_bytes) {
  *stored = long(e->Y.nvals);
  *ref_nnz = long(e->Y.nnz_ref);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  *device_bytes = long(total_b - free_b);
  return HDDM_OK;
}

int hddm_apply_global(hddm_engine* e, const double* u, double* out, int memkind) {
  return guarded(e, [&] {
    const cplx* du = in_ptr(e, u, memkind, e->d_f);
    GlobalArgs G{e->S.gnx, e->S.gny, 1.0 / (e->S.h * e->S.h), e->d_ga, e->d_k2};
    cplx* dst = memkind == HDDM_DEVICE ? reinterpret_cast<cplx*>(out) : e->d_tmp;
    launch_apply_global(G, du, dst, nullptr, nullptr, e->st);
    if (memkind != HDDM_DEVICE) out_copy(e, out, dst, memkind);
    CK(cudaStreamSynchronize(e->st));
  });
}

int hddm_solve_iterative(hddm_engine* e, const double* f, double tol, int max_steps,
                         int check_every, double* out, int memkind, hddm_stats* stats,
                         int* hist_step, double* hist_rel, double* hist_ms, int hist_cap,
                         int* hist_len) {
  return guarded(e, [&] {
    if (check_every < 1) check_every = 1;
    hddm_stats st{};
    st.relres = -1;
    st.factor_ms = e->factor_ms;
    const cplx* df = in_ptr(e, f, memkind, e->d_f);
    if (df != e->d_f)
      CK(cudaMemcpyAsync(e->d_f, df, e->ng * sizeof(cplx), cudaMemcpyDeviceToDevice, e->st));
    df = e->d_f;
    const double bnorm = e->device_norm(df);
    int nh = 0;
    e->reset_state();
    CK(cudaMemsetAsync(e->d_counts, 0, 2 * sizeof(long long), e->st));
    CK(cudaMemsetAsync(e->d_refine, 0, sizeof(int), e->st));
    CK(cudaMemsetAsync(e->d_maxrel, 0, sizeof(double), e->st));
    if (bnorm == 0) {
      st.converged = 1;
      st.relres = 0;
      CK(cudaMemsetAsync(e->d_asm, 0, e->ng * sizeof(cplx), e->st));
    } else {
      StepArgs A0 = e->step_args(1, df);
      launch_fany(A0, e->st);
      GlobalArgs G{e->S.gnx, e->S.gny, 1.0 / (e->S.h * e->S.h), e->d_ga, e->d_k2};
      for (int s = 1; s <= max_steps; ++s) {
        const double t0 = now_ms();
        e->run_step(s);
        st.steps = s;
        if (s % check_every == 0 || s == max_steps) {
          // residual_norm, ddm.cpp:237-242
          launch_apply_global(G, e->d_asm, nullptr, df, e->d_part, e->st);
          launch_finish_sum(e->d_part, 1, e->d_scal, e->st);
          CK(cudaMemcpyAsync(e->h_scal, e->d_scal, sizeof(double), cudaMemcpyDeviceToHost, e->st));
          CK(cudaStreamSynchronize(e->st));
          const double rel = std::sqrt(e->h_scal[0]) / bnorm;
          const double ms = now_ms() - t0;
          if (nh < hist_cap) {
            if (hist_step) hist_step[nh] = s;
            if (hist_rel) hist_rel[nh] = rel;
            if (hist_ms) hist_ms[nh] = ms;
          }
          ++nh;
          st.sweep_ms += ms;
          st.relres = rel;
          if (rel <= tol) {
            st.converged = 1;
            break;
          }
        } else {
          st.sweep_ms += now_ms() - t0;
        }
      }
    }
    out_copy(e, out, e->d_asm, memkind);
    long long cnt[2];
    read_counts(e, cnt);
    check_refine(e);
    st.solves = long(cnt[0]);
    st.skipped = long(cnt[1]);
    if (hist_len) *hist_len = nh;
    if (stats) *stats = st;
  });
}

int hddm_precondition(hddm_engine* e, const double* r, double* z, int ksteps, int memkind,
                      hddm_stats* stats) {
  return guarded(e, [&] {
    const cplx* dr = in_ptr(e, r, memkind, e->d_f);
    if (dr != e->d_f)
      CK(cudaMemcpyAsync(e->d_f, dr, e->ng * sizeof(cplx), cudaMemcpyDeviceToDevice, e->st));
    dr = e->d_f;
    const double t0 = now_ms();
    e->reset_state();
    CK(cudaMemsetAsync(e->d_counts, 0, 2 * sizeof(long long), e->st));
    CK(cudaMemsetAsync(e->d_refine, 0, sizeof(int), e->st));
    CK(cudaMemsetAsync(e->d_maxrel, 0, sizeof(double), e->st));
    StepArgs A0 = e->step_args(1, dr);
    launch_fany(A0, e->st);
    e->launches += 4;  // 3 flag fills + fany
    for (int s = 1; s <= ksteps; ++s) e->run_step(s);
    out_copy(e, z, e->d_asm, memkind);
    long long cnt[2];
    read_counts(e, cnt);
    check_refine(e);
    if (stats) {
      stats->solves += long(cnt[0]);
      stats->skipped += long(cnt[1]);
      stats->sweep_ms += now_ms() - t0;
      stats->factor_ms = e->factor_ms;
    }
  });
}

int hddm_fgmres(hddm_engine* e, const double* b, double* x, double tol, int max_iters,
                int restart, int ksteps, int memkind, hddm_fgmres_result* res, double* hist,
                int hist_cap, hddm_stats* pstats) {
  return guarded(e, [&] {
    const double tstart = now_ms();
    hddm_fgmres_result R{};
    R.relres = R.true_relres = -1;
    const long long n = e->ng;
    int mcap = restart > 0 ? restart : max_iters;
    if (mcap < 1) mcap = 1;
    e->ensure_krylov(mcap);
    // the workspace (and the cycle graph) may be wider than this call needs: H column j
    // is d_H[j*ld + i] with the workspace's leading dimension
    const int ld = e->kry_m + 1;
    cudaStream_t st = e->st;
    CK(cudaMemcpyAsync(e->d_b, b, n * sizeof(cplx),
                       memkind == HDDM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(e->d_x, 0, n * sizeof(cplx), st));
    CK(cudaMemsetAsync(e->d_refine, 0, sizeof(int), st));
    CK(cudaMemsetAsync(e->d_maxrel, 0, sizeof(double), st));
    CK(cudaMemsetAsync(e->d_counts, 0, 2 * sizeof(long long), st));
    const double bnorm = e->device_norm(e->d_b);
    GlobalArgs G{e->S.gnx, e->S.gny, 1.0 / (e->S.h * e->S.h), e->d_ga, e->d_k2};
    double sweep_ms = 0;
    e->kry_k_last = 0;
    if (e->d_hist_cap < max_iters) {  // the cycle graph holds the old buffer
      if (e->d_hist) e->dfree(e->d_hist);
      e->d_hist_cap = std::max(max_iters, 256);
      e->d_hist = e->dalloc<double>(e->d_hist_cap);
      if (e->kry_exec) {
        CK(cudaGraphExecDestroy(e->kry_exec));
        e->kry_exec = nullptr;
      }
    }
    if (bnorm == 0) {
      R.converged = 1;
      R.relres = R.true_relres = 0;
    } else {
      CK(cudaMemcpyAsync(e->d_r, e->d_b, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
      KryState ks{};
      ks.total = 0;
      ks.max_iters = max_iters;
      ks.tol = tol;
      ks.bnorm = bnorm;
      while (!ks.stop && ks.total < max_iters) {
        const int m = restart > 0 ? std::min(restart, max_iters - ks.total) : max_iters - ks.total;
        const double rnorm = e->device_norm(e->d_r);
        if (rnorm == 0) {
          ks.converged = 1;
          break;
        }
        // one restart cycle: V_0 = r / |r|, g = |r| e_0, then the Arnoldi iterations
        // as ONE graph launch (WHILE node, status on the device); the host reads the
        // cycle's status record once (krylov.cpp:53-109)
        e->h_scal[8] = rnorm;
        CK(cudaMemcpyAsync(e->d_scal + 8, e->h_scal + 8, sizeof(double), cudaMemcpyHostToDevice, st));
        launch_scale_div(e->V[0], e->d_r, e->d_scal + 8, n, st);
        launch_init_g(e->d_g, m, e->d_scal + 8, st);
        CK(cudaMemsetAsync(e->d_H, 0, sizeof(cplx) * size_t(e->kry_m) * ld, st));
        ks.j = 0;
        ks.m = m;
        ks.k = 0;
        ks.adv = 0;
        *e->h_ks = ks;
        CK(cudaMemcpyAsync(e->d_ks, e->h_ks, sizeof(KryState), cudaMemcpyHostToDevice, st));
        const double ts = now_ms();
        e->launch_kry_cycle(ksteps, m);
        CK(cudaMemcpyAsync(e->h_ks, e->d_ks, sizeof(KryState), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        sweep_ms += now_ms() - ts;
        const int before = ks.total;
        ks = *e->h_ks;
        if (e->kry_exec)  // iterations run by the cycle graph (a dead column runs too)
          e->launches += (long long)e->kry_iter_kernels * (ks.total - before + (ks.flags & 1));
        if (hist) {
          const int lo = std::min(before, hist_cap), hi = std::min(ks.total, hist_cap);
          if (hi > lo)
            CK(cudaMemcpy(hist + lo, e->d_hist + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToHost));
        }
        if (ks.total > before) R.relres = ks.relres;
        const int k = ks.k;
        e->kry_k_last = k;
        if (k > 0) {
          launch_backsolve(e->d_H, ld, e->d_g, e->d_y, k, st);
          launch_update_x(e->d_x, e->d_Zptr, e->d_y, k, n, st);
        }
        if (!ks.stop) {  // restart: the residual recomputed explicitly
          launch_apply_global(G, e->d_x, e->d_r, nullptr, nullptr, st);
          launch_bsub(e->d_r, e->d_b, n, st);
        }
      }
      R.iters = ks.total;
      R.converged = ks.converged;
      // true residual, krylov.cpp:126-131
      launch_apply_global(G, e->d_x, nullptr, e->d_b, e->d_part, st);
      launch_finish_sum(e->d_part, 1, e->d_scal, st);
      CK(cudaMemcpyAsync(e->h_scal, e->d_scal, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      R.true_relres = std::sqrt(e->h_scal[0]) / bnorm;
    }
    out_copy(e, x, e->d_x, memkind);
    long long cnt[2];
    read_counts(e, cnt);
    check_refine(e);
    R.wall_ms = now_ms() - tstart;
    if (res) *res = R;
    if (pstats) {
      pstats->solves += long(cnt[0]);
      pstats->skipped += long(cnt[1]);
      pstats->sweep_ms += sweep_ms;
      pstats->factor_ms = e->factor_ms;
    }
  });
}

// ---- sharded runs: one engine per rank, each solving its block of
// subdomains; the ranks exchange the solutions and zero flags of the subdomains at
// their block boundaries after every step and sum their assembled fields at the end
// (paper_1807_04180_b200/shard.py drives it over torch.distributed).
int hddm_set_owned(hddm_engine* e, const int* owned) {
  return guarded(e, [&] {
    std::vector<int> o(e->nsub, 1);
    if (owned)
      for (int t = 0; t < e->nsub; ++t) o[t] = owned[t] ? 1 : 0;
    CK(cudaMemcpyAsync(e->d_owned, o.data(), sizeof(int) * e->nsub, cudaMemcpyHostToDevice, e->st));
    CK(cudaStreamSynchronize(e->st));
  });
}

int hddm_precondition_begin(hddm_engine* e, const double* r, int memkind) {
  return guarded(e, [&] {
    const cplx* dr = in_ptr(e, r, memkind, e->d_f);
    if (dr != e->d_f)
      CK(cudaMemcpyAsync(e->d_f, dr, e->ng * sizeof(cplx), cudaMemcpyDeviceToDevice, e->st));
    e->reset_state();
    CK(cudaMemsetAsync(e->d_counts, 0, 2 * sizeof(long long), e->st));
    CK(cudaMemsetAsync(e->d_refine, 0, sizeof(int), e->st));
    CK(cudaMemsetAsync(e->d_maxrel, 0, sizeof(double), e->st));
    launch_fany(e->step_args(1, e->d_f), e->st);
  });
}

int hddm_step(hddm_engine* e, int s) {
  return guarded(e, [&] {
    if (s < 1 || s != e->last_step + 1) throw ConfigErr("steps run in order from 1 after hddm_precondition_begin");
    e->run_step(s);
  });
}

int hddm_halo_pack(hddm_engine* e, int s, const int* ts, int nts, double* buf, int* flags) {
  return guarded(e, [&] {
    if (s < 1 || s != e->last_step) throw ConfigErr("halo of a step that has not run");
    cplx* b = reinterpret_cast<cplx*>(buf);
    for (int k = 0; k < nts; ++k) {
      if (ts[k] < 0 || ts[k] >= e->nsub) throw ConfigErr("no such subdomain");
      e->get_vec(e->d_U[s % 3], ts[k], b + size_t(k) * e->nw, e->st);
      CK(cudaMemcpyAsync(flags + k, e->d_Z[s % 3] + ts[k], sizeof(int), cudaMemcpyDeviceToHost, e->st));
    }
    CK(cudaStreamSynchronize(e->st));
  });
}

int hddm_halo_unpack(hddm_engine* e, int s, const int* ts, int nts, const double* buf, const int* flags) {
  return guarded(e, [&] {
    if (s < 1 || s != e->last_step) throw ConfigErr("halo of a step that has not run");
    const cplx* b = reinterpret_cast<const cplx*>(buf);
    for (int k = 0; k < nts; ++k) {
      if (ts[k] < 0 || ts[k] >= e->nsub) throw ConfigErr("no such subdomain");
      e->put_vec(e->d_U[s % 3], ts[k], b + size_t(k) * e->nw, e->st);
      CK(cudaMemcpyAsync(e->d_Z[s % 3] + ts[k], flags + k, sizeof(int), cudaMemcpyHostToDevice, e->st));
    }
    CK(cudaStreamSynchronize(e->st));
  });
}

int hddm_set_step_hook(hddm_engine* e, hddm_step_hook fn, void* user) {
  return guarded(e, [&] {
    e->hook = fn;
    e->hook_user = user;
  });
}

int hddm_assembled(hddm_engine* e, double* buf, int write) {
  return guarded(e, [&] {
    CK(cudaMemcpyAsync(write ? static_cast<void*>(e->d_asm) : static_cast<void*>(buf),
                       write ? static_cast<const void*>(buf) : static_cast<const void*>(e->d_asm),
                       e->ng * sizeof(cplx), write ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
  });
}

int hddm_precondition_end(hddm_engine* e, double* z, int memkind, hddm_stats* stats) {
  return guarded(e, [&] {
    out_copy(e, z, e->d_asm, memkind);
    long long cnt[2];
    read_counts(e, cnt);
    check_refine(e);
    if (stats) {
      stats->solves += long(cnt[0]);
      stats->skipped += long(cnt[1]);
      stats->factor_ms = e->factor_ms;
    }
  });
}

int hddm_fgmres_z(hddm_engine* e, int j, double* out, int memkind) {
  return guarded(e, [&] {
    if (j < 0 || j >= e->kry_k_last) throw ConfigErr("no such preconditioned vector Z_j (last FGMRES cycle)");
    out_copy(e, out, e->Z[j], memkind);
    CK(cudaStreamSynchronize(e->st));
  });
}

int hddm_tap_subdomain(hddm_engine* e, int t, double* rhs, double* u, int* active) {
  return guarded(e, [&] {
    if (t < 0 || t >= e->nsub || e->last_step < 1) throw ConfigErr("no sweep to tap");
    const int s = e->last_step;
    std::vector<cplx> b(e->nw), x(e->nw);
    int z = 1;
    e->get_vec(e->d_B, t, b.data(), e->st);
    e->get_vec(e->d_U[s % 3], t, x.data(), e->st);
    CK(cudaMemcpyAsync(&z, e->d_Z[s % 3] + t, sizeof(int), cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    for (int k = 0; k < e->nw; ++k) {
      const int node = e->Y.perm[k];
      rhs[2 * node] = b[k].x;
      rhs[2 * node + 1] = b[k].y;
      u[2 * node] = x[k].x;
      u[2 * node + 1] = x[k].y;
    }
    *active = z ? 0 : 1;
  });
}

int hddm_class_solve(hddm_engine* e, int c, const double* b, double* x, double* relres) {
  return guarded(e, [&] {
    if (c < 0 || c >= e->ncls) throw ConfigErr("class index out of range");
    const int t = e->S.cls_rep[c];
    std::vector<cplx> bfo(e->nw);
    for (int k = 0; k < e->nw; ++k) {
      const int node = e->Y.perm[k];
      bfo[k] = cmk(b[2 * node], b[2 * node + 1]);
    }
    std::vector<int> zc(e->nsub, 1), aptr(e->ncls + 1, 0), alist(1, t);
    zc[t] = 0;
    for (int k = c + 1; k <= e->ncls; ++k) aptr[k] = 1;
    cudaStream_t st = e->st;
    e->put_vec(e->d_B, t, bfo.data(), st);
    CK(cudaMemcpyAsync(e->d_Z[0], zc.data(), sizeof(int) * e->nsub, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(e->d_act_ptr, aptr.data(), sizeof(int) * (e->ncls + 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(e->d_act_list, alist.data(), sizeof(int), cudaMemcpyHostToDevice, st));
    e->enqueue_solve(e->solve_args(e->d_B, e->d_U[0], e->d_Y, e->d_Z[0], 0), st);
    e->host_refine(e->d_B, e->d_U[0], e->d_Z[0]);
    std::vector<cplx> xf(e->nw);
    double rel = 0;
    e->get_vec(e->d_U[0], t, xf.data(), st);
    CK(cudaMemcpyAsync(&rel, e->d_relcur + t, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int k = 0; k < e->nw; ++k) {
      const int node = e->Y.perm[k];
      x[2 * node] = xf[k].x;
      x[2 * node + 1] = xf[k].y;
    }
    if (relres) *relres = rel;
    e->last_step = 0;
  });
}

int hddm_set_timing(hddm_engine* e, int enable) {
  return guarded(e, [&] {
    e->stage_resolve();
    e->timing = enable != 0;
    for (int k = 0; k < kStages; ++k) {
      e->stage_ms[k] = 0;
      e->stage_n[k] = 0;
    }
    e->launches = 0;
  });
}

int hddm_stage_times(hddm_engine* e, double* ms, long long* count, int cap, int* n) {
  return guarded(e, [&] {
    e->stage_resolve();
    for (int k = 0; k < kStages && k < cap; ++k) {
      ms[k] = e->stage_ms[k];
      if (count) count[k] = e->stage_n[k];
    }
    *n = kStages;
  });
}

long long hddm_launch_count(const hddm_engine* e) { return e->launches; }

const char* hddm_solver_desc(const hddm_engine* e) {
  (void)e;
  return "level-synchronous batched supernodal solve";
}

int hddm_fwd_entries(const hddm_engine* e, long long* full, long long* sparse_rhs) {
  if (!e || !full || !sparse_rhs) return 1;
  *full = e->fwd_entries_full ? e->fwd_entries_full : e->Y.nnz_stored;
  *sparse_rhs = e->plan.has_sparse ? e->fwd_entries_sparse : *full;
  return 0;
}

int hddm_time_solve(hddm_engine* e, int reps, double* ms_per_solve) {
  return guarded(e, [&] {
    // steady state: every subdomain active, right-hand sides of the last step,
    // the step graphs' per-class stream structure
    cudaStream_t st = e->st;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    set_solve_skip(profiling_env("HDDM_SKIP") ? std::atoi(profiling_env("HDDM_SKIP")) : 0,
                   profiling_env("HDDM_ONLY_TILE")
                       ? std::atoi(profiling_env("HDDM_ONLY_TILE"))
                       : (profiling_env("HDDM_ONLY_M") ? -2 - std::atoi(profiling_env("HDDM_ONLY_M")) : -1));
    // HDDM_ONLY_M=M: only the tile groups of M members (profiling aid)
    // HDDM_TIME_EMPTY: no RHS active -- every kernel exits after its setup, so
    // the time is the launch / dependency floor of the solve graph (profiling aid)
    const int on = profiling_env("HDDM_TIME_EMPTY") ? 1 : 0;
    SolveArgs SA = e->solve_args(e->d_B, e->d_C, e->d_Y, e->d_zero, on);
    // HDDM_TIME_SPARSE: the steady-state (steps >= 2) forward plan; B then holds the last
    // step's right-hand sides, which are nonzero only on the transfer patches
    if (std::getenv("HDDM_TIME_SPARSE") && e->plan.has_sparse) SA.sparse_rhs = 1;
    e->enqueue_solve(SA, st);
    set_solve_skip(0, -1);
    CK(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t x, x2 = nullptr;
    CK(cudaGraphInstantiate(&x, g, 0));
    // HDDM_TIME_PAIR (profiling aid, results invalid): two instances run
    // concurrently on two streams; the time per solve then shows how much idle
    // capacity the single solve graph leaves
    const bool pair = profiling_env("HDDM_TIME_PAIR") != nullptr;
    if (pair) CK(cudaGraphInstantiate(&x2, g, 0));
    CK(cudaGraphDestroy(g));
    CK(cudaGraphLaunch(x, st));  // warm-up
    cudaEvent_t a, b, j;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventCreate(&j));
    CK(cudaEventRecord(a, st));
    for (int r = 0; r < reps; ++r) {
      if (pair) {
        CK(cudaEventRecord(j, st));
        CK(cudaStreamWaitEvent(e->st2, j, 0));
        CK(cudaGraphLaunch(x2, e->st2));
      }
      CK(cudaGraphLaunch(x, st));
      if (pair) {
        CK(cudaEventRecord(j, e->st2));
        CK(cudaStreamWaitEvent(st, j, 0));
      }
    }
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    *ms_per_solve = ms / std::max(reps, 1) / (pair ? 2 : 1);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaEventDestroy(j);
    cudaGraphExecDestroy(x);
    if (x2) cudaGraphExecDestroy(x2);
  });
}

int hddm_solve_launches(const hddm_engine* e) { return const_cast<hddm_engine*>(e)->solve_launches(); }

int hddm_time_kernel(hddm_engine* e, int which, int reps, double* ms_per_launch) {
  return guarded(e, [&] {
    if (e->last_step < 3) throw ConfigErr("time_kernel needs a sweep sequence of at least 3 steps");
    if (which < 0 || which > 2) throw ConfigErr("time_kernel: 0 transfer, 1 residual check, 2 accumulate");
    // the state of the last step: its transfer (idempotent: rewrites the same patch
    // values), its residual check (writes scratch partials), its blend-accumulate into
    // a scratch field
    StepArgs A = e->step_args(e->last_step, e->d_f);
    A.asmb = e->d_tmp;
    const CheckArgs Cc = e->check_args(e->d_B, A.Ucur, A.zc, nullptr, true);
    auto run = [&] {
      if (which == 0)
        launch_transfer(A, e->st);
      else if (which == 1)
        launch_check_partials(Cc, e->st);
      else
        launch_accumulate(A, e->st);
    };
    run();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, e->st));
    for (int r = 0; r < std::max(reps, 1); ++r) run();
    CK(cudaEventRecord(b, e->st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    *ms_per_launch = ms / std::max(reps, 1);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int hddm_tune_fwd_shape(hddm_engine* e, int which, int level, int E) {
  return guarded(e, [&] {
    CK(cudaStreamSynchronize(e->st));
    set_fwd_shape(which, level, E);
    for (auto& g : e->step_exec)
      if (g) {
        CK(cudaGraphExecDestroy(g));
        g = nullptr;
      }
    if (e->kry_exec) {
      CK(cudaGraphExecDestroy(e->kry_exec));
      e->kry_exec = nullptr;
    }
  });
}

int hddm_refine_stats(const hddm_engine* e, double* max_local_relres, int* corrections) {
  *max_local_relres = e->last_max_rel;
  *corrections = e->last_refine_count;
  return HDDM_OK;
}

const char* hddm_stage_name(int i) { return i >= 0 && i < kStages ? kStageNames[i] : ""; }

void* hddm_stream(const hddm_engine* e) { return e->st; }

}  // extern "C"
