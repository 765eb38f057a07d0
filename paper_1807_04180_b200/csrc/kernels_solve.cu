// Batched multi-RHS supernodal triangular solves (the per-step hot path that
// replaces Factorization::solve -> solve_raw, proj/src/sparse.cpp:244-266).
//
// Level-synchronous over the nested-dissection tree: every kernel handles one
// level for ALL classes and ALL active member right-hand sides at once, one
// thread per (class, output item, member). Threads are ordered class-major,
// then item, then member, so the members of a class sharing a factor entry sit
// in the same warp (one load, broadcast), and consecutive output columns of a
// supernode read consecutive factor entries (coalesced). Each thread runs one
// short sequential dot product; hundreds of thousands of independent threads
// per level keep the memory system busy.
//
//   forward, leaves:      z_leaf = L_leaf^{-1} b_leaf              (band)
//   forward, separators:  y_r = b_r - (incoming run of row r) . z   (pull)
//                         z_s = Linv_s y_s                         (dense inverse)
//   backward, separators: w_j = z_j / D_j - sum_r L[r][j] x_r       (pull)
//                         x_s = Linv_s^T w_s
//   backward, leaves:     the same pull per leaf column, then a band
//                         back-substitution per leaf
//   ring (identity rows): x = b
// Every output has one writer and a fixed summation order: deterministic.
// Vectors are in factor order; RHS index = subdomain id, stride nw.
#include "dev.cuh"
#include "kernels.cuh"

namespace hddm {

namespace {

constexpr int kThreads = 256;

// thread -> (class c, item, RHS t); false past the end of the work list
__device__ __forceinline__ bool decode(const SolveArgs& A, int ncls, long long idx, int nitem,
                                       int& c, int& item, int& t) {
  const int* ap = A.act_ptr;
  if (idx >= (long long)ap[ncls] * nitem) return false;
  int lo = 0, hi = ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)ap[mid] * nitem <= idx) lo = mid; else hi = mid - 1;
  }
  c = lo;
  const int m = ap[c + 1] - ap[c];
  const long long r = idx - (long long)ap[c] * nitem;
  item = int(r / m);
  t = A.act_list[ap[c] + int(r - (long long)item * m)];
  return true;
}

__device__ __forceinline__ void csub_mul(cplx& acc, cplx l, cplx x) {
  acc.x -= l.x * x.x - l.y * x.y;
  acc.y -= l.x * x.y + l.y * x.x;
}

}  // namespace

// identity ring rows: x = b (thread per (class, ring position, member))
__global__ void __launch_bounds__(kThreads) k_ring(SolveArgs A, int ncls) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, A.nring, c, it, t)) return;
  const long long p = (long long)t * A.nw + it;
  A.X[p] = A.B[p];
}

// leaves, forward: z_i = b_i - sum_{q in [first_i, i)} L[i][q] z_q. The band is
// at most kBand wide (checked at setup), so the last kBand values live in a
// register window.
constexpr int kBand = 6;

__global__ void __launch_bounds__(kThreads) k_fwd_leaf(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const DevSn sn = A.sn[items[it].x];
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const cplx* b = A.B + (long long)t * A.nw + sn.c0;
  cplx* x = A.X + (long long)t * A.nw + sn.c0;
  cplx win[kBand + 1];  // win[d] = z_{i-d}
#pragma unroll
  for (int d = 0; d <= kBand; ++d) win[d] = cmk(0, 0);
  for (int i = 0; i < sn.n; ++i) {
    const int rt = sn.drow0 + i;
    const int first = A.row_first[rt];
    const cplx* L = vals + A.row_off[rt] - first;  // L[q] for q in [first, i)
    cplx acc = b[i];
#pragma unroll
    for (int d = 1; d <= kBand; ++d)
      if (i - d >= first) csub_mul(acc, ldf(L + i - d), win[d]);
#pragma unroll
    for (int d = kBand; d >= 2; --d) win[d] = win[d - 1];
    win[1] = acc;
    x[i] = acc;
  }
}

// separator rows, forward pull: Y[r] = B[r] - run(r) . X[src]
__global__ void __launch_bounds__(kThreads) k_fwd_pull(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const int2 item = items[it];
  const int pos = A.sn[item.x].c0 + item.y;
  const cplx* run = A.vals + (long long)c * A.nvals + A.run_off[pos];
  const cplx* X = A.X + (long long)t * A.nw;
  cplx acc = A.B[(long long)t * A.nw + pos];
  for (int e = A.seg_ptr[pos]; e < A.seg_ptr[pos + 1]; ++e) {
    const int2 sg = A.seg[e];
    const cplx* xs = X + sg.y;
    int j = 0;
    for (; j + 4 <= sg.x; j += 4) {
      const cplx l0 = ldf(run + j), l1 = ldf(run + j + 1), l2 = ldf(run + j + 2), l3 = ldf(run + j + 3);
      const cplx x0 = xs[j], x1 = xs[j + 1], x2 = xs[j + 2], x3 = xs[j + 3];
      csub_mul(acc, l0, x0);
      csub_mul(acc, l1, x1);
      csub_mul(acc, l2, x2);
      csub_mul(acc, l3, x3);
    }
    for (; j < sg.x; ++j) csub_mul(acc, ldf(run + j), xs[j]);
    run += sg.x;
  }
  A.Y[(long long)t * A.nw + pos] = acc;
}

// separator rows with long runs (top levels): one WARP per (class, row,
// member); lanes stride the run (coalesced), zidx gives each element's source.
__global__ void __launch_bounds__(kThreads) k_fwd_pull_warp(SolveArgs A, int ncls,
                                                            const int2* items, int nitem) {
  int c, it, t;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (!decode(A, ncls, w, nitem, c, it, t)) return;
  const int2 item = items[it];
  const int pos = A.sn[item.x].c0 + item.y;
  const long long r0 = A.run_off[pos];
  const int total = int(A.run_off[pos + 1] - r0);
  const cplx* run = A.vals + (long long)c * A.nvals + r0;
  const int* zi = A.zidx + r0;
  const cplx* X = A.X + (long long)t * A.nw;
  cplx acc0 = cmk(0, 0), acc1 = cmk(0, 0);
  int q = lane;
  for (; q + 32 < total; q += 64) {
    const cplx l0 = ldf(run + q), l1 = ldf(run + q + 32);
    const int i0 = __ldg(zi + q), i1 = __ldg(zi + q + 32);
    cfma(acc0, l0, X[i0]);
    cfma(acc1, l1, X[i1]);
  }
  if (q < total) cfma(acc0, ldf(run + q), X[__ldg(zi + q)]);
  const cplx sum = warp_sum(cadd(acc0, acc1));
  if (lane == 0) A.Y[(long long)t * A.nw + pos] = csub(A.B[(long long)t * A.nw + pos], sum);
}

// separator rows, forward diagonal: X[i] = Y[i] + sum_{j<i} Linv[i][j] Y[j]
__global__ void __launch_bounds__(kThreads) k_fwd_diag(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int i = item.y;
  const cplx* row = A.vals + (long long)c * A.nvals + sn.diag_off + (long long)i * (i - 1) / 2;
  const cplx* y = A.Y + (long long)t * A.nw + sn.c0;
  cplx acc = y[i];
  int j = 0;
  for (; j + 4 <= i; j += 4) {
    const cplx l0 = ldf(row + j), l1 = ldf(row + j + 1), l2 = ldf(row + j + 2), l3 = ldf(row + j + 3);
    cfma(acc, l0, y[j]);
    cfma(acc, l1, y[j + 1]);
    cfma(acc, l2, y[j + 2]);
    cfma(acc, l3, y[j + 3]);
  }
  for (; j < i; ++j) cfma(acc, ldf(row + j), y[j]);
  A.X[(long long)t * A.nw + sn.c0 + i] = acc;
}

// backward pull for column j of supernode s: w = Dinv[j] X[j] - sum_rows L[r][j] X[dst r]
// (dst = scratch target: Y for separators, X in place for leaves)
template <bool TO_X>
__global__ void __launch_bounds__(kThreads) k_bwd_pull(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int j = item.y;
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const cplx* X = A.X + (long long)t * A.nw;
  cplx acc = cmul(ldg(vals + sn.dinv_off + j), X[sn.c0 + j]);
  const BwRow* rows = A.bw + A.bw_ptr[item.x];
  const int nr = A.bw_ptr[item.x + 1] - A.bw_ptr[item.x];
  int k = 0;
  for (; k + 4 <= nr; k += 4) {
    BwRow d[4];
    cplx l[4], x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) d[u] = rows[k + u];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = j >= d[u].first;
      l[u] = ok ? ldf(vals + d[u].off + (j - d[u].first)) : cmk(0, 0);
      x[u] = ok ? X[d[u].dpos] : cmk(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) csub_mul(acc, l[u], x[u]);
  }
  for (; k < nr; ++k) {
    const BwRow d = rows[k];
    if (j >= d.first) csub_mul(acc, ldf(vals + d.off + (j - d.first)), X[d.dpos]);
  }
  (TO_X ? A.X : A.Y)[(long long)t * A.nw + sn.c0 + j] = acc;
}

// separator columns, backward diagonal: X[j] = Y[j] + sum_{i>j} Linv[i][j] Y[i]
__global__ void __launch_bounds__(kThreads) k_bwd_diag(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int j = item.y;
  const cplx* Linv = A.vals + (long long)c * A.nvals + sn.diag_off;
  const cplx* y = A.Y + (long long)t * A.nw + sn.c0;
  cplx acc = y[j], acc2 = cmk(0, 0);
  int i = j + 1;
  for (; i + 4 <= sn.n; i += 4) {
    const cplx l0 = ldf(Linv + (long long)i * (i - 1) / 2 + j);
    const cplx l1 = ldf(Linv + (long long)(i + 1) * i / 2 + j);
    const cplx l2 = ldf(Linv + (long long)(i + 2) * (i + 1) / 2 + j);
    const cplx l3 = ldf(Linv + (long long)(i + 3) * (i + 2) / 2 + j);
    const cplx y0 = y[i], y1 = y[i + 1], y2 = y[i + 2], y3 = y[i + 3];
    cfma(acc, l0, y0);
    cfma(acc2, l1, y1);
    cfma(acc, l2, y2);
    cfma(acc2, l3, y3);
  }
  for (; i < sn.n; ++i) cfma(acc, ldf(Linv + (long long)i * (i - 1) / 2 + j), y[i]);
  A.X[(long long)t * A.nw + sn.c0 + j] = cadd(acc, acc2);
}

// leaves, backward band back-substitution on w (held in X): for i = n-1..0:
// x_i = w_i; w_q -= L[i][q] x_i for q in [first_i, i). Register window of the
// next kBand pending w values.
__global__ void __launch_bounds__(kThreads) k_bwd_leaf(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const DevSn sn = A.sn[items[it].x];
  const cplx* vals = A.vals + (long long)c * A.nvals;
  cplx* x = A.X + (long long)t * A.nw + sn.c0;
  const int n = sn.n;
  cplx w[kBand + 1];  // w[d] = pending w_{i-d}
#pragma unroll
  for (int d = 0; d <= kBand; ++d) w[d] = (n - 1 - d >= 0) ? x[n - 1 - d] : cmk(0, 0);
  for (int i = n - 1; i >= 0; --i) {
    const cplx xi = w[0];
    x[i] = xi;
    const int rt = sn.drow0 + i;
    const int first = A.row_first[rt];
    const cplx* L = vals + A.row_off[rt] - first;
#pragma unroll
    for (int d = 1; d <= kBand; ++d)
      if (i - d >= first) csub_mul(w[d], ldf(L + i - d), xi);
#pragma unroll
    for (int d = 0; d < kBand; ++d) w[d] = w[d + 1];
    w[kBand] = (i - 1 - kBand >= 0) ? x[i - 1 - kBand] : cmk(0, 0);
  }
}

// ------------------------------------------------------------------ launcher
int solve_launch_count(const SolvePlan& P) {
  return 2 + 2 * int(P.fwd.size()) + 2 * int(P.bwd.size()) + 2;
}

static unsigned grid_for(long long work) {
  return unsigned((work + kThreads - 1) / kThreads);
}

void launch_solve(const SolveArgs& A, const SolvePlan& P, int ncls, int max_rhs,
                  cudaStream_t st) {
  k_ring<<<grid_for((long long)max_rhs * A.nring), kThreads, 0, st>>>(A, ncls);
  const SolveLevel& FL = P.fwd_leaf;
  k_fwd_leaf<<<grid_for((long long)max_rhs * FL.nitem), kThreads, 0, st>>>(A, ncls, FL.d_items,
                                                                          FL.nitem);
  for (const auto& L : P.fwd) {
    const unsigned g = grid_for((long long)max_rhs * L.nitem);
    if (L.warp_rows)
      k_fwd_pull_warp<<<grid_for((long long)max_rhs * L.nitem * 32), kThreads, 0, st>>>(
          A, ncls, L.d_items, L.nitem);
    else
      k_fwd_pull<<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
    k_fwd_diag<<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
  }
  for (const auto& L : P.bwd) {
    const unsigned g = grid_for((long long)max_rhs * L.nitem);
    k_bwd_pull<false><<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
    k_bwd_diag<<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
  }
  const SolveLevel& BC = P.bwd_leafcol;
  k_bwd_pull<true><<<grid_for((long long)max_rhs * BC.nitem), kThreads, 0, st>>>(
      A, ncls, BC.d_items, BC.nitem);
  const SolveLevel& BL = P.bwd_leaf;
  k_bwd_leaf<<<grid_for((long long)max_rhs * BL.nitem), kThreads, 0, st>>>(A, ncls, BL.d_items,
                                                                          BL.nitem);
}

}  // namespace hddm
