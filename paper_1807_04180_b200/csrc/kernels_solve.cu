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
  // act_ptr may be a per-class view (ap[0] != 0): offsets are relative to ap[0]
  const int* ap = A.act_ptr;
  const int a0 = ap[0];
  if (idx >= (long long)(ap[ncls] - a0) * nitem) return false;
  int lo = 0, hi = ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)(ap[mid] - a0) * nitem <= idx) lo = mid; else hi = mid - 1;
  }
  c = lo;
  const int m = ap[c + 1] - ap[c];
  const long long r = idx - (long long)(ap[c] - a0) * nitem;
  if (A.member_major) {  // consecutive threads: consecutive items of one RHS
    const int k = int(r / nitem);
    item = int(r - (long long)k * nitem);
    t = A.act_list[ap[c] + k];
  } else {               // consecutive threads: the members of one item
    item = int(r / m);
    t = A.act_list[ap[c] + int(r - (long long)item * m)];
  }
  return true;
}

// member-major decode: consecutive threads walk consecutive items of ONE right-
// hand side (backward sweeps: a warp covers consecutive columns, so the
// ancestor value x_r is a broadcast and the factor row a coalesced read)
__device__ __forceinline__ bool decode_mm(const SolveArgs& A, int ncls, long long idx, int nitem,
                                          int& c, int& item, int& t) {
  const int* ap = A.act_ptr;
  const int a0 = ap[0];
  if (idx >= (long long)(ap[ncls] - a0) * nitem) return false;
  int lo = 0, hi = ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)(ap[mid] - a0) * nitem <= idx) lo = mid; else hi = mid - 1;
  }
  c = lo;
  const long long r = idx - (long long)(ap[c] - a0) * nitem;
  const int k = int(r / nitem);
  item = int(r - (long long)k * nitem);
  t = A.act_list[ap[c] + k];
  return true;
}

__device__ __forceinline__ void csub_mul(cplx& acc, cplx l, cplx x) {
  acc.x -= l.x * x.x - l.y * x.y;
  acc.y -= l.x * x.y + l.y * x.x;
}

// sum_{q = start, start+step, ... < n} L[q] * X[zi[q]], software-pipelined:
// the next batch's factor values and source indices are in flight while the
// current batch's gathers are consumed.
template <int U>
__device__ __forceinline__ cplx gather_dot(const cplx* __restrict__ L, const int* __restrict__ zi,
                                           int start, int n, int step, const cplx* __restrict__ X) {
  cplx acc0 = cmk(0, 0), acc1 = cmk(0, 0);
  cplx l[U];
  int ix[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int q = start + u * step;
    const bool ok = q < n;
    l[u] = ok ? ldf(L + q) : cmk(0, 0);
    ix[u] = ok ? __ldg(zi + q) : -1;
  }
  for (int q0 = start; q0 < n; q0 += U * step) {
    cplx x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = ix[u] >= 0 ? X[ix[u]] : cmk(0, 0);
    cplx ln[U];
    int ixn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + (U + u) * step;
      const bool ok = q < n;
      ln[u] = ok ? ldf(L + q) : cmk(0, 0);
      ixn[u] = ok ? __ldg(zi + q) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cfma((u & 1) ? acc1 : acc0, l[u], x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      l[u] = ln[u];
      ix[u] = ixn[u];
    }
  }
  return cadd(acc0, acc1);
}

// sum over backward rows of L[r][j] * X[dst r] for column j, pipelined the
// same way (row descriptors of the next batch in flight)
template <int U>
__device__ __forceinline__ cplx bw_gather(const cplx* __restrict__ vals, const BwRow* __restrict__ rows,
                                          int start, int nr, int step, int j,
                                          const cplx* __restrict__ X) {
  cplx acc0 = cmk(0, 0), acc1 = cmk(0, 0);
  BwRow d[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int k = start + u * step;
    d[u] = k < nr ? rows[k] : BwRow{0, 1 << 30, 0};
  }
  for (int k0 = start; k0 < nr; k0 += U * step) {
    cplx l[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = j >= d[u].first;
      l[u] = ok ? ldf(vals + d[u].off + (j - d[u].first)) : cmk(0, 0);
      x[u] = ok ? X[d[u].dpos] : cmk(0, 0);
    }
    BwRow dn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + (U + u) * step;
      dn[u] = k < nr ? rows[k] : BwRow{0, 1 << 30, 0};
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cfma((u & 1) ? acc1 : acc0, l[u], x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = dn[u];
  }
  return cadd(acc0, acc1);
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

// separator rows, forward pull: Y[r] = B[r] - run(r) . X[src] (thread per row).
// rec[item] = (position, run length, run offset lo, hi): one load of setup.
__global__ void __launch_bounds__(kThreads) k_fwd_pull(SolveArgs A, int ncls, const int4* rec,
                                                       int nitem) {
  int c, it, t;
  if (!decode(A, ncls, (long long)blockIdx.x * blockDim.x + threadIdx.x, nitem, c, it, t)) return;
  const int4 R = __ldg(rec + it);
  const long long r0 = (long long)(unsigned)R.z | ((long long)R.w << 32);
  const cplx* run = A.vals + (long long)c * A.nvals + r0;
  const long long base = (long long)t * A.nw;
  const cplx s = gather_dot<4>(run, A.zidx + r0, 0, R.y, 1, A.X + base);
  A.Y[base + R.x] = csub(A.B[base + R.x], s);
}

// separator rows with long runs (top levels): one WARP per (class, row,
// member); lanes stride the run (coalesced), zidx gives each element's source.
__global__ void __launch_bounds__(kThreads) k_fwd_pull_warp(SolveArgs A, int ncls,
                                                            const int4* rec, int nitem) {
  int c, it, t;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (!decode(A, ncls, w, nitem, c, it, t)) return;
  const int4 R = __ldg(rec + it);
  const long long r0 = (long long)(unsigned)R.z | ((long long)R.w << 32);
  const cplx* run = A.vals + (long long)c * A.nvals + r0;
  const long long base = (long long)t * A.nw;
  const cplx part = gather_dot<4>(run, A.zidx + r0, lane, R.y, 32, A.X + base);
  const cplx sum = warp_sum(part);
  if (lane == 0) A.Y[base + R.x] = csub(A.B[base + R.x], sum);
}

// separator rows, sub-warp of G lanes per (class, row, member): each group
// reads its run in G-wide coalesced chunks; a 32-lane warp serves 32/G rows.
template <int G>
__global__ void __launch_bounds__(kThreads) k_fwd_pull_sub(SolveArgs A, int ncls,
                                                           const int2* items, int nitem) {
  int c, it, t;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int sl = threadIdx.x & (G - 1);
  const bool live = decode(A, ncls, gid, nitem, c, it, t);
  cplx acc = cmk(0, 0);
  int pos = 0;
  if (live) {
    const int2 item = items[it];
    pos = A.sn[item.x].c0 + item.y;
    const long long r0 = A.run_off[pos];
    const int total = int(A.run_off[pos + 1] - r0);
    const cplx* run = A.vals + (long long)c * A.nvals + r0;
    const int* zi = A.zidx + r0;
    const cplx* X = A.X + (long long)t * A.nw;
    cplx acc1 = cmk(0, 0);
    int q = sl;
    for (; q + G < total; q += 2 * G) {
      const cplx l0 = ldf(run + q), l1 = ldf(run + q + G);
      const int i0 = __ldg(zi + q), i1 = __ldg(zi + q + G);
      cfma(acc, l0, X[i0]);
      cfma(acc1, l1, X[i1]);
    }
    if (q < total) cfma(acc, ldf(run + q), X[__ldg(zi + q)]);
    acc = cadd(acc, acc1);
  }
#pragma unroll
  for (int m = G / 2; m > 0; m >>= 1) acc = cadd(acc, shfl_xor(acc, m));
  if (live && sl == 0) A.Y[(long long)t * A.nw + pos] = csub(A.B[(long long)t * A.nw + pos], acc);
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
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (!(A.bwd_mm ? decode_mm(A, ncls, idx, nitem, c, it, t) : decode(A, ncls, idx, nitem, c, it, t)))
    return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int j = item.y;
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const cplx* X = A.X + (long long)t * A.nw;
  cplx acc = cmul(ldg(vals + sn.dinv_off + j), X[sn.c0 + j]);
  const BwRow* rows = A.bw + A.bw_ptr[item.x];
  const int nr = A.bw_ptr[item.x + 1] - A.bw_ptr[item.x];
  acc = csub(acc, bw_gather<4>(vals, rows, 0, nr, 1, j, X));
  (TO_X ? A.X : A.Y)[(long long)t * A.nw + sn.c0 + j] = acc;
}

// separator columns, backward diagonal: X[j] = Y[j] + sum_{i>j} Linv[i][j] Y[i]
__global__ void __launch_bounds__(kThreads) k_bwd_diag(SolveArgs A, int ncls, const int2* items,
                                                       int nitem) {
  int c, it, t;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (!(A.bwd_mm ? decode_mm(A, ncls, idx, nitem, c, it, t) : decode(A, ncls, idx, nitem, c, it, t)))
    return;
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

// ---------------------------------------------------------- fused small separators
// Separators with n <= G lanes (deep levels): a group of G lanes per
// (class, separator, member) does the pull of its rows/columns and then the
// dense-inverse product through shuffles within the group -- one kernel per
// level, no scratch round trip. items: (separator, 0).
template <int G>
__global__ void __launch_bounds__(kThreads) k_fwd_small(SolveArgs A, int ncls, const int2* items,
                                                        int nitem) {
  int c, it, t;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int l = threadIdx.x & (G - 1);
  const bool live = decode(A, ncls, gid, nitem, c, it, t);
  const DevSn sn = A.sn[live ? items[it].x : 0];
  const bool row = live && l < sn.n;
  const cplx* vals = A.vals + (long long)(live ? c : 0) * A.nvals;
  cplx y = cmk(0, 0);
  if (row) {
    const int pos = sn.c0 + l;
    const cplx* run = vals + A.run_off[pos];
    const cplx* X = A.X + (long long)t * A.nw;
    y = A.B[(long long)t * A.nw + pos];
    for (int e = A.seg_ptr[pos]; e < A.seg_ptr[pos + 1]; ++e) {
      const int2 sg = A.seg[e];
      const cplx* xs = X + sg.y;
      int j = 0;
      for (; j + 4 <= sg.x; j += 4) {
        const cplx l0 = ldf(run + j), l1 = ldf(run + j + 1), l2 = ldf(run + j + 2), l3 = ldf(run + j + 3);
        const cplx x0 = xs[j], x1 = xs[j + 1], x2 = xs[j + 2], x3 = xs[j + 3];
        csub_mul(y, l0, x0);
        csub_mul(y, l1, x1);
        csub_mul(y, l2, x2);
        csub_mul(y, l3, x3);
      }
      for (; j < sg.x; ++j) csub_mul(y, ldf(run + j), xs[j]);
      run += sg.x;
    }
  }
  // z_l = y_l + sum_{j<l} Linv[l][j] y_j (y_j broadcast within the group)
  const cplx* Lrow = vals + sn.diag_off + (long long)l * (l - 1) / 2;
  cplx z = y;
  const int n = live ? sn.n : 0;
  for (int j = 0; j + 1 < n; ++j) {
    const cplx yj = cmk(__shfl_sync(0xffffffffu, y.x, j, G), __shfl_sync(0xffffffffu, y.y, j, G));
    if (row && j < l) cfma(z, ldf(Lrow + j), yj);
  }
  if (row) A.X[(long long)t * A.nw + sn.c0 + l] = z;
}

template <int G>
__global__ void __launch_bounds__(kThreads) k_bwd_small(SolveArgs A, int ncls, const int2* items,
                                                        int nitem) {
  int c, it, t;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int j = threadIdx.x & (G - 1);
  const bool live = decode(A, ncls, gid, nitem, c, it, t);
  const int sid = live ? items[it].x : 0;
  const DevSn sn = A.sn[sid];
  const bool col = live && j < sn.n;
  const cplx* vals = A.vals + (long long)(live ? c : 0) * A.nvals;
  cplx w = cmk(0, 0);
  if (col) {
    const cplx* X = A.X + (long long)t * A.nw;
    w = cmul(ldg(vals + sn.dinv_off + j), X[sn.c0 + j]);
    const BwRow* rows = A.bw + A.bw_ptr[sid];
    const int nr = A.bw_ptr[sid + 1] - A.bw_ptr[sid];
    int k = 0;
    for (; k + 4 <= nr; k += 4) {
      BwRow d[4];
      cplx lv[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) d[u] = rows[k + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = j >= d[u].first;
        lv[u] = ok ? ldf(vals + d[u].off + (j - d[u].first)) : cmk(0, 0);
        xv[u] = ok ? X[d[u].dpos] : cmk(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) csub_mul(w, lv[u], xv[u]);
    }
    for (; k < nr; ++k) {
      const BwRow d = rows[k];
      if (j >= d.first) csub_mul(w, ldf(vals + d.off + (j - d.first)), X[d.dpos]);
    }
  }
  // x_j = w_j + sum_{i>j} Linv[i][j] w_i
  const cplx* Linv = vals + sn.diag_off;
  cplx x = w;
  const int n = live ? sn.n : 0;
  for (int i = 1; i < n; ++i) {
    const cplx wi = cmk(__shfl_sync(0xffffffffu, w.x, i, G), __shfl_sync(0xffffffffu, w.y, i, G));
    if (col && i > j) cfma(x, ldf(Linv + (long long)i * (i - 1) / 2 + j), wi);
  }
  if (col) A.X[(long long)t * A.nw + sn.c0 + j] = x;
}

// ---------------------------------------------------------- split variants
// Levels whose per-output loops are long (top of the tree) use more threads per
// output so no single thread walks a long dependent chain.

// forward diagonal, one WARP per (class, row, member); lanes over j < i
__global__ void __launch_bounds__(kThreads) k_fwd_diag_warp(SolveArgs A, int ncls,
                                                            const int2* items, int nitem) {
  int c, it, t;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (!decode(A, ncls, w, nitem, c, it, t)) return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int i = item.y;
  const cplx* row = A.vals + (long long)c * A.nvals + sn.diag_off + (long long)i * (i - 1) / 2;
  const cplx* y = A.Y + (long long)t * A.nw + sn.c0;
  cplx acc = cmk(0, 0);
  for (int j = lane; j < i; j += 32) cfma(acc, ldf(row + j), y[j]);
  acc = warp_sum(acc);
  if (lane == 0) A.X[(long long)t * A.nw + sn.c0 + i] = cadd(y[i], acc);
}

// backward, one CTA per (class, 32-column chunk, member): lanes over columns,
// the 8 warps split the inner range, partial sums combined in fixed warp order.
// items: (supernode, first column of the chunk)
template <bool DIAG>
__global__ void __launch_bounds__(256) k_bwd_split(SolveArgs A, int ncls, const int2* items,
                                                   int nitem) {
  __shared__ cplx part[8][32];
  int c, it, t;
  if (!decode(A, ncls, blockIdx.x, nitem, c, it, t)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int j = item.y + lane;
  const bool ok = j < sn.n;
  const cplx* vals = A.vals + (long long)c * A.nvals;
  cplx acc = cmk(0, 0);
  if (DIAG) {
    // x_j = y_j + sum_{i>j} Linv[i][j] y_i ; warps split i
    const cplx* Linv = vals + sn.diag_off;
    const cplx* y = A.Y + (long long)t * A.nw + sn.c0;
    if (ok)
      for (int i = item.y + 1 + warp; i < sn.n; i += 8)
        if (i > j) cfma(acc, ldf(Linv + (long long)i * (i - 1) / 2 + j), y[i]);
  } else {
    // w_j = Dinv z_j - sum_rows L[r][j] x_r ; warps split the rows
    const cplx* X = A.X + (long long)t * A.nw;
    const BwRow* rows = A.bw + A.bw_ptr[item.x];
    const int nr = A.bw_ptr[item.x + 1] - A.bw_ptr[item.x];
    if (ok) acc = bw_gather<4>(vals, rows, warp, nr, 8, j, X);
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && ok) {
    cplx sum = part[0][lane];
    for (int w = 1; w < 8; ++w) sum = cadd(sum, part[w][lane]);
    const long long p = (long long)t * A.nw + sn.c0 + j;
    if (DIAG)
      A.X[p] = cadd(A.Y[p], sum);
    else
      A.Y[p] = csub(cmul(ldg(vals + sn.dinv_off + j), A.X[p]), sum);
  }
}

// ------------------------------------------------------------------ launcher
// One class's solve on one stream: the kernels see a single-class view
// (act_ptr and vals offset to class c), so their class decode is trivial.
void launch_solve_class(const SolveArgs& A0, const SolvePlan& P, int c, int members,
                        cudaStream_t st) {
  SolveArgs A = A0;
  A.act_ptr = A0.act_ptr + c;
  A.vals = A0.vals + (long long)c * A0.nvals;
  launch_solve(A, P, 1, members, st);
}

int solve_launch_count(const SolvePlan& P) {
  int n = 2 + 2;
  for (const auto& L : P.fwd) n += L.small_g ? 1 : 2;
  for (const auto& L : P.bwd) n += L.small_g ? 1 : 2;
  return n;
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
    if (L.small_g) {
      const long long w = (long long)max_rhs * L.nsmall * L.small_g;
      if (L.small_g == 8) k_fwd_small<8><<<grid_for(w), kThreads, 0, st>>>(A, ncls, L.d_small, L.nsmall);
      else if (L.small_g == 16) k_fwd_small<16><<<grid_for(w), kThreads, 0, st>>>(A, ncls, L.d_small, L.nsmall);
      else k_fwd_small<32><<<grid_for(w), kThreads, 0, st>>>(A, ncls, L.d_small, L.nsmall);
      continue;
    }
    const unsigned g = grid_for((long long)max_rhs * L.nitem);
    const unsigned gw = grid_for((long long)max_rhs * L.nitem * 32);
    const long long w = (long long)max_rhs * L.nitem;
    switch (L.group) {
      case 32: k_fwd_pull_warp<<<gw, kThreads, 0, st>>>(A, ncls, L.d_rec, L.nitem); break;
      case 16: k_fwd_pull_sub<16><<<grid_for(w * 16), kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem); break;
      case 8: k_fwd_pull_sub<8><<<grid_for(w * 8), kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem); break;
      case 4: k_fwd_pull_sub<4><<<grid_for(w * 4), kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem); break;
      default: k_fwd_pull<<<g, kThreads, 0, st>>>(A, ncls, L.d_rec, L.nitem); break;
    }
    if (L.warp_diag)
      k_fwd_diag_warp<<<gw, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
    else
      k_fwd_diag<<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
  }
  for (const auto& L : P.bwd) {
    if (L.small_g) {
      const long long w = (long long)max_rhs * L.nsmall * L.small_g;
      if (L.small_g == 8) k_bwd_small<8><<<grid_for(w), kThreads, 0, st>>>(A, ncls, L.d_small, L.nsmall);
      else if (L.small_g == 16) k_bwd_small<16><<<grid_for(w), kThreads, 0, st>>>(A, ncls, L.d_small, L.nsmall);
      else k_bwd_small<32><<<grid_for(w), kThreads, 0, st>>>(A, ncls, L.d_small, L.nsmall);
      continue;
    }
    const unsigned g = grid_for((long long)max_rhs * L.nitem);
    if (L.nchunk > 0) {
      const unsigned gc = unsigned((long long)max_rhs * L.nchunk);
      if (L.warp_rows)
        k_bwd_split<false><<<gc, 256, 0, st>>>(A, ncls, L.d_chunks, L.nchunk);
      else
        k_bwd_pull<false><<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
      if (L.warp_diag)
        k_bwd_split<true><<<gc, 256, 0, st>>>(A, ncls, L.d_chunks, L.nchunk);
      else
        k_bwd_diag<<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
    } else {
      k_bwd_pull<false><<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
      k_bwd_diag<<<g, kThreads, 0, st>>>(A, ncls, L.d_items, L.nitem);
    }
  }
  const SolveLevel& BC = P.bwd_leafcol;
  k_bwd_pull<true><<<grid_for((long long)max_rhs * BC.nitem), kThreads, 0, st>>>(
      A, ncls, BC.d_items, BC.nitem);
  const SolveLevel& BL = P.bwd_leaf;
  k_bwd_leaf<<<grid_for((long long)max_rhs * BL.nitem), kThreads, 0, st>>>(A, ncls, BL.d_items,
                                                                          BL.nitem);
}

}  // namespace hddm
