// Batched multi-RHS supernodal triangular solves (the per-step hot path that
// replaces Factorization::solve -> solve_raw, proj/src/sparse.cpp:244-266).
//
// Level-synchronous over the nested-dissection tree. The right-hand sides of a
// factor class are stored member-interleaved (VMap, dev.cuh), and the work of a
// class is cut into MEMBER TILES of up to 32 members; every kernel launch
// serves one tile (its descriptor travels in the kernel parameters, so a warp
// needs no setup loads). A warp's 32 lanes are split as R x E x M:
//   k = lane % M          member of the tile (consecutive lanes: consecutive
//                         members -> contiguous vector entries, one factor
//                         entry broadcast to all of them),
//   e = lane / M % E      element lane within one output (E > 1: the lanes
//                         stride a long run, partial sums reduced by shuffles),
//   r = lane / (E M)      output item (R items per warp).
// The host picks E and R per level and tile: singleton classes stride their
// runs with E lanes (coalesced factor / index / vector reads), multi-member
// tiles keep E = 1 deep in the tree (lanes over members already coalesce) and
// widen E near the root where runs are long and items few.
//
//   forward, leaves:      z_leaf = L_leaf^{-1} b_leaf              (band, registers)
//   forward, separators:  y_r = b_r - (incoming run of row r) . z   (pull)
//                         z_s = Linv_s y_s                         (dense inverse)
//   backward, separators: w_j = z_j / D_j - sum_r L[r][j] x_r       (pull, rows sorted
//                         x_s = Linv_s^T w_s                        by first column)
//   backward, leaves:     the same pull per leaf column, then a band
//                         back-substitution per leaf
//   ring (identity rows): x = b
// Every output has one writer and a fixed summation order: deterministic.
#include <algorithm>
#include <cstdlib>

#include "dev.cuh"
#include "kernels.cuh"

namespace hddm {

namespace {

#ifndef HDDM_SOLVE_THREADS
#define HDDM_SOLVE_THREADS 128  // measured best at config 4 (64-512 within 5%)
#endif
constexpr int kThreads = HDDM_SOLVE_THREADS;
#ifndef HDDM_UF
#define HDDM_UF 4
#endif
#ifndef HDDM_UB
#define HDDM_UB 4
#endif
constexpr int kUF = HDDM_UF;  // forward gathers in flight per lane
constexpr int kUB = HDDM_UB;  // backward rows in flight per lane
constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch: every solve kernel lets its successor in the
// stream launch as soon as all of its CTAs are resident (trigger), does its
// static setup (tile records, item lists, activity flags -- all written before
// the solve), and waits for its predecessor's completion before touching any
// vector or writing anything.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// one lane of a tile-group launch: warp w serves tile w / wpt of the group
// (wpt = warps per tile for this level), items (w % wpt) * R + r
struct TL {
  int r, e, k;    // item within the warp, element lane, member
  int c, m;       // class, member count (vector stride)
  long long cb;   // storage offset of (position 0, member k of the tile)
  long long it;   // item index of this lane
  bool act;       // lane maps to an active right-hand side
};

__device__ __forceinline__ void tile_fill(const SolveArgs& A, const TileArg& T, int ti, bool in,
                                          TL& L) {
  const TileRec* rec = T.rec + (in ? ti : 0);
  L.c = rec->c;
  L.m = rec->m;
  L.cb = rec->cb + L.k;
  const int t = rec->t[L.k];
  L.act = in && (A.flag[t] != 0) == (A.flag_on != 0);
}

// x / d for small x (x * d < 2^32) with mag = ceil(2^32 / d); d == 1: x
__device__ __forceinline__ unsigned udiv(unsigned x, int d, unsigned mag) {
  return d == 1 ? x : __umulhi(x, mag);
}

// the same, opaque to the optimiser: recomputed where it is used instead of being hoisted
// out of a loop into registers (k_bwd_stage's pair indices: 80 -> 126 registers if hoisted)
__device__ __forceinline__ unsigned udiv_here(unsigned x, int d, unsigned mag) {
  unsigned q;
  asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(q) : "r"(x), "r"(mag));
  return d == 1 ? x : q;
}

__device__ __forceinline__ TL tile_lane(const SolveArgs& A, const TileArg& T, int nitem) {
  // 32-bit unsigned arithmetic and host-side division magics: the lane decomposition
  // is on every warp's start-up path
  const unsigned lane = threadIdx.x & 31;
  const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned wpt = (unsigned(nitem) + unsigned(T.R) - 1u) / unsigned(T.R);
  const unsigned ti = w / wpt;
  TL L;
  const unsigned q = udiv(lane, T.M, T.magM);   // lane / M
  const unsigned qe = udiv(q, T.E, T.magE);     // lane / (M E)
  L.k = int(lane - q * unsigned(T.M));
  L.e = int(q - qe * unsigned(T.E));
  L.r = int(qe);
  L.it = (long long)(w - ti * wpt) * T.R + L.r;
  tile_fill(A, T, int(ti), int(ti) < T.ntile && L.r < T.R && L.it < nitem, L);
  return L;
}

__device__ __forceinline__ long long vat(const TL& L, int pos) {
  return L.cb + (long long)pos * L.m;
}

// sum over the E element lanes of each (item, member); result valid at e == 0
__device__ __forceinline__ cplx tile_reduce(cplx v, const TileArg& T, const TL& L) {
  for (int step = 1; step < T.E; step <<= 1) {
    const double ox = __shfl_down_sync(kFull, v.x, step * T.M);
    const double oy = __shfl_down_sync(kFull, v.y, step * T.M);
    if ((L.e & (2 * step - 1)) == 0 && L.e + step < T.E) v = cadd(v, cmk(ox, oy));
  }
  return v;
}

__device__ __forceinline__ void csub_mul(cplx& acc, cplx l, cplx x) {
  acc.x -= l.x * x.x - l.y * x.y;
  acc.y -= l.x * x.y + l.y * x.x;
}

// sum over a row's run segments of L[q] * X[(zb + q) * m]: a segment is a
// contiguous piece of the factor values against consecutive source positions,
// so no per-element index is loaded; lanes e, e+E, ... stride each segment with
// U loads of both operands in flight.
template <int U, bool PF>
__device__ __forceinline__ cplx seg_dot(const cplx* __restrict__ vals, const SegRec* __restrict__ sg,
                                        int ns, int e, int E, unsigned magE,
                                        const cplx* __restrict__ X, int m) {
  cplx acc0 = cmk(0, 0), acc1 = cmk(0, 0);
  const long long xs = (long long)E * m;  // vector stride per step: pointer increments only
  // PF (singleton tiles): the next segment's record is loaded behind this one's data, one
  // dependent round trip less per segment; member tiles keep the registers (measured)
  SegRec rn = (PF && ns > 0) ? sg[0] : SegRec{0, 0, 0};
  for (int k = 0; k < ns; ++k) {
    const SegRec r = PF ? rn : sg[k];
    if (PF && k + 1 < ns) rn = sg[k + 1];
    if (e >= r.len) continue;
    int n = int(udiv(unsigned(r.len - 1 - e), E, magE)) + 1;  // entries of this lane
    const cplx* lp = vals + r.off + e;
    const cplx* xp = X + (long long)(r.zb + e) * m;
    for (; n >= U; n -= U) {  // full batches of U
      cplx l[U], x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        l[u] = ldf(lp);
        x[u] = *xp;
        lp += E;
        xp += xs;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cfma((u & 1) ? acc1 : acc0, l[u], x[u]);
    }
    if (n > 0) {  // tail: one predicated batch
      cplx l[U], x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        l[u] = u < n ? ldf(lp) : cmk(0, 0);
        x[u] = u < n ? *xp : cmk(0, 0);
        lp += E;
        xp += xs;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cfma((u & 1) ? acc1 : acc0, l[u], x[u]);
    }
  }
  return cadd(acc0, acc1);
}

// forward result z at position p of supernode s: supernodes the sparse-RHS
// forward skipped hold z = 0 exactly and X is not cleared for them
__device__ __forceinline__ cplx zval(const SolveArgs& A, int s, long long p) {
  return (A.sn_live != nullptr && A.sn_live[s] == 0) ? cmk(0, 0) : A.X[p];
}

// sum over rows k = start, start+step, ... < nr of L[r][j] * X[dpos_r * m],
// row descriptors of the next batch in flight
template <int U>
__device__ __forceinline__ cplx bw_gather(const cplx* __restrict__ vals, const BwRow* __restrict__ rows,
                                          int start, int nr, int step, int j,
                                          const cplx* __restrict__ X, int m) {
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
      x[u] = ok ? X[(long long)d[u].dpos * m] : cmk(0, 0);
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

// identity ring rows: x = b (thread per (position, member))
__global__ void __launch_bounds__(kThreads) k_ring(SolveArgs A, TileArg T) {
  pdl_trigger();
  const TL L = tile_lane(A, T, A.nring);
  pdl_wait();
  if (!L.act) return;
  const long long p = vat(L, int(L.it));
  A.X[p] = A.B[p];
}

// leaves, forward: z_i = b_i - sum_{q in [first_i, i)} L[i][q] z_q. A leaf is a
// w x h box in natural order: row i stores columns [first_i, i) with first_i =
// i-1 in the first grid row and i-w after it (checked at setup), rows back to
// back from diag_off -- so the band streams with pointer arithmetic and the next
// row's entries and right-hand side are loaded while the current row computes.
// The last kBand values live in a register window. Thread per (leaf, member).
constexpr int kBand = 6;

__device__ __forceinline__ int leaf_first(int i, int w) { return i < w ? (i > 0 ? i - 1 : 0) : i - w; }

__global__ void __launch_bounds__(kThreads) k_fwd_leaf(SolveArgs A, TileArg T, const int2* items,
                                                       int nitem) {
  pdl_trigger();
  const TL L = tile_lane(A, T, nitem);
  const long long it = L.it;
  pdl_wait();
  if (!L.act) return;
  const DevSn sn = A.sn[items[it].x];
  const cplx* p = A.vals + (long long)L.c * A.nvals + sn.diag_off;  // row 0's entries
  const SVec<const cplx> b{A.B + vat(L, sn.c0), L.m};
  const SVec<cplx> x{A.X + vat(L, sn.c0), L.m};
  const int w = sn.lw, n = sn.n;
  cplx win[kBand + 1];  // win[d] = z_{i-d}
#pragma unroll
  for (int d = 0; d <= kBand; ++d) win[d] = cmk(0, 0);
  // current row's band: lv[d] = L[i][i-d] (0 outside the profile), bv = b_i
  cplx lv[kBand + 1], bv = n > 0 ? b[0] : cmk(0, 0);
#pragma unroll
  for (int d = 0; d <= kBand; ++d) lv[d] = cmk(0, 0);
  for (int i = 0; i < n; ++i) {
    const int cnt = i - leaf_first(i, w);  // entries of row i, L[i][i-d] = p[cnt - d]
    const cplx* pn = p + cnt;              // row i+1
    cplx ln[kBand + 1], bn = cmk(0, 0);
    const int cn = (i + 1 < n) ? i + 1 - leaf_first(i + 1, w) : 0;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) ln[d] = d <= cn ? ldf(pn + cn - d) : cmk(0, 0);
    if (i + 1 < n) bn = b[i + 1];
    if (i == 0) {
#pragma unroll
      for (int d = 1; d <= kBand; ++d) lv[d] = d <= cnt ? ldf(p + cnt - d) : cmk(0, 0);
    }
    cplx acc = bv;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) csub_mul(acc, lv[d], win[d]);
#pragma unroll
    for (int d = kBand; d >= 2; --d) win[d] = win[d - 1];
    win[1] = acc;
    x[i] = acc;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = ln[d];
    bv = bn;
    p = pn;
  }
}

// separator rows, forward pull: Y[r] = B[r] - run(r) . X[src].
// rec[item] = (position, first segment in A.fseg, segment count, -).
template <bool PF>
__global__ void __launch_bounds__(kThreads) k_fwd_pull(SolveArgs A, TileArg T, const int4* rec,
                                                       int nitem) {
  pdl_trigger();
  const TL L = tile_lane(A, T, nitem);
  const long long it = L.it;
  const bool live = L.act;
  pdl_wait();
  int4 R = make_int4(0, 0, 0, 0);
  cplx acc = cmk(0, 0);
  if (live) {
    R = __ldg(rec + it);
    acc = seg_dot<kUF, PF>(A.vals + (long long)L.c * A.nvals, A.fseg + R.y, R.z, L.e, T.E, T.magE, A.X + L.cb,
                       L.m);
  }
  if (T.E > 1) acc = tile_reduce(acc, T, L);
  if (live && L.e == 0) {
    const long long p = vat(L, R.x);
    A.Y[p] = csub(A.B[p], acc);
  }
}

// separator rows of member tiles, forward pull on the FP64 tensor cores:
// Y[r][k] = B[r][k] - sum_z L[r][z] X[z][k] for a block of up to 8 rows r of one
// separator and the tile's members k (n-blocks of 8), as mma.sync m8n8k4 f64
// (A = 8 rows x 4 columns of L, zero outside each row's run piece; B = 4 columns x 8
// members of X, contiguous in the member-interleaved layout; complex products as four
// real MMAs). A warp per (tile, block); the members' X of a column is read once per
// block instead of once per row (the L2 re-reads of the lane-per-member kernel).
__device__ __forceinline__ void dmma2(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NB>
__global__ void __launch_bounds__(256) k_fwd_pull_mma(SolveArgs A, TileArg T, const int4* __restrict__ rec,
                                                      const int4* __restrict__ blk, const MmaSeg* __restrict__ segs,
                                                      int nblk) {
  // CTA per (tile, block); the 8 warps split the k-steps (interleaved), their partial
  // accumulators combined in warp order
  __shared__ double part[8][32][NB * 4];
  pdl_trigger();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int ti = blockIdx.x / nblk;
  const int b = blockIdx.x - ti * nblk;
  // static tables first (written at setup): the block record and its first segment are in
  // flight while the activity flags resolve
  const int4 B = blk[b];  // (first item, rows, first segment, segments)
  const int g = lane >> 2, q = lane & 3;
  const bool grow = g < B.y;
  int zmin_n = 0, ulen_n = 0, lo_n = 0, hi_n = 0;
  long long vb_n = 0;
  if (B.w > 0) {
    const MmaSeg& S0 = segs[B.z];
    zmin_n = S0.zmin;
    ulen_n = S0.ulen;
    if (grow) {
      lo_n = S0.lo[g];
      hi_n = S0.hi[g];
      vb_n = S0.vb[g];
    }
  }
  pdl_wait();
  const TileRec* tr = T.rec + ti;
  const int M = T.M, m = tr->m;
  const long long cb = tr->cb;
  bool any = false;  // a tile without an active member does nothing (CTA-uniform)
  for (int k = 0; k < M; ++k) any |= (A.flag[tr->t[k]] != 0) == (A.flag_on != 0);
  if (!any) return;
  const cplx* vals = A.vals + (long long)tr->c * A.nvals;
  const cplx* X = A.X + cb;
  double cr[NB][2], ci[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) cr[nb][0] = cr[nb][1] = ci[nb][0] = ci[nb][1] = 0.0;
  for (int u = B.z; u < B.z + B.w; ++u) {
    // this segment's record was loaded one iteration ahead; the next one's goes out now
    const int zmin = zmin_n, ulen = ulen_n, lo = lo_n, hi = hi_n;
    const cplx* vrow = vals + vb_n;
    if (u + 1 < B.z + B.w) {
      const MmaSeg& S = segs[u + 1];
      zmin_n = S.zmin;
      ulen_n = S.ulen;
      if (grow) {
        lo_n = S.lo[g];
        hi_n = S.hi[g];
        vb_n = S.vb[g];
      }
    }
    for (int k0 = 4 * wp; k0 < ulen; k0 += 32) {
      const int z = zmin + k0 + q;
      const bool zin = k0 + q < ulen;
      const cplx a = (z >= lo && z < hi) ? ldf(vrow + z) : cmk(0, 0);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int mem = nb * 8 + g;
        const cplx x = (zin && mem < M) ? X[(long long)z * m + mem] : cmk(0, 0);
        dmma2(cr[nb][0], cr[nb][1], a.x, x.x);
        dmma2(cr[nb][0], cr[nb][1], -a.y, x.y);
        dmma2(ci[nb][0], ci[nb][1], a.x, x.y);
        dmma2(ci[nb][0], ci[nb][1], a.y, x.x);
      }
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    part[wp][lane][nb * 4 + 0] = cr[nb][0];
    part[wp][lane][nb * 4 + 1] = cr[nb][1];
    part[wp][lane][nb * 4 + 2] = ci[nb][0];
    part[wp][lane][nb * 4 + 3] = ci[nb][1];
  }
  __syncthreads();
  if (wp != 0 || g >= B.y) return;
  double sum[NB * 4];
#pragma unroll
  for (int v = 0; v < NB * 4; ++v) {
    double acc = part[0][lane][v];
    for (int k = 1; k < 8; ++k) acc += part[k][lane][v];
    sum[v] = acc;
  }
  const int pos = __ldg(rec + B.x + g).x;
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int mem = nb * 8 + 2 * q + h;
      if (mem >= M) continue;
      const long long p = cb + (long long)pos * m + mem;
      A.Y[p] = csub(A.B[p], cmk(sum[nb * 4 + h], sum[nb * 4 + 2 + h]));
    }
}

// separator rows of member tiles, forward dense inverse on the FP64 tensor cores:
// X[i][k] = Y[i][k] + sum_{j<i} Linv[i][j] Y[j][k] for a block of up to 8 rows i of one
// separator (the pull's row blocks), CTA per (tile, block), 8 warps splitting the
// k-steps, combined in warp order.
template <int NB>
__global__ void __launch_bounds__(256) k_fwd_diag_mma(SolveArgs A, TileArg T, const int2* __restrict__ items,
                                                      const int4* __restrict__ blk, int nblk) {
  __shared__ double part[8][32][NB * 4];
  pdl_trigger();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int ti = blockIdx.x / nblk;
  const int b = blockIdx.x - ti * nblk;
  pdl_wait();
  const TileRec* tr = T.rec + ti;
  const int M = T.M, m = tr->m;
  const long long cb = tr->cb;
  bool any = false;
  for (int k = 0; k < M; ++k) any |= (A.flag[tr->t[k]] != 0) == (A.flag_on != 0);
  if (!any) return;
  const int4 B = blk[b];
  const int2 it0 = items[B.x];
  const DevSn sn = A.sn[it0.x];
  const int i0 = it0.y;
  const int g = lane >> 2, q = lane & 3;
  const int i = i0 + g;
  const cplx* Linv = A.vals + (long long)tr->c * A.nvals + sn.diag_off;
  const cplx* lrow = Linv + (long long)i * (i - 1) / 2;
  const cplx* Yb = A.Y + cb + (long long)sn.c0 * m;
  double cr[NB][2], ci[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) cr[nb][0] = cr[nb][1] = ci[nb][0] = ci[nb][1] = 0.0;
  const int jend = i0 + B.y - 1;  // columns below the block's last row
  for (int k0 = 4 * wp; k0 < jend; k0 += 32) {
    const int j = k0 + q;
    const cplx a = (g < B.y && j < i) ? ldf(lrow + j) : cmk(0, 0);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int mem = nb * 8 + g;
      const cplx x = (j < jend && mem < M) ? Yb[(long long)j * m + mem] : cmk(0, 0);
      dmma2(cr[nb][0], cr[nb][1], a.x, x.x);
      dmma2(cr[nb][0], cr[nb][1], -a.y, x.y);
      dmma2(ci[nb][0], ci[nb][1], a.x, x.y);
      dmma2(ci[nb][0], ci[nb][1], a.y, x.x);
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    part[wp][lane][nb * 4 + 0] = cr[nb][0];
    part[wp][lane][nb * 4 + 1] = cr[nb][1];
    part[wp][lane][nb * 4 + 2] = ci[nb][0];
    part[wp][lane][nb * 4 + 3] = ci[nb][1];
  }
  __syncthreads();
  if (wp != 0 || g >= B.y) return;
  double sum[NB * 4];
#pragma unroll
  for (int v = 0; v < NB * 4; ++v) {
    double acc = part[0][lane][v];
    for (int k = 1; k < 8; ++k) acc += part[k][lane][v];
    sum[v] = acc;
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int mem = nb * 8 + 2 * q + h;
      if (mem >= M) continue;
      if ((A.flag[tr->t[mem]] != 0) != (A.flag_on != 0)) continue;
      const long long p = cb + (long long)(sn.c0 + i) * m + mem;
      A.X[p] = cadd(A.Y[p], cmk(sum[nb * 4 + h], sum[nb * 4 + 2 + h]));
    }
}

// separator rows, forward diagonal: X[i] = Y[i] + sum_{j<i} Linv[i][j] Y[j]
__global__ void __launch_bounds__(kThreads) k_fwd_diag(SolveArgs A, TileArg T, const int2* items,
                                                       int nitem) {
  pdl_trigger();
  const TL L = tile_lane(A, T, nitem);
  const long long it = L.it;
  const bool live = L.act;
  pdl_wait();
  int2 item = make_int2(0, 0);
  long long y0 = 0;
  cplx acc = cmk(0, 0), acc2 = cmk(0, 0);
  if (live) {
    item = items[it];
    const DevSn sn = A.sn[item.x];
    const int i = item.y;
    y0 = vat(L, sn.c0);
    const cplx* row = A.vals + (long long)L.c * A.nvals + sn.diag_off + (long long)i * (i - 1) / 2;
    const int E = T.E;
    const long long ys = (long long)E * L.m;
    const cplx* lp = row + L.e;
    const cplx* yp = A.Y + y0 + (long long)L.e * L.m;
    int j = L.e;
    for (; j + E < i; j += 2 * E) {
      const cplx l0 = ldf(lp), l1 = ldf(lp + E);
      const cplx v0 = *yp, v1 = yp[ys];
      cfma(acc, l0, v0);
      cfma(acc2, l1, v1);
      lp += 2 * E;
      yp += 2 * ys;
    }
    if (j < i) cfma(acc, ldf(lp), *yp);
  }
  acc = cadd(acc, acc2);
  if (T.E > 1) acc = tile_reduce(acc, T, L);
  if (live && L.e == 0) {
    const long long p = y0 + (long long)item.y * L.m;
    A.X[p] = cadd(A.Y[p], acc);
  }
}

// Member tiles' backward on the FP64 tensor cores, blocks of up to 8 columns j of one
// separator (lane group g = column), CTA per (tile, block), the 8 warps splitting the
// k-steps, partials combined in warp order:
//   pull:    Y[j][k] = Dinv_j z_j[k] - sum_r L[r][j] X[dst r][k] over the rows reaching
//            the block (a prefix of the first-column-sorted list; zero left of a row's
//            first column);
//   inverse: X[j][k] = Y[j][k] + sum_{i>j} Linv[i][j] Y[i][k].
template <int NB, bool DIAG>
__global__ void __launch_bounds__(256) k_bwd_mma(SolveArgs A, TileArg T, const int2* __restrict__ items,
                                                 const int4* __restrict__ blk, int nblk) {
  __shared__ double part[8][32][NB * 4];
  pdl_trigger();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int ti = blockIdx.x / nblk;
  const int b = blockIdx.x - ti * nblk;
  pdl_wait();
  const TileRec* tr = T.rec + ti;
  const int M = T.M, m = tr->m;
  const long long cb = tr->cb;
  bool any = false;
  for (int k = 0; k < M; ++k) any |= (A.flag[tr->t[k]] != 0) == (A.flag_on != 0);
  if (!any) return;
  const int4 B = blk[b];
  const int2 it0 = items[B.x];
  const DevSn sn = A.sn[it0.x];
  const int j0 = it0.y;
  const int g = lane >> 2, q = lane & 3;
  const int j = j0 + g;
  const bool col = g < B.y;
  const cplx* vals = A.vals + (long long)tr->c * A.nvals;
  double cr[NB][2], ci[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) cr[nb][0] = cr[nb][1] = ci[nb][0] = ci[nb][1] = 0.0;
  if (DIAG) {
    const cplx* Linv = vals + sn.diag_off;
    const cplx* Yb = A.Y + cb + (long long)sn.c0 * m;
    for (int i0 = j0 + 1 + 4 * wp; i0 < sn.n; i0 += 32) {
      // A: rows = the block's columns j (lane group g), k = rows i of Linv (lane q)
      const int ia = i0 + q;  // the Linv row this lane loads for its column j
      const cplx a = (col && ia < sn.n && ia > j) ? ldf(Linv + (long long)ia * (ia - 1) / 2 + j) : cmk(0, 0);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int mem = nb * 8 + g;
        const cplx x = (ia < sn.n && mem < M) ? Yb[(long long)ia * m + mem] : cmk(0, 0);
        dmma2(cr[nb][0], cr[nb][1], a.x, x.x);
        dmma2(cr[nb][0], cr[nb][1], -a.y, x.y);
        dmma2(ci[nb][0], ci[nb][1], a.x, x.y);
        dmma2(ci[nb][0], ci[nb][1], a.y, x.x);
      }
    }
  } else {
    const BwRow* rows = A.bw + A.bw_ptr[it0.x];
    const int nr = __ldg(A.bw_cnt + sn.c0 + j0 + B.y - 1);
    const cplx* Xb = A.X + cb;
    for (int r0 = 4 * wp; r0 < nr; r0 += 32) {
      const int rk = r0 + q;
      const BwRow d = rk < nr ? rows[rk] : BwRow{0, 1 << 30, 0};
      const cplx a = (col && j >= d.first) ? ldf(vals + d.off + (j - d.first)) : cmk(0, 0);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int mem = nb * 8 + g;
        const cplx x = (rk < nr && mem < M) ? Xb[(long long)d.dpos * m + mem] : cmk(0, 0);
        dmma2(cr[nb][0], cr[nb][1], a.x, x.x);
        dmma2(cr[nb][0], cr[nb][1], -a.y, x.y);
        dmma2(ci[nb][0], ci[nb][1], a.x, x.y);
        dmma2(ci[nb][0], ci[nb][1], a.y, x.x);
      }
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    part[wp][lane][nb * 4 + 0] = cr[nb][0];
    part[wp][lane][nb * 4 + 1] = cr[nb][1];
    part[wp][lane][nb * 4 + 2] = ci[nb][0];
    part[wp][lane][nb * 4 + 3] = ci[nb][1];
  }
  __syncthreads();
  if (wp != 0 || !col) return;
  double sum[NB * 4];
#pragma unroll
  for (int v = 0; v < NB * 4; ++v) {
    double acc = part[0][lane][v];
    for (int k = 1; k < 8; ++k) acc += part[k][lane][v];
    sum[v] = acc;
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int mem = nb * 8 + 2 * q + h;
      if (mem >= M) continue;
      const long long p = cb + (long long)(sn.c0 + j) * m + mem;
      const cplx s2 = cmk(sum[nb * 4 + h], sum[nb * 4 + 2 + h]);
      if (DIAG) {
        if ((A.flag[tr->t[mem]] != 0) != (A.flag_on != 0)) continue;
        A.X[p] = cadd(A.Y[p], s2);
      } else {
        A.Y[p] = csub(cmul(ldg(vals + sn.dinv_off + j), zval(A, it0.x, p)), s2);
      }
    }
}

// backward pull, thread per (column, member) (T.E == 1; items are columns):
// w_j = Dinv[j] X[j] - sum_rows L[r][j] X[dst r] into Y (in place into X for leaf
// columns). Rows are sorted by first stored column: column j walks only the
// rows that reach it.
template <bool TO_X>
__global__ void __launch_bounds__(kThreads) k_bwd_pull(SolveArgs A, TileArg T, const int2* items,
                                                       int nitem) {
  pdl_trigger();
  const TL L = tile_lane(A, T, nitem);
  const long long it = L.it;
  pdl_wait();
  if (!L.act) return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int j = item.y;
  const cplx* vals = A.vals + (long long)L.c * A.nvals;
  const BwRow* rows = A.bw + A.bw_ptr[item.x];
  const int nr = __ldg(A.bw_cnt + sn.c0 + j);
  const cplx acc = bw_gather<kUB>(vals, rows, 0, nr, 1, j, A.X + L.cb, L.m);
  const long long p = vat(L, sn.c0 + j);
  (TO_X ? A.X : A.Y)[p] = csub(cmul(ldg(vals + sn.dinv_off + j), zval(A, item.x, p)), acc);
}

// separator columns, backward diagonal: X[j] = Y[j] + sum_{i>j} Linv[i][j] Y[i]
// (thread per (column, member))
__global__ void __launch_bounds__(kThreads) k_bwd_diag(SolveArgs A, TileArg T, const int2* items,
                                                       int nitem) {
  pdl_trigger();
  const TL L = tile_lane(A, T, nitem);
  const long long it = L.it;
  pdl_wait();
  if (!L.act) return;
  const int2 item = items[it];
  const DevSn sn = A.sn[item.x];
  const int j = item.y;
  const int m = L.m;
  const cplx* yp = A.Y + vat(L, sn.c0 + j);
  cplx acc = *yp, acc2 = cmk(0, 0);
  int i = j + 1;
  // column j of the packed strictly-lower inverse (row i starts at i(i-1)/2):
  // rows i+1, i+2, i+3, i+4 are i, 2i+1, 3i+3, 4i+6 entries further
  const cplx* lp = A.vals + (long long)L.c * A.nvals + sn.diag_off + (long long)i * (i - 1) / 2 + j;
  yp += m;
  for (; i + 4 <= sn.n; i += 4) {
    const cplx l0 = ldf(lp);
    const cplx l1 = ldf(lp + i);
    const cplx l2 = ldf(lp + 2 * i + 1);
    const cplx l3 = ldf(lp + 3 * i + 3);
    const cplx y0 = yp[0], y1 = yp[m], y2 = yp[2 * m], y3 = yp[3 * m];
    cfma(acc, l0, y0);
    cfma(acc2, l1, y1);
    cfma(acc, l2, y2);
    cfma(acc2, l3, y3);
    lp += 4 * i + 6;
    yp += 4 * m;
  }
  for (; i < sn.n; ++i) {
    cfma(acc, ldf(lp), *yp);
    lp += i;
    yp += m;
  }
  A.X[vat(L, sn.c0 + j)] = cadd(acc, acc2);
}

// backward, CTA per (column group): lanes cover R = 32 / M columns x M members,
// the 8 warps split the inner range, partial sums combined in fixed warp order
// (top levels: few columns, long row lists / inverse columns). items: the
// group's first column.
constexpr int kSplitWarps = 8;  // k_bwd_split CTA: 8 warps share one column group

template <bool DIAG>
__global__ void __launch_bounds__(kSplitWarps * 32) k_bwd_split(SolveArgs A, TileArg T, const int2* items,
                                                        int nitem) {
  __shared__ cplx part[kSplitWarps][32];
  pdl_trigger();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = blockIdx.x / nitem;  // CTA per (tile, column group)
  TL L;
  L.r = int(udiv(unsigned(lane), T.M, T.magM));
  L.k = lane - L.r * T.M;
  L.e = 0;
  L.it = 0;
  tile_fill(A, T, ti, L.r < T.R, L);
  const int2 item = items[blockIdx.x - ti * nitem];
  const DevSn sn = A.sn[item.x];
  const int j = item.y + L.r;
  const bool ok = L.act && j < sn.n;
  const cplx* vals = A.vals + (long long)L.c * A.nvals;
  cplx acc = cmk(0, 0);
  pdl_wait();
  if (ok) {
    if (DIAG) {
      const cplx* Linv = vals + sn.diag_off;
      const SVec<const cplx> y{A.Y + vat(L, sn.c0), L.m};
      for (int i = j + 1 + warp; i < sn.n; i += kSplitWarps)
        cfma(acc, ldf(Linv + (long long)i * (i - 1) / 2 + j), y[i]);
    } else {
      const BwRow* rows = A.bw + A.bw_ptr[item.x];
      const int nr = __ldg(A.bw_cnt + sn.c0 + j);
      acc = bw_gather<kUB>(vals, rows, warp, nr, kSplitWarps, j, A.X + L.cb, L.m);
    }
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && ok) {
    cplx sum = part[0][lane];
    for (int w = 1; w < kSplitWarps; ++w) sum = cadd(sum, part[w][lane]);
    const long long p = vat(L, sn.c0 + j);
    if (DIAG)
      A.X[p] = cadd(A.Y[p], sum);
    else
      A.Y[p] = csub(cmul(ldg(vals + sn.dinv_off + j), zval(A, item.x, p)), sum);
  }
}

// backward pull, staged through shared memory. CTA per (tile, column chunk
// [j0, j1) of supernode s). The rows reaching the chunk (a prefix of the list
// sorted by first column) are processed RC at a time: their descriptors, the
// tile members' x values (M contiguous per row) and the rows' factor entries
// for the chunk columns (a dense RC x CW tile, zero left of each row's first
// column) are copied with cp.async -- no registers held per load, one wait per
// row chunk -- then every (column, member) pair accumulates from shared memory.
// Pairs below the CTA size split the rows S ways (fixed-order combine).
// w_j = Dinv[j] X[j] - sum_rows L[r][j] X[dst r] into Y (X for leaf columns).
#ifndef HDDM_STAGE_THREADS
#define HDDM_STAGE_THREADS 128
#endif
#ifndef HDDM_STAGE_KB
#define HDDM_STAGE_KB 24  // measured best at config 4 (20-24 KB: 8 CTAs per SM)
#endif
constexpr int kStageThreads = HDDM_STAGE_THREADS;

// MODE 0: w -> Y (a diagonal kernel follows); 1: leaf columns, w -> X; 2: every chunk is a
// whole separator (n <= 32 columns): w stays in shared memory and the dense-inverse product
// x_j = w_j + sum_{i>j} Linv[i][j] w_i follows in the same CTA (one kernel less per level)
template <int MODE>
__global__ void __launch_bounds__(kStageThreads) k_bwd_stage(SolveArgs A, TileArg T,
                                                             const int4* chunks, int nchunk,
                                                             int RC, int CWmax) {
  extern __shared__ __align__(16) unsigned char smem[];
  pdl_trigger();
  const int ti = blockIdx.x / nchunk;
  const int4 ch = chunks[blockIdx.x - ti * nchunk];  // (supernode, j0, j1, rows reaching j1 - 1)
  const TileRec* rec = T.rec + ti;
  const int M = T.M, m = rec->m;
  const long long cb = rec->cb;
  const int tid = threadIdx.x;
  {  // a tile without any active member does nothing (uniform over the CTA)
    const bool a = tid < M && (A.flag[rec->t[tid]] != 0) == (A.flag_on != 0);
    if (!__syncthreads_or(a)) return;
  }
  const DevSn sn = A.sn[ch.x];
  const int j0 = ch.y, CW = ch.z - ch.y;
  const BwRow* rows = A.bw + A.bw_ptr[ch.x];
  const int nre = ch.w;  // rows reaching the chunk's last column (a prefix of the sorted list)
  const cplx* vals = A.vals + (long long)rec->c * A.nvals;
  cplx* xs = reinterpret_cast<cplx*>(smem);            // [RC][M]
  cplx* ls = xs + (size_t)RC * M;                        // [RC][CW]
  BwRow* rd = reinterpret_cast<BwRow*>(ls + (size_t)RC * CWmax);  // [RC]
  cplx* red = reinterpret_cast<cplx*>(rd + RC);          // [kStageThreads] split partials
  const int P = CW * M;                                  // (column, member) pairs
  // small quotients through a float reciprocal: n / d = int((n + 0.5f) * (1 / d)), exact for
  // n, d <= 1024 (the distance to the next integer is >= 0.5 / d, the error < 2e-5)
  const float rP = __frcp_rn(float(P));
  const int S = P >= kStageThreads ? 1 : int((kStageThreads + 0.5f) * rP);  // row splits
  const int sp = int((tid + 0.5f) * rP), pp = tid - sp * P;  // split mode: row split, pair
  constexpr int kMaxQ = 1024 / kStageThreads;  // pairs per thread (P <= 32 x 32)
  cplx acc[kMaxQ];
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) acc[q] = cmk(0, 0);
  pdl_wait();
  // staging lanes on (row, member) and (row, column) grids: no divisions in the loops
  const int xr = int(udiv(unsigned(tid), M, T.magM)), xm = tid - xr * M;
  const int xrows = int(udiv(unsigned(kStageThreads), M, T.magM));
  const float rCW = __frcp_rn(float(CW));
  const int lr = int((tid + 0.5f) * rCW), lc = tid - lr * CW, lrows = int((kStageThreads + 0.5f) * rCW);
  const cplx* Xb = A.X + cb + xm;
  for (int k0 = 0; k0 < nre; k0 += RC) {
    const int kc = min(RC, nre - k0);
    for (int kk = tid; kk < kc; kk += kStageThreads) rd[kk] = rows[k0 + kk];
    __syncthreads();
    if (xr < xrows)
      for (int kk = xr; kk < kc; kk += xrows) cp_async16(xs + kk * M + xm, Xb + (long long)rd[kk].dpos * m);
    if (lr < lrows) {
      const int j = j0 + lc;
      for (int kk = lr; kk < kc; kk += lrows) {
        const BwRow d = rd[kk];
        if (j >= d.first)
          cp_async16(ls + kk * CW + lc, vals + d.off + (j - d.first));
        else
          ls[kk * CW + lc] = cmk(0, 0);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (S == 1) {
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q) {
        const int p = tid + q * kStageThreads;
        if (p < P) {
          const int jj = int(udiv_here(unsigned(p), M, T.magM)), mm = p - jj * M;
          cplx a = acc[q], a2 = cmk(0, 0);
          int kk = 0;
          for (; kk + 1 < kc; kk += 2) {
            cfma(a, ls[kk * CW + jj], xs[kk * M + mm]);
            cfma(a2, ls[(kk + 1) * CW + jj], xs[(kk + 1) * M + mm]);
          }
          if (kk < kc) cfma(a, ls[kk * CW + jj], xs[kk * M + mm]);
          acc[q] = cadd(a, a2);
        }
      }
    } else if (sp < S) {
      const int jj = pp / M, mm = pp - jj * M;
      cplx a = acc[0];
      for (int kk = sp; kk < kc; kk += S) cfma(a, ls[kk * CW + jj], xs[kk * M + mm]);
      acc[0] = a;
    }
    __syncthreads();
  }
  if (S > 1) {  // combine the row splits in fixed order
    red[tid] = acc[0];
    __syncthreads();
    if (tid < P) {
      cplx a = red[tid];
      for (int k = 1; k < S; ++k) a = cadd(a, red[tid + k * P]);
      acc[0] = a;
    }
  }
  if (MODE == 2) {
    cplx* ws = xs;  // [CW][M]: the pulled w of the whole separator (the staging loop ended on a barrier)
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) {
      const int p = tid + q * kStageThreads;
      if (p < P && (S == 1 || q == 0)) {
        const int jj = int(udiv_here(unsigned(p), M, T.magM)), mm = p - jj * M;
        const long long a = cb + (long long)(sn.c0 + jj) * m + mm;
        ws[p] = csub(cmul(ldg(vals + sn.dinv_off + jj), zval(A, ch.x, a)), acc[q]);
      }
    }
    __syncthreads();
    const cplx* Linv = vals + sn.diag_off;
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) {
      const int p = tid + q * kStageThreads;
      if (p < P && (S == 1 || q == 0)) {
        const int jj = int(udiv_here(unsigned(p), M, T.magM)), mm = p - jj * M;
        if ((A.flag[rec->t[mm]] != 0) == (A.flag_on != 0)) {
          cplx x = ws[p], x2 = cmk(0, 0);
          int i = jj + 1;
          const cplx* lp = Linv + (long long)i * (i - 1) / 2 + jj;  // column jj of the packed inverse
          const cplx* wp = ws + i * M + mm;
          for (; i + 2 <= CW; i += 2) {
            const cplx l0 = ldf(lp), l1 = ldf(lp + i);
            cfma(x, l0, wp[0]);
            cfma(x2, l1, wp[M]);
            lp += 2 * i + 1;
            wp += 2 * M;
          }
          if (i < CW) cfma(x, ldf(lp), wp[0]);
          A.X[cb + (long long)(sn.c0 + jj) * m + mm] = cadd(x, x2);
        }
      }
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) {
    const int p = tid + q * kStageThreads;
    if (p < P && (S == 1 || q == 0)) {
      const int jj = int(udiv_here(unsigned(p), M, T.magM)), mm = p - jj * M;
      if ((A.flag[rec->t[mm]] != 0) == (A.flag_on != 0)) {
        const int j = j0 + jj;
        const long long a = cb + (long long)(sn.c0 + j) * m + mm;
        (MODE == 1 ? A.X : A.Y)[a] = csub(cmul(ldg(vals + sn.dinv_off + j), zval(A, ch.x, a)), acc[q]);
      }
    }
  }
}

// leaves, backward band back-substitution on w (held in X): for i = n-1..0:
// x_i = w_i; w_q -= L[i][q] x_i for q in [first_i, i). Rows streamed from the
// end of the leaf's band (see k_fwd_leaf), the next row's entries in flight;
// register window of the next kBand pending w values. Thread per (leaf, member).
__global__ void __launch_bounds__(kThreads) k_bwd_leaf(SolveArgs A, TileArg T, const int2* items,
                                                       int nitem) {
  pdl_trigger();
  const TL L = tile_lane(A, T, nitem);
  const long long it = L.it;
  pdl_wait();
  if (!L.act) return;
  const DevSn sn = A.sn[items[it].x];
  const int w = sn.lw, n = sn.n;
  const cplx* base = A.vals + (long long)L.c * A.nvals + sn.diag_off;
  long long tot = 0;  // entries of the whole band
  for (int i = 0; i < n; ++i) tot += i - leaf_first(i, w);
  const cplx* p = base + tot;  // one past row n-1
  const SVec<cplx> x{A.X + vat(L, sn.c0), L.m};
  cplx wv[kBand + 1];  // wv[d] = pending w_{i-d}
#pragma unroll
  for (int d = 0; d <= kBand; ++d) wv[d] = (n - 1 - d >= 0) ? x[n - 1 - d] : cmk(0, 0);
  cplx lv[kBand + 1];
  {
    const int c = n > 0 ? n - 1 - leaf_first(n - 1, w) : 0;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = d <= c ? ldf(p - d) : cmk(0, 0);
    p -= c;  // start of row n-1
  }
  for (int i = n - 1; i >= 0; --i) {
    const int cn = i > 0 ? i - 1 - leaf_first(i - 1, w) : 0;  // row i-1
    cplx ln[kBand + 1];
#pragma unroll
    for (int d = 1; d <= kBand; ++d) ln[d] = d <= cn ? ldf(p - d) : cmk(0, 0);
    const cplx nxt = (i - 1 - kBand >= 0) ? x[i - 1 - kBand] : cmk(0, 0);
    const cplx xi = wv[0];
    x[i] = xi;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) csub_mul(wv[d], lv[d], xi);
#pragma unroll
    for (int d = 0; d < kBand; ++d) wv[d] = wv[d + 1];
    wv[kBand] = nxt;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = ln[d];
    p -= cn;
  }
}


// Separator diagonal blocks by substitution with L_ss itself (the reference's
// solve_raw order of operations, sparse.cpp:244-266) instead of an explicit
// inverse: the inverse's rounding amplification pushed first-pass residuals over
// refine's 1e-11 (config 4: 1.3e-11 with inverses, 5.5e-12 substituting, 8.2e-12
// in the reference), and every crossing costs a whole correction solve.
// A warp per (separator, member): lane l holds rows l, l+32, ... of the block in
// registers; step i broadcasts the finished x_i from its owner lane and every lane
// updates its rows below i with column i of L_ss (column-major packed: coalesced).
// The backward (L^T) sweep runs j = n-1..0 with row j of L_ss (row-major packed).
constexpr int kTrsvR = 2;  // rows per lane: separators up to 64 nodes

// CTA per (tile, separator): the block (n(n-1)/2 entries, column-major for the
// forward, row-major for the backward) is staged in shared memory once, then warp
// k sweeps member k's right-hand side through it.
template <bool BWD>
__global__ void __launch_bounds__(512) k_sep_trsv(SolveArgs A, TileArg T, const int2* __restrict__ seps,
                                                  int nsep) {
  extern __shared__ __align__(16) unsigned char smem[];
  cplx* Ls = reinterpret_cast<cplx*>(smem);
  const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int ti = blockIdx.x / nsep, is = blockIdx.x - ti * nsep;
  const TileRec* rec = T.rec + ti;
  const int s = seps[is].x;
  const DevSn sn = A.sn[s];
  const int n = sn.n, m = rec->m, M = T.M;
  const long long nl = (long long)n * (n - 1) / 2;
  const cplx* L = (BWD ? A.lss : A.lssc) + (long long)rec->c * A.nlss + A.lss_off[s];
  for (long long e = threadIdx.x; e < nl; e += blockDim.x) Ls[e] = ldf(L + e);
  __syncthreads();
  if (k >= M) return;
  if ((A.flag[rec->t[k]] != 0) != (A.flag_on != 0)) return;  // warp-uniform
  const long long vb = rec->cb + k + (long long)sn.c0 * m;
  cplx v[kTrsvR];
#pragma unroll
  for (int r = 0; r < kTrsvR; ++r) {
    const int i = lane + 32 * r;
    v[r] = i < n ? A.Y[vb + (long long)i * m] : cmk(0, 0);
  }
  if (!BWD) {
#pragma unroll
    for (int rs = 0; rs < kTrsvR; ++rs) {
      if (32 * rs >= n) break;
      for (int ii = 0; ii < 32; ++ii) {
        const int i = 32 * rs + ii;
        if (i >= n) break;
        const cplx xi = cmk(__shfl_sync(0xffffffffu, v[rs].x, ii), __shfl_sync(0xffffffffu, v[rs].y, ii));
        const cplx* col = Ls + (long long)i * (n - 1) - (long long)i * (i - 1) / 2 - (i + 1);  // col[kk] = L[kk][i]
#pragma unroll
        for (int r = rs; r < kTrsvR; ++r) {
          const int kk = lane + 32 * r;
          if (kk > i && kk < n) csub_mul(v[r], col[kk], xi);
        }
      }
    }
  } else {
#pragma unroll
    for (int rs = kTrsvR - 1; rs >= 0; --rs) {
      if (32 * rs >= n) continue;
      for (int jj = 31; jj >= 0; --jj) {
        const int j = 32 * rs + jj;
        if (j >= n) continue;
        const cplx xj = cmk(__shfl_sync(0xffffffffu, v[rs].x, jj), __shfl_sync(0xffffffffu, v[rs].y, jj));
        const cplx* row = Ls + (long long)j * (j - 1) / 2;  // row[i] = L[j][i], i < j
#pragma unroll
        for (int r = 0; r <= rs; ++r) {
          const int i = lane + 32 * r;
          if (i < j) csub_mul(v[r], row[i], xj);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kTrsvR; ++r) {
    const int i = lane + 32 * r;
    if (i < n) A.X[vb + (long long)i * m] = v[r];
  }
}

// count the launches of a solve without launching (solve_launch_count); per host thread,
// so a dry run never swallows another thread's launches
static thread_local bool g_dry = false;
static thread_local int g_count = 0;

template <bool BWD>
static void launch_sep_trsv(const SolveArgs& A, const TileArg& T, const SolveLevel& L, cudaStream_t st) {
  const size_t smem = size_t(L.nmax_sep) * (L.nmax_sep - 1) / 2 * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sep_trsv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_sep_trsv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr = true;
  }
  ++g_count;
  if (g_dry) return;
  k_sep_trsv<BWD><<<unsigned(T.ntile * L.nsep), 32 * T.M, smem, st>>>(A, T, (const int2*)L.d_seps, L.nsep);
}

// ------------------------------------------------------------------ launcher
static thread_local bool g_pdl = false;   // the chain being enqueued (SolvePlan::pdl)

// launch with programmatic stream serialization (see pdl_trigger / pdl_wait)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       cudaStream_t st, Args... args) {
  if (grid == 0) return;
  ++g_count;
  if (g_dry) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

static unsigned blocks_for(long long threads) {
  return unsigned((threads + kThreads - 1) / kThreads);
}

static int pow2_floor(long v) {
  int p = 1;
  while (2L * p <= v) p <<= 1;
  return p;
}

// lanes per output for a forward pull/diagonal level with mean inner length avg
// (tuning knobs HDDM_FWD_DIV / HDDM_FWD_WIDE). Two parameter sets: the full-RHS plan
// (step 1, class solves, refinement corrections) and the steady-state sparse-RHS plan of
// steps >= 2. Singleton tiles take E = avg / div lanes per row: re-measured on the round's
// final kernels (tools/run42.sh, run43.sh) div = 16 (full), 8 (sparse) and 2 for the inverse
// rows -- twice the lanes of the round-1 values: config 3 step 1.632 -> 1.414 ms, config 1
// 0.451 -> 0.383, config 2 0.721 -> 0.705; config 4 (member tiles: E from HDDM_FWD_WIDE)
// does not move, and per-level tuning (tools/tune_fwd_shapes.py) found no better point.
static long env_long(const char* name, long dflt) {
  const char* v = std::getenv(name);
  return v ? std::atol(v) : dflt;
}

static int fwd_lanes(int M, long avg, bool diag = false, bool sparse = false) {
  static const long div_pull = env_long("HDDM_FWD_DIV", 16), div_pull_sp = env_long("HDDM_FWD_DIV_SP", 8);
  static const long div_diag = env_long("HDDM_DIAG_DIV", 2);
  static const long wide = env_long("HDDM_FWD_WIDE", 16), wide_sp = env_long("HDDM_FWD_WIDE_SP", 6);
  const long div = diag ? div_diag : (sparse ? div_pull_sp : div_pull);
  if (M == 1) return std::max(1, std::min(32, pow2_floor(avg / div)));
  if (avg > (sparse ? wide_sp : wide)) return std::max(1, pow2_floor(32 / M));
  return 1;
}

// Lane shape of a forward level: the heuristic fwd_lanes, or (tuning aid) a per-level
// override for the steady-state (sparse-RHS) plan: HDDM_FWDP_E1 / HDDM_FWDP_EM (pulls of
// singleton / member tiles) and HDDM_FWDD_E1 / HDDM_FWDD_EM (inverse rows), comma lists
// of E per level (0: heuristic)
static std::vector<int> g_fwd_tab[4];

void set_fwd_shape(int which, int level, int E) {
  if (which < 0 || which > 3 || level < 0 || level > 64) return;
  std::vector<int>& t = g_fwd_tab[which];
  if (int(t.size()) <= level) t.resize(level + 1, 0);
  t[level] = E;
}

static int fwd_shape(int M, long avg, bool diag, bool sparse, int level) {
  const int E = fwd_lanes(M, avg, diag, sparse);
  if (!sparse) return E;
  std::vector<int>* tab = g_fwd_tab;
  static bool init = false;
  if (!init) {
    const char* names[4] = {"HDDM_FWDP_E1", "HDDM_FWDP_EM", "HDDM_FWDD_E1", "HDDM_FWDD_EM"};
    for (int k = 0; k < 4; ++k)
      if (const char* v = std::getenv(names[k]))
        for (const char* q = v; *q;) {
          tab[k].push_back(std::atoi(q));
          while (*q && *q != ',') ++q;
          if (*q) ++q;
        }
    init = true;
  }
  const std::vector<int>& t = tab[(diag ? 2 : 0) + (M > 1 ? 1 : 0)];
  if (level < int(t.size()) && t[level] > 0 && t[level] * M <= 32) return t[level];
  return E;
}

static TileArg with_shape(TileArg T, int E) {
  T.E = E;
  T.R = std::max(1, 32 / (E * T.M));
  tile_mags(T);
  return T;
}

// Profiling aid for hddm_time_solve (results invalid): HDDM_SKIP is a bit mask of kernel families
// left out of the solve -- 1 ring, 2 forward leaves, 4 forward pulls, 8 forward
// diagonals, 16 backward pulls, 32 backward diagonals, 64 leaf columns,
// 128 backward leaves -- so their marginal cost in the concurrent graph can be
// timed.
static int g_skip = 0, g_only = -1;
static int skip_mask() { return g_skip; }
void set_solve_skip(int mask, int only_tile) {
  g_skip = mask;
  g_only = only_tile;
}

// staged backward pull over a level's column chunks
template <int MODE>
static void launch_bwd_stage(const SolveArgs& A, const TileArg& T, const SolveLevel& L,
                             cudaStream_t st) {
  constexpr int kBudget = HDDM_STAGE_KB * 1024;  // staging buffer per CTA
  const int rowb = (T.M + L.cw_max + 1) * int(sizeof(cplx));
  const int RC = std::max(1, (kBudget - kStageThreads * int(sizeof(cplx))) / rowb);
  const size_t smem = size_t(RC) * rowb + kStageThreads * sizeof(cplx);
  launch_pdl(k_bwd_stage<MODE>, unsigned((long long)T.ntile * L.nchunk4), kStageThreads, smem, st,
             A, T, (const int4*)L.d_chunks4, L.nchunk4, RC, L.cw_max);
}

// one tile group's full solve on one stream
void launch_solve_group(const SolveArgs& A0, const SolvePlan& P, int g, cudaStream_t st) {
  const int skip = skip_mask();
  if (g_only >= 0 && g != g_only) return;
  if (g_only <= -2 && P.groups[g].M != -2 - g_only) return;  // HDDM_ONLY_M (time_solve only)
  const TileArg T1 = with_shape(P.groups[g], 1);  // thread per (item, member)
  g_pdl = P.pdl == 1 || (P.pdl == 2 && P.groups[g].M == 1);
  // substitution for the mid-size separators: tiles of at least this many members
  static const int subst_min_m = std::getenv("HDDM_SUBST_MIN_M") ? std::atoi(std::getenv("HDDM_SUBST_MIN_M")) : 2;
  const long long nt = T1.ntile;
  auto blocks = [nt](long long items, int R) { return blocks_for(nt * ((items + R - 1) / R) * 32); };
  // sparse RHS (steps >= 2): patch-free subtrees are skipped (z = 0, see zval)
  const bool sp = A0.sparse_rhs && P.has_sparse;
  SolveArgs A = A0;
  A.fseg = sp ? P.d_fseg_sp : P.d_fseg;
  A.sn_live = sp ? P.d_sn_live : nullptr;
  if (!(skip & 1)) {
    ++g_count;
    if (!g_dry) k_ring<<<blocks(A.nring, T1.R), kThreads, 0, st>>>(A, T1);
  }
  const SolveLevel& FL = sp ? P.fwd_leaf_sp : P.fwd_leaf;
  if (!(skip & 2) && FL.nitem > 0)
    launch_pdl(k_fwd_leaf, blocks(FL.nitem, T1.R), kThreads, 0, st, A, T1, (const int2*)FL.d_items,
               FL.nitem);
  const TileArg& TS = P.sub[g];  // 2-member sub-tiles (ntile 0: none)
  auto blocks_n = [](long long ntile, long long items, int R) {
    return blocks_for(ntile * ((items + R - 1) / R) * 32);
  };
  for (const auto& L : (sp ? P.fwd_sp : P.fwd)) {
    if (L.nitem == 0) continue;
    if (TS.ntile > 0 && L.avg_run > P.sub_run) {  // long rows: sub-tiles
      const TileArg Tp = with_shape(TS, fwd_lanes(TS.M, L.avg_run));
      if (!(skip & 4))
        launch_pdl(Tp.M == 1 ? k_fwd_pull<true> : k_fwd_pull<false>, blocks_n(Tp.ntile, L.nitem, Tp.R), kThreads, 0, st, A, Tp,
                   (const int4*)L.d_rec, L.nitem);
      const TileArg Td = with_shape(TS, fwd_lanes(TS.M, L.avg_diag, true));
      if (!(skip & 8))
        launch_pdl(k_fwd_diag, blocks_n(Td.ntile, L.nitem, Td.R), kThreads, 0, st, A, Td,
                   (const int2*)L.d_items, L.nitem);
      continue;
    }
    const int li = int(&L - (sp ? P.fwd_sp.data() : P.fwd.data()));
    // member tiles: the tensor-core pull (HDDM_MMA_PULL=0: the lane-per-member kernel)
    // on levels whose 8-row blocks pad the runs by at most HDDM_MMA_FILL
    static const bool mma_pull = !(std::getenv("HDDM_MMA_PULL") && std::getenv("HDDM_MMA_PULL")[0] == '0');
    static const double mma_fill = std::getenv("HDDM_MMA_FILL") ? std::atof(std::getenv("HDDM_MMA_FILL")) : 1.3;
    // the dense-inverse rows on the tensor cores for separators with long rows only
    static const long mma_diag_min = std::getenv("HDDM_MMA_DIAG_MIN") ? std::atol(std::getenv("HDDM_MMA_DIAG_MIN")) : 32;
    if (skip & 4) {
    } else if (mma_pull && T1.M >= 2 && T1.M <= 16 && L.nmblk > 0 && L.mma_fill <= mma_fill) {
      const unsigned g = unsigned(nt * L.nmblk);  // CTA per (tile, block)
      if (T1.M <= 8)
        launch_pdl(k_fwd_pull_mma<1>, g, 256, 0, st, A, T1, (const int4*)L.d_rec, (const int4*)L.d_mblk,
                   (const MmaSeg*)L.d_mseg, L.nmblk);
      else
        launch_pdl(k_fwd_pull_mma<2>, g, 256, 0, st, A, T1, (const int4*)L.d_rec, (const int4*)L.d_mblk,
                   (const MmaSeg*)L.d_mseg, L.nmblk);
    } else {
      const TileArg Tp = with_shape(T1, fwd_shape(T1.M, L.avg_run, false, sp, li));
      launch_pdl(Tp.M == 1 ? k_fwd_pull<true> : k_fwd_pull<false>, blocks(L.nitem, Tp.R), kThreads, 0, st, A, Tp, (const int4*)L.d_rec,
                 L.nitem);
    }
    if (skip & 8) {
    } else if (A.lss && L.nsep > 0 && T1.M >= subst_min_m && T1.M <= 16) {
      launch_sep_trsv<false>(A, T1, L, st);
    } else if (mma_pull && T1.M >= 2 && T1.M <= 16 && L.nmblk > 0 && L.avg_diag >= mma_diag_min) {
      const unsigned g = unsigned(nt * L.nmblk);
      if (T1.M <= 8)
        launch_pdl(k_fwd_diag_mma<1>, g, 256, 0, st, A, T1, (const int2*)L.d_items, (const int4*)L.d_mblk,
                   L.nmblk);
      else
        launch_pdl(k_fwd_diag_mma<2>, g, 256, 0, st, A, T1, (const int2*)L.d_items, (const int4*)L.d_mblk,
                   L.nmblk);
    } else {
      const TileArg Td = with_shape(T1, fwd_shape(T1.M, L.avg_diag, true, sp, li));
      launch_pdl(k_fwd_diag, blocks(L.nitem, Td.R), kThreads, 0, st, A, Td, (const int2*)L.d_items,
                 L.nitem);
    }
  }
  for (const auto& L : P.bwd) {
    // split kernels: one CTA per (tile, group of R = 32 / M consecutive columns)
    const auto grp = L.groups.find(T1.R);
    const bool has_grp = grp != L.groups.end();
    const unsigned gs = has_grp ? unsigned(nt * grp->second.first) : 0;
    // staging pays for multi-member tiles; singletons pull per thread (measured)
    static const int stage_min_m =
        std::getenv("HDDM_STAGE_MIN_M") ? std::atoi(std::getenv("HDDM_STAGE_MIN_M")) : 2;
    const bool staged = P.staged && T1.M >= stage_min_m;
    const bool use_sub = staged && TS.ntile > 0 && (long long)T1.ntile * L.nchunk4 < P.sub_bwd_ctas;
    static const bool mma_bwd = !(std::getenv("HDDM_MMA_BWD") && std::getenv("HDDM_MMA_BWD")[0] == '0');
    const bool mma_ok = mma_bwd && T1.M >= 2 && T1.M <= 16 && L.nmblk > 0;
    const unsigned gm = unsigned(nt * L.nmblk);
    // the pulls stay on the staged kernel (measured: the tensor-core pull 1.699 -> 1.731 ms
    // per config-4 step); HDDM_MMA_BPULL=1 selects it
    static const bool mma_bpull = std::getenv("HDDM_MMA_BPULL") && std::getenv("HDDM_MMA_BPULL")[0] == '1';
    static const long mma_bdiag_min =
        std::getenv("HDDM_MMA_DIAG_MIN") ? std::atol(std::getenv("HDDM_MMA_DIAG_MIN")) : 32;
    // small separators (one staged chunk each, dense inverse): pull and inverse product in
    // one kernel (HDDM_FUSE_BWD=0: two kernels)
    static const bool fuse_bwd = !(std::getenv("HDDM_FUSE_BWD") && std::getenv("HDDM_FUSE_BWD")[0] == '0');
    const bool trsv = A.lss && L.nsep > 0 && T1.M >= subst_min_m && T1.M <= 16;
    const bool fuse = fuse_bwd && staged && !use_sub && L.one_chunk && !trsv && !(skip & 48) &&
                      !(mma_ok && (mma_bpull || L.avg_diag >= mma_bdiag_min));
    if (skip & 16) {
    } else if (mma_ok && mma_bpull) {
      if (T1.M <= 8)
        launch_pdl(k_bwd_mma<1, false>, gm, 256, 0, st, A, T1, (const int2*)L.d_items, (const int4*)L.d_mblk, L.nmblk);
      else
        launch_pdl(k_bwd_mma<2, false>, gm, 256, 0, st, A, T1, (const int2*)L.d_items, (const int4*)L.d_mblk, L.nmblk);
    } else if (fuse) {
      launch_bwd_stage<2>(A, T1, L, st);
      continue;
    } else if (staged)
      launch_bwd_stage<0>(A, use_sub ? with_shape(TS, 1) : T1, L, st);
    else if (L.split_rows && has_grp)
      launch_pdl(k_bwd_split<false>, gs, kSplitWarps * 32, 0, st, A, T1, (const int2*)grp->second.second,
                 grp->second.first);
    else
      launch_pdl(k_bwd_pull<false>, blocks(L.nitem, T1.R), kThreads, 0, st, A, T1,
                 (const int2*)L.d_items, L.nitem);
    if (skip & 32) {
    } else if (A.lss && L.nsep > 0 && T1.M >= subst_min_m && T1.M <= 16) {
      launch_sep_trsv<true>(A, T1, L, st);
    } else if (mma_ok && L.avg_diag >= mma_bdiag_min) {
      if (T1.M <= 8)
        launch_pdl(k_bwd_mma<1, true>, gm, 256, 0, st, A, T1, (const int2*)L.d_items, (const int4*)L.d_mblk, L.nmblk);
      else
        launch_pdl(k_bwd_mma<2, true>, gm, 256, 0, st, A, T1, (const int2*)L.d_items, (const int4*)L.d_mblk, L.nmblk);
    } else if (L.split_diag && has_grp)
      launch_pdl(k_bwd_split<true>, gs, kSplitWarps * 32, 0, st, A, T1, (const int2*)grp->second.second,
                 grp->second.first);
    else
      launch_pdl(k_bwd_diag, blocks(L.nitem, T1.R), kThreads, 0, st, A, T1, (const int2*)L.d_items,
                 L.nitem);
  }
  const SolveLevel& BC = P.bwd_leafcol;
  if (!(skip & 64)) {
    static const int leaf_min_m =
        std::getenv("HDDM_LEAF_STAGE_MIN_M") ? std::atoi(std::getenv("HDDM_LEAF_STAGE_MIN_M")) : 2;
    if (P.staged && T1.M >= leaf_min_m)
      launch_bwd_stage<1>(A, T1, BC, st);
    else
      launch_pdl(k_bwd_pull<true>, blocks(BC.nitem, T1.R), kThreads, 0, st, A, T1,
                 (const int2*)BC.d_items, BC.nitem);
  }
  const SolveLevel& BL = P.bwd_leaf;
  if (!(skip & 128))
    launch_pdl(k_bwd_leaf, blocks(BL.nitem, T1.R), kThreads, 0, st, A, T1, (const int2*)BL.d_items,
               BL.nitem);
}

// kernels of one solve over all tile groups: a dry run of the launch logic
int solve_launch_count(const SolvePlan& P, const SolveArgs& A) {
  g_dry = true;
  g_count = 0;
  for (int g = 0; g < int(P.groups.size()); ++g) launch_solve_group(A, P, g, nullptr);
  g_dry = false;
  return g_count;
}

}  // namespace hddm
