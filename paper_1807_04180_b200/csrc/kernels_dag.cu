// Dataflow supernodal solve (the per-step hot path replacing Factorization::solve
// -> solve_raw, proj/src/sparse.cpp:244-266, for every subdomain of a step).
//
// ONE persistent kernel per solve: CTAs take tasks (tile, unit, sweep) from an
// atomic ticket in topological order (dag_plan.cu), wait for the task's own
// predecessors through release/acquire flags, run it, and publish it. A task
// holds the tile's members' vectors of its unit in shared memory:
//
//   forward (L z = b), per level of the unit, bottom-up:
//     gather   y_p = b_p - sum of the partials pushed into p (fixed order)
//     diagonal leaves: band substitution; separators: blocked -- z_b = Xinv_b y_b on
//              each kDiagBlk block (inverted at factor time), then the rows below
//              y_i -= L[i, b] z_b (column-major copy F: lanes over rows coalesce)
//     push     partial_r = L[r, s] . z_s for every block row r of s (column-major:
//              a lane per row, the supernode's z broadcast from shared memory),
//              into shared memory (inside the unit) or a global slot (leaving it;
//              a subtree unit first merges all its partials per target)
//   backward (L^T x = D^{-1} z), per level, top-down:
//     columns  w_j = z_j / D_j - sum_r L[r][j] x_r (row-major copy B: a lane per
//              column, the rows' x and descriptors staged in shared memory)
//     diagonal the transposed blocked solve
//
// Members of a tile beyond 8 are processed in groups of 8 (registers: one
// accumulator per member). Every output has one writer and a fixed summation
// order: results are deterministic. Data written by other CTAs (X, partials) is
// read through L2 (ld.global.cg) after the acquire; inner loops issue their
// factor loads in batches of kU before consuming them.
#include "dag.cuh"
#include "kernels.cuh"

namespace hddm {

namespace {

constexpr int kU = 8;       // loads in flight per lane in the gather loops
constexpr int kMG = 8;      // members per register group
constexpr int kLvSn = 64;   // supernodes of one level staged in shared memory
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// wait for a published task: relaxed polling, then one acquire fence
__device__ __forceinline__ void wait_done(const int* p) {
  while (ld_relaxed(p) == 0) __nanosleep(32);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ cplx ldcg(const cplx* p) { return __ldcg(p); }
// factor entries: shared memory (staged units) or global memory (generic load)
__device__ __forceinline__ cplx ldv(const cplx* p) { return *p; }

// ---- bulk copies (TMA engine) of a unit's factor values into shared memory
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// [src, src + bytes) -> dst (16-byte aligned, bytes a multiple of 16), completion on bar
// (the caller registered the bytes with mbar_expect_tx)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  while (bytes > 0) {
    const unsigned c = bytes > 32768u ? 32768u : bytes;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(d)),
                 "l"(s), "r"(c), "r"(smem_u32(bar))
                 : "memory");
    s += c;
    d += c;
    bytes -= c;
  }
}
__device__ __forceinline__ void csubmul(cplx& acc, cplx l, cplx x) {
  acc.x = fma(-l.x, x.x, acc.x);
  acc.x = fma(l.y, x.y, acc.x);
  acc.y = fma(-l.x, x.y, acc.y);
  acc.y = fma(-l.y, x.x, acc.y);
}

__device__ __forceinline__ int leaf_first(int i, int w) { return i < w ? (i > 0 ? i - 1 : 0) : i - w; }
constexpr int kBand = 6;  // a leaf row holds at most kBand entries (checked by the plan)

// bulk prefetch of [p, p + n) complex into L2
__device__ __forceinline__ void prefetch_range(const cplx* p, long long n) {
  const char* a = reinterpret_cast<const char*>(p);
  long long bytes = n * (long long)sizeof(cplx);
  while (bytes > 0) {
    const unsigned chunk = unsigned(bytes > 65536 ? 65536 : bytes);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(chunk) : "memory");
    a += chunk;
    bytes -= chunk;
  }
}

// Phase profile (profiling builds only, -DHDDM_DAG_PROF): thread 0 accumulates
// clock64 deltas between the CTA-wide barriers per task category
// (sweep, unit kind, M > 1) and phase; read with hddm_dag_profile.
#ifdef HDDM_DAG_PROF
__shared__ long long g_pacc[8];
__shared__ long long g_plast;
__shared__ long long g_ptail;  // end of the previous task: the gap to the next is phase 5
__shared__ int g_ptail_cat;
#define DPROF(ph)                     \
  do {                                \
    if (threadIdx.x == 0) {           \
      const long long t_ = clock64(); \
      g_pacc[ph] += t_ - g_plast;     \
      g_plast = t_;                   \
    }                                 \
  } while (0)
#else
#define DPROF(ph) \
  do {            \
  } while (0)
#endif

struct TaskCtx {
  DagTile T;
  DagUnit U;
  unsigned act;  // bit k: member k is an active right-hand side
};

// the supernodes of the current level (staged once per level)
struct LvCache {
  DagSn sn[kLvSn];
  int rb[kLvSn];  // offset of each one's rows in the level's row list
};

__device__ __forceinline__ void stage_level(const DagArgs& A, const DagDec& D, const DagLv& L, LvCache& c) {
  for (int i = threadIdx.x; i < L.ns; i += blockDim.x) {
    c.sn[i] = D.lvsn[L.s0 + i];
    c.rb[i] = D.lsr[L.s0 + i];
  }
  __syncthreads();
}

// ---------------------------------------------------------------- leaves
// band forward substitution of one leaf for one member (stride M in y): row i+1's
// entries are loaded while row i computes; the last kBand z values in registers
__device__ __forceinline__ void leaf_fwd(cplx* y, int M, const cplx* band, int n, int w) {
  cplx win[kBand + 1];
#pragma unroll
  for (int d = 0; d <= kBand; ++d) win[d] = cmk(0, 0);
  cplx lv[kBand + 1];
  const cplx* p = band;
  {
    const int c0 = 0;  // row 0 has no entries
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = d <= c0 ? ldv(p + c0 - d) : cmk(0, 0);
  }
  for (int i = 0; i < n; ++i) {
    const int cnt = i - leaf_first(i, w);
    const cplx* pn = p + cnt;
    const int cn = (i + 1 < n) ? i + 1 - leaf_first(i + 1, w) : 0;
    cplx ln[kBand + 1];
#pragma unroll
    for (int d = 1; d <= kBand; ++d) ln[d] = d <= cn ? ldv(pn + cn - d) : cmk(0, 0);
    cplx acc = y[(long long)i * M];
#pragma unroll
    for (int d = 1; d <= kBand; ++d) csubmul(acc, lv[d], win[d]);
#pragma unroll
    for (int d = kBand; d >= 2; --d) win[d] = win[d - 1];
    win[1] = acc;
    y[(long long)i * M] = acc;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = ln[d];
    p = pn;
  }
}

// band back substitution on w (held in y, stride M): x_i = w_i, w_q -= L[i][q] x_i
__device__ __forceinline__ void leaf_bwd(cplx* y, int M, const cplx* band, int n, int w) {
  long long tot = 0;
  for (int i = 0; i < n; ++i) tot += i - leaf_first(i, w);
  const cplx* p = band + tot;  // one past row n-1
  cplx wv[kBand + 1];
#pragma unroll
  for (int d = 0; d <= kBand; ++d) wv[d] = (n - 1 - d >= 0) ? y[(long long)(n - 1 - d) * M] : cmk(0, 0);
  cplx lv[kBand + 1];
  {
    const int c = n > 0 ? n - 1 - leaf_first(n - 1, w) : 0;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = d <= c ? ldv(p - d) : cmk(0, 0);
    p -= c;
  }
  for (int i = n - 1; i >= 0; --i) {
    const int cn = i > 0 ? i - 1 - leaf_first(i - 1, w) : 0;
    cplx ln[kBand + 1];
#pragma unroll
    for (int d = 1; d <= kBand; ++d) ln[d] = d <= cn ? ldv(p - d) : cmk(0, 0);
    const cplx nxt = (i - 1 - kBand >= 0) ? y[(long long)(i - 1 - kBand) * M] : cmk(0, 0);
    const cplx xi = wv[0];
    y[(long long)i * M] = xi;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) csubmul(wv[d], lv[d], xi);
#pragma unroll
    for (int d = 0; d < kBand; ++d) wv[d] = wv[d + 1];
    wv[kBand] = nxt;
#pragma unroll
    for (int d = 1; d <= kBand; ++d) lv[d] = ln[d];
    p -= cn;
  }
}


// ---------------------------------------------------------------- forward
// push of a level of a unit whose values sit in shared memory: thread per (block
// row, member), the row's column-major entries and z from shared memory; cof holds
// the column offsets of the unit's positions
__device__ __forceinline__ void push_staged(const DagArgs& A, const DagDec& D, const DagLv& L,
                                            const LvCache& lc, const TaskCtx& C, const cplx* VF,
                                            const cplx* ys, const int* cof, cplx* sl, cplx* Pv) {
  const int M = C.T.M;
  const int pos0 = C.U.pos0;
  for (int idx = threadIdx.x; idx < L.nrow * M; idx += blockDim.x) {
    const int f = idx / M, k = idx - f * M;
    const int4 q4 = __ldg(D.lrm + L.r0 + f);  // (dpos, first, boff, si)
    const DagSn& S = lc.sn[q4.w];
    const int rr = f - lc.rb[q4.w];
    const cplx* colp = VF + S.frows + rr;
    const int* co = cof + (S.c0 - pos0);
    const cplx* z = ys + (long long)(S.c0 - pos0) * M + k;
    cplx acc = cmk(0, 0), acc2 = cmk(0, 0);
    int q = q4.y;
    for (; q + 1 < S.n; q += 2) {
      cfma(acc, colp[co[q]], z[(long long)q * M]);
      cfma(acc2, colp[co[q + 1]], z[(long long)(q + 1) * M]);
    }
    if (q < S.n) cfma(acc, colp[co[q]], z[(long long)q * M]);
    acc = cadd(acc, acc2);
    const int r = S.rs0 + rr;
    if (C.U.kind == 0)
      sl[(long long)(r - C.U.row0) * M + k] = acc;
    else
      Pv[(long long)(-D.row_slot[r] - 1) * M + k] = acc;
  }
}


// ---------------------------------------------------------------- backward
// columns of a level of a unit whose values sit in shared memory: thread per
// (column, member); ws holds z (bulk-loaded) and the x of the levels above, xs the x
// of the outside positions the rows reach (bulk-loaded)
__device__ void bwd_columns_staged(const DagArgs& A, const DagDec& D, const DagLv& L, const LvCache& lc,
                                   const TaskCtx& C, const cplx* VB, cplx* ws, const cplx* xs, bool zero_z) {
  const int M = C.T.M;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int pos0 = C.U.pos0;
  const int per = L.nmax * M;
  for (int idx = tid; idx < L.ns * per; idx += nt) {
    const int si = idx / per, rem = idx - si * per, j = rem / M, k = rem - j * M;
    const DagSn& S = lc.sn[si];
    if (j >= S.n) continue;
    const int pos = S.c0 + j;
    cplx* wp = ws + (long long)(pos - pos0) * M + k;
    const cplx z = zero_z ? cmk(0, 0) : *wp;
    const cplx* vrow = VB + S.brows + j;
    cplx acc = cmk(0, 0), acc2 = cmk(0, 0);
    const int fb = L.r0 + lc.rb[si], fe = fb + S.nrs;
    for (int f = fb; f < fe; ++f) {
      const int4 q = __ldg(D.lrm + f);  // (dpos, first, boff, si)
      if (q.y > j) break;               // rows sorted by first column
      const int src = __ldg(D.lrx + f);
      const cplx x = src >= 0 ? ws[(long long)src * M + k] : xs[(long long)(-src - 1) * M + k];
      cfma((f & 1) ? acc2 : acc, vrow[q.z - q.y], x);
    }
    acc = cadd(acc, acc2);
    *wp = csub(cmul(ldv(VB + S.bdinv + j), z), acc);
  }
}


// ---------------------------------------------------------------- separators
// Blocked forward substitution z = L_ss^{-1} y of the level's separators, all in
// shared memory (ys) with the panels of the forward copy at V (dev.cuh layout):
//   per panel b: z_b = Xinv_b y_b, then y_i -= L[i, b] z_b for the rows below.
__device__ void diag_fwd_staged(const LvCache& lc, const DagLv& L, const cplx* V, cplx* ys, int pos0, int M) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nb = (L.nmax + kDiagBlk - 1) / kDiagBlk;
  for (int b = 0; b < nb; ++b) {
    const int b0 = b * kDiagBlk;
    constexpr int kReg = 4;
    cplx zr[kReg];
    int zi[kReg];
    const int per = min(kDiagBlk, L.nmax - b0) * M;
    int nz = 0;
    for (int idx = tid; idx < L.ns * per && nz < kReg; idx += nt, ++nz) {
      const int si = idx / per, rem = idx - si * per, ii = rem / M, k = rem - ii * M;
      const DagSn& S = lc.sn[si];
      zi[nz] = -1;
      const int b1 = min(S.n, b0 + kDiagBlk), bw = b1 - b0;
      if (b0 + ii >= S.n) continue;
      const cplx* y = ys + (long long)(S.c0 - pos0 + b0) * M + k;
      const cplx* X = V + S.fdiag + fpanel_off(S.n, b);  // column-major strictly lower, size bw
      cplx acc = y[(long long)ii * M], acc2 = cmk(0, 0);
      for (int jj = 0; jj < ii; ++jj)
        cfma((jj & 1) ? acc2 : acc, X[(long long)jj * (bw - 1) - (long long)jj * (jj - 1) / 2 + (ii - jj - 1)],
             y[(long long)jj * M]);
      zr[nz] = cadd(acc, acc2);
      zi[nz] = int((S.c0 - pos0 + b0 + ii) * M + k);
    }
    __syncthreads();
    for (int u = 0; u < nz; ++u)
      if (zi[u] >= 0) ys[zi[u]] = zr[u];
    __syncthreads();
    if (b + 1 < nb) {  // rows below the block
      const int per2 = (L.nmax - b0 - kDiagBlk) * M;
      for (int idx = tid; idx < L.ns * per2; idx += nt) {
        const int si = idx / per2, rem = idx - si * per2, ii = rem / M, k = rem - ii * M;
        const DagSn& S = lc.sn[si];
        const int b1 = b0 + kDiagBlk, i = b1 + ii;
        if (i >= S.n) continue;
        const int bw = kDiagBlk, nl = S.n - b1;
        const cplx* Lb = V + S.fdiag + fpanel_off(S.n, b) + (long long)bw * (bw - 1) / 2 + ii;
        cplx* y = ys + (long long)(S.c0 - pos0) * M + k;
        cplx acc = y[(long long)i * M], acc2 = cmk(0, 0);
        for (int jj = 0; jj < bw; ++jj)
          csubmul((jj & 1) ? acc2 : acc, Lb[(long long)jj * nl], y[(long long)(b0 + jj) * M]);
        y[(long long)i * M] = cadd(acc, acc2);
      }
      __syncthreads();
    }
  }
}

// Blocked backward substitution x = L_ss^{-T} w, panels from the last (backward copy):
//   w_b -= L[below, b]^T x_below, then x_b = Xinv_b^T w_b.
__device__ void diag_bwd_staged(const LvCache& lc, const DagLv& L, const cplx* V, cplx* ws, int pos0, int M) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nb = (L.nmax + kDiagBlk - 1) / kDiagBlk;
  for (int b = nb - 1; b >= 0; --b) {
    const int b0 = b * kDiagBlk;
    const int per = min(kDiagBlk, L.nmax - b0) * M;
    if (b + 1 < nb) {
      for (int idx = tid; idx < L.ns * per; idx += nt) {
        const int si = idx / per, rem = idx - si * per, jj = rem / M, k = rem - jj * M;
        const DagSn& S = lc.sn[si];
        const int b1 = min(S.n, b0 + kDiagBlk), bw = b1 - b0;
        if (b0 + jj >= S.n || b1 >= S.n) continue;
        const cplx* Lb = V + S.bdiag + bpanel_off(S.n, b) + jj;  // row-major rows below
        cplx* w = ws + (long long)(S.c0 - pos0) * M + k;
        cplx acc = w[(long long)(b0 + jj) * M], acc2 = cmk(0, 0);
        for (int i = b1; i < S.n; ++i)
          csubmul(((i - b1) & 1) ? acc2 : acc, Lb[(long long)(i - b1) * bw], w[(long long)i * M]);
        w[(long long)(b0 + jj) * M] = cadd(acc, acc2);
      }
      __syncthreads();
    }
    constexpr int kReg = 4;
    cplx xr[kReg];
    int xi[kReg];
    int nx = 0;
    for (int idx = tid; idx < L.ns * per && nx < kReg; idx += nt, ++nx) {
      const int si = idx / per, rem = idx - si * per, jj = rem / M, k = rem - jj * M;
      const DagSn& S = lc.sn[si];
      xi[nx] = -1;
      if (b0 + jj >= S.n) continue;
      const int b1 = min(S.n, b0 + kDiagBlk), bw = b1 - b0;
      const cplx* X = V + S.bdiag + bpanel_off(S.n, b) + (long long)(S.n - b1) * bw;  // row-major
      const cplx* w = ws + (long long)(S.c0 - pos0 + b0) * M + k;
      cplx acc = w[(long long)jj * M], acc2 = cmk(0, 0);
      for (int ii = jj + 1; ii < bw; ++ii)
        cfma((ii & 1) ? acc2 : acc, X[(long long)ii * (ii - 1) / 2 + jj], w[(long long)ii * M]);
      xr[nx] = cadd(acc, acc2);
      xi[nx] = int((S.c0 - pos0 + b0 + jj) * M + k);
    }
    __syncthreads();
    for (int u = 0; u < nx; ++u)
      if (xi[u] >= 0) ws[xi[u]] = xr[u];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- staged units
// The unit's factor values were bulk-copied into shared memory (voff) with its
// right-hand sides (forward) or its z and the outside x its rows reach (backward).
__device__ void fwd_staged(const DagArgs& A, cplx* sm, const TaskCtx& C, LvCache& lc) {
  const DagTile& T = C.T;
  const DagUnit& U = C.U;
  const DagDec& D = A.dec[T.dec];
  const int M = T.M, m = T.m;
  const int tid = threadIdx.x, nt = blockDim.x;
  cplx* ys = sm;                          // [npos][M]: b, then y, then z
  cplx* sl = sm + (long long)U.npos * M;  // [nrow][M]: partials of the unit's rows
  const cplx* VF = reinterpret_cast<const cplx*>(reinterpret_cast<const char*>(sm) + U.voff) - U.f0;
  cplx* Xv = A.X + T.cb;
  cplx* Pv = A.P + T.pbase;
  int* cof = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + U.cof);
  for (int i = tid; i < U.npos; i += nt) cof[i] = __ldg(A.col_off + U.pos0 + i);
  for (int l = 0; l < U.nlv; ++l) {
    const DagLv L = D.lv[U.lv0 + l];
    stage_level(A, D, L, lc);
    // gather: y = b - incoming partials (in_ref order): shared slots inside the unit,
    // global slots for a single unit
    if (l > 0 || U.kind == 1) {
      const int per = L.nmax * M;
      for (int idx = tid; idx < L.ns * per; idx += nt) {
        const int si = idx / per, rem = idx - si * per, j = rem / M, k = rem - j * M;
        const DagSn& S = lc.sn[si];
        if (j >= S.n) continue;
        const int pos = S.c0 + j;
        cplx* yp = ys + (long long)(pos - U.pos0) * M + k;
        cplx y = *yp;
        const int e1 = __ldg(D.in_ptr + pos + 1);
        for (int e = __ldg(D.in_ptr + pos); e < e1; ++e) {
          const int ref = __ldg(D.in_ref + e);
          if (ref >= 0)
            y = csub(y, sl[(long long)ref * M + k]);
          else if (!A.sparse || __ldg(D.in_live + e))
            y = csub(y, ldcg(Pv + (long long)(-ref - 1) * M + k));
        }
        *yp = y;
      }
      __syncthreads();
    }
    DPROF(1);
    if (L.kind == 0) {
      for (int idx = tid; idx < L.ns * M; idx += nt) {  // leaves: band substitution
        const int si = idx / M, k = idx - si * M;
        const DagSn& S = lc.sn[si];
        leaf_fwd(ys + (long long)(S.c0 - U.pos0) * M + k, M, VF + S.fdiag, S.n, S.lw);
      }
      __syncthreads();
    } else {
      diag_fwd_staged(lc, L, VF, ys, U.pos0, M);
    }
    DPROF(2);
    {  // z -> X (active members; the backward reads it)
      const int per = L.nmax * M;
      for (int idx = tid; idx < L.ns * per; idx += nt) {
        const int si = idx / per, rem = idx - si * per, j = rem / M, k = rem - j * M;
        const DagSn& S = lc.sn[si];
        if (j >= S.n || !((C.act >> k) & 1)) continue;
        const int pos = S.c0 + j;
        Xv[(long long)pos * m + k] = ys[(long long)(pos - U.pos0) * M + k];
      }
    }
    push_staged(A, D, L, lc, C, VF, ys, cof, sl, Pv);
    __syncthreads();
    DPROF(3);
  }
  if (U.kind == 0) {  // partials leaving the subtree: merged per target, row order
    for (int idx = tid; idx < U.nex * M; idx += nt) {
      const int e = idx / M, k = idx - e * M;
      const DagExt E = D.ext[U.ex0 + e];
      cplx s = cmk(0, 0);
      for (int q = 0; q < E.nsrc; ++q) s = cadd(s, sl[(long long)D.ext_src[E.src0 + q] * M + k]);
      Pv[(long long)E.gslot * M + k] = s;
    }
    __syncthreads();
    DPROF(4);
  }
}

__device__ void bwd_staged(const DagArgs& A, cplx* sm, const TaskCtx& C, LvCache& lc) {
  const DagTile& T = C.T;
  const DagUnit& U = C.U;
  const DagDec& D = A.dec[T.dec];
  const int M = T.M, m = T.m;
  const int tid = threadIdx.x, nt = blockDim.x;
  cplx* ws = sm;  // [npos][M]: z, then w, then x
  const cplx* xs = sm + (long long)U.npos * M;
  const cplx* VB = reinterpret_cast<const cplx*>(reinterpret_cast<const char*>(sm) + U.voff) - U.b0;
  cplx* Xv = A.X + T.cb;
  const bool zero_z = A.sparse && !U.live;  // the forward skipped the unit: z = 0
  for (int l = U.nlv - 1; l >= 0; --l) {
    const DagLv L = D.lv[U.lv0 + l];
    stage_level(A, D, L, lc);
    bwd_columns_staged(A, D, L, lc, C, VB, ws, xs, zero_z);
    __syncthreads();
    DPROF(1);
    if (L.kind == 0) {
      for (int idx = tid; idx < L.ns * M; idx += nt) {  // leaves: band back substitution
        const int si = idx / M, k = idx - si * M;
        const DagSn& S = lc.sn[si];
        leaf_bwd(ws + (long long)(S.c0 - U.pos0) * M + k, M, VB + S.bdiag, S.n, S.lw);
      }
      __syncthreads();
    } else {
      diag_bwd_staged(lc, L, VB, ws, U.pos0, M);
    }
    DPROF(2);
    {  // x -> X
      const int per = L.nmax * M;
      for (int idx = tid; idx < L.ns * per; idx += nt) {
        const int si = idx / per, rem = idx - si * per, j = rem / M, k = rem - j * M;
        const DagSn& S = lc.sn[si];
        if (j >= S.n || !((C.act >> k) & 1)) continue;
        const int pos = S.c0 + j;
        Xv[(long long)pos * m + k] = ws[(long long)(pos - U.pos0) * M + k];
      }
    }
    __syncthreads();
    DPROF(3);
  }
}

// ---------------------------------------------------------------- streamed units
// One big separator whose values do not fit shared memory: its chunk list (plan)
// is streamed through two buffers by the TMA engine (warp 0 issues chunk c + 2 while
// the CTA works on chunk c + 1), every thread computing from shared memory.
constexpr int kAcc = kDagAcc;  // accumulator items per thread (the plan bounds n*mg, rows*mg)

struct Stream {
  const DagChunk* ch;
  int nc;
  unsigned char* buf[2];
  unsigned long long* bar;  // 2 barriers
  unsigned* par;            // their parities (per thread, advanced in lockstep)
};

__device__ __forceinline__ void stream_issue(const DagArgs& A, const TaskCtx& C, const Stream& Sx, int c,
                                             const cplx* base, int rs0) {
  // warp 0 only
  const int lane = threadIdx.x & 31;
  const DagChunk q = Sx.ch[c];
  const int M = C.T.M, m = C.T.m;
  unsigned char* dst = Sx.buf[c & 1];
  unsigned long long* bar = Sx.bar + (c & 1);
  const unsigned vb = unsigned(q.cnt) * unsigned(sizeof(cplx));
  const unsigned xb = q.kind == 3 ? unsigned(q.z - q.a) * M * unsigned(sizeof(cplx)) : 0u;
  const unsigned mb = q.kind == 3 ? unsigned((2 * (q.z - q.a) * 4 + 15) & ~15) : 0u;
  if (lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, vb + xb + mb);
    bulk_copy(dst, base + q.off, vb, bar);
    if (mb) bulk_copy(dst + vb + xb, A.dec[C.T.dec].cmeta + q.meta, mb, bar);
  }
  if (q.kind == 3) {  // the rows' x (final: written by the units above)
    __syncwarp();
    const cplx* Xv = A.X + C.T.cb;
    for (int r = q.a + lane; r < q.z; r += 32)
      bulk_copy(dst + vb + (unsigned)(r - q.a) * M * sizeof(cplx),
                Xv + (long long)__ldg(A.row_dpos + rs0 + r) * m, unsigned(M * sizeof(cplx)), bar);
  }
}

__device__ __forceinline__ void stream_wait(const Stream& Sx, int c) {
#ifdef HDDM_DAG_PROF
  const long long t0 = clock64();
#endif
  mbar_wait(Sx.bar + (c & 1), Sx.par[c & 1] & 1);
  Sx.par[c & 1] += 1;
#ifdef HDDM_DAG_PROF
  if (threadIdx.x == 0) g_pacc[4] += clock64() - t0;  // time waiting for chunks (phase 4)
#endif
}

__device__ void fwd_stream(const DagArgs& A, cplx* sm, const TaskCtx& C, LvCache& lc, unsigned long long* bars,
                           unsigned* par) {
  const DagTile& T = C.T;
  const DagUnit& U = C.U;
  const DagDec& D = A.dec[T.dec];
  const int M = T.M, m = T.m;
  const int tid = threadIdx.x, nt = blockDim.x;
  const DagLv L = D.lv[U.lv0];
  stage_level(A, D, L, lc);
  const DagSn& S = lc.sn[0];
  const int n = S.n;
  cplx* ys = sm;  // [n][M]
  int* cof = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + U.cof);
  unsigned char* sb = reinterpret_cast<unsigned char*>(sm);
  const Stream Sx{D.ch + U.fc0, U.nfc, {sb + U.buf, sb + U.buf + U.bufb}, bars, par};
  const cplx* VFg = A.vF + (long long)T.c * A.nvF;
  for (int i = tid; i < n; i += nt) cof[i] = __ldg(A.col_off + S.c0 + i);
  const cplx* Bv = A.B + T.cb;
  cplx* Xv = A.X + T.cb;
  cplx* Pv = A.P + T.pbase;
  {
    // incoming partial refs of the supernode's positions (contiguous in in_ref) into
    // chunk buffer 0 (dead refs -- steps >= 2, source unit skipped -- as 0), then
    // y = b - sum of the partials, loads kU at a time
    const int e0 = __ldg(D.in_ptr + S.c0), e1 = __ldg(D.in_ptr + S.c0 + n);
    int* refs = reinterpret_cast<int*>(Sx.buf[0]);
    for (int e = e0 + tid; e < e1; e += nt)
      refs[e - e0] = (!A.sparse || __ldg(D.in_live + e)) ? __ldg(D.in_ref + e) : 0;
    __syncthreads();
    for (int idx = tid; idx < n * M; idx += nt) {
      const int j = idx / M, k = idx - j * M;
      const int pos = S.c0 + j;
      cplx y = Bv[(long long)pos * m + k];
      const int a = __ldg(D.in_ptr + pos) - e0, z = __ldg(D.in_ptr + pos + 1) - e0;
      for (int e = a; e < z; e += kU) {
        cplx v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int ref = e + u < z ? refs[e + u] : 0;
          v[u] = ref < 0 ? ldcg(Pv + (long long)(-ref - 1) * M + k) : cmk(0, 0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) y = csub(y, v[u]);
      }
      ys[idx] = y;
    }
    __syncthreads();
  }
  if (tid < 32) {  // the first two chunks
    if (Sx.nc > 0) stream_issue(A, C, Sx, 0, VFg, S.rs0);
    if (Sx.nc > 1) stream_issue(A, C, Sx, 1, VFg, S.rs0);
  }
  DPROF(1);
  // the diagonal panels (chunks of kinds 0 and 1) ...
  int c = 0;
  for (; c < Sx.nc && Sx.ch[c].kind <= 1; ++c) {
    stream_wait(Sx, c);
    const DagChunk q = Sx.ch[c];
    const cplx* V = reinterpret_cast<const cplx*>(Sx.buf[c & 1]);
    if (q.kind == 0) {  // z_b = Xinv_b y_b
      const int b0 = q.a, bw = q.z - q.a, per = bw * M;
      cplx zr[4];
      int zi[4];
      int nz = 0;
      for (int idx = tid; idx < per && nz < 4; idx += nt, ++nz) {
        const int ii = idx / M, k = idx - ii * M;
        const cplx* y = ys + (long long)b0 * M + k;
        cplx a0 = y[(long long)ii * M], a1 = cmk(0, 0);
        for (int jj = 0; jj < ii; ++jj)
          cfma((jj & 1) ? a1 : a0, V[(long long)jj * (bw - 1) - (long long)jj * (jj - 1) / 2 + (ii - jj - 1)],
               y[(long long)jj * M]);
        zr[nz] = cadd(a0, a1);
        zi[nz] = (b0 + ii) * M + k;
      }
      __syncthreads();
      for (int u = 0; u < nz; ++u) ys[zi[u]] = zr[u];
    } else {  // rows below panel b: y_i -= L[i, a..z) z_{a..z)
      const int b1 = min(n, (q.b + 1) * kDiagBlk), nl = n - b1;
      for (int idx = tid; idx < nl * M; idx += nt) {
        const int ii = idx / M, k = idx - ii * M;
        cplx* yp = ys + (long long)(b1 + ii) * M + k;
        const cplx* vp = V + ii;
        const cplx* zp = ys + (long long)q.a * M + k;
        cplx a0 = *yp, a1 = cmk(0, 0);
        const int nj = q.z - q.a;
        for (int j = 0; j < nj; ++j) csubmul((j & 1) ? a1 : a0, vp[(long long)j * nl], zp[(long long)j * M]);
        *yp = cadd(a0, a1);
      }
    }
    __syncthreads();
    if (tid < 32 && c + 2 < Sx.nc) stream_issue(A, C, Sx, c + 2, VFg, S.rs0);
  }
  DPROF(2);
  for (int idx = tid; idx < n * M; idx += nt) {  // z -> X
    const int j = idx / M, k = idx - j * M;
    if ((C.act >> k) & 1) Xv[(long long)(S.c0 + j) * m + k] = ys[idx];
  }
  // ... then the block rows (kind 2), once per member group: partial_r += L[r][q] z_q,
  // register accumulators for the items (row, member of the group)
  while (c < Sx.nc) {
    const int g = Sx.ch[c].b;
    const int k0 = g * kDagMG, mg = min(kDagMG, M - k0);
    cplx acc[kAcc];
#pragma unroll
    for (int u = 0; u < kAcc; ++u) acc[u] = cmk(0, 0);
    for (; c < Sx.nc && Sx.ch[c].b == g; ++c) {
      stream_wait(Sx, c);
      const DagChunk q = Sx.ch[c];
      const cplx* V = reinterpret_cast<const cplx*>(Sx.buf[c & 1]);
      const int c0 = cof[q.a];
#pragma unroll
      for (int u = 0; u < kAcc; ++u) {
        const int it = tid + u * nt;
        const int rr = it / mg, k = k0 + it - rr * mg;
        if (rr < S.nrs) {
          const int first = __ldg(A.row_first + S.rs0 + rr);
          cplx a = acc[u];
          for (int qq = max(q.a, first); qq < q.z; ++qq) cfma(a, V[cof[qq] - c0 + rr], ys[(long long)qq * M + k]);
          acc[u] = a;
        }
      }
      __syncthreads();
      if (tid < 32 && c + 2 < Sx.nc) stream_issue(A, C, Sx, c + 2, VFg, S.rs0);
    }
#pragma unroll
    for (int u = 0; u < kAcc; ++u) {
      const int it = tid + u * nt;
      const int rr = it / mg, k = k0 + it - rr * mg;
      if (rr < S.nrs) Pv[(long long)(-D.row_slot[S.rs0 + rr] - 1) * M + k] = acc[u];
    }
  }
  __syncthreads();
  DPROF(3);
}

__device__ __forceinline__ void bwd_write_w(const cplx (&acc)[kAcc], cplx* ws, const cplx* dinv, int n, int M,
                                            int k0, int mg, bool zero_z) {
#pragma unroll
  for (int u = 0; u < kAcc; ++u) {
    const int it = threadIdx.x + u * blockDim.x;
    const int j = it / mg, k = k0 + it - j * mg;
    if (j < n) {
      cplx* wp = ws + (long long)j * M + k;
      const cplx z = zero_z ? cmk(0, 0) : *wp;
      *wp = csub(cmul(__ldg(dinv + j), z), acc[u]);
    }
  }
  __syncthreads();
}

__device__ void bwd_stream(const DagArgs& A, cplx* sm, const TaskCtx& C, LvCache& lc, unsigned long long* bars,
                           unsigned* par) {
  const DagTile& T = C.T;
  const DagUnit& U = C.U;
  const DagDec& D = A.dec[T.dec];
  const int M = T.M, m = T.m;
  const int tid = threadIdx.x, nt = blockDim.x;
  const DagLv L = D.lv[U.lv0];
  stage_level(A, D, L, lc);
  const DagSn& S = lc.sn[0];
  const int n = S.n;
  cplx* ws = sm;  // [n][M]: z (bulk-loaded), then w, then x
  unsigned char* sb = reinterpret_cast<unsigned char*>(sm);
  const Stream Sx{D.ch + U.bc0, U.nbc, {sb + U.buf, sb + U.buf + U.bufb}, bars, par};
  const cplx* VBg = A.vB + (long long)T.c * A.nvB;
  if (tid < 32) {
    if (Sx.nc > 0) stream_issue(A, C, Sx, 0, VBg, S.rs0);
    if (Sx.nc > 1) stream_issue(A, C, Sx, 1, VBg, S.rs0);
  }
  cplx* Xv = A.X + T.cb;
  const bool zero_z = A.sparse && !U.live;
  int c = 0;
  // block rows (kind 3), once per member group: w_j = z_j / D_j - sum_r L[r][j] x_r,
  // register accumulators for the items (column, member of the group)
  while (c < Sx.nc && Sx.ch[c].kind == 3) {
    const int g = Sx.ch[c].b;
    const int k0 = g * kDagMG, mg = min(kDagMG, M - k0);
    cplx acc[kAcc];
#pragma unroll
    for (int u = 0; u < kAcc; ++u) acc[u] = cmk(0, 0);
    for (; c < Sx.nc && Sx.ch[c].kind == 3 && Sx.ch[c].b == g; ++c) {
      stream_wait(Sx, c);
      const DagChunk q = Sx.ch[c];
      const cplx* V = reinterpret_cast<const cplx*>(Sx.buf[c & 1]);
      const cplx* xb = V + q.cnt;  // values, then the rows' x, then (first, offset) pairs
      const int2* rm = reinterpret_cast<const int2*>(xb + (long long)(q.z - q.a) * M);
      const int nr = q.z - q.a;
#pragma unroll
      for (int u = 0; u < kAcc; ++u) {
        const int it = tid + u * nt;
        const int j = it / mg, k = k0 + it - j * mg;
        if (j < n) {
          cplx a0 = acc[u], a1 = cmk(0, 0);
          for (int r = 0; r < nr; ++r) {
            const int2 fo = rm[r];
            if (fo.x > j) break;  // rows sorted by first column
            cfma((r & 1) ? a1 : a0, V[fo.y + (j - fo.x)], xb[(long long)r * M + k]);
          }
          acc[u] = cadd(a0, a1);
        }
      }
      __syncthreads();
      if (tid < 32 && c + 2 < Sx.nc) stream_issue(A, C, Sx, c + 2, VBg, S.rs0);
    }
    bwd_write_w(acc, ws, VBg + S.bdinv, n, M, k0, mg, zero_z);
  }
  if (S.nrs == 0) {  // no block rows: w = z / D
    cplx acc[kAcc];
#pragma unroll
    for (int u = 0; u < kAcc; ++u) acc[u] = cmk(0, 0);
    for (int k0 = 0; k0 < M; k0 += kDagMG) bwd_write_w(acc, ws, VBg + S.bdinv, n, M, k0, min(kDagMG, M - k0), zero_z);
  }
  for (; c < Sx.nc; ++c) {  // the diagonal panels from the last (kinds 4 and 5)
    stream_wait(Sx, c);
    const DagChunk q = Sx.ch[c];
    const cplx* V = reinterpret_cast<const cplx*>(Sx.buf[c & 1]);
    const int b0 = q.b * kDiagBlk, b1 = min(n, b0 + kDiagBlk), bw = b1 - b0;
    if (q.kind == 4) {  // w_b -= L[a..z, b]^T x_{a..z}
      for (int idx = tid; idx < bw * M; idx += nt) {
        const int jj = idx / M, k = idx - jj * M;
        cplx* wp = ws + (long long)(b0 + jj) * M + k;
        const cplx* vp = V + jj;
        const cplx* xp = ws + (long long)q.a * M + k;
        cplx a0 = *wp, a1 = cmk(0, 0);
        const int ni = q.z - q.a;
        for (int i = 0; i < ni; ++i) csubmul((i & 1) ? a1 : a0, vp[(long long)i * bw], xp[(long long)i * M]);
        *wp = cadd(a0, a1);
      }
    } else {  // x_b = Xinv_b^T w_b
      cplx xr[4];
      int xi[4];
      int nx = 0;
      for (int idx = tid; idx < bw * M && nx < 4; idx += nt, ++nx) {
        const int jj = idx / M, k = idx - jj * M;
        const cplx* w = ws + (long long)b0 * M + k;
        cplx a0 = w[(long long)jj * M], a1 = cmk(0, 0);
        for (int ii = jj + 1; ii < bw; ++ii)
          cfma((ii & 1) ? a1 : a0, V[(long long)ii * (ii - 1) / 2 + jj], w[(long long)ii * M]);
        xr[nx] = cadd(a0, a1);
        xi[nx] = (b0 + jj) * M + k;
      }
      __syncthreads();
      for (int u = 0; u < nx; ++u) ws[xi[u]] = xr[u];
    }
    __syncthreads();
    if (tid < 32 && c + 2 < Sx.nc) stream_issue(A, C, Sx, c + 2, VBg, S.rs0);
  }
  DPROF(2);
  for (int idx = tid; idx < n * M; idx += nt) {  // x -> X
    const int j = idx / M, k = idx - j * M;
    if ((C.act >> k) & 1) Xv[(long long)(S.c0 + j) * m + k] = ws[idx];
  }
  __syncthreads();
  DPROF(3);
}

}  // namespace

__global__ void __launch_bounds__(kDagThreads, 2) k_dag(const __grid_constant__ DagArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  cplx* sm = reinterpret_cast<cplx*>(dsm);
  __shared__ int s_t;
  __shared__ TaskCtx s_c;
  __shared__ LvCache s_lc;
  // 0: values (+ b) of a staged unit; 1: z (+ outside x) of a backward; 2, 3: the chunk buffers
  __shared__ __align__(8) unsigned long long s_bar[4];
  if (threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) mbar_init(&s_bar[i]);
#ifdef HDDM_DAG_PROF
  if (threadIdx.x == 0) g_ptail_cat = -1;
#endif
  __syncthreads();
  unsigned phase0 = 0, phase1 = 0;
  unsigned spar[2] = {0, 0};
  if (threadIdx.x == 0) s_t = atomicAdd(A.ticket, 1);
  __syncthreads();
  for (;;) {
    const int t = s_t;
    if (t >= A.ntask) return;
    const DagTask T = A.task[t];
    int nxt = 0;
    __syncthreads();  // every thread has read s_t
    if (threadIdx.x < 32) {  // warp 0: descriptors, bulk loads, dependency wait
      const int lane = threadIdx.x;
      if (lane == 0) {
        nxt = atomicAdd(A.ticket, 1);  // the next task's ticket, consumed at the end of this one
#ifdef HDDM_DAG_PROF
        {
          const long long now = clock64();
          if (g_ptail_cat >= 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(A.prof) + g_ptail_cat * 8 + 5,
                      (unsigned long long)(now - g_ptail));
          for (int q = 0; q < 8; ++q) g_pacc[q] = 0;
          g_plast = now;
          if (A.trace) {
            unsigned long long gt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            A.trace[8 * t + 0] = (long long)gt;
            A.trace[8 * t + 2] = smid;
            A.trace[8 * t + 3] = blockIdx.x + 1000000LL * A.dec[A.tile[T.tile].dec].unit[T.unit].height;
          }
        }
#endif
        s_c.T = A.tile[T.tile];
        s_c.U = A.dec[s_c.T.dec].unit[T.unit];
        unsigned act = 0;
        for (int k = 0; k < s_c.T.M; ++k)
          if ((A.flag[s_c.T.t[k]] != 0) == (A.flag_on != 0)) act |= 1u << k;
        if (T.kind == 0 && A.sparse && !s_c.U.live) act = 0;  // z = 0 exactly: nothing to do
        s_c.act = act;
      }
      __syncwarp();
      const DagTile& Tl = s_c.T;
      const DagUnit& U = s_c.U;
      const int M = Tl.M, m = Tl.m;
      const bool staged = s_c.act && U.voff >= 0;
      if (staged) {
        // factor values (+ the right-hand sides in the forward): independent of the
        // predecessors, so issued before the wait
        const cplx* src = T.kind == 0 ? A.vF + (long long)Tl.c * A.nvF + U.f0 : A.vB + (long long)Tl.c * A.nvB + U.b0;
        const long long n = T.kind == 0 ? U.f1 - U.f0 : U.b1 - U.b0;
        const unsigned vb = unsigned(n * sizeof(cplx));
        const unsigned bb = T.kind == 0 ? unsigned(U.npos) * M * unsigned(sizeof(cplx)) : 0u;
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&s_bar[0], vb + bb);
          bulk_copy(dsm + U.voff, src, vb, &s_bar[0]);
        }
        __syncwarp();
        if (T.kind == 0) {
          const cplx* Bv = A.B + Tl.cb + (long long)U.pos0 * m;
          if (m == M) {
            if (lane == 0) bulk_copy(dsm, Bv, bb, &s_bar[0]);
          } else {
            for (int p = lane; p < U.npos; p += 32)
              bulk_copy(reinterpret_cast<cplx*>(dsm) + (long long)p * M, Bv + (long long)p * m,
                        unsigned(M * sizeof(cplx)), &s_bar[0]);
          }
        }
      }
      if (lane == 0) {
        if (T.dep0 >= 0) wait_done(A.done + T.dep0);
        if (T.dep1 >= 0) wait_done(A.done + T.dep1);
      }
      __syncwarp();
      if (s_c.act && T.kind == 1) {
        // backward: the unit's z (written by its forward) and, staged units, the x of
        // the outside positions its rows reach (written by the units above)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const unsigned zb = unsigned(U.npos) * M * unsigned(sizeof(cplx));
        const unsigned xb = staged ? unsigned(U.nxe) * M * unsigned(sizeof(cplx)) : 0u;
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&s_bar[1], zb + xb);
        }
        __syncwarp();
        const cplx* Xv = A.X + Tl.cb;
        cplx* ws = reinterpret_cast<cplx*>(dsm);
        if (m == M) {
          if (lane == 0) bulk_copy(ws, Xv + (long long)U.pos0 * m, zb, &s_bar[1]);
        } else {
          for (int p = lane; p < U.npos; p += 32)
            bulk_copy(ws + (long long)p * M, Xv + (long long)(U.pos0 + p) * m, unsigned(M * sizeof(cplx)), &s_bar[1]);
        }
        if (staged) {
          cplx* xs = ws + (long long)U.npos * M;
          for (int e = lane; e < U.nxe; e += 32)
            bulk_copy(xs + (long long)e * M, Xv + (long long)__ldg(A.dec[Tl.dec].xe + U.xe0 + e) * m,
                      unsigned(M * sizeof(cplx)), &s_bar[1]);
        }
      }
    }
    __syncthreads();
    if (s_c.act) {
      if (s_c.U.voff >= 0) {
        mbar_wait(&s_bar[0], phase0 & 1);
        ++phase0;
      }
      if (T.kind == 1) {
        mbar_wait(&s_bar[1], phase1 & 1);
        ++phase1;
      }
    }
    DPROF(0);
    if (s_c.act) {
      if (s_c.U.voff >= 0) {
        if (T.kind == 0)
          fwd_staged(A, sm, s_c, s_lc);
        else
          bwd_staged(A, sm, s_c, s_lc);
      } else {
        if (T.kind == 0)
          fwd_stream(A, sm, s_c, s_lc, &s_bar[2], spar);
        else
          bwd_stream(A, sm, s_c, s_lc, &s_bar[2], spar);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // publish (release: the CTA's writes, ordered before it by the barrier)
      st_release(A.done + t, 1);
      s_t = nxt;
#ifdef HDDM_DAG_PROF
      if (A.trace) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        A.trace[8 * t + 1] = (long long)gt;
        for (int q = 0; q < 4; ++q) A.trace[8 * t + 4 + q] = g_pacc[q + 1];
      }
      if (A.prof) {
        const int cat = T.kind * 4 + s_c.U.kind * 2 + (s_c.T.M > 1 ? 1 : 0);
        for (int q = 0; q < 5; ++q)
          atomicAdd(reinterpret_cast<unsigned long long*>(A.prof) + cat * 8 + q, (unsigned long long)g_pacc[q]);
        atomicAdd(reinterpret_cast<unsigned long long*>(A.prof) + cat * 8 + 7, 1ull);
        g_ptail_cat = cat;
        g_ptail = clock64();
      }
#endif
    }
    __syncthreads();
  }
}

// identity ring rows x = b for every tile (before the dataflow kernel)
__global__ void k_dag_ring(DagArgs A, int nring) {
  const DagTile T = A.tile[blockIdx.y];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nring * T.M; idx += gridDim.x * blockDim.x) {
    const int pos = idx / T.M, k = idx - pos * T.M;
    if ((A.flag[T.t[k]] != 0) != (A.flag_on != 0)) continue;
    const long long e = T.cb + (long long)pos * T.m + k;
    A.X[e] = A.B[e];
  }
}

int dag_grid(int smem_bytes) {
  static int grid = 0, smem_done = -1;
  if (smem_done != smem_bytes) {
    cudaFuncSetAttribute(k_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    int per_sm = 0, dev = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dag, kDagThreads, smem_bytes);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    grid = std::max(1, per_sm) * nsm;
    smem_done = smem_bytes;
  }
  return grid;
}

void launch_dag_solve(const DagArgs& A, int ntile, int nring, cudaStream_t st) {
  cudaMemsetAsync(A.ticket, 0, sizeof(int), st);
  cudaMemsetAsync(A.done, 0, sizeof(int) * size_t(A.ntask), st);
  k_dag_ring<<<dim3((nring * kDagMaxM + 255) / 256, ntile), 256, 0, st>>>(A, nring);
  k_dag<<<dag_grid(A.smem_bytes), kDagThreads, A.smem_bytes, st>>>(A);
}

}  // namespace hddm
