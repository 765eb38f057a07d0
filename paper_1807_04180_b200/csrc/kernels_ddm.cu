// DDM step kernels: zero-flag bookkeeping, the fused gather-sources kernel
// (restrict_owned + 8-direction add_transfer + scale_rhs), the blend-accumulate,
// the local-solve residual check, the global stencil and deterministic
// reductions.
//
// Reference semantics reproduced (proj/src/ddm.cpp:174-242, transfer.cpp:7-88):
//   * step 1 only sees f (restrict_owned on the owned rectangle);
//   * edge transfers read step s-1, corner transfers read step s-2;
//   * a subdomain is skipped iff it has no nonzero owned f (step 1) and every
//     in-range source is zero-flagged; values of transferred sources are never
//     inspected;
//   * the assembled field adds w_x w_y u_t in ascending t at every node.
#include "dev.cuh"
#include "kernels.cuh"

namespace hddm {

namespace {

constexpr int kRedBlocks = kReduceBlocks;
__constant__ int kDI[8] = {+1, -1, 0, 0, +1, -1, +1, -1};  // source offsets in
__constant__ int kDJ[8] = {0, 0, +1, -1, +1, +1, -1, -1};  // kGatherOrder L,R,D,U,DL,DR,UL,UR

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) r += sh[i];
  return r;  // valid in thread 0
}

}  // namespace

int reduce_blocks() { return kRedBlocks; }

// fany[t] = owned rectangle of f holds a nonzero (restrict_owned, ddm.cpp:159-172)
__global__ void k_fany(StepArgs A) {
  const int t = blockIdx.x;
  const DevSub S = A.sub[t];
  const int w = S.own1 - S.own0 + 1, h = S.own3 - S.own2 + 1;
  int any = 0;
  for (int k = threadIdx.x; k < w * h && !any; k += blockDim.x) {
    const int P = S.own0 + k % w, Q = S.own2 + k / w;
    const cplx v = A.f[(long long)Q * A.gnx + P];
    any = (v.x != 0.0 || v.y != 0.0);
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) const_cast<int*>(A.fany)[t] = any;
}

void launch_fany(const StepArgs& A, cudaStream_t st) {
  k_fany<<<A.nsub, 256, 0, st>>>(A);
}

// zero flags, active lists per class, solve/skip counters (ddm.cpp:187-207)
__global__ void k_flags(StepArgs A, int ncls) {
  extern __shared__ int sh[];  // ncls counts
  __shared__ int nown;
  if (threadIdx.x == 0) nown = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < A.nsub; t += blockDim.x) {
    if (A.owned && !A.owned[t]) {  // another engine's subdomain (sharded run)
      A.zc[t] = 1;
      continue;
    }
    atomicAdd(&nown, 1);
    const DevSub S = A.sub[t];
    int any = (A.step == 1) ? A.fany[t] : 0;
    for (int d = 0; d < 8; ++d) {
      const int si = S.i + kDI[d], sj = S.j + kDJ[d];
      if (si < 0 || si >= A.n1 || sj < 0 || sj >= A.n2) continue;
      const int src = sj * A.n1 + si;
      if (!(d >= 4 ? A.zp2 : A.zp1)[src]) any = 1;
    }
    A.zc[t] = any ? 0 : 1;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncls; c += blockDim.x) {
    int cnt = 0;
    for (int k = A.cls_ptr[c]; k < A.cls_ptr[c + 1]; ++k) cnt += A.zc[A.cls_mem[k]] ? 0 : 1;
    sh[c] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int c = 0; c < ncls; ++c) {
      A.act_ptr[c] = acc;
      acc += sh[c];
    }
    A.act_ptr[ncls] = acc;
    A.counts[0] += acc;
    A.counts[1] += nown - acc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncls; c += blockDim.x) {
    int o = A.act_ptr[c];
    for (int k = A.cls_ptr[c]; k < A.cls_ptr[c + 1]; ++k)
      if (!A.zc[A.cls_mem[k]]) A.act_list[o++] = A.cls_mem[k];
  }
}

void launch_flags(const StepArgs& A, int ncls, cudaStream_t st) {
  k_flags<<<1, 256, sizeof(int) * ncls, st>>>(A, ncls);
}

// ------------------------------------------------------------ gather sources
// Right-hand side assembly in two passes (restrict_owned + add_transfer +
// scale_rhs, ddm.cpp:183-205, transfer.cpp:64-88, discretize.cpp:162-172):
//  (1) every window node: B = J * f_owned (step 1) or 0; ring rows 0;
//  (2) only nodes of the union of the 8 transfer patches (a structural list,
//      identical for every window): B = J * (f_owned - sum_d L_t(beta_d v_d))
//      over the in-range, non-zero-flagged sources in kGatherOrder.
__global__ void __launch_bounds__(256) k_rhs_base(StepArgs A) {
  // storage order: the members of a class at one position are adjacent
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= A.vm.total) return;
  int t, pos;
  vdecode(A.vm, e, t, pos);
  if (A.zc[t]) return;
  cplx v = cmk(0, 0);
  if (A.step == 1) {
    const int node = A.perm[pos];
    const int lp = node % A.wnx, lq = node / A.wnx;
    if (lp > 0 && lq > 0 && lp < A.wnx - 1 && lq < A.wny - 1) {
      const DevSub T = A.sub[t];
      const int P = T.wx0 + lp, Q = T.wy0 + lq;
      if (P >= T.own0 && P <= T.own1 && Q >= T.own2 && Q <= T.own3) {
        const cplx* sa = A.sa + (long long)t * A.sa_stride;
        v = cmul(cmul(sa[lp], sa[2 * A.wnx + lq]), A.f[(long long)Q * A.gnx + P]);
      }
    }
  }
  A.B[e] = v;
}

#ifndef HDDM_XFER_MINB
#define HDDM_XFER_MINB 3  // register cap for occupancy: measured -8% per step with the check
#endif
// Block table (StepArgs::xblk): block -> (class c, first member slot k0, members M <= 32,
// first patch node u0). Thread tid serves member k0 + tid % M at patch node u0 + tid / M:
// the members of a class at one position are adjacent in the interleaved layout, so a
// warp's loads of a neighbour's solution and its stores of B are contiguous runs of M
// values (sources of adjacent members are adjacent members of the source's class on a
// regular partition), and the structural tables and the class coefficients are
// broadcast loads. Members of a class have bitwise-identical window operators (the
// class criterion), so alpha and k^2 come from the class representative.
__global__ void __launch_bounds__(256, HDDM_XFER_MINB) k_rhs_transfer(StepArgs A) {
  const int4 blk = __ldg(A.xblk + blockIdx.x);
  const int c = blk.x, M = blk.z;
  const int pi = threadIdx.x / M;
  const int u = blk.w + pi;
  if (pi >= 256 / M || u >= A.npatch) return;
  const int c0 = __ldg(A.vm.cptr + c);
  const int t = __ldg(A.vm.cmem + c0 + blk.y + threadIdx.x % M);
  if (A.zc[t]) return;
  const int node = __ldg(A.pnode + u);
  const int mask = __ldg(A.pmask + u);
  const int tpos = __ldg(A.pinv + node);
  const int lp = node % A.wnx, lq = node / A.wnx;
  const DevSub T = A.sub[t];
  const cplx* sa = A.sa + (long long)__ldg(A.vm.cmem + c0) * A.sa_stride;
  const cplx a1 = sa[lp], a2 = sa[2 * A.wnx + lq];
  const cplx ia1w = sa[A.wnx + lp - 1], ia1e = sa[A.wnx + lp];
  const cplx ia2s = sa[2 * A.wnx + A.wny + lq - 1], ia2n = sa[2 * A.wnx + A.wny + lq];
  const cplx jac = cmul(a1, a2);
  const double k2 = __ldg(A.k2c + (long long)c * A.nw + tpos);
  const cplx ex = cscale(a2, A.ih2), ey = cscale(a1, A.ih2);
  const cplx cE = cmul(ex, ia1e), cW = cmul(ex, ia1w), cN = cmul(ey, ia2n), cS = cmul(ey, ia2s);
  cplx val = cmk(0, 0);
  if (A.step == 1) {
    const int P = T.wx0 + lp, Q = T.wy0 + lq;
    if (P >= T.own0 && P <= T.own1 && Q >= T.own2 && Q <= T.own3) val = A.f[(long long)Q * A.gnx + P];
  }
  bool any = false;
  for (int d = 0; d < 8; ++d) {
    if (!((mask >> d) & 1)) continue;
    const int di = kDI[d], dj = kDJ[d];
    const int si = T.i + di, sj = T.j + dj;
    if (si < 0 || si >= A.n1 || sj < 0 || sj >= A.n2) continue;
    const int src = sj * A.n1 + si;
    const bool corner = d >= 4;
    if ((corner ? A.zp2 : A.zp1)[src]) continue;
    any = true;
    const SVec<const cplx> V = vview(corner ? A.Up2 : A.Up1, A.vm, src);
    // structural tables: source positions of the 5 stencil points (-1 outside the
    // source window) and transfer_beta (partition.cpp:131-152) at them -- the same
    // for every window, since windows are offset by whole cores
    const int* xp = A.xfer_pos + (u * 8 + d) * 5;
    const double* xb = A.xfer_beta + (u * 8 + d) * 5;
    cplx w5[5];  // C, E, W, N, S
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int pos = __ldg(xp + k);
      const cplx v = pos >= 0 ? V[pos] : cmk(0, 0);
      w5[k] = cscale(v, __ldg(xb + k));  // beta >= 0: a zero v stays the same zero
    }
    const cplx uc = w5[0];
    // DiscreteOperator::stencil (discretize.hpp:43-54)
    cplx tt = cmul(cE, csub(w5[1], uc));
    tt = csub(tt, cmul(cW, csub(uc, w5[2])));
    tt = cadd(tt, cmul(cN, csub(w5[3], uc)));
    tt = csub(tt, cmul(cS, csub(uc, w5[4])));
    val = csub(val, cadd(cdiv(tt, jac), cscale(uc, k2)));
  }
  // step 1: the base value J f stays where no source contributes; later steps
  // write every patch node (0 without a contribution), so B stays zero off the
  // patches after the one clear at step 2
  if (any)
    vview(A.B, A.vm, t)[tpos] = cmul(jac, val);
  else if (A.step != 1)
    vview(A.B, A.vm, t)[tpos] = cmk(0, 0);
}

void launch_transfer(const StepArgs& A, cudaStream_t st) {
  k_rhs_transfer<<<A.nxblk, 256, 0, st>>>(A);
}

void launch_gather(const StepArgs& A, cudaStream_t st) {
  // steps >= 2 see no f: every base value is 0. Step 2 clears all of B at memset
  // speed (right-hand sides of inactive subdomains are never read); from step 3
  // on B is already zero off the transfer patches, which the transfer rewrites.
  if (A.step == 1)
    k_rhs_base<<<unsigned((A.vm.total + 255) / 256), 256, 0, st>>>(A);
  else if (A.step == 2)
    cudaMemsetAsync(A.B, 0, size_t(A.vm.total) * sizeof(cplx), st);
  k_rhs_transfer<<<A.nxblk, 256, 0, st>>>(A);
}

// ------------------------------------------------------------ accumulate
#ifndef HDDM_ACC_MINB
#define HDDM_ACC_MINB 1
#endif
__global__ void __launch_bounds__(256, HDDM_ACC_MINB) k_accumulate(StepArgs A) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)A.gnx * A.gny) return;
  const int P = int(idx % A.gnx), Q = int(idx / A.gnx);
  cplx acc = A.asmb[idx];
  bool touched = false;
  for (int b = 0; b < 4; ++b) {
    const int j = A.rowcov[4 * Q + b];
    if (j < 0) break;
    for (int a = 0; a < 4; ++a) {
      const int i = A.colcov[4 * P + a];
      if (i < 0) break;
      const int t = j * A.n1 + i;
      if (A.zc[t]) continue;
      const DevSub T = A.sub[t];
      const double wy = A.wy[(long long)t * A.wny + (Q - T.wy0)];
      if (wy == 0.0) continue;
      const double w = A.wx[(long long)t * A.wnx + (P - T.wx0)] * wy;
      if (w == 0.0) continue;
      const cplx u = vview((const cplx*)A.Ucur, A.vm, t)[A.pinv[(Q - T.wy0) * A.wnx + (P - T.wx0)]];
      acc.x = __dadd_rn(acc.x, __dmul_rn(w, u.x));
      acc.y = __dadd_rn(acc.y, __dmul_rn(w, u.y));
      touched = true;
    }
  }
  if (touched) A.asmb[idx] = acc;
}

void launch_accumulate(const StepArgs& A, cudaStream_t st) {
  const long long n = (long long)A.gnx * A.gny;
  k_accumulate<<<unsigned((n + 255) / 256), 256, 0, st>>>(A);
}

// ------------------------------------------------------------ residual check
#ifndef HDDM_CHECK_MINB
#define HDDM_CHECK_MINB 3
#endif
#ifndef HDDM_CHECK_UNROLL
#define HDDM_CHECK_UNROLL 1
#endif
constexpr int kCheckUnroll = HDDM_CHECK_UNROLL;
// (A x)_pos for the J-scaled assembled matrix of subdomain t's window
// (discretize.cpp:98-160): identity ring rows, ring columns dropped;
// from structural tables: window coordinates (lp < 0: ring row)
// and neighbour positions (S, W, E, N; -1 where the coupling is dropped) per
// factor-order position, k^2 of the class window in factor order
// coefficients of row (lp, lq): diagonal, S, W, E, N
__device__ __forceinline__ void row_coefs(int2 lpq, int wnx, int wny, double ih2, const cplx* sa,
                                          double k2, cplx cf[5]) {
  const int lp = lpq.x, lq = lpq.y;
  const cplx* a1n = sa;
  const cplx* ia1h = sa + wnx;
  const cplx* a2n = sa + 2 * wnx;
  const cplx* ia2h = sa + 2 * wnx + wny;
  const cplx ew = cscale(cmul(a2n[lq], ia1h[lp - 1]), ih2);
  const cplx ee = cscale(cmul(a2n[lq], ia1h[lp]), ih2);
  const cplx es = cscale(cmul(a1n[lp], ia2h[lq - 1]), ih2);
  const cplx en = cscale(cmul(a1n[lp], ia2h[lq]), ih2);
  cf[0] = cadd(cmk(-(ew.x + ee.x + es.x + en.x), -(ew.y + ee.y + es.y + en.y)),
               cscale(cmul(a1n[lp], a2n[lq]), k2));
  cf[1] = es;
  cf[2] = ew;
  cf[3] = ee;
  cf[4] = en;
}

template <class XV>
__device__ __forceinline__ cplx ax_apply(XV X, int pos, int4 nb, const cplx cf[5]) {
  const cplx xc = X[pos];
  const cplx xs = nb.x >= 0 ? X[nb.x] : cmk(0, 0), xw = nb.y >= 0 ? X[nb.y] : cmk(0, 0);
  const cplx xe = nb.z >= 0 ? X[nb.z] : cmk(0, 0), xn = nb.w >= 0 ? X[nb.w] : cmk(0, 0);
  cplx ax = cmul(cf[0], xc);
  if (nb.x >= 0) cfma(ax, cf[1], xs);
  if (nb.y >= 0) cfma(ax, cf[2], xw);
  if (nb.z >= 0) cfma(ax, cf[3], xe);
  if (nb.w >= 0) cfma(ax, cf[4], xn);
  return ax;
}

template <class XV>
__device__ __forceinline__ cplx ax_row_t(XV X, int pos, int wnx, int wny, double ih2,
                                         const cplx* sa, double k2, int2 lpq, int4 nb) {
  if (lpq.x < 0) return X[pos];
  cplx cf[5];
  row_coefs(lpq, wnx, wny, ih2, sa, k2, cf);
  return ax_apply(X, pos, nb, cf);
}

// Row coefficients of a class window, tabulated once (classes with several members: every
// member's check re-reads them as broadcast loads instead of re-forming them from the
// alpha arrays): tab[pos * 5 + (C, S, W, E, N)]; ring rows (1, 0, 0, 0, 0).
__global__ void __launch_bounds__(256) k_build_ctab(CheckArgs A, int c, cplx* tab) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= A.nw) return;
  const int2 lq = A.lpq[pos];
  cplx cf[5] = {cmk(1, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
  if (lq.x >= 0)
    row_coefs(lq, A.wnx, A.wny, A.ih2, A.sa + (long long)A.vm.cmem[A.vm.cptr[c]] * A.sa_stride,
              A.k2c[(long long)c * A.nw + pos], cf);
  for (int k = 0; k < 5; ++k) tab[(long long)pos * 5 + k] = cf[k];
}

void launch_build_ctab(const CheckArgs& A, int c, cplx* tab, cudaStream_t st) {
  k_build_ctab<<<(A.nw + 255) / 256, 256, 0, st>>>(A, c, tab);
}

// Residual partials of members [k0, k0 + M) of class c over position chunk
// blockIdx.x: thread t serves member k0 + t % M at positions t / M,
// t / M + 256 / M, ... of the chunk (a warp reads consecutive members:
// contiguous addresses). Members of a class have bitwise-identical window
// operators (the class criterion), so the coefficients come from the class
// representative. Per-member sums combine in fixed thread order.
__device__ __forceinline__ void check_block(const CheckArgs& A, int c, int k0, int M, double* sr,
                                            double* sb) {
  const int c0 = A.vm.cptr[c], m = A.vm.cptr[c + 1] - c0;
  const int tid = threadIdx.x;
  const int per = 256 / M;  // positions per sweep of the block (M <= 256)
  const int k = k0 + tid % M, pi = tid / M;
  const int t = A.vm.cmem[c0 + k];
  const bool act = pi < per && (A.only ? A.only[t] != 0 : !A.zc[t]);
  double r2 = 0, b2 = 0;
  if (act) {
    const int rep = A.vm.cmem[c0];
    const cplx* sa = A.sa + (long long)rep * A.sa_stride;
    const double* k2c = A.k2c + (long long)c * A.nw;
    const SVec<const cplx> X{A.X + A.vm.cbase[c] + k, m};
    const SVec<const cplx> Bv{A.B + A.vm.cbase[c] + k, m};
    const int chunk = (A.nw + A.nchunk - 1) / A.nchunk;
    const int p0 = blockIdx.x * chunk, p1 = min(A.nw, p0 + chunk);
    const long long toff = A.ctab_off ? __ldg(A.ctab_off + c) : -1;  // uniform per block
    if (toff >= 0) {
      // tabulated coefficients: five broadcast loads per position
      const cplx* ct = A.ctab + toff;
      int pos = p0 + pi;
      int4 nb_n = make_int4(-1, -1, -1, -1);
      if (pos < p1) nb_n = __ldg(A.nbr + pos);
      for (; pos < p1; pos += per) {
        const int4 nb = nb_n;
        const int pn = pos + per;
        if (pn < p1) nb_n = __ldg(A.nbr + pn);
        const cplx b = (A.bmask && !__ldg(A.bmask + pos)) ? cmk(0, 0) : Bv[pos];
        cplx cf[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) cf[q] = ct[(long long)pos * 5 + q];
        b2 += cnorm2(b);
        r2 += cnorm2(csub(b, ax_apply(X, pos, nb, cf)));
      }
    } else {
    // the next position's structural tables are loaded one iteration ahead, so
    // the vector / coefficient loads of a position (which depend on them) are
    // the only round trip per iteration
    int pos = p0 + pi;
    int2 lq_n = make_int2(-1, 0);
    int4 nb_n = make_int4(-1, -1, -1, -1);
    double k2_n = 0;
    if (pos < p1) {
      lq_n = __ldg(A.lpq + pos);
      nb_n = __ldg(A.nbr + pos);
      k2_n = __ldg(k2c + pos);
    }
#pragma unroll kCheckUnroll
    for (; pos < p1; pos += per) {
      const int2 lq = lq_n;
      const int4 nb = nb_n;
      const double k2 = k2_n;
      const int pn = pos + per;
      if (pn < p1) {
        lq_n = __ldg(A.lpq + pn);
        nb_n = __ldg(A.nbr + pn);
        k2_n = __ldg(k2c + pn);
      }
      const cplx b = (A.bmask && !__ldg(A.bmask + pos)) ? cmk(0, 0) : Bv[pos];
      b2 += cnorm2(b);
      const cplx ax = ax_row_t(X, pos, A.wnx, A.wny, A.ih2, sa, k2, lq, nb);
      r2 += cnorm2(csub(b, ax));
    }
    }
  }
  sr[tid] = r2;
  sb[tid] = b2;
  __syncthreads();
  if (tid < M) {
    double R = 0, Bs = 0;
    for (int q = tid; q < per * M; q += M) {
      R += sr[q];
      Bs += sb[q];
    }
    const int tk = A.vm.cmem[c0 + k0 + tid];
    A.part[((long long)tk * A.nchunk + blockIdx.x) * 2 + 0] = R;
    A.part[((long long)tk * A.nchunk + blockIdx.x) * 2 + 1] = Bs;
  }
}

__global__ void k_finish_init(CheckArgs A, RefineArgs R, int* done);

// all members of class blockIdx.y, 256 at a time (a thread per member and position)
__global__ void __launch_bounds__(256, HDDM_CHECK_MINB) k_check(CheckArgs A) {
  __shared__ double sr[256], sb[256];
  const int c = blockIdx.y;
  const int m = A.vm.cptr[c + 1] - A.vm.cptr[c];
  for (int k0 = 0; k0 < m; k0 += 256) {
    check_block(A, c, k0, min(256, m - k0), sr, sb);
    __syncthreads();
  }
}

// the members of tile blockIdx.y of a tile group (right after that group's solve)
__global__ void __launch_bounds__(256, HDDM_CHECK_MINB) k_check_tiles(CheckArgs A, TileArg G) {
  __shared__ double sr[256], sb[256];
  const TileRec* r = G.rec + blockIdx.y;
  const int c = r->c;
  check_block(A, c, int(r->cb - A.vm.cbase[c]), G.M, sr, sb);
}

void launch_check_tiles(const CheckArgs& A, const TileArg& G, cudaStream_t st) {
  if (G.ntile == 0) return;
  k_check_tiles<<<dim3(A.nchunk, G.ntile), 256, 0, st>>>(A, G);
}

// per-RHS rel + refinement init from partials already written (after the
// per-group checks of the forked solve)
void launch_finish_init(const CheckArgs& A, const RefineArgs& R, int* done, cudaStream_t st) {
  cudaMemsetAsync(R.any, 0, sizeof(int), st);
  k_finish_init<<<unsigned((A.nsub * 32 + 255) / 256), 256, 0, st>>>(A, R, done);
}

__global__ void k_check_finish(CheckArgs A, int nsub) {
  for (int t = threadIdx.x; t < nsub; t += blockDim.x) {
    double r2 = 0, b2 = 0;
    for (int k = 0; k < A.nchunk; ++k) {
      r2 += A.part[((long long)t * A.nchunk + k) * 2];
      b2 += A.part[((long long)t * A.nchunk + k) * 2 + 1];
    }
    const double rel = b2 > 0 ? sqrt(r2) / sqrt(b2) : 0.0;
    A.rel[t] = rel;
    if (rel > 1e-11) atomicAdd(A.refine_flag, 1);
    // max_rel: deterministic (max is order-free); atomicMax on the bit pattern of a
    // nonnegative double preserves ordering
    atomicMax(reinterpret_cast<unsigned long long*>(A.max_rel),
              (unsigned long long)__double_as_longlong(rel));
  }
}

__device__ __forceinline__ void set_cond(unsigned long long h, int v) {
  if (h) cudaGraphSetConditional(cudaGraphConditionalHandle(h), unsigned(v));
}

// check_finish + refine_init in one pass: a warp per right-hand side sums its
// partials (fixed tree order), records rel for the stopping statistics and the
// refinement state; the last block to finish sets the WHILE condition.
__global__ void k_finish_init(CheckArgs A, RefineArgs R, int* done) {
  const int lane = threadIdx.x & 31;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int need = 0;
  if (t < A.nsub) {
    double r2 = 0, b2 = 0;
    for (int k = lane; k < A.nchunk; k += 32) {
      r2 += A.part[((long long)t * A.nchunk + k) * 2];
      b2 += A.part[((long long)t * A.nchunk + k) * 2 + 1];
    }
    r2 = warp_sum(r2);
    b2 = warp_sum(b2);
    if (lane == 0) {
      const double rel = b2 > 0 ? sqrt(r2) / sqrt(b2) : 0.0;
      A.rel[t] = rel;
      if (rel > 1e-11) atomicAdd(A.refine_flag, 1);
      atomicMax(reinterpret_cast<unsigned long long*>(A.max_rel),
                (unsigned long long)__double_as_longlong(rel));
      need = (!R.zc[t] && b2 > 0 && rel > 1e-11) ? 1 : 0;
      R.rel_cur[t] = rel;
      R.need[t] = need;
      R.ncorr[t] = 0;
      R.undo[t] = 0;
    }
  }
  const int any = __syncthreads_or(need);
  if (threadIdx.x == 0) {
    if (any) atomicOr(R.any, 1);
    __threadfence();
    if (atomicAdd(done, 1) == int(gridDim.x) - 1) {  // last block: all flags are in
      __threadfence();
      set_cond(R.cond, *reinterpret_cast<volatile int*>(R.any));
      *done = 0;
    }
  }
}

void launch_check_init(const CheckArgs& A, const RefineArgs& R, int* done, cudaStream_t st) {
  dim3 g(A.nchunk, A.vm.ncls);
  k_check<<<g, 256, 0, st>>>(A);
  cudaMemsetAsync(R.any, 0, sizeof(int), st);
  k_finish_init<<<unsigned((A.nsub * 32 + 255) / 256), 256, 0, st>>>(A, R, done);
}

void launch_check_partials(const CheckArgs& A, cudaStream_t st) {
  dim3 g(A.nchunk, A.vm.ncls);
  k_check<<<g, 256, 0, st>>>(A);
}

void launch_check(const CheckArgs& A, cudaStream_t st) {
  dim3 g(A.nchunk, A.vm.ncls);
  k_check<<<g, 256, 0, st>>>(A);
  k_check_finish<<<1, 256, 0, st>>>(A, A.nsub);
}

// ------------------------------------------------------------ refinement

// first pass done: rel[t] from the check partials; start refining RHS above 1e-11
__global__ void k_refine_init(RefineArgs R) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < R.nsub; t += blockDim.x) {
    double r2 = 0, b2 = 0;
    for (int k = 0; k < R.nchunk; ++k) {
      r2 += R.part[((long long)t * R.nchunk + k) * 2];
      b2 += R.part[((long long)t * R.nchunk + k) * 2 + 1];
    }
    const double rel = b2 > 0 ? sqrt(r2) / sqrt(b2) : 0.0;
    const int nd = (!R.zc[t] && b2 > 0 && rel > 1e-11) ? 1 : 0;
    R.rel_cur[t] = rel;
    R.need[t] = nd;
    R.ncorr[t] = 0;
    R.undo[t] = 0;
    if (nd) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *R.any = any;
    set_cond(R.cond, any);
  }
}

// R = B - A X for the refining RHS
__global__ void __launch_bounds__(256) k_refine_resid(RefineArgs R) {
  const int t = blockIdx.y;
  if (!R.need[t]) return;
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= R.nw) return;
  const int c = R.sub[t].cls;
  const SVec<const cplx> X = vview((const cplx*)R.X, R.vm, t);
  const cplx ax = ax_row_t(X, pos, R.wnx, R.wny, R.ih2, R.sa + (long long)t * R.sa_stride,
                           __ldg(R.k2c + (long long)c * R.nw + pos), __ldg(R.lpq + pos),
                           __ldg(R.nbr + pos));
  const long long p = (X.p - R.X) + (long long)pos * X.s;
  R.R[p] = csub(R.B[p], ax);
}

// X += C for the refining RHS
__global__ void __launch_bounds__(256) k_refine_apply(RefineArgs R) {
  const int t = blockIdx.y;  // only the refining RHS do work
  if (!R.need[t]) return;
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= R.nw) return;
  const long long p = __ldg(R.vm.base + t) + (long long)pos * __ldg(R.vm.str + t);
  R.X[p] = cadd(R.X[p], R.C[p]);
}

// after the re-check: the reference's stagnation / stopping rules
__global__ void k_refine_decide(RefineArgs R) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < R.nsub; t += blockDim.x) {
    if (!R.need[t]) continue;
    const int nc = ++R.ncorr[t];
    atomicAdd(reinterpret_cast<unsigned long long*>(R.nfix), 1ULL);
    if (nc >= 12) {  // the reference's loop ends after its 12th correction
      R.need[t] = 0;
      continue;
    }
    double r2 = 0, b2 = 0;
    for (int k = 0; k < R.nchunk; ++k) {
      r2 += R.part[((long long)t * R.nchunk + k) * 2];
      b2 += R.part[((long long)t * R.nchunk + k) * 2 + 1];
    }
    const double rn = b2 > 0 ? sqrt(r2) / sqrt(b2) : 0.0;
    const double rel = R.rel_cur[t];
    if (rn >= 0.5 * rel) {  // stagnation: stop, undoing a correction that hurt
      if (rn > rel) R.undo[t] = 1;
      R.rel_cur[t] = rn < rel ? rn : rel;  // refine returns min(r, rel)
      R.need[t] = 0;
    } else {
      R.rel_cur[t] = rn;
      if (rn <= 1e-11) R.need[t] = 0;
    }
    if (R.need[t]) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *R.any = any;
    set_cond(R.cond, any);
  }
}

__global__ void __launch_bounds__(256) k_refine_undo(RefineArgs R) {
  const int t = blockIdx.y;
  if (!R.undo[t]) return;  // flag cleared by the next init
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= R.nw) return;
  const long long p = __ldg(R.vm.base + t) + (long long)pos * __ldg(R.vm.str + t);
  R.X[p] = csub(R.X[p], R.C[p]);
}

void launch_refine_init(const RefineArgs& R, cudaStream_t st) {
  k_refine_init<<<1, 256, 0, st>>>(R);
}
void launch_refine_prep(const RefineArgs& R, cudaStream_t st) {
  dim3 g((R.nw + 255) / 256, R.nsub);
  k_refine_resid<<<g, 256, 0, st>>>(R);
}
void launch_refine_apply(const RefineArgs& R, cudaStream_t st) {
  k_refine_apply<<<dim3((R.nw + 255) / 256, R.nsub), 256, 0, st>>>(R);
}
void launch_refine_decide(const RefineArgs& R, cudaStream_t st) {
  k_refine_decide<<<1, 256, 0, st>>>(R);
}
void launch_refine_undo(const RefineArgs& R, cudaStream_t st) {
  k_refine_undo<<<dim3((R.nw + 255) / 256, R.nsub), 256, 0, st>>>(R);
}

// ------------------------------------------------------------ global stencil
// DiscreteOperator::apply (discretize.cpp:81-96) on the global window; when f is
// given, also per-block partial sums of |f - L u|^2 (residual_norm, ddm.cpp:237-242).
__device__ __forceinline__ void apply_global_body(const GlobalArgs& G, const cplx* u, cplx* out,
                                                  const cplx* f, double* part) {
  __shared__ double sh[32];
  const long long n = (long long)G.gnx * G.gny;
  const cplx* a1n = G.ga;
  const cplx* ia1h = G.ga + G.gnx;
  const cplx* a2n = G.ga + 2 * G.gnx;
  const cplx* ia2h = G.ga + 2 * G.gnx + G.gny;
  double acc = 0;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int p = int(idx % G.gnx), q = int(idx / G.gnx);
    cplx o;
    if (p == 0 || q == 0 || p == G.gnx - 1 || q == G.gny - 1) {
      o = u[idx];
    } else {
      const cplx uc = u[idx];
      const cplx ex = cscale(a2n[q], G.ih2);
      const cplx ey = cscale(a1n[p], G.ih2);
      cplx tt = cmul(cmul(ex, ia1h[p]), csub(u[idx + 1], uc));
      tt = csub(tt, cmul(cmul(ex, ia1h[p - 1]), csub(uc, u[idx - 1])));
      tt = cadd(tt, cmul(cmul(ey, ia2h[q]), csub(u[idx + G.gnx], uc)));
      tt = csub(tt, cmul(cmul(ey, ia2h[q - 1]), csub(uc, u[idx - G.gnx])));
      o = cadd(cdiv(tt, cmul(a1n[p], a2n[q])), cscale(uc, G.k2[idx]));
    }
    if (out) out[idx] = o;
    if (f) acc += cnorm2(csub(f[idx], o));
  }
  if (part) {
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) k_apply_global(GlobalArgs G, const cplx* u, cplx* out,
                                                      const cplx* f, double* part) {
  apply_global_body(G, u, out, f, part);
}

// out = L u with u = U[*jp + du], out = O[*jp + dout] (device-resident Krylov index)
__global__ void __launch_bounds__(256) k_apply_global_ind(GlobalArgs G, cplx* const* U, int du,
                                                          cplx* const* O, int dout, const int* jp) {
  const int j = *jp;
  apply_global_body(G, U[j + du], O[j + dout], nullptr, nullptr);
}

void launch_apply_global(const GlobalArgs& G, const cplx* u, cplx* out, const cplx* f,
                         double* part, cudaStream_t st) {
  k_apply_global<<<kRedBlocks, 256, 0, st>>>(G, u, out, f, part);
}

void launch_apply_global_ind(const GlobalArgs& G, cplx* const* U, int du, cplx* const* O, int dout,
                             const int* jp, cudaStream_t st) {
  k_apply_global_ind<<<kRedBlocks, 256, 0, st>>>(G, U, du, O, dout, jp);
}

// ------------------------------------------------------------ reductions
__global__ void __launch_bounds__(256) k_nrm2_part(const cplx* v, long long n, double* part) {
  __shared__ double sh[32];
  double acc = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc += cnorm2(v[i]);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dot_part(const cplx* a, const cplx* b, long long n,
                                                  double* part) {
  __shared__ double sh[32];
  double re = 0, im = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const cplx x = a[i], y = b[i];  // conj(x) * y
    re += x.x * y.x + x.y * y.y;
    im += x.x * y.y - x.y * y.x;
  }
  const double s0 = block_sum(re, sh);
  const double s1 = block_sum(im, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

// one warp sums the partials in a fixed order
__global__ void k_finish_sum(const double* part, int ncomp, double* out) {
  const int lane = threadIdx.x;
  for (int c = 0; c < ncomp; ++c) {
    double acc = 0;
    for (int i = lane; i < kRedBlocks; i += 32) acc += part[i * ncomp + c];
    acc = warp_sum(acc);
    if (lane == 0) out[c] = acc;
  }
}

void launch_nrm2_part(const cplx* v, long long n, double* part, cudaStream_t st) {
  k_nrm2_part<<<kRedBlocks, 256, 0, st>>>(v, n, part);
}
void launch_dot_part(const cplx* a, const cplx* b, long long n, double* part, cudaStream_t st) {
  k_dot_part<<<kRedBlocks, 256, 0, st>>>(a, b, n, part);
}
void launch_finish_sum(const double* part, int ncomp, double* out, cudaStream_t st) {
  k_finish_sum<<<1, 32, 0, st>>>(part, ncomp, out);
}

}  // namespace hddm
