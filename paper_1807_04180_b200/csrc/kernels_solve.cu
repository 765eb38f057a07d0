// Batched multi-RHS supernodal triangular solves (the per-step hot path that
// replaces Factorization::solve -> solve_raw, proj/src/sparse.cpp:244-266).
//
// All subdomains of a class share one factor; a CTA reads each factor entry
// once and applies it to every active member right-hand side of that class
// (up to MC per pass). Both sweeps are written in "pull" form so that every
// output value is produced by one thread in a fixed summation order:
// deterministic, no atomics.
//
//   forward, leaves:      z_leaf = L_leaf^{-1} b_leaf           (band, sequential)
//   forward, separators:  y_s = b_s - sum_{d desc.} L_{s,d} z_d  (pull)
//                         z_s = Linv_s y_s                      (dense inverse)
//   backward, separators: w_s = D_s^{-1} z_s - sum_{a anc.} L_{a,s}^T x_a
//                         x_s = Linv_s^T w_s
//   backward, leaves:     same, with a band back-substitution
//   ring (identity rows): x = b
//
// Work split: the maximal ND subtrees of at most np_max nodes (contiguous
// position ranges in postorder) are solved by ONE CTA each with the member
// vectors resident in shared memory for the whole subtree (k_*_subtree);
// only the separators above them go through level-synchronous kernels
// (k_fwd_pull/diag, k_bwd_pull/diag), whose pulls read subtree results from HBM.
// Vectors are in factor order; RHS index = subdomain id, stride nw.
#include "dev.cuh"
#include "kernels.cuh"

namespace hddm {

namespace {

constexpr int MR = 8;         // member right-hand sides per register pass (top levels)
constexpr int kSubWarps = 8;  // warps per CTA of the subtree kernels

__device__ __forceinline__ int load_members(const SolveArgs& A, int c, int* sm) {
  const int b = A.act_ptr[c], e = A.act_ptr[c + 1];
  for (int k = threadIdx.x; k < e - b; k += blockDim.x) sm[k] = A.act_list[b + k];
  __syncthreads();
  return e - b;
}

__device__ __forceinline__ void csub_mul(cplx& acc, cplx l, cplx x) {
  acc.x -= l.x * x.x - l.y * x.y;
  acc.y -= l.x * x.y + l.y * x.x;
}

// Stage the segment table of a forward run into per-warp shared memory.
__device__ __forceinline__ int stage_segs(const SolveArgs& A, int pos, int2* segs, int lane) {
  const int s0 = A.seg_ptr[pos], ns = A.seg_ptr[pos + 1] - s0;
  for (int i = lane; i < ns; i += 32) segs[i] = A.seg[s0 + i];
  __syncwarp();
  return ns;
}

// sum_q run[q] * z(src(q)) over one contiguous incoming run (single RHS); the
// lanes walk the run in stride 32 and track their segment incrementally.
template <class ZGet>
__device__ __forceinline__ cplx run_dot(const cplx* __restrict__ run, const int2* segs, int ns,
                                        int total, ZGet zget, int lane) {
  cplx acc = cmk(0, 0);
  int k = 0, segstart = 0;
  int2 sg = ns > 0 ? segs[0] : make_int2(0, 0);
  for (int q = lane; q < total; q += 32) {
    while (q >= segstart + sg.x) {
      segstart += sg.x;
      sg = segs[++k];
    }
    cfma(acc, ldg(run + q), zget(sg.y + (q - segstart)));
  }
  return warp_sum(acc);
}

// sum over a supernode's backward rows of L[r][j] * x(dst r) (single RHS),
// four rows per batch so their loads are in flight together.
template <class XGet>
__device__ __forceinline__ cplx bw_dot(const cplx* __restrict__ vals, const BwRow* __restrict__ rows,
                                       int nrows, int j, XGet xget) {
  cplx acc = cmk(0, 0);
  int k = 0;
  constexpr int U = 8;
  for (; k + U <= nrows; k += U) {
    BwRow d[U];
    cplx l[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = rows[k + u];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      l[u] = j >= d[u].first ? ldg(vals + d[u].off + (j - d[u].first)) : cmk(0, 0);
      x[u] = xget(d[u].dpos);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cfma(acc, l[u], x[u]);
  }
  for (; k < nrows; ++k) {
    const BwRow d = rows[k];
    if (j >= d.first) cfma(acc, ldg(vals + d.off + (j - d.first)), xget(d.dpos));
  }
  return acc;
}

// L2 prefetch of the factor data phase ph will read (forward: the leaves'
// bands / the separators' incoming runs and inverses; backward: the rows of the
// phase's supernodes and their inverses). Issued one phase ahead.
__device__ __forceinline__ void prefetch_phase(const SolveArgs& A, const SubtreeArgs& T,
                                               const cplx* vals, int ph, bool fwd, int lane) {
  const Phase P = T.ph[ph];
  const int2* items = T.items + P.it0;
  for (int q = lane; q < P.nit; q += 32) {
    const int2 it = items[q];
    if (P.kind == 1 && it.y != 0) continue;  // one entry per separator
    const DevSn sn = A.sn[it.x];
    if (sn.kind == 0) {
      // [1/D | band] is contiguous
      const long long e = A.row_off[sn.drow0 + sn.n - 1] + (sn.n - 1 - A.row_first[sn.drow0 + sn.n - 1]);
      if (fwd) prefetch_l2(vals + sn.dinv_off, unsigned((e - sn.dinv_off) * sizeof(cplx)));
    } else {
      const long long e = sn.diag_off + (long long)sn.n * (sn.n - 1) / 2;
      prefetch_l2(vals + sn.dinv_off, unsigned((e - sn.dinv_off) * sizeof(cplx)));
      if (fwd) {
        const long long r0 = A.run_off[sn.c0], r1 = A.run_off[sn.c0 + sn.n];
        prefetch_l2(vals + r0, unsigned((r1 - r0) * sizeof(cplx)));
      }
    }
    if (!fwd) {
      for (int r = A.bw_ptr[it.x]; r < A.bw_ptr[it.x + 1]; ++r) {
        const BwRow d = A.bw[r];
        prefetch_l2(vals + d.off, unsigned((sn.n - d.first) * sizeof(cplx)));
      }
    }
  }
}

}  // namespace

// ====================================================================== subtrees
//
// One WARP per (class, subtree, right-hand side): the warp keeps the subtree's
// slice of its vector in shared memory and walks the phases bottom-up
// (forward) or top-down (backward) with only __syncwarp between phases, so the
// many independent warps on an SM hide each other's latency. Warps are ordered
// class-major, then subtree, then member: the warps of one CTA mostly share a
// (class, subtree), so the factor lines they stream are served from L1/L2
// after the first touch (HBM sees each factor once per pass).

// warp-list prefix over classes: wprefix[c] = sum_{c'<c} m_c' * nsubtree
__global__ void k_wprefix(const int* act_ptr, int ncls, int nsubtree, int* wprefix) {
  if (threadIdx.x != 0) return;
  int acc = 0;
  for (int c = 0; c < ncls; ++c) {
    wprefix[c] = acc;
    acc += (act_ptr[c + 1] - act_ptr[c]) * nsubtree;
  }
  wprefix[ncls] = acc;
}

__device__ __forceinline__ bool decode_warp(const SolveArgs& A, const int* wprefix, int ncls,
                                            int w, int& c, int& tau, int& t) {
  if (w >= wprefix[ncls]) return false;
  int lo = 0, hi = ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (wprefix[mid] <= w) lo = mid; else hi = mid - 1;
  }
  c = lo;
  const int m = A.act_ptr[c + 1] - A.act_ptr[c];
  const int r = w - wprefix[c];
  tau = r / m;
  t = A.act_list[A.act_ptr[c] + (r - tau * m)];
  return true;
}

__device__ __forceinline__ size_t subtree_warp_words(const SubtreeArgs& T) {
  // z[np_max] + scr[items_max] (cplx) + segs[seg_max] (int2 = half a cplx)
  return (size_t)T.np_max + T.items_max + (T.seg_max + 1) / 2;
}

__global__ void __launch_bounds__(256, 3) k_fwd_subtree(SolveArgs A, SubtreeArgs T,
                                                     const int* wprefix, int ncls) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c, tau, t;
  if (!decode_warp(A, wprefix, ncls, blockIdx.x * kSubWarps + warp, c, tau, t)) return;
  const SubtreeInfo info = T.st[tau];
  const int np = info.np, p0 = info.p0;
  cplx* z = reinterpret_cast<cplx*>(s_raw) + (size_t)warp * subtree_warp_words(T);
  cplx* scr = z + T.np_max;
  int2* segs = reinterpret_cast<int2*>(scr + T.items_max);
  const cplx* vals = A.vals + (long long)c * A.nvals;
  {
    const cplx* src = A.B + (long long)t * A.nw + p0;
    for (int i = lane; i < np; i += 32) z[i] = src[i];
  }
  __syncwarp();
  prefetch_phase(A, T, vals, info.ph0, true, lane);
  for (int ph = info.ph0; ph < info.ph0 + info.nph; ++ph) {
    if (ph + 1 < info.ph0 + info.nph) prefetch_phase(A, T, vals, ph + 1, true, lane);
    const Phase P = T.ph[ph];
    if ((T.dbg >> (P.kind == 0 ? 0 : 1)) & 1) continue;
    const int2* items = T.items + P.it0;
    if (P.kind == 0) {
      // leaves: lane per leaf, band forward substitution
      for (int li = lane; li < P.nit; li += 32) {
        const DevSn sn = A.sn[items[li].x];
        cplx* zb = z + (sn.c0 - p0);
        for (int i = 0; i < sn.n; ++i) {
          const int rt = sn.drow0 + i;
          const int first = A.row_first[rt];
          const cplx* L = vals + A.row_off[rt] - first;
          cplx acc = zb[i];
          for (int q = first; q < i; ++q) csub_mul(acc, ldg(L + q), zb[q]);
          zb[i] = acc;
        }
      }
      __syncwarp();
      continue;
    }
    // separator rows: y = b - (incoming run) . z. A warp walks four rows at a
    // time with its lanes over the run elements (coalesced loads, eight
    // independent global loads per lane per step); zidx gives each element's
    // source position.
    for (int g = 0; g < P.nit; g += 4) {
      const cplx* run[4];
      const int* zi[4];
      int tot[4], pos[4];
      int maxlen = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tot[k] = 0;
        pos[k] = -1;
        if (g + k < P.nit) {
          const int2 item = items[g + k];
          pos[k] = A.sn[item.x].c0 + item.y;
          const long long r0 = A.run_off[pos[k]];
          run[k] = vals + r0;
          zi[k] = A.zidx + r0;
          tot[k] = int(A.run_off[pos[k] + 1] - r0);
          maxlen = max(maxlen, tot[k]);
        } else {
          run[k] = vals;
          zi[k] = A.zidx;
        }
      }
      cplx acc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = cmk(0, 0);
      for (int q = lane; q < maxlen; q += 32) {
        cplx l[4];
        int ix[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool ok = q < tot[k];
          l[k] = ok ? ldg(run[k] + q) : cmk(0, 0);
          ix[k] = ok ? __ldg(zi[k] + q) - p0 : 0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) cfma(acc[k], l[k], z[ix[k]]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const cplx sum = warp_sum(acc[k]);
        if (lane == 0 && pos[k] >= 0) scr[g + k] = csub(z[pos[k] - p0], sum);
      }
    }
    __syncwarp();
    for (int it = lane; it < P.nit; it += 32) {
      const int2 item = items[it];
      z[A.sn[item.x].c0 + item.y - p0] = scr[it];
    }
    __syncwarp();
    // z_s = Linv_s y_s, lane per row, to scratch
    for (int it = lane; it < P.nit; it += 32) {
      const int2 item = items[it];
      const DevSn sn = A.sn[item.x];
      const int i = item.y;
      const cplx* row = vals + sn.diag_off + (long long)i * (i - 1) / 2;
      const cplx* ys = z + (sn.c0 - p0);
      cplx acc = ys[i];
      for (int j = 0; j < i; ++j) cfma(acc, ldg(row + j), ys[j]);
      scr[it] = acc;
    }
    __syncwarp();
    for (int it = lane; it < P.nit; it += 32) {
      const int2 item = items[it];
      z[A.sn[item.x].c0 + item.y - p0] = scr[it];
    }
    __syncwarp();
  }
  {
    cplx* dst = A.X + (long long)t * A.nw + p0;
    for (int i = lane; i < np; i += 32) dst[i] = z[i];
  }
}

__global__ void __launch_bounds__(256, 3) k_bwd_subtree(SolveArgs A, SubtreeArgs T,
                                                     const int* wprefix, int ncls) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c, tau, t;
  if (!decode_warp(A, wprefix, ncls, blockIdx.x * kSubWarps + warp, c, tau, t)) return;
  const SubtreeInfo info = T.st[tau];
  const int np = info.np, p0 = info.p0;
  cplx* z = reinterpret_cast<cplx*>(s_raw) + (size_t)warp * subtree_warp_words(T);
  cplx* scr = z + T.np_max;
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const cplx* Xg = A.X + (long long)t * A.nw;
  for (int i = lane; i < np; i += 32) z[i] = Xg[p0 + i];
  __syncwarp();
  auto xget = [&](int dpos) {
    return (dpos >= p0 && dpos < p0 + np) ? z[dpos - p0] : Xg[dpos];
  };
  for (int ph = info.ph0 + info.nph - 1; ph >= info.ph0; --ph) {
    const Phase P = T.ph[ph];
    if ((T.dbg >> (P.kind == 0 ? 2 : 3)) & 1) continue;
    if (P.kind == 0) {
      // leaf columns: w_j = Dinv_j z_j - sum_r L[r][j] x_r, lane per column
      // (lanes of one leaf read consecutive columns of each row: coalesced)
      {
        const int2* cols = T.items + P.ic0;
        for (int q = lane; q < P.nic; q += 32) {
          const int2 it = cols[q];
          const DevSn sn = A.sn[it.x];
          const int j = it.y;
          const int b0 = A.bw_ptr[it.x];
          const cplx sm = bw_dot(vals, A.bw + b0, A.bw_ptr[it.x + 1] - b0, j, xget);
          // each (leaf, column) is owned by one lane and only reads x outside the
          // leaf, so the update is in place
          z[sn.c0 + j - p0] = csub(cmul(ldg(vals + sn.dinv_off + j), z[sn.c0 + j - p0]), sm);
        }
      }
      __syncwarp();
      // band back-substitution, lane per leaf
      const int2* items = T.items + P.it0;
      for (int li = lane; li < P.nit; li += 32) {
        const DevSn sn = A.sn[items[li].x];
        cplx* zb = z + (sn.c0 - p0);
        for (int i = sn.n - 1; i >= 0; --i) {
          const cplx xi = zb[i];
          const int rt = sn.drow0 + i;
          const int first = A.row_first[rt];
          const cplx* L = vals + A.row_off[rt] - first;
          for (int q = first; q < i; ++q) csub_mul(zb[q], ldg(L + q), xi);
        }
      }
      __syncwarp();
      continue;
    }
    const int2* items = T.items + P.it0;
    // separator columns: w = Dinv z - sum L^T x, lane per column, to scratch
    for (int q = lane; q < P.nit; q += 32) {
      const int2 item = items[q];
      const DevSn sn = A.sn[item.x];
      const int j = item.y;
      const int b0 = A.bw_ptr[item.x];
      const cplx s = bw_dot(vals, A.bw + b0, A.bw_ptr[item.x + 1] - b0, j, xget);
      scr[q] = csub(cmul(ldg(vals + sn.dinv_off + j), z[sn.c0 + j - p0]), s);
    }
    __syncwarp();
    // x_s = Linv_s^T w_s (items of one separator are contiguous, column order)
    for (int q = lane; q < P.nit; q += 32) {
      const int2 item = items[q];
      const DevSn sn = A.sn[item.x];
      const int j = item.y;
      const cplx* Linv = vals + sn.diag_off;
      const int q0 = q - j;
      cplx acc = scr[q];
      for (int i = j + 1; i < sn.n; ++i)
        cfma(acc, ldg(Linv + (long long)i * (i - 1) / 2 + j), scr[q0 + i]);
      z[sn.c0 + j - p0] = acc;
    }
    __syncwarp();
  }
  {
    cplx* dst = A.X + (long long)t * A.nw + p0;
    for (int i = lane; i < np; i += 32) dst[i] = z[i];
  }
}

// ====================================================================== top levels

// Forward pull for separator rows: Y[r] = B[r] - run . X (MR members per pass).
// Warp per row, two run elements per lane per iteration; the source position of
// every run element comes from the structural zidx array (shared by all
// classes, so it stays L2-resident).
__global__ void __launch_bounds__(256) k_fwd_pull(SolveArgs A, const Task* tasks) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const Task T = tasks[blockIdx.x];
  const DevSn sn = A.sn[T.s];
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int r = T.a + warp; r < T.b; r += nwarp) {
    const int pos = sn.c0 + r;
    const long long r0 = A.run_off[pos];
    const cplx* run = vals + r0;
    const int* zi = A.zidx + r0;
    const int total = int(A.run_off[pos + 1] - r0);
    for (int mb = 0; mb < m; mb += MR) {
      const int mc = min(MR, m - mb);
      cplx acc[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
      int q = lane;
      for (; q + 32 < total; q += 64) {
        const cplx l0 = ldg(run + q), l1 = ldg(run + q + 32);
        const int i0 = __ldg(zi + q), i1 = __ldg(zi + q + 32);
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          if (k < mc) {
            const cplx* Xk = A.X + (long long)s_mem[mb + k] * A.nw;
            cfma(acc[k], l0, Xk[i0]);
            cfma(acc[k], l1, Xk[i1]);
          }
        }
      }
      if (q < total) {
        const cplx l0 = ldg(run + q);
        const int i0 = __ldg(zi + q);
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (k < mc) cfma(acc[k], l0, A.X[(long long)s_mem[mb + k] * A.nw + i0]);
      }
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        if (k < mc) {
          const cplx sum = warp_sum(acc[k]);
          if (lane == k) {
            const long long base = (long long)s_mem[mb + k] * A.nw;
            A.Y[base + pos] = csub(A.B[base + pos], sum);
          }
        }
      }
    }
  }
}

// Forward diagonal for separator rows: X[i] = Y[i] + sum_{k<i} Linv[i][k] Y[k].
__global__ void __launch_bounds__(256) k_fwd_diag(SolveArgs A, const Task* tasks) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const Task T = tasks[blockIdx.x];
  const DevSn sn = A.sn[T.s];
  const cplx* Linv = A.vals + (long long)c * A.nvals + sn.diag_off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int i = T.a + warp; i < T.b; i += nwarp) {
    const cplx* row = Linv + (long long)i * (i - 1) / 2;
    for (int mb = 0; mb < m; mb += MR) {
      const int mc = min(MR, m - mb);
      cplx acc[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
      for (int j = lane; j < i; j += 32) {
        const cplx l = ldg(row + j);
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (k < mc) cfma(acc[k], l, A.Y[(long long)s_mem[mb + k] * A.nw + sn.c0 + j]);
      }
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        if (k < mc) {
          const cplx s = warp_sum(acc[k]);
          if (lane == k) {
            const long long p = (long long)s_mem[mb + k] * A.nw + sn.c0 + i;
            A.X[p] = cadd(A.Y[p], s);
          }
        }
      }
    }
  }
}

// Backward pull for separator columns: Y[j] = Dinv[j] X[j] - sum_rows L[r][j] x_r.
// Lane per column (32-column tasks); the supernode's backward rows are split
// over the warps and the per-warp partial sums are combined in fixed warp order.
__global__ void __launch_bounds__(256) k_bwd_pull(SolveArgs A, const Task* tasks) {
  extern __shared__ int s_mem[];
  __shared__ cplx part[8][MR][32];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const Task T = tasks[blockIdx.x];
  const DevSn sn = A.sn[T.s];
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int j = T.a + lane;
  const bool colok = j < T.b;
  const int r0 = A.bw_ptr[T.s], r1 = A.bw_ptr[T.s + 1];
  for (int mb = 0; mb < m; mb += MR) {
    const int mc = min(MR, m - mb);
    cplx acc[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
    if (colok) {
      int r = r0 + warp;
      for (; r + nwarp < r1; r += 2 * nwarp) {
        const BwRow d0 = A.bw[r], d1 = A.bw[r + nwarp];
        const cplx l0 = j >= d0.first ? ldg(vals + d0.off + (j - d0.first)) : cmk(0, 0);
        const cplx l1 = j >= d1.first ? ldg(vals + d1.off + (j - d1.first)) : cmk(0, 0);
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          if (k < mc) {
            const cplx* Xk = A.X + (long long)s_mem[mb + k] * A.nw;
            cfma(acc[k], l0, Xk[d0.dpos]);
            cfma(acc[k], l1, Xk[d1.dpos]);
          }
        }
      }
      if (r < r1) {
        const BwRow d = A.bw[r];
        if (j >= d.first) {
          const cplx l = ldg(vals + d.off + (j - d.first));
#pragma unroll
          for (int k = 0; k < MR; ++k)
            if (k < mc) cfma(acc[k], l, A.X[(long long)s_mem[mb + k] * A.nw + d.dpos]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < MR; ++k) part[warp][k][lane] = acc[k];
    __syncthreads();
    if (warp == 0 && colok) {
      for (int k = 0; k < mc; ++k) {
        cplx s = part[0][k][lane];
        for (int w = 1; w < nwarp; ++w) s = cadd(s, part[w][k][lane]);
        const long long p = (long long)s_mem[mb + k] * A.nw + sn.c0 + j;
        A.Y[p] = csub(cmul(ldg(vals + sn.dinv_off + j), A.X[p]), s);
      }
    }
    __syncthreads();
  }
}

// Backward diagonal for separator columns: X[j] = Y[j] + sum_{i>j} Linv[i][j] Y[i].
// Lane per column (32-column tasks), rows i split over the warps, per-warp
// partial sums combined in fixed warp order.
__global__ void __launch_bounds__(256) k_bwd_diag(SolveArgs A, const Task* tasks) {
  extern __shared__ int s_mem[];
  __shared__ cplx part[8][MR][32];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const Task T = tasks[blockIdx.x];
  const DevSn sn = A.sn[T.s];
  const cplx* Linv = A.vals + (long long)c * A.nvals + sn.diag_off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int j = T.a + lane;
  const bool colok = j < T.b;
  for (int mb = 0; mb < m; mb += MR) {
    const int mc = min(MR, m - mb);
    cplx acc[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
    if (colok) {
      for (int i = T.a + 1 + warp; i < sn.n; i += nwarp) {
        if (i <= j) continue;
        const cplx l = ldg(Linv + (long long)i * (i - 1) / 2 + j);
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (k < mc) cfma(acc[k], l, A.Y[(long long)s_mem[mb + k] * A.nw + sn.c0 + i]);
      }
    }
#pragma unroll
    for (int k = 0; k < MR; ++k) part[warp][k][lane] = acc[k];
    __syncthreads();
    if (warp == 0 && colok) {
      for (int k = 0; k < mc; ++k) {
        cplx s = part[0][k][lane];
        for (int w = 1; w < nwarp; ++w) s = cadd(s, part[w][k][lane]);
        const long long p = (long long)s_mem[mb + k] * A.nw + sn.c0 + j;
        A.X[p] = cadd(A.Y[p], s);
      }
    }
    __syncthreads();
  }
}

// identity ring rows: x = b
__global__ void k_ring(SolveArgs A) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < A.nring * m; g += gridDim.x * blockDim.x) {
    const int k = g / A.nring, r = g - k * A.nring;
    const long long p = (long long)s_mem[k] * A.nw + r;
    A.X[p] = A.B[p];
  }
}

// ------------------------------------------------------------------ launcher
int solve_launch_count(const SolvePlan& P) {
  return 2 + 2 + 2 * int(P.fwd.size()) + 2 * int(P.bwd.size());
}

static void launch_subtrees(const SolveArgs& A, const SolvePlan& P, int ncls, int max_rhs,
                            bool fwd, cudaStream_t st) {
  const size_t words = (size_t)P.sub.np_max + P.sub.items_max + (P.sub.seg_max + 1) / 2;
  const size_t smem = sizeof(cplx) * kSubWarps * words;
  const long long warps = (long long)max_rhs * P.nsubtree;
  const unsigned grid = unsigned((warps + kSubWarps - 1) / kSubWarps);
  if (grid == 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fwd_subtree, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_bwd_subtree, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  if (fwd)
    k_fwd_subtree<<<grid, 32 * kSubWarps, smem, st>>>(A, P.sub, P.d_wprefix, ncls);
  else
    k_bwd_subtree<<<grid, 32 * kSubWarps, smem, st>>>(A, P.sub, P.d_wprefix, ncls);
}

void launch_solve(const SolveArgs& A, const SolvePlan& P, int ncls, int max_members,
                  int max_rhs, cudaStream_t st) {
  const size_t smem = sizeof(int) * size_t(max_members);
  {
    dim3 g((A.nring * max_members + 255) / 256, ncls);
    k_ring<<<g, 256, smem, st>>>(A);
  }
  k_wprefix<<<1, 32, 0, st>>>(A.act_ptr, ncls, P.nsubtree, P.d_wprefix);
  launch_subtrees(A, P, ncls, max_rhs, true, st);
  for (const auto& L : P.fwd) {
    dim3 g(L.ntask, ncls);
    k_fwd_pull<<<g, 256, smem, st>>>(A, L.d_tasks);
    k_fwd_diag<<<g, 256, smem, st>>>(A, L.d_tasks);
  }
  for (const auto& L : P.bwd) {
    dim3 g(L.ntask32, ncls);
    k_bwd_pull<<<g, 256, smem, st>>>(A, L.d_tasks32);
    k_bwd_diag<<<g, 256, smem, st>>>(A, L.d_tasks32);
  }
  launch_subtrees(A, P, ncls, max_rhs, false, st);
}

}  // namespace hddm
