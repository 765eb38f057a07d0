// Batched multi-RHS supernodal triangular solves (the per-step hot path that
// replaces Factorization::solve -> solve_raw, proj/src/sparse.cpp:244-266).
//
// All subdomains of a class share one factor; every kernel reads a factor
// entry ONCE per CTA pass and applies it to all active member right-hand sides
// of that class (up to MR at a time). Both sweeps are written in "pull" form so
// that every output value is produced by exactly one thread in a fixed
// summation order: deterministic, no atomics.
//
//   forward, leaves:      z_leaf = L_leaf^{-1} b_leaf         (band, sequential)
//   forward, separators:  y_s = b_s - sum_{d desc.} L_{s,d} z_d  (pull)
//                         z_s = Linv_s y_s                    (dense inverse)
//   backward, separators: w_s = D_s^{-1} z_s - sum_{a anc.} L_{a,s}^T x_a
//                         x_s = Linv_s^T w_s
//   backward, leaves:     same, with a band back-substitution
//   ring (identity rows): x = b
//
// Vectors are in factor order; RHS index = subdomain id, stride nw.
#include "dev.cuh"
#include "kernels.cuh"

namespace hddm {

namespace {

constexpr int MR = 8;  // member right-hand sides per register pass

__device__ __forceinline__ int load_members(const SolveArgs& A, int c, int* sm) {
  const int b = A.act_ptr[c], e = A.act_ptr[c + 1];
  for (int k = threadIdx.x; k < e - b; k += blockDim.x) sm[k] = A.act_list[b + k];
  __syncthreads();
  return e - b;
}

}  // namespace

// Forward pull for separator rows: Y[r] = B[r] - sum L z. Warp per row.
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
    const int e0 = A.rin_ptr[pos], e1 = A.rin_ptr[pos + 1];
    for (int mb = 0; mb < m; mb += MR) {
      const int mc = min(MR, m - mb);
      cplx acc[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
      for (int e = e0; e < e1; ++e) {
        const RowIn in = A.rin[e];
        const int first = A.row_first[in.rowtab];
        const cplx* L = vals + A.row_off[in.rowtab] - first;
        for (int j = first + lane; j < in.src_n; j += 32) {
          const cplx l = ldg(L + j);
#pragma unroll
          for (int k = 0; k < MR; ++k)
            if (k < mc) cfma(acc[k], l, A.X[(long long)s_mem[mb + k] * A.nw + in.src_c0 + j]);
        }
      }
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        if (k < mc) {
          const cplx s = warp_sum(acc[k]);
          if (lane == 0) {
            const long long base = (long long)s_mem[mb + k] * A.nw;
            A.Y[base + pos] = csub(A.B[base + pos], s);
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
          if (lane == 0) {
            const long long p = (long long)s_mem[mb + k] * A.nw + sn.c0 + i;
            A.X[p] = cadd(A.Y[p], s);
          }
        }
      }
    }
  }
}

// Backward pull for separator columns: Y[j] = Dinv[j] X[j] - sum_b L_b[.][j]^T x.
// Thread per column.
__global__ void __launch_bounds__(256) k_bwd_pull(SolveArgs A, const Task* tasks) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const Task T = tasks[blockIdx.x];
  const DevSn sn = A.sn[T.s];
  const cplx* vals = A.vals + (long long)c * A.nvals;
  for (int j = T.a + threadIdx.x; j < T.b; j += blockDim.x) {
    const cplx dinv = ldg(vals + sn.dinv_off + j);
    for (int mb = 0; mb < m; mb += MR) {
      const int mc = min(MR, m - mb);
      cplx acc[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
      for (int b = sn.blk0; b < sn.blk0 + sn.nblk; ++b) {
        const DevBlk B = A.blk[b];
        const int dst_c0 = A.sn[B.dst].c0 + B.r0;
        for (int r = 0; r < B.nr; ++r) {
          const int first = A.row_first[B.row0 + r];
          if (j < first) continue;
          const cplx l = ldg(vals + A.row_off[B.row0 + r] + (j - first));
#pragma unroll
          for (int k = 0; k < MR; ++k)
            if (k < mc) cfma(acc[k], l, A.X[(long long)s_mem[mb + k] * A.nw + dst_c0 + r]);
        }
      }
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        if (k < mc) {
          const long long p = (long long)s_mem[mb + k] * A.nw + sn.c0 + j;
          A.Y[p] = csub(cmul(dinv, A.X[p]), acc[k]);
        }
      }
    }
  }
}

// Backward diagonal for separator columns: X[j] = Y[j] + sum_{i>j} Linv[i][j] Y[i].
__global__ void __launch_bounds__(256) k_bwd_diag(SolveArgs A, const Task* tasks) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const Task T = tasks[blockIdx.x];
  const DevSn sn = A.sn[T.s];
  const cplx* Linv = A.vals + (long long)c * A.nvals + sn.diag_off;
  for (int j = T.a + threadIdx.x; j < T.b; j += blockDim.x) {
    for (int mb = 0; mb < m; mb += MR) {
      const int mc = min(MR, m - mb);
      cplx acc[MR];
#pragma unroll
      for (int k = 0; k < MR; ++k) acc[k] = cmk(0, 0);
      for (int i = j + 1; i < sn.n; ++i) {
        const cplx l = ldg(Linv + (long long)i * (i - 1) / 2 + j);
#pragma unroll
        for (int k = 0; k < MR; ++k)
          if (k < mc) cfma(acc[k], l, A.Y[(long long)s_mem[mb + k] * A.nw + sn.c0 + i]);
      }
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        if (k < mc) {
          const long long p = (long long)s_mem[mb + k] * A.nw + sn.c0 + j;
          A.X[p] = cadd(A.Y[p], acc[k]);
        }
      }
    }
  }
}

// Leaves (and the identity ring): one thread per (leaf, member).
// forward: z_i = b_i - sum_{k in [first_i, i)} L[i][k] z_k
__global__ void __launch_bounds__(128) k_fwd_leaf(SolveArgs A, const int* leaves, int nleaf) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  // ring: identity rows (x = b)
  const int nring_work = A.nring * m;
  const int nleaf_work = nleaf * m;
  if (gid < nleaf_work) {
    const int li = gid / m, k = gid % m;
    const DevSn sn = A.sn[leaves[li]];
    const long long base = (long long)s_mem[k] * A.nw + sn.c0;
    for (int i = 0; i < sn.n; ++i) {
      const int rt = sn.drow0 + i;
      const int first = A.row_first[rt];
      const cplx* L = vals + A.row_off[rt] - first;
      cplx z = A.B[base + i];
      for (int q = first; q < i; ++q) {
        const cplx l = ldg(L + q);
        const cplx zq = A.X[base + q];
        z.x -= l.x * zq.x - l.y * zq.y;
        z.y -= l.x * zq.y + l.y * zq.x;
      }
      A.X[base + i] = z;
    }
  } else if (gid < nleaf_work + nring_work) {
    const int g = gid - nleaf_work;
    const int k = g / A.nring, r = g % A.nring;
    const long long p = (long long)s_mem[k] * A.nw + r;
    A.X[p] = A.B[p];
  }
}

// backward: w_j = Dinv_j z_j - sum_blocks L^T x ; x = L_leaf^{-T} w
__global__ void __launch_bounds__(128) k_bwd_leaf(SolveArgs A, const int* leaves, int nleaf) {
  extern __shared__ int s_mem[];
  const int c = blockIdx.y;
  const int m = load_members(A, c, s_mem);
  if (m == 0) return;
  const cplx* vals = A.vals + (long long)c * A.nvals;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nleaf * m) return;
  const int li = gid / m, k = gid % m;
  const DevSn sn = A.sn[leaves[li]];
  const long long rbase = (long long)s_mem[k] * A.nw;
  const long long base = rbase + sn.c0;
  cplx w[36];
#pragma unroll 1
  for (int j = 0; j < sn.n; ++j) w[j] = cmul(ldg(vals + sn.dinv_off + j), A.X[base + j]);
  for (int b = sn.blk0; b < sn.blk0 + sn.nblk; ++b) {
    const DevBlk B = A.blk[b];
    const int dst_c0 = A.sn[B.dst].c0 + B.r0;
    for (int r = 0; r < B.nr; ++r) {
      const int first = A.row_first[B.row0 + r];
      const cplx* L = vals + A.row_off[B.row0 + r] - first;
      const cplx xr = A.X[rbase + dst_c0 + r];
#pragma unroll 1
      for (int j = first; j < sn.n; ++j) {
        const cplx l = ldg(L + j);
        w[j].x -= l.x * xr.x - l.y * xr.y;
        w[j].y -= l.x * xr.y + l.y * xr.x;
      }
    }
  }
#pragma unroll 1
  for (int i = sn.n - 1; i >= 0; --i) {
    const cplx xi = w[i];
    A.X[base + i] = xi;
    const int rt = sn.drow0 + i;
    const int first = A.row_first[rt];
    const cplx* L = vals + A.row_off[rt] - first;
#pragma unroll 1
    for (int q = first; q < i; ++q) {
      const cplx l = ldg(L + q);
      w[q].x -= l.x * xi.x - l.y * xi.y;
      w[q].y -= l.x * xi.y + l.y * xi.x;
    }
  }
}

// ------------------------------------------------------------------ launcher
void launch_solve(const SolveArgs& A, const SolvePlan& P, int ncls, int max_members,
                  cudaStream_t st) {
  const size_t smem = sizeof(int) * size_t(max_members);
  {
    const int work = (P.nleaf + A.nring) * max_members;
    dim3 g((work + 127) / 128, ncls);
    k_fwd_leaf<<<g, 128, smem, st>>>(A, P.d_leaves, P.nleaf);
  }
  for (size_t l = 0; l < P.fwd.size(); ++l) {
    const auto& L = P.fwd[l];
    dim3 g(L.ntask, ncls);
    k_fwd_pull<<<g, 256, smem, st>>>(A, L.d_tasks);
    k_fwd_diag<<<g, 256, smem, st>>>(A, L.d_tasks);
  }
  for (size_t l = 0; l < P.bwd.size(); ++l) {
    const auto& L = P.bwd[l];
    dim3 g(L.ntask, ncls);
    k_bwd_pull<<<g, 256, smem, st>>>(A, L.d_tasks);
    k_bwd_diag<<<g, 256, smem, st>>>(A, L.d_tasks);
  }
  {
    const int work = P.nleaf * max_members;
    dim3 g((work + 127) / 128, ncls);
    k_bwd_leaf<<<g, 128, smem, st>>>(A, P.d_leaves, P.nleaf);
  }
}

}  // namespace hddm
