// Batched multifrontal numeric LDL^T (unconjugated, no pivoting) of every
// operator class, replacing factor_ldlt (proj/src/sparse.cpp:110-174). One CTA
// per (class, supernode) of a tree level; levels run bottom-up. The pivot order
// is the reference's: supernodes are the nd_rec calls (sparse.cpp:20-57) and the
// pivots inside a supernode are eliminated in factor order, so L and D equal the
// reference's up to rounding.
//
// Per supernode s with front F = [own columns | update rows]:
//   F  = A[front, s] (scattered)  +  extend-add of the children's update blocks
//   partial right-looking LDL^T over the first n columns
//   emit 1/D, the diagonal part (separator: dense inverse of the unit-lower
//   block; leaf: its band profile) and the profile rows of every block
//   the trailing (rows x rows) part stays in the workspace for the parent.
// FP64 on the CUDA cores: B200's FP64 tensor (DMMA) rate equals its FP64 FMA
// rate, and these fronts are at most ~300 wide, so the update is written as a
// plain warp-per-row FMA sweep.
#include <algorithm>

#include "dev.cuh"
#include "kernels.cuh"

namespace hddm {

__global__ void __launch_bounds__(512) k_factor_node(FactorArgs A, const int* nodes) {
  extern __shared__ cplx s_col[];  // 2 * Fn
  const int s = nodes[blockIdx.x];
  const int c = blockIdx.y;
  const DevSn sn = A.sn[s];
  const int n = sn.n, Fn = sn.n + sn.nrows;
  cplx* F = A.front + (long long)c * A.front_words + sn.front_off;
  cplx* vals = A.vals + (long long)c * A.nvals;
  cplx* colv = s_col;
  cplx* lv = s_col + Fn;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;

  for (long long idx = tid; idx < (long long)Fn * Fn; idx += nt) F[idx] = cmk(0, 0);
  __syncthreads();
  const cplx* av = A.aval + (long long)c * A.naent;
  for (int e = sn.aent0 + tid; e < sn.aent1; e += nt)
    F[(long long)A.aent_i[e] * Fn + A.aent_j[e]] = av[e];
  __syncthreads();
  for (int k = 0; k < 2; ++k) {
    const int ch = k == 0 ? sn.child0 : sn.child1;
    if (ch < 0) continue;
    const DevSn cs = A.sn[ch];
    const int cF = cs.n + cs.nrows;
    const cplx* CF = A.front + (long long)c * A.front_words + cs.front_off;
    const int* map = A.extadd + cs.extadd0;
    for (int a = warp; a < cs.nrows; a += nwarp) {
      const int ma = map[a];
      const cplx* src = CF + (long long)(cs.n + a) * cF + cs.n;
      for (int b = lane; b <= a; b += 32) {
        cplx* dst = F + (long long)ma * Fn + map[b];
        *dst = cadd(*dst, src[b]);
      }
    }
    __syncthreads();
  }
  // partial factorization of the first n pivots
  for (int k = 0; k < n; ++k) {
    const cplx d = F[(long long)k * Fn + k];
    if (d.x == 0.0 && d.y == 0.0) {
      if (tid == 0) A.status[c] = 1;
      return;
    }
    for (int i = k + 1 + tid; i < Fn; i += nt) {
      const cplx ci = F[(long long)i * Fn + k];
      const cplx li = cdiv(ci, d);
      colv[i] = ci;
      lv[i] = li;
      F[(long long)i * Fn + k] = li;
    }
    __syncthreads();
    for (int i = k + 1 + warp; i < Fn; i += nwarp) {
      const cplx li = lv[i];
      cplx* row = F + (long long)i * Fn;
      for (int j = k + 1 + lane; j <= i; j += 32) {
        const cplx cj = colv[j];
        cplx v = row[j];
        v.x -= li.x * cj.x - li.y * cj.y;
        v.y -= li.x * cj.y + li.y * cj.x;
        row[j] = v;
      }
    }
    __syncthreads();
  }
  // emit 1/D
  for (int j = tid; j < n; j += nt)
    vals[sn.dinv_off + j] = cdiv(cmk(1.0, 0.0), F[(long long)j * Fn + j]);
  // diagonal part
  if (sn.kind == 1) {
    // dense inverse of the unit-lower block, column j per thread:
    // X[i][j] = -(L[i][j] + sum_{q=j+1}^{i-1} L[i][q] X[q][j])
    cplx* Xp = vals + sn.diag_off;  // packed strictly lower, row-major
    if (A.lss && A.lss_off[s] >= 0) {  // the block itself, row- and column-major packed
      cplx* Lp = A.lss + (long long)blockIdx.y * A.nlss + A.lss_off[s];
      cplx* Lc = A.lssc + (long long)blockIdx.y * A.nlss + A.lss_off[s];
      for (int i = tid; i < n; i += nt)
        for (int j = 0; j < i; ++j) {
          const cplx v = F[(long long)i * Fn + j];
          Lp[(long long)i * (i - 1) / 2 + j] = v;
          Lc[(long long)j * (n - 1) - (long long)j * (j - 1) / 2 + (i - j - 1)] = v;
        }
    }
    for (int j = tid; j < n; j += nt) {
      for (int i = j + 1; i < n; ++i) {
        const cplx* Li = F + (long long)i * Fn;
        cplx acc = Li[j];
        for (int q = j + 1; q < i; ++q) cfma(acc, Li[q], Xp[(long long)q * (q - 1) / 2 + j]);
        Xp[(long long)i * (i - 1) / 2 + j] = cmk(-acc.x, -acc.y);
      }
    }
  } else {
    for (int i = warp; i < n; i += nwarp) {
      const int first = A.row_first[sn.drow0 + i];
      cplx* dst = vals + A.row_off[sn.drow0 + i] - first;
      for (int q = first + lane; q < i; q += 32) dst[q] = F[(long long)i * Fn + q];
    }
  }
  // blocks (rows owned by ancestors)
  for (int b = sn.blk0; b < sn.blk0 + sn.nblk; ++b) {
    const DevBlk B = A.blk[b];
    for (int r = warp; r < B.nr; r += nwarp) {
      const int first = A.row_first[B.row0 + r];
      cplx* dst = vals + A.row_off[B.row0 + r] - first;
      const cplx* src = F + (long long)(B.front0 + r) * Fn;
      for (int j = first + lane; j < n; j += 32) dst[j] = src[j];
    }
  }
}

size_t factor_smem_limit() { return 200 * 1024; }

void launch_factor_level(const FactorArgs& A, const int* d_nodes, int nnodes, int ncls, int fmax,
                         cudaStream_t st) {
  // the two pivot-column buffers of the largest front (the host rejects fronts
  // beyond factor_smem_limit())
  dim3 g(nnodes, ncls);
  const size_t smem = 2 * sizeof(cplx) * size_t(std::max(fmax, 1));
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(k_factor_node, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr = smem;
  }
  k_factor_node<<<g, 512, smem, st>>>(A, d_nodes);
}

}  // namespace hddm
