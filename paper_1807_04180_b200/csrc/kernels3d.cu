// sm_100a kernels of the 3-D path (BASELINE config 5): the batched multifrontal
// LDL^T of every class (dense fronts: blocked partial factorization, FP64
// trailing updates), the dense supernodal forward / backward solves that apply
// it every DDM step, and the 3-D DDM step stages (26-direction source transfer,
// blend-accumulate, 7-point residuals, refinement). The math is the restatement
// oracle/hddm_oracle3.c (the reference has no 3-D code); every output has one
// writer and a fixed summation order, so results are deterministic.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "kernels3d.cuh"

namespace hddm3 {

using hddm::cadd;
using hddm::cdiv;
using hddm::cfma;
using hddm::cmk;
using hddm::cmul;
using hddm::cnorm2;
using hddm::cscale;
using hddm::csub;

namespace {

__device__ __forceinline__ cplx ldf(const cplx* p) { return __ldcs(p); }
__device__ __forceinline__ cplx warp_sum(cplx v) { return hddm::warp_sum(v); }

// column start of column j in a packed strictly-lower column-major n x n block
__host__ __device__ __forceinline__ long long colstart(int j, int n) {
  return (long long)j * (2LL * n - j - 1) / 2;
}

}  // namespace

// ================================================================ factorization
// Front of supernode s: (2n + r) x (n + r), column major, ld = 2n + r. Rows:
// own columns [0, n), the supernode's rows [n, n + r), identity rows E [n + r, 2n + r).

__global__ void __launch_bounds__(256) k3f_scatter(Fac3Args F, const int* lv) {
  const DSn3 S = F.sn[lv[blockIdx.x]];
  const int c = F.cls0 + blockIdx.y;
  cplx* fr = F.fronts + blockIdx.y * F.fw + S.front_off;
  const long long ld = 2LL * S.n + S.r;
  const cplx* av = F.aval + (long long)c * F.naent;
  for (int e = S.aent0 + threadIdx.x; e < S.aent1; e += blockDim.x)
    fr[(long long)F.aent_j[e] * ld + F.aent_i[e]] = av[e];
  for (int i = threadIdx.x; i < S.n; i += blockDim.x) fr[(long long)i * ld + S.n + S.r + i] = cmk(1, 0);
}

// extend-add of child `slot`'s contribution block: column b of the child's
// trailing r x r block into the parent front (CTA per column, rows a >= b)
__global__ void __launch_bounds__(256) k3f_extadd(Fac3Args F, const int* lv, int slot) {
  const DSn3 P = F.sn[lv[blockIdx.y]];
  const int ch = slot ? P.ch1 : P.ch0;
  if (ch < 0) return;
  const DSn3 C = F.sn[ch];
  const int b = blockIdx.x;
  if (b >= C.r) return;
  const cplx* cf = F.fronts + blockIdx.z * F.fw + C.front_off;
  cplx* pf = F.fronts + blockIdx.z * F.fw + P.front_off;
  const long long ldc = 2LL * C.n + C.r, ldp = 2LL * P.n + P.r;
  const int* ext = F.ext + C.ext_off;
  const int jb = ext[b];
  const cplx* src = cf + (long long)(C.n + b) * ldc + C.n;
  cplx* dst = pf + (long long)jb * ldp;
  for (int a = b + threadIdx.x; a < C.r; a += blockDim.x) {
    const long long i = ext[a];
    dst[i] = cadd(dst[i], src[a]);
  }
}

// LDL^T of the kNB x kNB diagonal block at (k0, k0) in shared memory
__global__ void __launch_bounds__(256) k3f_dfac(Fac3Args F, const int* lv, int k0) {
  __shared__ cplx Sb[kNB * kNB];
  const DSn3 S = F.sn[lv[blockIdx.x]];
  if (S.n <= k0) return;
  const int b = min(kNB, S.n - k0);
  cplx* fr = F.fronts + blockIdx.y * F.fw + S.front_off;
  const long long ld = 2LL * S.n + S.r;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    Sb[j * kNB + i] = i >= j ? fr[(long long)(k0 + j) * ld + k0 + i] : cmk(0, 0);
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    const cplx d = Sb[j * kNB + j];
    for (int i = j + 1 + threadIdx.x; i < b; i += blockDim.x) Sb[j * kNB + i] = cdiv(Sb[j * kNB + i], d);
    __syncthreads();
    // a_ik -= (l_ij d_j) l_kj for j < k <= i
    const int m = b - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e % m, k = j + 1 + e / m;
      if (k <= i) Sb[k * kNB + i] = csub(Sb[k * kNB + i], cmul(cmul(Sb[j * kNB + i], d), Sb[j * kNB + k]));
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    if (i >= j) fr[(long long)(k0 + j) * ld + k0 + i] = Sb[j * kNB + i];
  }
}

// panel rows below the diagonal block: l_i = a_i L_kk^-T D^-1 (thread per row):
// own rows [k0+b, n), the rows [n, n+r) and the identity rows E_e, e < k0 + b
__global__ void __launch_bounds__(256) k3f_trsm(Fac3Args F, const int* lv, int k0) {
  __shared__ cplx Ls[kNB * kNB];
  __shared__ cplx Ds[kNB];
  const DSn3 S = F.sn[lv[blockIdx.y]];
  if (S.n <= k0) return;
  const int b = min(kNB, S.n - k0);
  cplx* fr = F.fronts + blockIdx.z * F.fw + S.front_off;
  const long long ld = 2LL * S.n + S.r;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    Ls[j * kNB + i] = fr[(long long)(k0 + j) * ld + k0 + i];
  }
  __syncthreads();
  if (threadIdx.x < b) Ds[threadIdx.x] = Ls[threadIdx.x * kNB + threadIdx.x];
  __syncthreads();
  const int nown = S.n - k0 - b, ne = min(S.n, k0 + b);
  const int tot = nown + S.r + ne;
  const int ia = blockIdx.x * blockDim.x + threadIdx.x;
  if (ia >= tot) return;
  const long long row = ia < nown ? k0 + b + ia : (ia < nown + S.r ? S.n + (ia - nown) : S.n + S.r + (ia - nown - S.r));
  cplx w[kNB];
  cplx* base = fr + (long long)k0 * ld + row;
#pragma unroll
  for (int c = 0; c < kNB; ++c) w[c] = c < b ? base[(long long)c * ld] : cmk(0, 0);
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    if (c >= b) break;
    cplx v = w[c];
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      if (t >= c) break;
      v = csub(v, cmul(w[t], Ls[t * kNB + c]));
    }
    w[c] = v;
  }
#pragma unroll
  for (int c = 0; c < kNB; ++c)
    if (c < b) base[(long long)c * ld] = cdiv(w[c], Ds[c]);
}

// trailing update C_ij -= sum_c (l_ic d_c) l_jc over 64 x 64 tiles: the lower
// triangle of [k0+b, n+r)^2, then the identity rows E_e (e < k0 + b) against
// the own columns [k0+b, n). 256 threads, 4 x 4 complex outputs each.
constexpr int kTile = 64;
__global__ void __launch_bounds__(256) k3f_update(Fac3Args F, const int* lv, int k0) {
  extern __shared__ __align__(16) unsigned char smem3[];
  cplx (*As)[kTile] = reinterpret_cast<cplx (*)[kTile]>(smem3);
  cplx (*Bs)[kTile] = reinterpret_cast<cplx (*)[kTile]>(smem3 + sizeof(cplx) * kNB * kTile);
  const DSn3 S = F.sn[lv[blockIdx.y]];
  if (S.n <= k0) return;
  const int b = min(kNB, S.n - k0);
  const int t0 = k0 + b;
  const int M = S.n + S.r - t0;  // trailing size
  const int T = (M + kTile - 1) / kTile;
  const long long nmain = (long long)T * (T + 1) / 2;
  const int ne = min(S.n, t0);
  const int TE = (ne + kTile - 1) / kTile;
  const int TC = S.n > t0 ? (S.n - t0 + kTile - 1) / kTile : 0;
  const long long tid = blockIdx.x;
  long long rbase, cbase;  // front row / column of the tile's first output
  int rlim, clim;          // rows / columns valid in the tile
  if (tid < nmain) {
    int ti = int((sqrt(8.0 * double(tid) + 1.0) - 1.0) * 0.5);
    while ((long long)(ti + 1) * (ti + 2) / 2 <= tid) ++ti;
    while ((long long)ti * (ti + 1) / 2 > tid) --ti;
    const int tj = int(tid - (long long)ti * (ti + 1) / 2);
    rbase = t0 + ti * kTile;
    cbase = t0 + tj * kTile;
    rlim = min(kTile, S.n + S.r - int(rbase));
    clim = min(kTile, S.n + S.r - int(cbase));
  } else if (tid < nmain + (long long)TE * TC) {
    const long long u = tid - nmain;
    const int te = int(u / TC), tc = int(u % TC);
    rbase = S.n + S.r + te * kTile;
    cbase = t0 + tc * kTile;
    rlim = min(kTile, ne - te * kTile);
    clim = min(kTile, S.n - (t0 + tc * kTile));
  } else {
    return;
  }
  cplx* fr = F.fronts + blockIdx.z * F.fw + S.front_off;
  const long long ld = 2LL * S.n + S.r;
  // stage: As[c][i] = l(rbase+i, k0+c) * d_c, Bs[c][j] = l(cbase+j, k0+c)
  for (int e = threadIdx.x; e < kNB * kTile; e += blockDim.x) {
    const int i = e % kTile, c = e / kTile;
    cplx a = cmk(0, 0), bb = cmk(0, 0);
    if (c < b) {
      const cplx* col = fr + (long long)(k0 + c) * ld;
      const cplx d = col[k0 + c];
      if (i < rlim) a = cmul(col[rbase + i], d);
      if (i < clim) bb = col[cbase + i];
    }
    As[c][i] = a;
    Bs[c][i] = bb;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  cplx acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = cmk(0, 0);
#pragma unroll 4
  for (int c = 0; c < b; ++c) {
    cplx a[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = As[c][ty + 16 * u];
#pragma unroll
    for (int v = 0; v < 4; ++v) bv[v] = Bs[c][tx + 16 * v];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) cfma(acc[u][v], a[u], bv[v]);
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int j = tx + 16 * v;
    if (j >= clim) continue;
    cplx* col = fr + (cbase + j) * ld + rbase;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = ty + 16 * u;
      if (i < rlim) col[i] = csub(col[i], acc[u][v]);
    }
  }
}

// The same trailing update on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64):
// these fronts are genuinely dense contractions (north_star item 1). Complex
// products as four real MMAs: Cr += Wr Lr^T - Wi Li^T, Ci += Wr Li^T + Wi Lr^T.
// CTA tile 64 x 64, 8 warps of 32 x 16 (4 x 2 blocks of 8 x 8), K = the panel
// width in steps of 4; shared-memory rows padded to 66 so the fragment loads of a
// quarter warp hit distinct banks.
constexpr int kTileP = kTile + 2;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256) k3f_update_mma(Fac3Args F, const int* lv, int k0) {
  extern __shared__ __align__(16) unsigned char smem3[];
  cplx (*As)[kTileP] = reinterpret_cast<cplx (*)[kTileP]>(smem3);
  cplx (*Bs)[kTileP] = reinterpret_cast<cplx (*)[kTileP]>(smem3 + sizeof(cplx) * kNB * kTileP);
  const DSn3 S = F.sn[lv[blockIdx.y]];
  if (S.n <= k0) return;
  const int b = min(kNB, S.n - k0);
  const int t0 = k0 + b;
  const int M = S.n + S.r - t0;
  const int T = (M + kTile - 1) / kTile;
  const long long nmain = (long long)T * (T + 1) / 2;
  const int ne = min(S.n, t0);
  const int TE = (ne + kTile - 1) / kTile;
  const int TC = S.n > t0 ? (S.n - t0 + kTile - 1) / kTile : 0;
  const long long tid = blockIdx.x;
  long long rbase, cbase;
  int rlim, clim;
  if (tid < nmain) {
    int ti = int((sqrt(8.0 * double(tid) + 1.0) - 1.0) * 0.5);
    while ((long long)(ti + 1) * (ti + 2) / 2 <= tid) ++ti;
    while ((long long)ti * (ti + 1) / 2 > tid) --ti;
    const int tj = int(tid - (long long)ti * (ti + 1) / 2);
    rbase = t0 + ti * kTile;
    cbase = t0 + tj * kTile;
    rlim = min(kTile, S.n + S.r - int(rbase));
    clim = min(kTile, S.n + S.r - int(cbase));
  } else if (tid < nmain + (long long)TE * TC) {
    const long long u = tid - nmain;
    const int te = int(u / TC), tc = int(u % TC);
    rbase = S.n + S.r + te * kTile;
    cbase = t0 + tc * kTile;
    rlim = min(kTile, ne - te * kTile);
    clim = min(kTile, S.n - (t0 + tc * kTile));
  } else {
    return;
  }
  cplx* fr = F.fronts + blockIdx.z * F.fw + S.front_off;
  const long long ld = 2LL * S.n + S.r;
  for (int e = threadIdx.x; e < kNB * kTile; e += blockDim.x) {
    const int i = e % kTile, c = e / kTile;
    cplx a = cmk(0, 0), bb = cmk(0, 0);
    if (c < b) {
      const cplx* col = fr + (long long)(k0 + c) * ld;
      const cplx d = col[k0 + c];
      if (i < rlim) a = cmul(col[rbase + i], d);
      if (i < clim) bb = col[cbase + i];
    }
    As[c][i] = a;
    Bs[c][i] = bb;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = (w >> 2) * 32, c0 = (w & 3) * 16;
  const int g = lane >> 2, q = lane & 3;
  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) cr[u][v][0] = cr[u][v][1] = ci[u][v][0] = ci[u][v][1] = 0.0;
  const int ksteps = (b + 3) / 4;
  for (int kk = 0; kk < ksteps; ++kk) {
    const int c = kk * 4 + q;
    cplx a[4], l[2];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = As[c][r0 + u * 8 + g];
#pragma unroll
    for (int v = 0; v < 2; ++v) l[v] = Bs[c][c0 + v * 8 + g];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        dmma(cr[u][v][0], cr[u][v][1], a[u].x, l[v].x);
        dmma(cr[u][v][0], cr[u][v][1], -a[u].y, l[v].y);
        dmma(ci[u][v][0], ci[u][v][1], a[u].x, l[v].y);
        dmma(ci[u][v][0], ci[u][v][1], a[u].y, l[v].x);
      }
  }
#pragma unroll
  for (int v = 0; v < 2; ++v)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = c0 + v * 8 + q * 2 + h;
      if (j >= clim) continue;
      cplx* col = fr + (cbase + j) * ld + rbase;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = r0 + u * 8 + g;
        if (i < rlim) col[i] = csub(col[i], cmk(cr[u][v][h], ci[u][v][h]));
      }
    }
}

// factor values of the finished fronts: D, the packed inverse of the unit-lower
// diagonal block (Linv_ij = L_E(j, i) d_i), the panel (column major)
__global__ void __launch_bounds__(256) k3f_extract(Fac3Args F, const int* lv) {
  const DSn3 S = F.sn[lv[blockIdx.y]];
  const int c = F.cls0 + blockIdx.z;
  const cplx* fr = F.fronts + blockIdx.z * F.fw + S.front_off;
  const long long ld = 2LL * S.n + S.r;
  cplx* v = F.vals + (long long)c * F.nvals;
  cplx* vt = F.valsT + (long long)c * F.nvals;
  const long long nd = (long long)S.n * S.n, tot = nd + (long long)S.r * S.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nd) {
      const int i = int(e % S.n), j = int(e / S.n);
      if (i == j) {
        v[S.c0 + j] = fr[(long long)j * ld + j];
        vt[S.c0 + j] = v[S.c0 + j];
      } else if (i > j) {
        const cplx di = fr[(long long)i * ld + i];
        const cplx x = cmul(fr[(long long)i * ld + S.n + S.r + j], di);
        v[S.linv_off + colstart(j, S.n) + (i - j - 1)] = x;
        vt[S.linv_off + (long long)i * (i - 1) / 2 + j] = x;
      }
    } else {
      const long long q = e - nd;
      const int k = int(q % S.r), j = int(q / S.r);
      const cplx x = fr[(long long)j * ld + S.n + k];
      v[S.pan_off + (long long)j * S.r + k] = x;
      vt[S.pan_off + (long long)k * S.n + j] = x;
    }
  }
}

void f3_scatter(const Fac3Args& F, const int* lv, int nlv, int nb, cudaStream_t st) {
  if (nlv) k3f_scatter<<<dim3(nlv, nb), 256, 0, st>>>(F, lv);
}
void f3_extadd(const Fac3Args& F, const int* lv, int nlv, int nb, int slot, int maxr, cudaStream_t st) {
  if (nlv && maxr) k3f_extadd<<<dim3(maxr, nlv, nb), 256, 0, st>>>(F, lv, slot);
}
void f3_dfac(const Fac3Args& F, const int* lv, int nlv, int nb, int k0, cudaStream_t st) {
  if (nlv) k3f_dfac<<<dim3(nlv, nb), 256, 0, st>>>(F, lv, k0);
}
void f3_trsm(const Fac3Args& F, const int* lv, int nlv, int nb, int k0, int maxrows, cudaStream_t st) {
  if (nlv && maxrows > 0) k3f_trsm<<<dim3((maxrows + 255) / 256, nlv, nb), 256, 0, st>>>(F, lv, k0);
}
void f3_update(const Fac3Args& F, const int* lv, int nlv, int nb, int k0, long long maxtiles,
               cudaStream_t st) {
  // DMMA by default; HDDM3_FACTOR_FMA=1 selects the CUDA-core kernel (same math)
  static const bool fma = std::getenv("HDDM3_FACTOR_FMA") != nullptr;
  constexpr size_t smem = 2 * sizeof(cplx) * kNB * kTile;
  constexpr size_t smemp = 2 * sizeof(cplx) * kNB * kTileP;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3f_update, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k3f_update_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemp));
    attr = true;
  }
  if (!(nlv && maxtiles > 0)) return;
  if (fma)
    k3f_update<<<dim3(unsigned(maxtiles), nlv, nb), 256, smem, st>>>(F, lv, k0);
  else
    k3f_update_mma<<<dim3(unsigned(maxtiles), nlv, nb), 256, smemp, st>>>(F, lv, k0);
}
void f3_extract(const Fac3Args& F, const int* lv, int nlv, int nb, long long maxent, cudaStream_t st) {
  if (!nlv) return;
  const unsigned gx = unsigned(std::min<long long>(std::max<long long>(1, (maxent + 255) / 256), 4096));
  k3f_extract<<<dim3(gx, nlv, nb), 256, 0, st>>>(F, lv);
}

// ================================================================ solves
// Grid: (task, class, member group). The members of class c in group g are
// cls_mem[cls_ptr[c] + g*MG + k], k < MG; a member takes part iff its flag says so.
namespace {
template <int MG>
struct Mem {
  int t[MG];
  int cnt;
};
template <int MG>
__device__ __forceinline__ Mem<MG> members(const Solve3Args& A) {
  Mem<MG> m;
  const int c = blockIdx.y, g = blockIdx.z;
  const int p0 = A.cls_ptr[c], p1 = A.cls_ptr[c + 1];
  m.cnt = 0;
#pragma unroll
  for (int k = 0; k < MG; ++k) {
    const int q = p0 + g * MG + k;
    m.t[k] = -1;
    if (q < p1) {
      const int t = A.cls_mem[q];
      if ((A.flag[t] != 0) == (A.flag_on != 0)) m.t[m.cnt++] = t;
    }
  }
  return m;
}
}  // namespace

// Programmatic dependent launch (on by default; HDDM3_PDL=0 off): a solve kernel lets
// its successor launch at once and waits for its predecessor before touching a vector.
__device__ __forceinline__ void pdl_trigger3() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait3() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// shell (identity rows): x = b
// Leaves (no children, at most 32 nodes) fused, a warp per leaf, lane = node:
//   forward:  x = Linv b (y_j broadcast by shuffles), then the panel rows
//             u_k = -sum_j L_kj x_j (lane = row, x_j by shuffles): no assembly pass and
//             no round trip between the two products;
//   backward: w_j = z_j / d_j - sum_k L_kj x_rows(k) (the ancestors' x gathered
//             directly), then x = Linv^T w (w_i by shuffles).
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_fleaf(Solve3Args A, const Task3* tk) {
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Task3 T = tk[blockIdx.x * 8 + w];
  if (T.b <= T.a) return;
  const int n = T.n, r = T.r, i = lane;
  const cplx* vals = A.vals + (long long)blockIdx.y * A.nvals;
  const cplx* L = vals + T.linv;
  cplx x[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) x[q] = (q < m.cnt && i < n) ? A.B[(long long)m.t[q] * A.nw + T.c0 + i] : cmk(0, 0);
  cplx acc[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) acc[q] = x[q];
  for (int j = 0; j + 1 < n; ++j) {
    const cplx l = (i < n && j < i) ? ldf(L + colstart(j, n) + (i - j - 1)) : cmk(0, 0);
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      if (q >= m.cnt) break;
      const cplx yj = cmk(__shfl_sync(0xffffffffu, x[q].x, j), __shfl_sync(0xffffffffu, x[q].y, j));
      cfma(acc[q], l, yj);
    }
  }
#pragma unroll
  for (int q = 0; q < MG; ++q) {
    if (q >= m.cnt) break;
    x[q] = acc[q];
    if (i < n) A.X[(long long)m.t[q] * A.nw + T.c0 + i] = x[q];
  }
  const cplx* P = vals + T.pan;
  for (int k0 = 0; k0 < r; k0 += 32) {
    const int k = k0 + lane;
    cplx u[MG];
#pragma unroll
    for (int q = 0; q < MG; ++q) u[q] = cmk(0, 0);
    for (int j = 0; j < n; ++j) {
      const cplx l = k < r ? ldf(P + (long long)j * r + k) : cmk(0, 0);
#pragma unroll
      for (int q = 0; q < MG; ++q) {
        if (q >= m.cnt) break;
        const cplx xj = cmk(__shfl_sync(0xffffffffu, x[q].x, j), __shfl_sync(0xffffffffu, x[q].y, j));
        cfma(u[q], l, xj);
      }
    }
    if (k < r)
#pragma unroll
      for (int q = 0; q < MG; ++q) {
        if (q >= m.cnt) break;
        A.U[(long long)m.t[q] * A.nupd + T.upd + k] = cmk(-u[q].x, -u[q].y);
      }
  }
}

template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_bleaf(Solve3Args A, const Task3* tk) {
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Task3 T = tk[blockIdx.x * 8 + w];
  if (T.b <= T.a) return;
  const int n = T.n, r = T.r, j = lane;
  const bool col = j < n;
  const cplx* valsT = A.valsT + (long long)blockIdx.y * A.nvals;
  const cplx* PT = valsT + T.pan;
  const int* rows = A.rows_all + T.rows;
  cplx acc[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) acc[q] = cmk(0, 0);
  for (int k = 0; k < r; ++k) {
    const cplx l = col ? ldf(PT + (long long)k * n + j) : cmk(0, 0);
    const int pr = rows[k];
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      if (q >= m.cnt) break;
      cfma(acc[q], l, A.X[(long long)m.t[q] * A.nw + pr]);
    }
  }
  const cplx d = A.vals[(long long)blockIdx.y * A.nvals + T.c0 + (col ? j : 0)];
  cplx wv[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) {
    wv[q] = cmk(0, 0);
    if (q < m.cnt && col) wv[q] = csub(cdiv(A.X[(long long)m.t[q] * A.nw + T.c0 + j], d), acc[q]);
    acc[q] = wv[q];
  }
  const cplx* LT = valsT + T.linv;
  for (int i = 1; i < n; ++i) {
    const cplx l = (col && i > j) ? ldf(LT + (long long)i * (i - 1) / 2 + j) : cmk(0, 0);
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      if (q >= m.cnt) break;
      const cplx wi = cmk(__shfl_sync(0xffffffffu, wv[q].x, i), __shfl_sync(0xffffffffu, wv[q].y, i));
      cfma(acc[q], l, wi);
    }
  }
  if (!col) return;
#pragma unroll
  for (int q = 0; q < MG; ++q) {
    if (q >= m.cnt) break;
    A.X[(long long)m.t[q] * A.nw + T.c0 + j] = acc[q];
  }
}

template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_ring(Solve3Args A) {
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  for (int k = 0; k < m.cnt; ++k) {
    const long long o = (long long)m.t[k] * A.nw;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.nshell; i += gridDim.x * blockDim.x)
      A.X[o + i] = A.B[o + i];
  }
}

// forward assembly of the own entries: Y = b + the children's update vectors
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_fasm(Solve3Args A, const Task3* tk) {
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const Task3 T = tk[blockIdx.x];
  const int i = T.a + threadIdx.x;
  if (i >= T.b) return;
  const int m0 = A.cmap0[T.cmap + i], m1 = A.cmap1[T.cmap + i];
  for (int k = 0; k < m.cnt; ++k) {
    const long long o = (long long)m.t[k] * A.nw + T.c0 + i;
    const cplx* u = A.U + (long long)m.t[k] * A.nupd;
    cplx y = A.B[o];
    if (m0 >= 0) y = cadd(y, u[m0]);
    if (m1 >= 0) y = cadd(y, u[m1]);
    A.Y[o] = y;
  }
}

namespace {
// sum over columns j = j0, j0+1, j0+2, j0+3, j0 + jstep, ... < jend of L(row, j) v_q[j]
// for the rows of one lane; get(j) returns the lane's factor entry (0 when the lane
// has none)
template <int MG, class G>
__device__ __forceinline__ void col_sweep(const Mem<MG>& m, const cplx* const* v, int jfirst, int jstep, int jend,
                                          G get, cplx* acc) {
  for (int j0 = jfirst; j0 < jend; j0 += jstep) {
    cplx l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) l[u] = j0 + u < jend ? get(j0 + u) : cmk(0, 0);
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      if (q >= m.cnt) break;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < jend) cfma(acc[q], l[u], v[q][j0 + u]);
    }
  }
}
}  // namespace

// forward inverse rows: x_i = y_i + sum_{j<i} Linv_ij y_j (lane = row). CTA tasks:
// 32 rows, the 8 warps take interleaved 4-column groups, partials combined in warp
// order; warp tasks: one warp sweeps all columns of its rows.
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_fdiag(Solve3Args A, const Task3* tk, int nbig) {
  __shared__ cplx part[8][MG][32];
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool big = int(blockIdx.x) < nbig;
  const Task3 T = tk[big ? blockIdx.x : nbig + (blockIdx.x - nbig) * 8 + w];
  if (!big && T.b <= T.a) return;  // padding warp task
  const int i = T.a + lane;
  const bool row = i < T.b;
  const cplx* L = A.vals + (long long)blockIdx.y * A.nvals + T.linv;
  const cplx* y[MG];
#pragma unroll
  for (int k = 0; k < MG; ++k) y[k] = A.Y + (long long)(k < m.cnt ? m.t[k] : m.t[0]) * A.nw + T.c0;
  cplx acc[MG];
#pragma unroll
  for (int k = 0; k < MG; ++k) acc[k] = cmk(0, 0);
  const int n = T.n;
  auto get = [&](int j) { return (row && j < i) ? ldf(L + colstart(j, n) + (i - j - 1)) : cmk(0, 0); };
  col_sweep(m, y, big ? 4 * w : 0, big ? 32 : 4, T.b - 1, get, acc);
  if (big) {
#pragma unroll
    for (int k = 0; k < MG; ++k) part[w][k][lane] = acc[k];
    __syncthreads();
    if (w != 0) return;
#pragma unroll
    for (int k = 0; k < MG; ++k) {
      cplx s = part[0][k][lane];
      for (int q = 1; q < 8; ++q) s = cadd(s, part[q][k][lane]);
      acc[k] = s;
    }
  }
  if (!row) return;
#pragma unroll
  for (int k = 0; k < MG; ++k) {
    if (k >= m.cnt) break;
    const long long o = (long long)m.t[k] * A.nw + T.c0 + i;
    A.X[o] = cadd(A.Y[o], acc[k]);
  }
}

// forward panel rows: u_k = (children's updates of row k) - sum_j L_kj x_j (lane = row)
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_fpanel(Solve3Args A, const Task3* tk, int nbig) {
  __shared__ cplx part[8][MG][32];
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool big = int(blockIdx.x) < nbig;
  const Task3 T = tk[big ? blockIdx.x : nbig + (blockIdx.x - nbig) * 8 + w];
  if (!big && T.b <= T.a) return;
  const int k = T.a + lane;
  const bool row = k < T.b;
  const cplx* L = A.vals + (long long)blockIdx.y * A.nvals + T.pan;
  const cplx* x[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) x[q] = A.X + (long long)(q < m.cnt ? m.t[q] : m.t[0]) * A.nw + T.c0;
  cplx acc[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) acc[q] = cmk(0, 0);
  const int r = T.r;
  auto get = [&](int j) { return row ? ldf(L + (long long)j * r + k) : cmk(0, 0); };
  col_sweep(m, x, big ? 4 * w : 0, big ? 32 : 4, T.n, get, acc);
  if (big) {
#pragma unroll
    for (int q = 0; q < MG; ++q) part[w][q][lane] = acc[q];
    __syncthreads();
    if (w != 0) return;
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      cplx s = part[0][q][lane];
      for (int v = 1; v < 8; ++v) s = cadd(s, part[v][q][lane]);
      acc[q] = s;
    }
  }
  if (!row) return;
  const int m0 = A.cmap0[T.cmap + T.n + k], m1 = A.cmap1[T.cmap + T.n + k];
#pragma unroll
  for (int q = 0; q < MG; ++q) {
    if (q >= m.cnt) break;
    cplx* u = A.U + (long long)m.t[q] * A.nupd;
    cplx c = cmk(0, 0);
    if (m0 >= 0) c = cadd(c, u[m0]);
    if (m1 >= 0) c = cadd(c, u[m1]);
    u[T.upd + k] = csub(c, acc[q]);
  }
}

// backward gather of the ancestors' solution at the supernode's rows into U
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_bgather(Solve3Args A, const Task3* tk) {
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const Task3 T = tk[blockIdx.x];
  const int k = T.a + threadIdx.x;
  if (k >= T.b) return;
  const int P = A.rows_all[T.rows + k];
  for (int q = 0; q < m.cnt; ++q)
    A.U[(long long)m.t[q] * A.nupd + T.upd + k] = A.X[(long long)m.t[q] * A.nw + P];
}

// backward panel columns: w_j = z_j / d_j - sum_k L_kj x_rows(k), lane = column on
// the row-major copy (coalesced across columns); CTA tasks: 8 warps split the rows
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_bpanel(Solve3Args A, const Task3* tk, int nbig) {
  __shared__ cplx part[8][MG][32];
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool big = int(blockIdx.x) < nbig;
  const Task3 T = tk[big ? blockIdx.x : nbig + (blockIdx.x - nbig) * 8 + w];
  if (!big && T.b <= T.a) return;
  const int j = T.a + lane;
  const bool col = j < T.b;
  const cplx* LT = A.valsT + (long long)blockIdx.y * A.nvals + T.pan;
  const cplx* u[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) u[q] = A.U + (long long)(q < m.cnt ? m.t[q] : m.t[0]) * A.nupd + T.upd;
  cplx acc[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) acc[q] = cmk(0, 0);
  const int n = T.n;
  auto get = [&](int k) { return col ? ldf(LT + (long long)k * n + j) : cmk(0, 0); };
  col_sweep(m, u, big ? 4 * w : 0, big ? 32 : 4, T.r, get, acc);
  if (big) {
#pragma unroll
    for (int q = 0; q < MG; ++q) part[w][q][lane] = acc[q];
    __syncthreads();
    if (w != 0) return;
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      cplx s = part[0][q][lane];
      for (int v = 1; v < 8; ++v) s = cadd(s, part[v][q][lane]);
      acc[q] = s;
    }
  }
  if (!col) return;
  const cplx d = A.vals[(long long)blockIdx.y * A.nvals + T.c0 + j];
#pragma unroll
  for (int q = 0; q < MG; ++q) {
    if (q >= m.cnt) break;
    const long long o = (long long)m.t[q] * A.nw + T.c0 + j;
    A.Y[o] = csub(cdiv(A.X[o], d), acc[q]);
  }
}

// backward inverse columns: x_j = w_j + sum_{i>j} Linv_ij w_i, lane = column on the
// row-major packed copy; CTA tasks: 8 warps split the rows
template <int MG>
__global__ void __launch_bounds__(256, MG == 1 ? 4 : 3) k3s_bdiag(Solve3Args A, const Task3* tk, int nbig) {
  __shared__ cplx part[8][MG][32];
  pdl_trigger3();
  const Mem<MG> m = members<MG>(A);
  pdl_wait3();
  if (!m.cnt) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool big = int(blockIdx.x) < nbig;
  const Task3 T = tk[big ? blockIdx.x : nbig + (blockIdx.x - nbig) * 8 + w];
  if (!big && T.b <= T.a) return;
  const int j = T.a + lane;
  const bool col = j < T.b;
  const cplx* LT = A.valsT + (long long)blockIdx.y * A.nvals + T.linv;
  const cplx* y[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) y[q] = A.Y + (long long)(q < m.cnt ? m.t[q] : m.t[0]) * A.nw + T.c0;
  cplx acc[MG];
#pragma unroll
  for (int q = 0; q < MG; ++q) acc[q] = cmk(0, 0);
  auto get = [&](int i) { return (col && i > j) ? ldf(LT + (long long)i * (i - 1) / 2 + j) : cmk(0, 0); };
  col_sweep(m, y, T.a + 1 + (big ? 4 * w : 0), big ? 32 : 4, T.n, get, acc);
  if (big) {
#pragma unroll
    for (int q = 0; q < MG; ++q) part[w][q][lane] = acc[q];
    __syncthreads();
    if (w != 0) return;
#pragma unroll
    for (int q = 0; q < MG; ++q) {
      cplx s = part[0][q][lane];
      for (int v = 1; v < 8; ++v) s = cadd(s, part[v][q][lane]);
      acc[q] = s;
    }
  }
  if (!col) return;
#pragma unroll
  for (int q = 0; q < MG; ++q) {
    if (q >= m.cnt) break;
    A.X[(long long)m.t[q] * A.nw + T.c0 + j] = cadd(y[q][j], acc[q]);
  }
}

// measured 4.552 -> 4.517 ms per config-5 solve; HDDM3_PDL=0 switches it off
static bool g_pdl3 = !(std::getenv("HDDM3_PDL") && std::getenv("HDDM3_PDL")[0] == '0');
template <typename... KArgs, typename... Args>
static void launch3(void (*k)(KArgs...), dim3 grid, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl3 ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}
template <int MG>
static void s3t_ring(const Solve3Args& A, int ncls, int ng, cudaStream_t st) {
  launch3(k3s_ring<MG>, dim3(std::max(1, std::min(64, (A.nshell + 255) / 256)), ncls, ng), st, A);
}
template <int MG>
static void s3t_fasm(const Solve3Args& A, const Task3* t, int nt, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_fasm<MG>, dim3(nt, ncls, ng), st, A, t);
}
template <int MG>
static void s3t_fdiag(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_fdiag<MG>, dim3(nbig + (nt - nbig + 7) / 8, ncls, ng), st, A, t, nbig);
}
template <int MG>
static void s3t_fpanel(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_fpanel<MG>, dim3(nbig + (nt - nbig + 7) / 8, ncls, ng), st, A, t, nbig);
}
template <int MG>
static void s3t_fleaf(const Solve3Args& A, const Task3* t, int nt, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_fleaf<MG>, dim3(nt / 8, ncls, ng), st, A, t);
}
template <int MG>
static void s3t_bleaf(const Solve3Args& A, const Task3* t, int nt, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_bleaf<MG>, dim3(nt / 8, ncls, ng), st, A, t);
}
template <int MG>
static void s3t_bgather(const Solve3Args& A, const Task3* t, int nt, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_bgather<MG>, dim3(nt, ncls, ng), st, A, t);
}
template <int MG>
static void s3t_bpanel(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_bpanel<MG>, dim3(nbig + (nt - nbig + 7) / 8, ncls, ng), st, A, t, nbig);
}
template <int MG>
static void s3t_bdiag(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ng, cudaStream_t st) {
  if (nt) launch3(k3s_bdiag<MG>, dim3(nbig + (nt - nbig + 7) / 8, ncls, ng), st, A, t, nbig);
}


// member groups of 4 right-hand sides, or 1 when every class has one member (config 5:
// fewer registers, 4 CTAs per SM)
void s3_ring(const Solve3Args& A, int ncls, int ng, cudaStream_t st) {
  if (A.mg == 1) s3t_ring<1>(A, ncls, ng, st); else s3t_ring<kMG>(A, ncls, ng, st);
}
#define S3_DISPATCH(name)                                                                       \
  void s3_##name(const Solve3Args& A, const Task3* t, int nt, int ncls, int ng, cudaStream_t st) { \
    if (A.mg == 1) s3t_##name<1>(A, t, nt, ncls, ng, st); else s3t_##name<kMG>(A, t, nt, ncls, ng, st); \
  }
#define S3_DISPATCH_B(name)                                                                     \
  void s3_##name(const Solve3Args& A, const Task3* t, int nt, int nbig, int ncls, int ng,         \
                 cudaStream_t st) {                                                             \
    if (A.mg == 1) s3t_##name<1>(A, t, nt, nbig, ncls, ng, st);                                 \
    else s3t_##name<kMG>(A, t, nt, nbig, ncls, ng, st);                                         \
  }
S3_DISPATCH(fasm)
S3_DISPATCH(fleaf)
S3_DISPATCH(bleaf)
S3_DISPATCH(bgather)
S3_DISPATCH_B(fdiag)
S3_DISPATCH_B(fpanel)
S3_DISPATCH_B(bpanel)
S3_DISPATCH_B(bdiag)

// ================================================================ DDM step
// source offsets in gather order (hddm_oracle3.c kO3): 6 faces, 12 edges, 8 vertices
__constant__ signed char kO3[26][3] = {
    {+1, 0, 0}, {-1, 0, 0}, {0, +1, 0}, {0, -1, 0}, {0, 0, +1}, {0, 0, -1},
    {+1, +1, 0}, {-1, +1, 0}, {+1, -1, 0}, {-1, -1, 0},
    {+1, 0, +1}, {-1, 0, +1}, {+1, 0, -1}, {-1, 0, -1},
    {0, +1, +1}, {0, -1, +1}, {0, +1, -1}, {0, -1, -1},
    {+1, +1, +1}, {-1, +1, +1}, {+1, -1, +1}, {-1, -1, +1},
    {+1, +1, -1}, {-1, +1, -1}, {+1, -1, -1}, {-1, -1, -1}};

namespace {
__device__ __forceinline__ int sub_index(const Step3Args& A, int i, int j, int k) {
  return (k * A.n[1] + j) * A.n[0] + i;
}
__device__ __forceinline__ bool shell3(const int* nn, int p, int q, int r) {
  return p == 0 || q == 0 || r == 0 || p == nn[0] - 1 || q == nn[1] - 1 || r == nn[2] - 1;
}
}  // namespace

// any nonzero source value in subdomain t's owned box (restrict_owned, ddm.cpp:159-172)
__global__ void __launch_bounds__(256) k3d_fany(Step3Args A) {
  __shared__ int any;
  const int t = blockIdx.x;
  const Sub3Dev s = A.sub[t];
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  const int ex = s.own1[0] - s.own0[0] + 1, ey = s.own1[1] - s.own0[1] + 1, ez = s.own1[2] - s.own0[2] + 1;
  const long long tot = (long long)ex * ey * ez;
  int loc = 0;
  for (long long e = threadIdx.x; e < tot && !loc; e += blockDim.x) {
    const int p = s.own0[0] + int(e % ex), q = s.own0[1] + int((e / ex) % ey), r = s.own0[2] + int(e / ((long long)ex * ey));
    const cplx v = A.f[((long long)r * A.gn[1] + q) * A.gn[0] + p];
    loc = v.x != 0.0 || v.y != 0.0;
  }
  if (loc) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) A.fany[t] = any;
}

// zero flags of this step and the solve / skip counts (sweep, ddm.cpp:187-207)
__global__ void k3d_flags(Step3Args A) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < A.nsub; t += gridDim.x * blockDim.x) {
    const Sub3Dev s = A.sub[t];
    bool any = A.step == 1 && A.fany[t];
    for (int d = 0; d < 26 && !any; ++d) {
      int si[3];
      bool ok = true;
      for (int a = 0; a < 3; ++a) {
        si[a] = s.ix[a] + kO3[d][a];
        ok = ok && si[a] >= 0 && si[a] < A.n[a];
      }
      if (!ok) continue;
      const int lag = (kO3[d][0] != 0) + (kO3[d][1] != 0) + (kO3[d][2] != 0);
      if (!A.zp[lag - 1][sub_index(A, si[0], si[1], si[2])]) any = true;
    }
    A.zc[t] = any ? 0 : 1;
    atomicAdd((unsigned long long*)&A.counts[any ? 0 : 1], 1ull);
  }
}

namespace {
// class coefficient pointers
struct CoefP {
  const cplx* an[3];
  const cplx* iah[3];
};
__device__ __forceinline__ CoefP coefs(const cplx* cop, int stride, int cls, const int* nn) {
  CoefP c;
  const cplx* b = cop + (long long)cls * stride;
  c.an[0] = b;
  c.an[1] = b + nn[0];
  c.an[2] = b + nn[0] + nn[1];
  c.iah[0] = b + nn[0] + nn[1] + nn[2];
  c.iah[1] = c.iah[0] + nn[0];
  c.iah[2] = c.iah[1] + nn[1];
  return c;
}
__device__ __forceinline__ cplx jac3(const CoefP& K, int p, int q, int r) {
  return cmul(cmul(K.an[0][p], K.an[1][q]), K.an[2][r]);
}
}  // namespace

// right-hand sides (sweep, ddm.cpp:174-205 in 3-D), two passes: (1) every window
// node of an active subdomain: b = J f on the owned box at step 1, else 0 (shell 0);
// (2) the nodes of the union of the 26 transfer patches (structural tables built on the
// host): b = J (f_owned - sum_d L_t(beta_d v_src)) over the directions in gather order
// whose source exists and is not zero-flagged, the source values and tapers of the 7
// stencil points read from the tables. Thread per (node, t).
__global__ void __launch_bounds__(256) k3d_rhs_base(Step3Args A) {
  const int t = blockIdx.y;
  if (A.zc[t]) return;
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= A.nw) return;
  const int v = A.perm[pos];
  const int nx = A.nn[0], ny = A.nn[1];
  const int p = v % nx, q = (v / nx) % ny, r = v / (nx * ny);
  cplx b = cmk(0, 0);
  if (A.step == 1 && !shell3(A.nn, p, q, r)) {
    const Sub3Dev s = A.sub[t];
    const int P[3] = {s.w0[0] + p, s.w0[1] + q, s.w0[2] + r};
    bool own = true;
    for (int a = 0; a < 3; ++a) own = own && P[a] >= s.own0[a] && P[a] <= s.own1[a];
    if (own) {
      const CoefP K = coefs(A.cop, A.cop_stride, s.cls, A.nn);
      b = cmul(jac3(K, p, q, r), A.f[((long long)P[2] * A.gn[1] + P[1]) * A.gn[0] + P[0]]);
    }
  }
  A.B[(long long)t * A.nw + pos] = b;
}

__global__ void __launch_bounds__(128) k3d_rhs_xfer(Step3Args A) {
  const int t = blockIdx.y;
  if (A.zc[t]) return;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= A.npatch) return;
  const int v = A.pnode[u];
  const int nx = A.nn[0], ny = A.nn[1];
  const int p = v % nx, q = (v / nx) % ny, r = v / (nx * ny);
  const Sub3Dev s = A.sub[t];
  cplx acc = cmk(0, 0);
  if (A.step == 1) {
    const int P[3] = {s.w0[0] + p, s.w0[1] + q, s.w0[2] + r};
    bool own = true;
    for (int a = 0; a < 3; ++a) own = own && P[a] >= s.own0[a] && P[a] <= s.own1[a];
    if (own) acc = A.f[((long long)P[2] * A.gn[1] + P[1]) * A.gn[0] + P[0]];
  }
  const CoefP K = coefs(A.cop, A.cop_stride, s.cls, A.nn);
  const cplx ex = cscale(cmul(K.an[1][q], K.an[2][r]), A.ih2);
  const cplx ey = cscale(cmul(K.an[0][p], K.an[2][r]), A.ih2);
  const cplx ez = cscale(cmul(K.an[0][p], K.an[1][q]), A.ih2);
  const cplx jac = jac3(K, p, q, r);
  for (int e = A.pent[u]; e < A.pent[u + 1]; ++e) {
    const int d = A.edir[e];
    int si[3];
    bool ok = true;
    for (int a = 0; a < 3; ++a) {
      si[a] = s.ix[a] + kO3[d][a];
      ok = ok && si[a] >= 0 && si[a] < A.n[a];
    }
    if (!ok) continue;
    const int lag = (kO3[d][0] != 0) + (kO3[d][1] != 0) + (kO3[d][2] != 0);
    const int src = sub_index(A, si[0], si[1], si[2]);
    if (A.zp[lag - 1][src]) continue;
    const cplx* vs = A.Up[lag - 1] + (long long)src * A.nw;
    const int* sp = A.esrc + 7LL * e;
    const double* bt = A.ebeta + 7LL * e;
    cplx w[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const int ps = sp[k];
      const cplx x = ps >= 0 ? vs[ps] : cmk(0, 0);
      w[k] = (x.x != 0.0 || x.y != 0.0) ? cscale(x, bt[k]) : cmk(0, 0);
    }
    // L-form 7-point stencil with the target's coefficients (hddm_oracle3.c stencil3)
    const cplx uc = w[0];
    cplx tt = cmul(cmul(ex, K.iah[0][p]), csub(w[1], uc));
    tt = csub(tt, cmul(cmul(ex, K.iah[0][p - 1]), csub(uc, w[2])));
    tt = cadd(tt, cmul(cmul(ey, K.iah[1][q]), csub(w[3], uc)));
    tt = csub(tt, cmul(cmul(ey, K.iah[1][q - 1]), csub(uc, w[4])));
    tt = cadd(tt, cmul(cmul(ez, K.iah[2][r]), csub(w[5], uc)));
    tt = csub(tt, cmul(cmul(ez, K.iah[2][r - 1]), csub(uc, w[6])));
    acc = csub(acc, cadd(cdiv(tt, jac), cscale(uc, A.k2)));
  }
  A.B[(long long)t * A.nw + A.pinv[v]] = cmul(jac, acc);
}

// blend-accumulate (accumulate_weighted in 3-D): thread per global node, the
// covering active subdomains in ascending t
__global__ void __launch_bounds__(256) k3d_accumulate(Step3Args A, const double* wts) {
  const long long n = (long long)A.gn[0] * A.gn[1] * A.gn[2];
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int P[3] = {int(g % A.gn[0]), int((g / A.gn[0]) % A.gn[1]), int(g / ((long long)A.gn[0] * A.gn[1]))};
    int cv[3][2];
    for (int a = 0; a < 3; ++a) {
      const int* c = A.cov + 2LL * (a == 0 ? 0 : (a == 1 ? A.gn[0] : A.gn[0] + A.gn[1]));
      cv[a][0] = c[2 * P[a]];
      cv[a][1] = c[2 * P[a] + 1];
    }
    cplx acc = A.asmb[g];
    bool touched = false;
    for (int kk = 0; kk < 2; ++kk) {
      const int k = cv[2][kk];
      if (k < 0) continue;
      for (int jj = 0; jj < 2; ++jj) {
        const int j = cv[1][jj];
        if (j < 0) continue;
        for (int ii = 0; ii < 2; ++ii) {
          const int i = cv[0][ii];
          if (i < 0) continue;
          const int t = sub_index(A, i, j, k);
          if (A.zc[t]) continue;
          const Sub3Dev s = A.sub[t];
          const int l[3] = {P[0] - s.w0[0], P[1] - s.w0[1], P[2] - s.w0[2]};
          const double* wt = wts + (long long)t * (A.nn[0] + A.nn[1] + A.nn[2]);
          const double wz = wt[A.nn[0] + A.nn[1] + l[2]];
          if (wz == 0) continue;
          const double wy = wt[A.nn[0] + l[1]];
          if (wy == 0) continue;
          const double w = wt[l[0]] * wy * wz;
          if (w == 0) continue;
          const cplx u = A.Ucur[(long long)t * A.nw + A.pinv[(l[2] * A.nn[1] + l[1]) * A.nn[0] + l[0]]];
          acc = cadd(acc, cscale(u, w));
          touched = true;
        }
      }
    }
    if (touched) A.asmb[g] = acc;
  }
}

void d3_fany(const Step3Args& A, cudaStream_t st) { k3d_fany<<<A.nsub, 256, 0, st>>>(A); }
void d3_flags(const Step3Args& A, cudaStream_t st) { k3d_flags<<<1, 256, 0, st>>>(A); }
void d3_rhs(const Step3Args& A, cudaStream_t st) {
  k3d_rhs_base<<<dim3((A.nw + 255) / 256, A.nsub), 256, 0, st>>>(A);
  if (A.npatch) k3d_rhs_xfer<<<dim3((A.npatch + 127) / 128, A.nsub), 128, 0, st>>>(A);
}
void d3_accumulate(const Step3Args& A, cudaStream_t st) {
  k3d_accumulate<<<hddm::reduce_blocks(), 256, 0, st>>>(A, A.wts);
}

// ---------------------------------------------------------------- global operator
namespace {
__device__ __forceinline__ double block_sum3(double v, double* sh) {
  v = hddm::warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) r += sh[i];
  return r;
}

__device__ __forceinline__ void apply3_body(const Glob3Args& G, const cplx* u, cplx* out, const cplx* f,
                                            double* part) {
  __shared__ double sh[32];
  const long long sx = G.gn[0], sxy = (long long)G.gn[0] * G.gn[1];
  const long long n = sxy * G.gn[2];
  const cplx* a1 = G.ga;
  const cplx* a2 = a1 + G.gn[0];
  const cplx* a3 = a2 + G.gn[1];
  const cplx* i1 = a3 + G.gn[2];
  const cplx* i2 = i1 + G.gn[0];
  const cplx* i3 = i2 + G.gn[1];
  double acc = 0;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int p = int(idx % sx), q = int((idx / sx) % G.gn[1]), r = int(idx / sxy);
    cplx o;
    if (shell3(G.gn, p, q, r)) {
      o = u[idx];
    } else {
      const cplx uc = u[idx];
      const cplx ex = cscale(cmul(a2[q], a3[r]), G.ih2);
      const cplx ey = cscale(cmul(a1[p], a3[r]), G.ih2);
      const cplx ez = cscale(cmul(a1[p], a2[q]), G.ih2);
      cplx tt = cmul(cmul(ex, i1[p]), csub(u[idx + 1], uc));
      tt = csub(tt, cmul(cmul(ex, i1[p - 1]), csub(uc, u[idx - 1])));
      tt = cadd(tt, cmul(cmul(ey, i2[q]), csub(u[idx + sx], uc)));
      tt = csub(tt, cmul(cmul(ey, i2[q - 1]), csub(uc, u[idx - sx])));
      tt = cadd(tt, cmul(cmul(ez, i3[r]), csub(u[idx + sxy], uc)));
      tt = csub(tt, cmul(cmul(ez, i3[r - 1]), csub(uc, u[idx - sxy])));
      o = cadd(cdiv(tt, cmul(cmul(a1[p], a2[q]), a3[r])), cscale(uc, G.k2));
    }
    if (out) out[idx] = o;
    if (f) acc += cnorm2(csub(f[idx], o));
  }
  if (part) {
    const double s = block_sum3(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}
}  // namespace

__global__ void __launch_bounds__(256) k3d_apply(Glob3Args G, const cplx* u, cplx* out, const cplx* f,
                                                 double* part) {
  apply3_body(G, u, out, f, part);
}
__global__ void __launch_bounds__(256) k3d_apply_ind(Glob3Args G, cplx* const* U, int du, cplx* const* O,
                                                     int dout, const int* jp) {
  const int j = *jp;
  apply3_body(G, U[j + du], O[j + dout], nullptr, nullptr);
}
void d3_apply_global(const Glob3Args& G, const cplx* u, cplx* out, const cplx* f, double* part,
                     cudaStream_t st) {
  k3d_apply<<<hddm::reduce_blocks(), 256, 0, st>>>(G, u, out, f, part);
}
void d3_apply_global_ind(const Glob3Args& G, cplx* const* U, int du, cplx* const* O, int dout,
                         const int* jp, cudaStream_t st) {
  k3d_apply_ind<<<hddm::reduce_blocks(), 256, 0, st>>>(G, U, du, O, dout, jp);
}

// ---------------------------------------------------------------- residual check / refine
// r = b - A x with the J-scaled assembled rows (hddm_oracle3.c op3_assemble, columns
// ascending), per (t, chunk) partial sums of |r|^2 and |b|^2; optionally R = r.
__global__ void __launch_bounds__(256) k3c_partials(Chk3Args C, int write_resid) {
  __shared__ double sh[32];
  const int t = blockIdx.y;
  const bool on = (C.flag[t] != 0) == (C.flag_on != 0);
  if (!on) return;  // uniform per CTA
  const Sub3Dev s = C.sub[t];
  const CoefP K = coefs(C.cop, C.cop_stride, s.cls, C.nn);
  const int nx = C.nn[0], ny = C.nn[1], sxy = nx * ny;
  const long long o = (long long)t * C.nw;
  double rr = 0, bb = 0;
  const int per = (C.nw + C.nchunk - 1) / C.nchunk;
  const int p0 = blockIdx.x * per, p1 = min(C.nw, p0 + per);
  for (int pos = p0 + threadIdx.x; pos < p1; pos += blockDim.x) {
    const int v = C.perm[pos];
    const int p = v % nx, q = (v / nx) % ny, r = v / sxy;
    const cplx b = C.B[o + pos];
    cplx ax;
    if (shell3(C.nn, p, q, r)) {
      ax = C.X[o + pos];
    } else {
      const cplx yz = cmul(K.an[1][q], K.an[2][r]), xz = cmul(K.an[0][p], K.an[2][r]),
                 xy = cmul(K.an[0][p], K.an[1][q]);
      const cplx cw = cscale(cmul(yz, K.iah[0][p - 1]), C.ih2);
      const cplx ce = cscale(cmul(yz, K.iah[0][p]), C.ih2);
      const cplx cs = cscale(cmul(xz, K.iah[1][q - 1]), C.ih2);
      const cplx cn = cscale(cmul(xz, K.iah[1][q]), C.ih2);
      const cplx cb = cscale(cmul(xy, K.iah[2][r - 1]), C.ih2);
      const cplx ct = cscale(cmul(xy, K.iah[2][r]), C.ih2);
      const cplx sum6 = cadd(cadd(cadd(cadd(cadd(cw, ce), cs), cn), cb), ct);
      const cplx diag = cadd(cmk(-sum6.x, -sum6.y), cscale(jac3(K, p, q, r), C.k2));
      cplx a = cmk(0, 0);
      if (r > 1) a = cadd(a, cmul(cb, C.X[o + C.pinv[v - sxy]]));
      if (q > 1) a = cadd(a, cmul(cs, C.X[o + C.pinv[v - nx]]));
      if (p > 1) a = cadd(a, cmul(cw, C.X[o + C.pinv[v - 1]]));
      a = cadd(a, cmul(diag, C.X[o + pos]));
      if (p < nx - 2) a = cadd(a, cmul(ce, C.X[o + C.pinv[v + 1]]));
      if (q < ny - 2) a = cadd(a, cmul(cn, C.X[o + C.pinv[v + nx]]));
      if (r < C.nn[2] - 2) a = cadd(a, cmul(ct, C.X[o + C.pinv[v + sxy]]));
      ax = a;
    }
    const cplx res = csub(b, ax);
    if (write_resid) C.R[o + pos] = res;
    rr += cnorm2(res);
    bb += cnorm2(b);
  }
  const double s0 = block_sum3(rr, sh);
  const double s1 = block_sum3(bb, sh);
  if (threadIdx.x == 0) {
    C.part[((long long)t * C.nchunk + blockIdx.x) * 2] = s0;
    C.part[((long long)t * C.nchunk + blockIdx.x) * 2 + 1] = s1;
  }
}

namespace {
__device__ __forceinline__ double rel_of(const Chk3Args& C, int t) {
  double rr = 0, bb = 0;
  for (int k = 0; k < C.nchunk; ++k) {
    rr += C.part[((long long)t * C.nchunk + k) * 2];
    bb += C.part[((long long)t * C.nchunk + k) * 2 + 1];
  }
  return bb > 0 ? sqrt(rr) / sqrt(bb) : 0.0;
}
}  // namespace

// refine's first residual (it = 0): rel, need = rel > 1e-11
__global__ void k3c_first(Chk3Args C) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < C.nsub; t += blockDim.x) {
    const bool on = (C.flag[t] != 0) == (C.flag_on != 0);
    int nd = 0;
    if (on) {
      const double r = rel_of(C, t);
      C.rel_prev[t] = r;
      atomicMax((unsigned long long*)C.max_rel, __double_as_longlong(r));
      nd = r > 1e-11 ? 1 : 0;
      if (nd) atomicAdd(C.corr_count, 1);
    }
    C.need[t] = nd;
    C.ncorr[t] = 0;
    C.undo[t] = 0;
    if (nd) any = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *C.any = any;
    if (C.cond) cudaGraphSetConditional(cudaGraphConditionalHandle(C.cond), any ? 1u : 0u);
  }
}

__global__ void __launch_bounds__(256) k3c_apply(Chk3Args C) {
  const int t = blockIdx.y;
  if (!C.need[t]) return;
  const long long o = (long long)t * C.nw;
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < C.nw; pos += gridDim.x * blockDim.x)
    C.X[o + pos] = cadd(C.X[o + pos], C.C[o + pos]);
}

// after a correction: the stagnation rule (rr >= 0.5 rel: stop, undo if worse),
// the threshold and the 12-pass cap of refine (sparse.cpp:268-292)
__global__ void k3c_decide(Chk3Args C) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < C.nsub; t += blockDim.x) {
    if (!C.need[t]) continue;
    const int it = ++C.ncorr[t];
    int nd = 0;
    if (it < 12) {
      const double r = rel_of(C, t), prev = C.rel_prev[t];
      if (r >= 0.5 * prev) {  // return r < rel ? r : rel, undoing a worse correction
        if (r > prev)
          C.undo[t] = 1;
        else
          C.rel_prev[t] = r;
      } else {
        C.rel_prev[t] = r;
        nd = r > 1e-11 ? 1 : 0;
      }
    }
    if (nd) {
      any = 1;
      atomicAdd(C.corr_count, 1);
    }
    C.need[t] = nd;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *C.any = any;
    if (C.cond) cudaGraphSetConditional(cudaGraphConditionalHandle(C.cond), any ? 1u : 0u);
  }
}

__global__ void __launch_bounds__(256) k3c_undo(Chk3Args C) {
  const int t = blockIdx.y;
  if (!C.undo[t]) return;
  const long long o = (long long)t * C.nw;
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < C.nw; pos += gridDim.x * blockDim.x)
    C.X[o + pos] = csub(C.X[o + pos], C.C[o + pos]);
}

__global__ void k3c_clear_undo(Chk3Args C) {
  for (int t = threadIdx.x; t < C.nsub; t += blockDim.x) C.undo[t] = 0;
}

void c3_partials(const Chk3Args& C, int write_resid, cudaStream_t st) {
  k3c_partials<<<dim3(C.nchunk, C.nsub), 256, 0, st>>>(C, write_resid);
}
void c3_first(const Chk3Args& C, cudaStream_t st) { k3c_first<<<1, 256, 0, st>>>(C); }
void c3_apply(const Chk3Args& C, cudaStream_t st) {
  k3c_apply<<<dim3(std::min(256, (C.nw + 255) / 256), C.nsub), 256, 0, st>>>(C);
}
void c3_decide(const Chk3Args& C, cudaStream_t st) { k3c_decide<<<1, 256, 0, st>>>(C); }
void c3_undo(const Chk3Args& C, cudaStream_t st) {
  k3c_undo<<<dim3(std::min(256, (C.nw + 255) / 256), C.nsub), 256, 0, st>>>(C);
  k3c_clear_undo<<<1, 256, 0, st>>>(C);
}

}  // namespace hddm3
