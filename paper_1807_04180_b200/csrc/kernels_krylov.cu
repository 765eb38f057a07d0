// Device-resident flexible GMRES building blocks (fgmres, proj/src/krylov.cpp:24-133).
// V, Z, the Hessenberg matrix, Givens rotations, g and the iteration state
// (KryState) stay in HBM; a restart cycle is one CUDA graph launch whose WHILE node
// runs the Arnoldi iterations, and the host reads the status record once per cycle.
//
// Modified Gram-Schmidt keeps the reference's sequential recurrence
// (h_ij = <V_i, w>, w -= h_ij V_i for i = 0..j): each pass fuses the axpy of
// step i with the dot of step i+1 (or the final norm), deterministic block
// partials + fixed-order finish.
#include "dev.cuh"
#include "kernels.cuh"
#include "kernels_krylov.cuh"

namespace hddm {

namespace {
__device__ __forceinline__ double block_sum_k(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) r += sh[i];
  return r;
}
}  // namespace

// out = in / s  (s = *scal)
__global__ void k_scale_div(cplx* out, const cplx* in, const double* scal, long long n) {
  const double s = *scal;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = cmk(in[i].x / s, in[i].y / s);
}
void launch_scale_div(cplx* out, const cplx* in, const double* scal, long long n,
                      cudaStream_t st) {
  k_scale_div<<<reduce_blocks(), 256, 0, st>>>(out, in, scal, n);
}

__global__ void k_sqrt(const double* in, double* out) { *out = sqrt(*in); }
void launch_sqrt(const double* in, double* out, cudaStream_t st) {
  k_sqrt<<<1, 1, 0, st>>>(in, out);
}

// r = b - r
__global__ void k_bsub(cplx* r, const cplx* b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    r[i] = csub(b[i], r[i]);
}
void launch_bsub(cplx* r, const cplx* b, long long n, cudaStream_t st) {
  k_bsub<<<reduce_blocks(), 256, 0, st>>>(r, b, n);
}

// x[t] += y_l Z_l[t] for l = 0..k-1 in order (krylov.cpp:118-119)
__global__ void k_update_x(cplx* x, const cplx* const* Z, const cplx* y, int k, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    cplx xi = x[i];
    for (int l = 0; l < k; ++l) xi = cadd(xi, cmul(y[l], Z[l][i]));
    x[i] = xi;
  }
}
void launch_update_x(cplx* x, const cplx* const* Z, const cplx* y, int k, long long n,
                     cudaStream_t st) {
  k_update_x<<<reduce_blocks(), 256, 0, st>>>(x, Z, y, k, n);
}

namespace {
__device__ double cabs_d(cplx a) { return hypot(a.x, a.y); }
__device__ __forceinline__ int reduce_blocks_dev() { return kReduceBlocks; }
}  // namespace

// back substitution H y = g (krylov.cpp:111-117); H column-major by j with
// leading dimension ld (H[l*ld + i] = H[l][i] of the reference)
__global__ void k_backsolve(const cplx* H, int ld, const cplx* g, cplx* y, int k) {
  for (int i = k - 1; i >= 0; --i) {
    cplx s = g[i];
    for (int l = i + 1; l < k; ++l) s = csub(s, cmul(H[(long long)l * ld + i], y[l]));
    y[i] = cdiv(s, H[(long long)i * ld + i]);
  }
}
void launch_backsolve(const cplx* H, int ld, const cplx* g, cplx* y, int k, cudaStream_t st) {
  k_backsolve<<<1, 1, 0, st>>>(H, ld, g, y, k);
}

// g[0] = rnorm (real), rest zero
__global__ void k_init_g(cplx* g, int m, const double* rnorm) {
  for (int i = threadIdx.x; i <= m; i += blockDim.x) g[i] = cmk(i == 0 ? *rnorm : 0.0, 0.0);
}
void launch_init_g(cplx* g, int m, const double* rnorm, cudaStream_t st) {
  k_init_g<<<1, 128, 0, st>>>(g, m, rnorm);
}

// ------------------------------------------------------------ graph-resident cycle
__global__ void k_kry_load(KryArgs K, cplx* f) {
  const cplx* v = K.V[K.ks->j];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < K.n;
       i += (long long)gridDim.x * blockDim.x)
    f[i] = v[i];
}
void launch_kry_load(const KryArgs& K, cplx* f, cudaStream_t st) {
  k_kry_load<<<reduce_blocks(), 256, 0, st>>>(K, f);
}

__global__ void k_kry_store(KryArgs K, const cplx* src) {
  cplx* z = K.Z[K.ks->j];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < K.n;
       i += (long long)gridDim.x * blockDim.x)
    z[i] = src[i];
}
void launch_kry_store(const KryArgs& K, const cplx* src, cudaStream_t st) {
  k_kry_store<<<reduce_blocks(), 256, 0, st>>>(K, src);
}

// partials of <V0, w>, w = V[j+1]
__global__ void __launch_bounds__(256) k_kry_dot0(KryArgs K) {
  __shared__ double sh[32];
  const int j = K.ks->j;
  const cplx* a = K.V[0];
  const cplx* b = K.V[j + 1];
  double re = 0, im = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < K.n;
       i += (long long)gridDim.x * blockDim.x) {
    const cplx x = a[i], y = b[i];  // conj(x) * y
    re += x.x * y.x + x.y * y.y;
    im += x.x * y.y - x.y * y.x;
  }
  const double s0 = block_sum_k(re, sh);
  const double s1 = block_sum_k(im, sh);
  if (threadIdx.x == 0) {
    K.part[2 * blockIdx.x] = s0;
    K.part[2 * blockIdx.x + 1] = s1;
  }
}

// fixed-order sum of the partials into H[j][i] (ncomp 2) or hlast^2 (ncomp 1);
// i < 0: the first dot (H[j][0])
__global__ void k_kry_finish(KryArgs K, int i) {
  const int j = K.ks->j;
  const int lane = threadIdx.x;
  if (i > j) return;
  const bool norm = i == j;
  const int ncomp = norm ? 1 : 2;
  double acc[2] = {0, 0};
  for (int c = 0; c < ncomp; ++c) {
    double a = 0;
    for (int b = lane; b < reduce_blocks_dev(); b += 32) a += K.part[b * ncomp + c];
    acc[c] = warp_sum(a);
  }
  if (lane == 0) {
    if (norm)
      K.ks->hlast2 = acc[0];
    else
      K.H[(long long)j * K.ld + i + 1] = cmk(acc[0], acc[1]);
  }
}

// MGS step i: w -= H[j][i] V_i, then partials of <V_{i+1}, w> (i < j) or |w|^2
__global__ void __launch_bounds__(256) k_kry_axpy_dot(KryArgs K, int i) {
  __shared__ double sh[32];
  const int j = K.ks->j;
  if (i > j) return;  // uniform: this unrolled step is beyond the current column
  cplx* w = K.V[j + 1];
  const cplx* Vi = K.V[i];
  const cplx* Vn = i < j ? K.V[i + 1] : nullptr;
  const cplx hv = K.H[(long long)j * K.ld + i];
  double a = 0, b = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < K.n;
       t += (long long)gridDim.x * blockDim.x) {
    cplx x = w[t];
    x = csub(x, cmul(hv, Vi[t]));  // w[t] -= hij * V[i][t]  (krylov.cpp:66)
    w[t] = x;
    if (Vn) {
      const cplx y = Vn[t];
      a += y.x * x.x + y.y * x.y;
      b += y.x * x.y - y.y * x.x;
    } else {
      a += cnorm2(x);
    }
  }
  const double s0 = block_sum_k(a, sh);
  const double s1 = block_sum_k(b, sh);
  if (threadIdx.x == 0) {
    if (Vn) {
      K.part[2 * blockIdx.x] = s0;
      K.part[2 * blockIdx.x + 1] = s1;
    } else {
      K.part[blockIdx.x] = s0;
    }
  }
}

void launch_kry_first_dot(const KryArgs& K, cudaStream_t st) {
  k_kry_dot0<<<reduce_blocks(), 256, 0, st>>>(K);
  k_kry_finish<<<1, 32, 0, st>>>(K, -1);
}

void launch_kry_mgs(const KryArgs& K, int i, cudaStream_t st) {
  k_kry_axpy_dot<<<reduce_blocks(), 256, 0, st>>>(K, i);
  k_kry_finish<<<1, 32, 0, st>>>(K, i);
}

// Givens step of column j and the cycle's stop rules (krylov.cpp:68-109); sets the
// WHILE condition of the cycle graph.
__global__ void k_kry_givens(KryArgs K) {
  KryState& S = *K.ks;
  const int j = S.j;
  cplx* Hc = K.H + (long long)j * K.ld;
  double* cs = K.cs;
  cplx* sn = K.sn;
  cplx* g = K.g;
  const double hlast = sqrt(S.hlast2);
  Hc[j + 1] = cmk(hlast, 0.0);
  for (int i = 0; i < j; ++i) {
    const cplx a = Hc[i], c = Hc[i + 1];
    Hc[i] = cadd(cscale(a, cs[i]), cmul(sn[i], c));
    Hc[i + 1] = cadd(cmul(cmk(-sn[i].x, sn[i].y), a), cscale(c, cs[i]));
  }
  const cplx a = Hc[j], c = Hc[j + 1];
  const double t = sqrt(cnorm2(a) + cnorm2(c));
  int cont = 0;
  S.hlast = hlast;
  if (t == 0) {  // dead column: dropped, stop
    S.flags |= 1;
    S.stop = 1;
  } else {
    if (a.x == 0.0 && a.y == 0.0) {
      cs[j] = 0;
      const double ac = cabs_d(c);
      sn[j] = cmk(c.x / ac, -c.y / ac);
    } else {
      const double aa = cabs_d(a);
      cs[j] = aa / t;
      const cplx u = cmk(a.x / aa, a.y / aa);
      const cplx v = cmul(u, cconj(c));
      sn[j] = cmk(v.x / t, v.y / t);
    }
    Hc[j] = cadd(cscale(a, cs[j]), cmul(sn[j], c));
    Hc[j + 1] = cmk(0, 0);
    const cplx gj = g[j];
    g[j + 1] = cmul(cmk(-sn[j].x, sn[j].y), gj);
    g[j] = cscale(gj, cs[j]);
    S.relres = cabs_d(g[j + 1]) / S.bnorm;
    K.hist[S.total] = S.relres;
    S.total += 1;
    S.k = j + 1;
    if (S.relres <= S.tol) {
      S.converged = 1;
      S.stop = 1;
    } else if (hlast == 0) {  // invariant subspace
      S.flags |= 2;
      S.stop = 1;
    } else {
      cont = (j + 1 < S.m) ? 1 : 0;
    }
  }
  if (K.cond) cudaGraphSetConditional(cudaGraphConditionalHandle(K.cond), unsigned(cont));
  S.adv = cont;
}
void launch_kry_givens(const KryArgs& K, cudaStream_t st) {
  k_kry_givens<<<1, 1, 0, st>>>(K);
}

// V[j+1] = w / hlast and j++ when the cycle continues (krylov.cpp:107-108)
__global__ void k_kry_scale(KryArgs K) {
  const KryState& S = *K.ks;
  if (!S.adv) return;
  cplx* w = K.V[S.j + 1];
  const double s = S.hlast;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < K.n;
       i += (long long)gridDim.x * blockDim.x)
    w[i] = cmk(w[i].x / s, w[i].y / s);
}
__global__ void k_kry_advance(KryArgs K) {
  if (K.ks->adv) K.ks->j += 1;
}
void launch_kry_next(const KryArgs& K, cudaStream_t st) {
  k_kry_scale<<<reduce_blocks(), 256, 0, st>>>(K);
  k_kry_advance<<<1, 1, 0, st>>>(K);
}

}  // namespace hddm
