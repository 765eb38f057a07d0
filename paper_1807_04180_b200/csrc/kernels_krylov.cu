// Device-resident flexible GMRES building blocks (fgmres, proj/src/krylov.cpp:24-133).
// V, Z, the Hessenberg matrix, Givens rotations and g stay in HBM; the host
// only reads one small status record per iteration to decide termination.
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

// w -= h * Vi ; then partials of <Vn, w> (Vn != null) or of |w|^2
__global__ void __launch_bounds__(256) k_axpy_dot(cplx* w, const cplx* Vi, const cplx* h,
                                                  const cplx* Vn, long long n, double* part) {
  __shared__ double sh[32];
  const cplx hv = *h;
  double a = 0, b = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const cplx v = Vi[i];
    cplx x = w[i];
    // w[t] -= hij * V[i][t]  (krylov.cpp:66)
    const cplx p = cmul(hv, v);
    x = csub(x, p);
    w[i] = x;
    if (Vn) {
      const cplx y = Vn[i];
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
      part[2 * blockIdx.x] = s0;
      part[2 * blockIdx.x + 1] = s1;
    } else {
      part[blockIdx.x] = s0;
    }
  }
}

void launch_axpy_dot(cplx* w, const cplx* Vi, const cplx* h, const cplx* Vn, long long n,
                     double* part, cudaStream_t st) {
  k_axpy_dot<<<reduce_blocks(), 256, 0, st>>>(w, Vi, h, Vn, n, part);
}

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
}  // namespace

// Givens step of column j (krylov.cpp:68-109). H column j holds h_0j..h_jj in
// Hc[0..j], and hlast^2 in *hlast2. Writes status: [0] relres, [1] flags
// (bit0 dead column, bit1 hlast == 0), [2] hlast.
__global__ void k_givens(cplx* Hc, const double* hlast2, double* cs, cplx* sn, cplx* g,
                         int j, double bnorm, double* status, double* hlast_out) {
  const double hlast = sqrt(*hlast2);
  Hc[j + 1] = cmk(hlast, 0.0);
  for (int i = 0; i < j; ++i) {
    const cplx a = Hc[i], c = Hc[i + 1];
    Hc[i] = cadd(cscale(a, cs[i]), cmul(sn[i], c));
    Hc[i + 1] = cadd(cmul(cmk(-sn[i].x, sn[i].y), a), cscale(c, cs[i]));
  }
  const cplx a = Hc[j], c = Hc[j + 1];
  const double t = sqrt(cnorm2(a) + cnorm2(c));
  int flags = 0;
  if (t == 0) {
    flags |= 1;
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
    status[0] = cabs_d(g[j + 1]) / bnorm;
  }
  if (hlast == 0) flags |= 2;
  status[1] = flags;
  status[2] = hlast;
  *hlast_out = hlast;
}
void launch_givens(cplx* Hc, const double* hlast2, double* cs, cplx* sn, cplx* g, int j,
                   double bnorm, double* status, double* hlast_out, cudaStream_t st) {
  k_givens<<<1, 1, 0, st>>>(Hc, hlast2, cs, sn, g, j, bnorm, status, hlast_out);
}

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

}  // namespace hddm
