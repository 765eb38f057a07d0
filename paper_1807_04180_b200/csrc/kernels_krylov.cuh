#pragma once
#include "dev.cuh"

namespace hddm {
void launch_axpy_dot(cplx* w, const cplx* Vi, const cplx* h, const cplx* Vn, long long n,
                     double* part, cudaStream_t st);
void launch_scale_div(cplx* out, const cplx* in, const double* scal, long long n,
                      cudaStream_t st);
void launch_sqrt(const double* in, double* out, cudaStream_t st);
void launch_bsub(cplx* r, const cplx* b, long long n, cudaStream_t st);
void launch_update_x(cplx* x, const cplx* const* Z, const cplx* y, int k, long long n,
                     cudaStream_t st);
void launch_givens(cplx* Hc, const double* hlast2, double* cs, cplx* sn, cplx* g, int j,
                   double bnorm, double* status, double* hlast_out, cudaStream_t st);
void launch_backsolve(const cplx* H, int ld, const cplx* g, cplx* y, int k, cudaStream_t st);
void launch_init_g(cplx* g, int m, const double* rnorm, cudaStream_t st);
}  // namespace hddm
