#pragma once
#include "dev.cuh"

namespace hddm {
void launch_scale_div(cplx* out, const cplx* in, const double* scal, long long n,
                      cudaStream_t st);
void launch_sqrt(const double* in, double* out, cudaStream_t st);
void launch_bsub(cplx* r, const cplx* b, long long n, cudaStream_t st);
void launch_update_x(cplx* x, const cplx* const* Z, const cplx* y, int k, long long n,
                     cudaStream_t st);
void launch_backsolve(const cplx* H, int ld, const cplx* g, cplx* y, int k, cudaStream_t st);
void launch_init_g(cplx* g, int m, const double* rnorm, cudaStream_t st);

// Device-resident state of one FGMRES restart cycle (krylov.cpp:53-109): the
// Arnoldi index j, the iteration counters and the stop decision live in HBM, so a
// whole cycle runs as one CUDA graph (a WHILE node over the iterations) with no
// host round trip; the host reads this record once per cycle.
struct KryState {
  int j;          // current column
  int m;          // columns available this cycle
  int total;      // iterations so far (all cycles)
  int max_iters;
  int k;          // usable columns of this cycle
  int stop;       // 1: converged / dead column / invariant subspace -> no restart
  int converged;
  int flags;      // bit0 dead column, bit1 hlast == 0
  int adv;        // the cycle continues: scale V[j+1] and advance j
  double tol, bnorm, relres, hlast, hlast2;
};
struct KryArgs {
  KryState* ks;
  cplx* const* V;   // m + 1 pointers
  cplx* const* Z;   // m pointers
  cplx* H;          // column j at H + j * ld
  int ld;
  cplx* g;
  cplx* sn;
  double* cs;
  double* hist;     // per iteration: recursive relres
  double* part;
  long long n;
  unsigned long long cond;  // WHILE handle of the cycle graph
};
void launch_kry_load(const KryArgs& K, cplx* f, cudaStream_t st);         // f = V[j]
void launch_kry_store(const KryArgs& K, const cplx* src, cudaStream_t st); // Z[j] = src
void launch_kry_first_dot(const KryArgs& K, cudaStream_t st);   // H[j][0] = <V0, w>
void launch_kry_mgs(const KryArgs& K, int i, cudaStream_t st);  // step i of MGS (no-op if i > j)
void launch_kry_givens(const KryArgs& K, cudaStream_t st);      // Givens, status, WHILE condition
void launch_kry_next(const KryArgs& K, cudaStream_t st);        // V[j+1] /= hlast; j++
}  // namespace hddm
