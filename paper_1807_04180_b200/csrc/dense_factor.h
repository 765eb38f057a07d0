// Batched multifrontal LDL^T of every class with dense fronts (kernels3d.cu k3f_*),
// shared by the 3-D engine and the 2-D engine's dense solver: classes in batches sized
// to a workspace budget, fronts level by level (height): assemble (scatter A,
// extend-add the children's contribution blocks), blocked partial factorization of the
// own columns with the identity rows riding along (their panel yields the inverse of
// the diagonal block), extraction of D, the inverse blocks and the panels in the
// forward (column-major) and backward (row-major) layouts.
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "engine3d.h"
#include "kernels3d.cuh"

namespace hddm3 {

// E provides dalloc<T>(n), upload(vector), dfree(p); d_sn = Y's supernodes on the device;
// aval = the assembled entries of Y's scatter lists, class-major
template <class E>
void dense_factorize(E& e, const Sym3& Y, const DSn3* d_sn, int ncls, const std::vector<cplx>& aval,
                     cplx*& d_vals, cplx*& d_valsT, cudaStream_t st) {
  const int nsn = int(Y.sn.size());
  const long long naent = (long long)Y.aent_i.size();
  auto ck = [](cudaError_t x) {
    if (x != cudaSuccess) throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(x));
  };
  cplx* d_aval = e.upload(aval);
  int* d_ai = e.upload(Y.aent_i);
  int* d_aj = e.upload(Y.aent_j);
  int* d_ext = e.upload(Y.ext);
  d_vals = e.template dalloc<cplx>(size_t(ncls) * Y.nvals);
  d_valsT = e.template dalloc<cplx>(size_t(ncls) * Y.nvals);
  ck(cudaMemsetAsync(d_vals, 0, sizeof(cplx) * size_t(ncls) * Y.nvals, st));
  ck(cudaMemsetAsync(d_valsT, 0, sizeof(cplx) * size_t(ncls) * Y.nvals, st));
  // levels by height
  std::vector<std::vector<int>> lv(Y.max_height + 1);
  for (int s = 0; s < nsn; ++s) lv[Y.sn[s].height].push_back(s);
  std::vector<int*> d_lv;
  for (auto& v : lv) d_lv.push_back(e.upload(v));
  // batch of classes within the workspace budget
  size_t freeb = 0, totb = 0;
  ck(cudaMemGetInfo(&freeb, &totb));
  const double budget = std::min(0.6 * double(freeb), 64.0 * (1ull << 30));
  const double per = double(Y.front_words) * sizeof(cplx);
  int nb = int(std::max(1.0, std::min(double(ncls), std::floor(budget / per))));
  if (per > budget) throw std::runtime_error("front workspace of one class exceeds device memory");
  cplx* fronts = e.template dalloc<cplx>(size_t(nb) * Y.front_words);
  Fac3Args F;
  F.sn = d_sn;
  F.fronts = fronts;
  F.fw = Y.front_words;
  F.aent_i = d_ai;
  F.aent_j = d_aj;
  F.aval = d_aval;
  F.naent = naent;
  F.ext = d_ext;
  F.vals = d_vals;
  F.valsT = d_valsT;
  F.nvals = Y.nvals;
  for (int c0 = 0; c0 < ncls; c0 += nb) {
    const int nbc = std::min(nb, ncls - c0);
    F.cls0 = c0;
    ck(cudaMemsetAsync(fronts, 0, sizeof(cplx) * size_t(nbc) * Y.front_words, st));
    for (int h = 0; h <= Y.max_height; ++h) {
      const int nl = int(lv[h].size());
      if (!nl) continue;
      int maxn = 0, maxcr = 0;
      long long maxent = 0;
      for (int s : lv[h]) {
        const Sn3& a = Y.sn[s];
        maxn = std::max(maxn, a.n);
        for (int k = 0; k < a.nch; ++k) maxcr = std::max(maxcr, int(Y.sn[a.ch[k]].rows.size()));
        maxent = std::max(maxent, (long long)a.n * a.n + (long long)a.rows.size() * a.n);
      }
      f3_scatter(F, d_lv[h], nl, nbc, st);
      f3_extadd(F, d_lv[h], nl, nbc, 0, maxcr, st);
      f3_extadd(F, d_lv[h], nl, nbc, 1, maxcr, st);
      for (int k0 = 0; k0 < maxn; k0 += kNB) {
        int maxrows = 0;
        long long maxtiles = 0;
        for (int s : lv[h]) {
          const Sn3& a = Y.sn[s];
          if (a.n <= k0) continue;
          const int b = std::min(kNB, a.n - k0), r = int(a.rows.size());
          const int ne = std::min(a.n, k0 + b);
          maxrows = std::max(maxrows, (a.n - k0 - b) + r + ne);
          const long long M = a.n + r - k0 - b, T = (M + 63) / 64;
          const long long TE = (ne + 63) / 64, TC = a.n > k0 + b ? (a.n - k0 - b + 63) / 64 : 0;
          maxtiles = std::max(maxtiles, T * (T + 1) / 2 + TE * TC);
        }
        f3_dfac(F, d_lv[h], nl, nbc, k0, st);
        f3_trsm(F, d_lv[h], nl, nbc, k0, maxrows, st);
        f3_update(F, d_lv[h], nl, nbc, k0, maxtiles, st);
      }
      f3_extract(F, d_lv[h], nl, nbc, maxent, st);
      ck(cudaGetLastError());
    }
  }
  ck(cudaStreamSynchronize(st));
  e.dfree(fronts);
  e.dfree(d_aval);
  e.dfree(d_ai);
  e.dfree(d_aj);
  e.dfree(d_ext);
  for (int* p : d_lv) e.dfree(p);
}

}  // namespace hddm3
