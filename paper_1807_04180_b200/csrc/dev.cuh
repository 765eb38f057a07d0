// Device-side helpers and POD tables shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace hddm {

typedef double2 cplx;

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return cmk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cmk(a.x, -a.y); }
__host__ __device__ __forceinline__ double cnorm2(cplx a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// a / b (operands here are O(1)..O(1e8) pivots/Jacobians; no overflow scaling)
__host__ __device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  const double d = b.x * b.x + b.y * b.y;
  return cmk((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ cplx shfl_xor(cplx v, int m) {
  return cmk(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
__device__ __forceinline__ cplx warp_sum(cplx v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = cadd(v, shfl_xor(v, m));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ cplx ldg(const cplx* p) { return __ldg(p); }
// factor entries are streamed once per pass: evict-first in L1/L2 so the
// per-subdomain vectors (reused across levels) stay cached
__device__ __forceinline__ cplx ldf(const cplx* p) { return __ldcs(p); }

// Non-blocking prefetch of the 128-byte lines covering [p, p + n) into L1.
__device__ __forceinline__ void prefetch_lines(const cplx* p, int n) {
  const char* a = reinterpret_cast<const char*>(p);
  const char* e = reinterpret_cast<const char*>(p + n);
  for (const char* q = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(127));
       q < e; q += 128)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
}

// Asynchronous bulk prefetch of a contiguous global range into L2 (TMA path,
// sm_90+). p must be 16-byte aligned and bytes a multiple of 16.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  if (bytes == 0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Asynchronous 16-byte global -> shared copy (cp.async, L2 only): no register
// staging, so a CTA can keep thousands of copies in flight.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------ vector layout
// Per-subdomain vectors (B, X, Y, U, R, C; factor order) are stored member-
// interleaved per class: element (t, pos) lives at base[t] + pos * str[t], with
// str[t] = the member count of t's class and base[t] = class offset + member
// slot. Threads walking the members of one (class, item) touch consecutive
// addresses; the factor entry they share is one broadcast load.
struct VMap {
  const long long* base;  // per RHS t
  const int* str;         // per RHS t
  const long long* cbase; // per class c (ncls + 1): storage offset of the class block
  const int* cptr;        // class membership CSR; slot k of class c is cmem[cptr[c] + k]
  const int* cmem;
  int ncls;
  long long total;        // storage length (= nsub * nw)
};

// storage index e -> (RHS t, position pos)
__device__ __forceinline__ void vdecode(const VMap& m, long long e, int& t, int& pos) {
  int lo = 0, hi = m.ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(m.cbase + mid) <= e) lo = mid; else hi = mid - 1;
  }
  const int c0 = __ldg(m.cptr + lo), nm = __ldg(m.cptr + lo + 1) - c0;
  const long long r = e - __ldg(m.cbase + lo);
  pos = int(r / nm);
  t = __ldg(m.cmem + c0 + int(r - (long long)pos * nm));
}

template <class T>
struct SVec {  // strided view of one subdomain's vector
  T* p;
  int s;
  __device__ __forceinline__ T& operator[](long long i) const { return p[i * s]; }
  __device__ __forceinline__ SVec operator+(long long i) const { return {p + i * s, s}; }
};

template <class T>
__device__ __forceinline__ SVec<T> vview(T* v, const VMap& m, int t) {
  return {v + __ldg(m.base + t), __ldg(m.str + t)};
}

// ------------------------------------------------------------ device tables
struct DevSn {
  int kind, c0, n, nrows;
  int blk0, nblk, drow0, parent;
  int child0, child1, extadd0, aent0;
  int aent1, lw;  // lw: leaf width (leaf band rows start at i-1 / i-lw)
  long long diag_off, dinv_off, front_off;
};

struct DevBlk {
  int src, dst, r0, nr, row0, front0;
};

// one solve task: supernode s, rows/columns [a, b)
struct Task {
  int s, a, b, pad;
};

// backward row of a supernode's block: value offset of the row's first stored
// column, that column, and the destination (ancestor) position
struct BwRow {
  long long off;
  int first, dpos;
};

// forward run segment: value offset (per class), length, first source position
struct SegRec {
  long long off;
  int len, zb;
};

struct DevSub {
  int i, j, cx0, cx1, cy0, cy1, wx0, wy0;
  int lint, rint, bint, tint;
  int own0, own1, own2, own3;
  int cls, pad0, pad1, pad2;
};

// quintic taper beta0, proj/src/partition.cpp:7-11
__host__ __device__ __forceinline__ double beta0(double t) {
  if (t <= 0) return 1.0;
  if (t >= 1) return 0.0;
  return 1.0 - t * t * t * (10.0 - 15.0 * t + 6.0 * t * t);
}

}  // namespace hddm
