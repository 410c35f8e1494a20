// common.cuh — shared device helpers for the sm_100a kernels of liblra.so.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/lra.h"

#define LRA_NT 512          // threads of the maxvol / C-A CTAs
#define LRA_QMAX 64         // largest k = l handled by the on-chip (cluster / grid) tiers
#define LRA_QMAX_ALL 112    // largest k = l handled at all (global-memory tier; the nucleus's H and V fit in shared memory)

// ------------------------------------------------------- index checks (diagnostic builds)
// Built with -DLRA_CHECK_IDX=1: data-dependent row / column indices are range-checked before
// use; the first violation (kernel id, problem, index value, bound) is recorded in
// lra::g_idx_err and the index is clamped so the kernel does not fault.
#ifndef LRA_CHECK_IDX
#define LRA_CHECK_IDX 0
#endif
namespace lra {
static __device__ long long g_idx_err[4];   // one per translation unit (no relocatable device code)
}
#if LRA_CHECK_IDX
#define LRA_CHKIDX(kid, prob, v, N)                                                            \
  do {                                                                                         \
    if ((v) < 0 || (v) >= (N)) {                                                               \
      if (atomicCAS((unsigned long long *)&lra::g_idx_err[0], 0ull, (unsigned long long)(kid)) == 0ull) { \
        lra::g_idx_err[1] = (long long)(prob);                                                 \
        lra::g_idx_err[2] = (long long)(v);                                                    \
        lra::g_idx_err[3] = (long long)(N);                                                    \
      }                                                                                        \
      (v) = 0;                                                                                 \
    }                                                                                          \
  } while (0)
#else
#define LRA_CHKIDX(kid, prob, v, N) do { } while (0)
#endif

// ----------------------------------------------------------------------------- complex
struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx cmake(double r, double i) { return cplx{r, i}; }

// IEEE-ordered operations without FMA contraction, so the cold LUP reproduces the
// oracle's numpy arithmetic (one multiply, one subtract) bit for bit (reading C23).
__device__ __forceinline__ double rsub_mul(double a, double f, double b) {
  return __dsub_rn(a, __dmul_rn(f, b));  // a - f*b
}
__device__ __forceinline__ cplx cmul_nofma(cplx a, cplx b) {
  return cplx{__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
              __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
// Smith's algorithm (numpy's complex division order).
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  double ar = fabs(b.re), ai = fabs(b.im);
  if (ar >= ai) {
    if (ar == 0.0 && ai == 0.0) return cplx{a.re / ar, a.im / ai};
    double rat = b.im / b.re;
    double scl = 1.0 / __dadd_rn(b.re, __dmul_rn(b.im, rat));
    return cplx{__dmul_rn(__dadd_rn(a.re, __dmul_rn(a.im, rat)), scl),
                __dmul_rn(__dsub_rn(a.im, __dmul_rn(a.re, rat)), scl)};
  } else {
    double rat = b.re / b.im;
    double scl = 1.0 / __dadd_rn(b.im, __dmul_rn(b.re, rat));
    return cplx{__dmul_rn(__dadd_rn(__dmul_rn(a.re, rat), a.im), scl),
                __dmul_rn(__dsub_rn(__dmul_rn(a.im, rat), a.re), scl)};
  }
}
__device__ __forceinline__ double cabs_(cplx a) { return hypot(a.re, a.im); }

// ------------------------------------------------------------- scalar trait for maxvol
template <typename T> struct Sc;
template <> struct Sc<double> {
  static __device__ __forceinline__ double abs(double x) { return fabs(x); }
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double one() { return 1.0; }
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  static __device__ __forceinline__ double sub_mul(double a, double f, double b) { return rsub_mul(a, f, b); }
  static __device__ __forceinline__ double fsub_mul(double a, double f, double b) { return fma(-f, b, a); }
  static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
};
template <> struct Sc<cplx> {
  static __device__ __forceinline__ double abs(cplx x) { return cabs_(x); }
  static __device__ __forceinline__ cplx zero() { return cplx{0.0, 0.0}; }
  static __device__ __forceinline__ cplx one() { return cplx{1.0, 0.0}; }
  static __device__ __forceinline__ cplx div(cplx a, cplx b) { return cdiv(a, b); }
  static __device__ __forceinline__ cplx sub_mul(cplx a, cplx f, cplx b) {
    cplx p = cmul_nofma(f, b);
    return cplx{__dsub_rn(a.re, p.re), __dsub_rn(a.im, p.im)};
  }
  static __device__ __forceinline__ cplx fsub_mul(cplx a, cplx f, cplx b) {
    return cplx{fma(-f.re, b.re, fma(f.im, b.im, a.re)), fma(-f.re, b.im, fma(-f.im, b.re, a.im))};
  }
  static __device__ __forceinline__ cplx mul(cplx a, cplx b) {
    return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  }
};

// ------------------------------------------------------------------- warp reductions
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --------------------------------------------------------------- dense operand access
__device__ __forceinline__ double wload(const void *w, int dtype, int64_t ldw, int64_t i, int64_t j) {
  return dtype == LRA_F32 ? (double)__ldg((const float *)w + j * ldw + i)
                          : __ldg((const double *)w + j * ldw + i);
}

// Entry oracle of the factored operand W = A*B + E (config 4): sum_t A[i,t] B[t,j] + E_ij.
struct FactOp {
  const double *fa, *fb;
  int64_t m, p;
  const int64_t *rowptr, *col;
  const double *val;
  __device__ double at(int64_t i, int64_t j) const {
    double s = 0.0;
    for (int64_t t = 0; t < p; ++t) s = fma(__ldg(fa + t * m + i), __ldg(fb + j * p + t), s);
    int64_t lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
    while (lo < hi) {  // binary search in the (ascending) columns of row i
      int64_t mid = (lo + hi) >> 1;
      int64_t c = __ldg(col + mid);
      if (c == j) return s + __ldg(val + mid);
      if (c < j) lo = mid + 1; else hi = mid;
    }
    return s;
  }
};

// Generic operand view passed by value to kernels.
struct OpView {
  int kind, dtype;
  int64_t m, n;
  const void *w;
  int64_t ldw;
  FactOp f;
  __device__ __forceinline__ double at(int64_t i, int64_t j) const {
    return kind == LRA_OP_DENSE ? wload(w, dtype, ldw, i, j) : f.at(i, j);
  }
};
