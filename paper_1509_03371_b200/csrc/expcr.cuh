// expcr.cuh -- exp(double) rounded once from a double-double evaluation (softmax_forward's
// glibc exp, layers.hpp:236), shared by the side kernels (layers.cu) and MALIS (malis.cu).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace graft {
namespace expcr {

// ---- exp(double) correctly rounded (double-double evaluation) ------------------------------
// softmax_forward uses glibc's exp (layers.hpp:236), which is correctly rounded except in
// rare cases; CUDA's exp() is a 1-ulp approximation. This evaluates exp to ~2^-98 relative
// and rounds once, so it equals a correctly rounded exp for all but ~2^-45 of arguments.
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dadd_rn(s, -a);
  const double e = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
  return {s, e};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dadd_rn(b, -__dadd_rn(s, -a))};
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = __dmul_rn(a.hi, b.hi);
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return fast_two_sum(p, e);
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_div_int(dd a, double n) {  // n small positive integer
  const double q1 = __ddiv_rn(a.hi, n);
  const double r = __fma_rn(-q1, n, a.hi);  // exact remainder
  const double q2 = __ddiv_rn(__dadd_rn(r, a.lo), n);
  return fast_two_sum(q1, q2);
}

// exp(x) = t * 2^k with t in double-double (|x| within the finite range, x != 0).
__device__ inline dd exp_dd_core(double x, int* k) {
  const double L1 = 0x1.62e42fee00000p-1;   // ln2 high part (32 significant bits)
  const double L2 = 0x1.a39ef35793c76p-33;  // next 53 bits
  const double L3 = 0x1.cc01f97b57a08p-87;  // remainder
  const double kd = rint(__dmul_rn(x, 1.4426950408889634));
  // r = x - k*ln2 in double-double; x - k*L1 is exact (Sterbenz / 32-bit L1).
  const double r0 = __fma_rn(-kd, L1, x);
  const double p_hi = __dmul_rn(kd, L2);
  const double p_lo = __fma_rn(kd, L2, -p_hi);
  dd r = two_sum(r0, -p_hi);
  r.lo = __dadd_rn(__dadd_rn(r.lo, -p_lo), -__dmul_rn(kd, L3));
  r = fast_two_sum(r.hi, r.lo);
  // q = r / 256, exp(q) by Horner 1 + q(1 + q/2(1 + q/3(... (1 + q/12)))) in dd, then ^256.
  const dd q = {ldexp(r.hi, -8), ldexp(r.lo, -8)};
  dd t = {1.0, 0.0};
  for (int n = 12; n >= 1; --n) {
    t = dd_div_int(dd_mul(q, t), static_cast<double>(n));
    t = dd_add({1.0, 0.0}, t);
  }
  for (int i = 0; i < 8; ++i) t = dd_mul(t, t);
  *k = static_cast<int>(kd);
  return t;
}

__device__ inline double exp_cr(double x) {
  if (x != x) return x;
  if (x == 0.0) return 1.0;
  if (x > 709.782712893384) return CUDART_INF;
  if (x < -745.1332191019412) return 0.0;
  int k = 0;
  const dd t = exp_dd_core(x, &k);
  const double y = __dadd_rn(t.hi, t.lo);
  return ldexp(y, k);
}

}  // namespace expcr
}  // namespace graft
