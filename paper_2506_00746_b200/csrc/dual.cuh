// dual<T>: forward-mode dual number (value, derivative) — the device
// counterpart of "MFEM's internal dual number type" (
// Table 1 "MFEM" column). Operator overloading confines AD to
// the pointwise operator D; P, G, B stay plain linear code.
//
// Supported ops: + - * / with dual or scalar, negation, sqrt, pow(dual, real).
// Rules: (a,a')(b,b') = (ab, a'b + ab');  (a,a')/(b,b') = (a/b, (a' - (a/b) b')/b);
//        sqrt(a,a') = (s, a'/(2s));       pow((a,a'), e) = (a^e, e a^e a'/a)
//        (e == 0 -> (1,0); e == 1 -> identity; e == 0.5 -> sqrt; sec. DESIGN.md A13).
#pragma once
#include <cmath>

#ifndef FEOD_HD
#ifdef __CUDACC__
#define FEOD_HD __host__ __device__ __forceinline__
#else
#define FEOD_HD inline   // host-only compilation (tests/test_dual_host.py)
#endif
#endif

namespace feod {

template <class T>
struct dual {
  T v, d;
  FEOD_HD dual() : v(0), d(0) {}
  FEOD_HD dual(T value) : v(value), d(0) {}
  FEOD_HD dual(T value, T deriv) : v(value), d(deriv) {}
};

template <class T> FEOD_HD dual<T> operator+(dual<T> a, dual<T> b) { return {a.v + b.v, a.d + b.d}; }
template <class T> FEOD_HD dual<T> operator-(dual<T> a, dual<T> b) { return {a.v - b.v, a.d - b.d}; }
template <class T> FEOD_HD dual<T> operator-(dual<T> a) { return {-a.v, -a.d}; }
template <class T> FEOD_HD dual<T> operator*(dual<T> a, dual<T> b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
template <class T> FEOD_HD dual<T> operator/(dual<T> a, dual<T> b) {
  const T q = a.v / b.v;
  return {q, (a.d - q * b.d) / b.v};
}
template <class T> FEOD_HD dual<T> operator+(dual<T> a, T b) { return {a.v + b, a.d}; }
template <class T> FEOD_HD dual<T> operator+(T a, dual<T> b) { return {a + b.v, b.d}; }
template <class T> FEOD_HD dual<T> operator-(dual<T> a, T b) { return {a.v - b, a.d}; }
template <class T> FEOD_HD dual<T> operator-(T a, dual<T> b) { return {a - b.v, -b.d}; }
template <class T> FEOD_HD dual<T> operator*(dual<T> a, T b) { return {a.v * b, a.d * b}; }
template <class T> FEOD_HD dual<T> operator*(T a, dual<T> b) { return {a * b.v, a * b.d}; }
template <class T> FEOD_HD dual<T> operator/(dual<T> a, T b) { return {a.v / b, a.d / b}; }
template <class T> FEOD_HD dual<T>& operator+=(dual<T>& a, dual<T> b) { a = a + b; return a; }

// At a.v == 0 the derivative is taken as 0: the only way to reach it is the p-Laplacian
// with eps = 0 at a zero gradient, where the flux tangent's limit is 0 (reading A20).
template <class T> FEOD_HD dual<T> sqrt(dual<T> a) {
  const T s = ::sqrt(a.v);
  return {s, s > T(0) ? a.d / (T(2) * s) : T(0)};
}

// pow with a real exponent; the special cases keep p = 2, 3, 4 exact and cheap.
template <class T> FEOD_HD dual<T> pow(dual<T> a, T e) {
  if (e == T(0)) return {T(1), T(0)};
  if (e == T(1)) return a;
  if (e == T(0.5)) return sqrt(a);
  const T pv = ::pow(a.v, e);
  return {pv, a.v != T(0) ? e * pv * a.d / a.v : T(0)};   // a.v == 0: reading A20
}

// Plain-double versions so the same flux template instantiates with T = double.
FEOD_HD double pow_special(double a, double e) {
  if (e == 0.0) return 1.0;
  if (e == 1.0) return a;
  if (e == 0.5) return ::sqrt(a);
  return ::pow(a, e);
}
template <class T> FEOD_HD dual<T> pow_special(dual<T> a, T e) { return pow(a, e); }

// The same with the exponent's special case decided once per handle (OpParams::pcase:
// 0 -> e = 0, 1 -> e = 1, 2 -> e = 0.5, 3 -> general): one integer test per point.
FEOD_HD double pow_case(double a, double e, int pc) {
  if (pc == 1) return a;
  if (pc == 2) return ::sqrt(a);
  if (pc == 0) return 1.0;
  return ::pow(a, e);
}
// sqrt of a dual through one reciprocal square root (device): s = a r, s' = a' r / 2 with
// r = 1/sqrt(a) -- no division, no libdevice special-case paths; a == 0 gives (0, 0)
// (reading A20)
template <class T> FEOD_HD dual<T> sqrt_rs(dual<T> a) {
#ifdef __CUDA_ARCH__
  // r from the hardware approximation (MUFU.RSQ64H, ~20 correct bits) and two Newton steps
  // r <- r (3/2 - a r^2 / 2) (~40, then full double precision); a <= 0 (only a == 0 occurs,
  // reading A20) takes the branch-free zero below
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"((double)a.v));
  const double h = -0.5 * a.v;
  r = r * fma(h * r, r, 1.5);
  r = r * fma(h * r, r, 1.5);
  const bool pos = a.v > T(0);
  return {pos ? a.v * r : T(0), pos ? (T(0.5) * a.d) * r : T(0)};
#else
  return sqrt(a);
#endif
}
template <class T> FEOD_HD dual<T> pow_case(dual<T> a, T e, int pc) {
  if (pc == 1) return a;
  if (pc == 2) return sqrt_rs(a);
  if (pc == 0) return {T(1), T(0)};
  const T pv = ::pow(a.v, e);
  return {pv, a.v != T(0) ? e * pv * a.d / a.v : T(0)};   // a.v == 0: reading A20
}

FEOD_HD double value(double a) { return a; }
template <class T> FEOD_HD T value(dual<T> a) { return a.v; }

}  // namespace feod
