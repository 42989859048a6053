// x^y to ~2^-90 relative error in double-double arithmetic, with a rounding
// certificate: the device half of the bit-identical weight synthesiser (row
// f4, weights.cpp:116-122 calls glibc pow).
//
// glibc 2.39's pow is not correctly rounded (its header states < 0.52 ULP for
// results of this magnitude), and its tables are not restated here.  Instead:
// the true value t = x^y is bracketed to far below an ulp; when t lies more
// than 1/32 ulp away from every rounding midpoint, ANY result within 0.53 ULP
// of t that is a double is RN(t), so glibc's result is known without running
// it.  The other draws (~1/16 of them, and every draw with |y ln x| > 64, where
// glibc's own bound widens) are flagged and the caller runs the host's libm on
// exactly those (synth.cu).
//
// All FP64 contractions are explicit (__fma_rn / fma): the build uses
// -fmad=false.
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define DD_HD __host__ __device__ __forceinline__
#else
#define DD_HD inline
#endif

namespace clg {
namespace dd {

struct D2 {
  double h, l;
};

DD_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

DD_HD D2 two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
DD_HD D2 quick_two_sum(double a, double b) {  // |a| >= |b|
  const double s = a + b;
  return {s, b - (s - a)};
}
DD_HD D2 two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma_(a, b, -p)};
}
DD_HD D2 add(D2 a, D2 b) {
  D2 s = two_sum(a.h, b.h);
  const D2 t = two_sum(a.l, b.l);
  s.l += t.h;
  s = quick_two_sum(s.h, s.l);
  s.l += t.l;
  return quick_two_sum(s.h, s.l);
}
DD_HD D2 add_d(D2 a, double b) {
  D2 s = two_sum(a.h, b);
  s.l += a.l;
  return quick_two_sum(s.h, s.l);
}
DD_HD D2 mul(D2 a, D2 b) {
  D2 p = two_prod(a.h, b.h);
  p.l += a.h * b.l + a.l * b.h;
  return quick_two_sum(p.h, p.l);
}
DD_HD D2 mul_d(D2 a, double b) {
  D2 p = two_prod(a.h, b);
  p.l = fma_(a.l, b, p.l);
  return quick_two_sum(p.h, p.l);
}

// ln 2 as a double-double
constexpr double kLn2Hi = 0x1.62e42fefa39efp-1;
constexpr double kLn2Lo = 0x1.abc9e3b39803fp-56;
constexpr double kInvLn2 = 0x1.71547652b82fep+0;

// 1/j! for j = 3..11 (hi, lo): set once by the host (long double quotient,
// 2^-64 relative, which the r^j <= 2^-22 factor takes below 2^-86)
struct ExpCoef {
  double h[12], l[12];
};

inline ExpCoef make_exp_coef() {
  ExpCoef c{};
  long double f = 1.0L;
  for (int j = 1; j < 12; ++j) {
    f *= static_cast<long double>(j);
    const long double q = 1.0L / f;
    c.h[j] = static_cast<double>(q);
    c.l[j] = static_cast<double>(q - static_cast<long double>(c.h[j]));
  }
  c.h[0] = 1.0;
  c.l[0] = 0.0;
  return c;
}

// exp(a) - 1 scaled: returns e with exp(a) = (1 + e) * 2^k.  |a| < 700.
DD_HD D2 expm1_reduced(D2 a, const ExpCoef& cf, int& k) {
  const double kd = rint(a.h * kInvLn2);
  k = static_cast<int>(kd);
  // r = a - k ln2, |r| <= 0.35; then r / 64
  D2 r = add(a, mul_d(D2{-kLn2Hi, -kLn2Lo}, kd));
  r.h *= 0x1p-6;
  r.l *= 0x1p-6;
  // p = r + r^2/2 + r^3/3! + ... + r^11/11!   (Horner from the top, dd)
  D2 p{cf.h[11], cf.l[11]};
#pragma unroll
  for (int j = 10; j >= 1; --j) p = add(mul(p, r), D2{cf.h[j], cf.l[j]});
  p = mul(p, r);
  // (1 + p)^2 - 1 = 2p + p^2, six times
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const D2 q = mul(p, p);
    p = add(D2{2.0 * p.h, 2.0 * p.l}, q);
  }
  return p;
}

// ln(x) for finite x > 0 (normal), as a double-double.  l0 is any double
// within a few ulps of ln(m) (libm / CUDA log): one Newton step in dd
// removes its error:  ln m = l0 + ln(m e^{-l0}) = l0 + t - t^2/2, |t| < 2^-50.
DD_HD D2 log_dd(double x, const ExpCoef& cf) {
  int e;
  double m = frexp(x, &e);  // [0.5, 1)
  if (m < 0.70710678118654752) {
    m *= 2.0;
    --e;
  }
  const double l0 = log(m);
  int k;
  const D2 em1 = expm1_reduced(D2{-l0, 0.0}, cf, k);  // e^{-l0} = (1+em1) 2^k
  const double ms = ldexp(m, k);                      // exact
  // t = ms (1 + em1) - 1 = (ms - 1) + ms em1
  const D2 t = add_d(mul_d(em1, ms), ms - 1.0);  // ms - 1 exact (Sterbenz range or ms == 1)
  const D2 t2 = mul(t, t);
  D2 lm = add(D2{l0, 0.0}, add(t, D2{-0.5 * t2.h, -0.5 * t2.l}));
  const D2 el = mul_d(D2{kLn2Hi, kLn2Lo}, static_cast<double>(e));
  return add(el, lm);
}

// x^y.  Returns RN candidate `r`; *certain is false when the double-double
// value lies within 1/32 ulp of a rounding midpoint (or r is a power of two,
// or outside the normal range handled here).
DD_HD double pow_certified(double x, double y, const ExpCoef& cf, bool* certain) {
  const D2 lx = log_dd(x, cf);
  const D2 a = mul_d(lx, y);
  if (!(fabs(a.h) < 690.0)) {
    *certain = false;
    return 0.0;
  }
  int k;
  const D2 em1 = expm1_reduced(a, cf, k);
  const D2 v = add_d(em1, 1.0);  // in (0.7, 1.42)
  const double r = ldexp(v.h, k);
  // ulp of v.h: v.h in [0.5,1) -> 2^-53, [1,2) -> 2^-52
  const double ulp = v.h < 1.0 ? 0x1p-53 : 0x1p-52;
  const bool pow2 = v.h == 1.0 || v.h == 0.5;
  // glibc's bound grows with |y ln x| (its log carries ~1.5 * 2^-68 relative error into the
  // exponent): 0.511 + |a| * 1.5 * 2^-15 ULP stays below 0.5 + 1/32 only for moderate |a|
  *certain = !pow2 && fabs(a.h) <= 64.0 && fabs(v.l) < (0.5 - 1.0 / 32.0) * ulp;
  return r;
}

}  // namespace dd
}  // namespace clg
