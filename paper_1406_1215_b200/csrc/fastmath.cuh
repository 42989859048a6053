// Fast FP64 pieces for the reference-stream sampler that stay BIT-EXACT with
// the reference by construction: each fast result either provably equals the
// reference's value or the caller falls back to the reference expression.
//
//   log_fast(x)       x in (0,1): |rel err| <= ~2^-49 (128-entry table of
//                     reciprocal centres + a degree-7 log1p series on
//                     |t| <= 2^-8; x >= 15/16 goes through log1m_series)
//   log1m_fast(p)     log1p(-p), p in (0,1), same bound (degree-7/15 series
//                     for p < 1/16, else log(1-p) with the exact residual)
//   rcp_fast(x)       1/x to ~2^-52 (float seed + two Newton steps)
//   div_S(prod)       RN(prod / S) from a correctly rounded 1/S plus one FMA
//                     correction, certified by an exact residual
//   accept_ref(r,q,p) r < RN(q / p) decided from the FMA residual q - r p,
//                     falling back to __ddiv_rn only inside the tie band
#pragma once

#include "common.cuh"

namespace clg {

constexpr int kLogTable = 128;

// inv_c[i] = RN(1 / c_i), c_i = 1 + (i + 1/2)/128;  nlog_inv[i] = -log(inv_c[i])
struct LogTable {
  double inv_c[kLogTable];
  double nlog_inv[kLogTable];
};

// log1p(-p) for 0 <= p < 1/16: -p * sum_{k=0}^{15} p^k / (k+1)  (trunc < 2^-64 p)
// Estrin's scheme (dependency depth ~5 instead of 16: this sits on the
// reference-stream chain's critical path p -> skip -> v -> w[v] -> q = p).
// For p < 2^-7 the first 8 terms suffice (truncation < p^8 / 9 < 2^-59).
__device__ __forceinline__ double log1m_series(double p) {
  const double p2 = p * p, p4 = p2 * p2;
  if (p < 0x1p-7) {
    const double a0 = __fma_rn(p, 0.5, 1.0);
    const double a1 = __fma_rn(p, 1.0 / 4.0, 1.0 / 3.0);
    const double a2 = __fma_rn(p, 1.0 / 6.0, 1.0 / 5.0);
    const double a3 = __fma_rn(p, 1.0 / 8.0, 1.0 / 7.0);
    return -p * __fma_rn(p4, __fma_rn(p2, a3, a2), __fma_rn(p2, a1, a0));
  }
  const double p8 = p4 * p4;
  // pairs c_k + c_{k+1} p with c_k = 1/(k+1)
  const double a0 = __fma_rn(p, 0.5, 1.0);
  const double a1 = __fma_rn(p, 1.0 / 4.0, 1.0 / 3.0);
  const double a2 = __fma_rn(p, 1.0 / 6.0, 1.0 / 5.0);
  const double a3 = __fma_rn(p, 1.0 / 8.0, 1.0 / 7.0);
  const double a4 = __fma_rn(p, 1.0 / 10.0, 1.0 / 9.0);
  const double a5 = __fma_rn(p, 1.0 / 12.0, 1.0 / 11.0);
  const double a6 = __fma_rn(p, 1.0 / 14.0, 1.0 / 13.0);
  const double a7 = __fma_rn(p, 1.0 / 16.0, 1.0 / 15.0);
  const double b0 = __fma_rn(p2, a1, a0);
  const double b1 = __fma_rn(p2, a3, a2);
  const double b2 = __fma_rn(p2, a5, a4);
  const double b3 = __fma_rn(p2, a7, a6);
  const double c0 = __fma_rn(p4, b1, b0);
  const double c1 = __fma_rn(p4, b3, b2);
  return -p * __fma_rn(p8, c1, c0);
}

// log(x) for x in (0, 1)
__device__ __forceinline__ double log_fast(double x, const LogTable& T) {
  if (x >= 0.9375) return log1m_series(1.0 - x);  // 1 - x exact (Sterbenz)
  long long b = __double_as_longlong(x);
  int E = static_cast<int>((b >> 52) & 0x7ff);
  if (E == 0) {  // subnormal: rescale
    x = x * 0x1p54;
    b = __double_as_longlong(x);
    E = static_cast<int>((b >> 52) & 0x7ff) - 54;
  }
  E -= 1023;
  const int i = static_cast<int>((b >> 45) & (kLogTable - 1));
  const double m = __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double t = __fma_rn(m, T.inv_c[i], -1.0);  // |t| <= ~2^-8
  // log1p(t) = t * (1 - t/2 + t^2/3 - ... + t^6/7)
  double s = __fma_rn(t, 1.0 / 7.0, -1.0 / 6.0);
  s = __fma_rn(t, s, 1.0 / 5.0);
  s = __fma_rn(t, s, -1.0 / 4.0);
  s = __fma_rn(t, s, 1.0 / 3.0);
  s = __fma_rn(t, s, -0.5);
  s = __fma_rn(t, s, 1.0);
  const double lt = t * s;
  const double ln2_hi = 0x1.62e42fefa39efp-1;
  const double ln2_lo = 0x1.abc9e3b39803fp-56;
  const double e = static_cast<double>(E);
  return __fma_rn(e, ln2_hi, T.nlog_inv[i] + __fma_rn(e, ln2_lo, lt));
}

// log1p(-p) for p in (0, 1)
__device__ __forceinline__ double log1m_fast(double p, const LogTable& T) {
  if (p < 0.0625) return log1m_series(p);
  const double t = 1.0 - p;          // rounded; t <= 15/16
  const double e = (1.0 - t) - p;    // exact residual (Fast2Sum, 1 >= p)
  return log_fast(t, T) + e / t;     // log(t + e) = log t + e/t + O((e/t)^2)
}

// 1/x to ~2^-52 relative: float reciprocal seed + two Newton steps (the
// skip ratio only needs ~2^-48; __drcp_rn's exact rounding costs ~3x more).
__device__ __forceinline__ double rcp_fast(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-30 && ax < 1e30)) return __drcp_rn(x);
  double y = static_cast<double>(__frcp_rn(static_cast<float>(x)));
  double e = __fma_rn(-x, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-x, y, 1.0);
  return __fma_rn(y, e, y);
}

// RN(prod / S) given invS = RN(1/S).  Falls back to __ddiv_rn when the
// residual cannot certify the result (power-of-two quotient, extreme ranges).
__device__ __forceinline__ double div_S(double prod, double S, double invS) {
  const double q0 = prod * invS;
  const double r0 = __fma_rn(-q0, S, prod);
  const double q1 = __fma_rn(r0, invS, q0);
  const double r1 = __fma_rn(-q1, S, prod);  // exact when q1 is within an ulp
  const long long qb = __double_as_longlong(q1);
  const int qe = static_cast<int>((qb >> 52) & 0x7ff);
  if (qe <= 54 || qe >= 0x7fe || (qb & 0x000fffffffffffffLL) == 0 || !(prod > 0x1p-900))
    return __ddiv_rn(prod, S);
  const double ulp = __longlong_as_double(static_cast<long long>(qe - 52) << 52);
  if (fabs(r1) < S * ulp * 0.4990234375) return q1;  // strictly inside half an ulp
  return __ddiv_rn(prod, S);
}

// r < RN(q / p) for r in (0,1), 0 < q <= p <= 1.
__device__ __forceinline__ bool accept_ref(double r, double q, double p) {
  const double t = __fma_rn(-r, p, q);  // RN(q - r p): sign exact
  if (t < 0.0) return false;            // q/p < r  =>  RN(q/p) <= r
  if (t > p * 0x1p-51) return true;     // q/p > r + 2^-51 > r + ulp(r)
  return r < __ddiv_rn(q, p);
}

}  // namespace clg
