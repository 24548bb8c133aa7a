// Correctly rounded pow(x, y) for x >= 0 (the power-cost map, cost.hpp:58-68,
// and axis costs, cost.hpp:36-40), host and device.
//
// x^y = exp(y ln x) evaluated in double-double (about 2^-100 relative), then
// rounded once to the nearest double. The reference calls glibc's pow, which
// is not correctly rounded: measured on this image, 31 of 40,000 samples of
// pow(x, 2.0) and about 0.08 % of pow(x, y) for the exponents 1/(p-1) differ
// from the correctly rounded value by one ulp (tests/test_oracle.py keeps the
// measurement). Bitwise agreement with glibc would need glibc's own code, so
// results here equal the reference to within one ulp per pow call.
//
// Steps: ln m for x = m 2^e, m in [1/sqrt2, sqrt2), by one Newton step on the
// double log (l1 = l0 + (m - e^l0) / e^l0 with e^l0 in double-double); e ln 2
// from a triple-double ln 2; exp of a double-double by k ln 2 + r reduction,
// r / 32 Taylor (12 terms, Horner) and five squarings.
#pragma once

#include <math.h>

#include "dct_line.h"  // BFM_HD

namespace bfmpow {

struct dd {
  double hi, lo;
};

BFM_HD dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
BFM_HD dd fast_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
BFM_HD dd two_prod(double a, double b) {
  const double p = a * b;
#if defined(__CUDA_ARCH__)
  return {p, __fma_rn(a, b, -p)};
#else
  return {p, fma(a, b, -p)};
#endif
}
BFM_HD dd add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return fast_two_sum(s.hi, s.lo);
}
BFM_HD dd mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return fast_two_sum(p.hi, p.lo);
}
BFM_HD dd mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return fast_two_sum(p.hi, p.lo);
}
BFM_HD dd div_d(dd a, double b) {  // a / b, b a small exact integer here
  const double q1 = a.hi / b;
  const dd p = two_prod(q1, b);
  const double r = ((a.hi - p.hi) - p.lo) + a.lo;
  return fast_two_sum(q1, r / b);
}

// ln 2 = L2_HI + L2_MID + L2_LO (triple double)
constexpr double L2_HI = 0x1.62e42fefa39efp-1;
constexpr double L2_MID = 0x1.abc9e3b39803fp-56;
constexpr double L2_LO = 0x1.7b57a079a1934p-111;

// exp of a double-double with |t| < 709
BFM_HD dd exp_dd(dd t) {
  const double k = rint(t.hi / L2_HI);
  // r = t - k ln 2, each product exact (two_prod) or below 2^-110 relative
  dd r = add(t, {-two_prod(k, L2_HI).hi, -two_prod(k, L2_HI).lo});
  r = add(r, {-two_prod(k, L2_MID).hi, -two_prod(k, L2_MID).lo});
  r = add(r, {-(k * L2_LO), 0.0});
  // r / 32, Taylor to r^12 / 12! (Horner), then square five times
  const dd s = {r.hi * 0.03125, r.lo * 0.03125};
  dd p = {1.0, 0.0};
  for (int n = 12; n >= 1; --n) p = add({1.0, 0.0}, div_d(mul(p, s), static_cast<double>(n)));
  for (int i = 0; i < 5; ++i) p = mul(p, p);
  const int ki = static_cast<int>(k);
  return {ldexp(p.hi, ki), ldexp(p.lo, ki)};
}

// ln x (x > 0 finite, normal) in double-double
BFM_HD dd log_dd(double x) {
  int e = 0;
  double m = frexp(x, &e);  // m in [0.5, 1)
  if (m < 0.70710678118654752440) {
    m *= 2.0;
    e -= 1;
  }
  const double l0 = log(m);
  const dd E = exp_dd({l0, 0.0});
  // correction (m - E) / E: m - E.hi is exact (E.hi is within an ulp or two of m)
  const double c = ((m - E.hi) - E.lo) / E.hi;
  dd lm = two_sum(l0, c);
  const double ed = static_cast<double>(e);
  dd el = two_prod(ed, L2_HI);
  el = add(el, two_prod(ed, L2_MID));
  el = add(el, {ed * L2_LO, 0.0});
  return add(el, lm);
}

// x^y for x >= 0, y > 0 (the exponents the power costs use)
BFM_HD double pow_cr(double x, double y) {
  if (!(x > 0.0)) return x == 0.0 ? 0.0 : x * y;  // 0 -> 0; NaN propagates
  if (isinf(x)) return x;
  if (y == 1.0) return x;
  if (y == 2.0) {  // exactly rounded square
    return x * x;
  }
  // subnormal x: scale into the normal range (x = xs 2^-64)
  double xs = x;
  double shift = 0.0;
  if (xs < 2.2250738585072014e-308) {
    xs = x * 18446744073709551616.0;  // 2^64, exact
    shift = -64.0;
  }
  dd l = log_dd(xs);
  if (shift != 0.0) l = add(l, mul_d({L2_HI, L2_MID}, shift));
  const dd t = mul_d(l, y);
  if (t.hi > 709.78) return INFINITY;
  if (t.hi < -745.2) return 0.0;
  const dd r = exp_dd(t);
  return r.hi + r.lo;
}

}  // namespace bfmpow
