// Error-free transforms and exact sign / round-down of short double sums,
// usable on host and device. Semantics follow the reference's exact.hpp
// (/root/reference/proj/include/bfm/exact.hpp:32-73 two_sum/two_prod, :89-106
// zero-eliminating grow, :167-179 round_down toward -inf with -0 -> +0) but
// the implementation is organised for the GPU: fixed-size register arrays,
// a certified double-double fast path for the final rounding, and the full
// expansion path only when the fast path cannot decide.
//
// Everything here must be compiled without FMA contraction (-fmad=false on
// device, -ffp-contract=off on host); two_prod uses an explicit fma, which is
// exact (as in exact.hpp:52-56).
#pragma once

#include <math.h>
#include <stdint.h>

#include "dct_line.h"  // BFM_HD

namespace bfmx {

BFM_HD void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

BFM_HD void two_prod(double a, double b, double& p, double& e) {
  p = a * b;
#if defined(__CUDA_ARCH__)
  e = __fma_rn(a, b, -p);
#else
  e = fma(a, b, -p);
#endif
}

// Neighbouring doubles by bit manipulation (finite inputs; x == 0 handled).
BFM_HD double bits_to_double(long long b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(b);
#else
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
#endif
}
BFM_HD long long double_to_bits(double x) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(x);
#else
  long long b;
  __builtin_memcpy(&b, &x, 8);
  return b;
#endif
}
BFM_HD double next_down(double x) {
  if (x == 0.0) return -4.9406564584124654e-324;
  const long long b = double_to_bits(x);
  return bits_to_double(x > 0.0 ? b - 1 : b + 1);
}
BFM_HD double next_up(double x) {
  if (x == 0.0) return 4.9406564584124654e-324;
  const long long b = double_to_bits(x);
  return bits_to_double(x > 0.0 ? b + 1 : b - 1);
}

// Fixed-capacity nonoverlapping expansion (increasing magnitude, zero-free).
template <int Cap>
struct Exp {
  double q[Cap];
  int n;
  BFM_HD void clear() { n = 0; }
  BFM_HD void grow(double b) {
    if (b == 0.0) return;
    double acc = b;
    int o = 0;
    for (int i = 0; i < n; ++i) {
      double s, e;
      two_sum(acc, q[i], s, e);
      acc = s;
      if (e != 0.0) q[o++] = e;
    }
    if (acc != 0.0) q[o++] = acc;
    n = o;
  }
  BFM_HD int sign() const { return n == 0 ? 0 : (q[n - 1] > 0.0 ? 1 : -1); }
  BFM_HD double approx() const {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += q[i];
    return s;
  }
};

// Sign of (sum a[0..na) - sum b[0..nb)), exact. na + nb <= 24. (Out of line
// on the device: reached only when two candidates need an exact compare.)
#if defined(__CUDACC__)
static __host__ __device__ __noinline__
#else
inline
#endif
int sign_diff(const double* a, int na, const double* b, int nb) {
  Exp<24> e;
  e.clear();
  for (int i = 0; i < na; ++i) e.grow(a[i]);
  for (int i = 0; i < nb; ++i) e.grow(-b[i]);
  return e.sign();
}

// Slow exact round-down of a sum of m <= 16 doubles (rare: kept out of line
// on the device so the kernels' hot code stays small).
#if defined(__CUDACC__)
static __host__ __device__ __noinline__
#else
inline
#endif
double round_down_slow(const double* t, int m) {
  Exp<16> e;
  e.clear();
  for (int i = 0; i < m; ++i) e.grow(t[i]);
  if (e.sign() == 0) return 0.0;
  double d = e.approx();
  // Adjust d until d <= value < next_up(d).
  for (int guard = 0; guard < 64; ++guard) {
    Exp<17> f;
    f.clear();
    for (int i = 0; i < e.n; ++i) f.grow(e.q[i]);
    f.grow(-d);
    if (f.sign() < 0) {
      d = next_down(d);
      continue;
    }
    const double up = next_up(d);
    Exp<17> g;
    g.clear();
    for (int i = 0; i < e.n; ++i) g.grow(e.q[i]);
    g.grow(-up);
    if (g.sign() >= 0) {
      d = up;
      continue;
    }
    break;
  }
  return d == 0.0 ? 0.0 : d;
}

// Largest double <= t[0] + ... + t[m-1] (exact), -0 -> +0. Certified
// double-double fast path; falls back to the expansion path.
BFM_HD double round_down_sum(const double* t, int m) {
  double s = t[0];
  double E = 0.0, absE = 0.0;
  for (int i = 1; i < m; ++i) {
    double ns, e;
    two_sum(s, t[i], ns, e);
    s = ns;
    E += e;
    absE += fabs(e);
  }
  if (absE == 0.0) return s == 0.0 ? 0.0 : s;  // value == s exactly
  double S2, r1;
  two_sum(s, E, S2, r1);
  const double bound = (2.0 * m) * 1.1102230246251565e-16 * absE;
  if (fabs(r1) > bound) {
    const double r = r1 < 0.0 ? next_down(S2) : S2;
    return r == 0.0 ? 0.0 : r;
  }
  return round_down_slow(t, m);
}

// RD(a + b) for two doubles.
BFM_HD double round_down2(double a, double b) {
  double s, e;
  two_sum(a, b, s, e);
  const double r = e < 0.0 ? next_down(s) : s;
  return r == 0.0 ? 0.0 : r;
}

}  // namespace bfmx
