// Host-side construction of the per-axis DCT line plans (twiddle tables,
// digit-reversal map, radix schedule). Shared by the device Poisson solver
// (which uploads these exact tables) and the oracle FFTW shim, so both sides
// consume bit-identical constants. See dct_line.h for the algorithm.
#pragma once

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "dct_line.h"

namespace bfmdct {

// Largest extent handled by the direct O(n^2) form (its table is n*n doubles).
constexpr int kNaiveMaxN = 2048;

struct HostLinePlan {
  LinePlan plan;  // table pointers refer to the vectors below
  std::vector<cplx> wm, cs, wn;
  std::vector<int> rev;
  std::vector<double> cosmat;

  HostLinePlan() = default;
  HostLinePlan(const HostLinePlan&) = delete;
  HostLinePlan& operator=(const HostLinePlan&) = delete;

  void build(int n) {
    constexpr double kPi = 3.14159265358979323846;
    plan = LinePlan{};
    plan.n = n;
    int m = n / 2;
    bool smooth = (n % 2 == 0) && m >= 1;
    int rest = m;
    while (smooth && rest % 2 == 0) rest /= 2;
    while (smooth && rest % 3 == 0) rest /= 3;
    smooth = smooth && rest == 1;
    if (smooth) {
      plan.kind = kFft;
      plan.m = m;
      // Radix schedule: 4s, then a 2 if needed, then 3s.
      int a = m, ns = 0;
      int twos = 0, threes = 0;
      while (a % 2 == 0) { a /= 2; ++twos; }
      while (a % 3 == 0) { a /= 3; ++threes; }
      for (int i = 0; i < twos / 2; ++i) plan.radix[ns++] = 4;
      if (twos % 2) plan.radix[ns++] = 2;
      for (int i = 0; i < threes; ++i) plan.radix[ns++] = 3;
      plan.nstages = ns;
      int L = m;
      for (int s = 0; s < ns; ++s) {
        plan.span[s] = L;
        L /= plan.radix[s];
      }
      wm.resize(m);
      for (int j = 0; j < m; ++j) {
        const double t = 2.0 * kPi * static_cast<double>(j) / static_cast<double>(m);
        wm[j] = cplx{std::cos(t), -std::sin(t)};
      }
      rev.resize(m);
      for (int k = 0; k < m; ++k) {
        int pos = 0, kk = k, LL = m;
        for (int s = 0; s < ns; ++s) {
          const int r = plan.radix[s];
          LL /= r;
          pos += (kk % r) * LL;
          kk /= r;
        }
        rev[k] = pos;
      }
      cs.resize(m + 1);
      wn.resize(m + 1);
      for (int k = 0; k <= m; ++k) {
        const double t = kPi * static_cast<double>(k) / (2.0 * n);
        cs[k] = cplx{std::cos(t), std::sin(t)};
        const double u = 2.0 * kPi * static_cast<double>(k) / static_cast<double>(n);
        wn[k] = cplx{std::cos(u), std::sin(u)};
      }
      plan.wm = wm.data();
      plan.rev = rev.data();
      plan.cs = cs.data();
      plan.wn = wn.data();
    } else {
      if (n > kNaiveMaxN)
        throw std::invalid_argument("DCT: extent " + std::to_string(n) +
                                    " is neither 2*(2^a 3^b) nor <= 2048");
      plan.kind = kNaive;
      cosmat.resize(static_cast<size_t>(n) * n);
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
          cosmat[static_cast<size_t>(k) * n + j] =
              std::cos(kPi * static_cast<double>(k) * (2.0 * j + 1.0) / (2.0 * n));
      plan.cosmat = cosmat.data();
    }
  }
};

// Sequential single-line transforms (CPU). x is read and y written with the
// given stride; x and y may alias. scratch holds >= max(m, n) complex values.
inline void dct2_line_cpu(const LinePlan& p, double* x, long stride, cplx* scratch) {
  if (p.kind == kFft) {
    for (int q = 0; q < p.m; ++q) dct2_pack(p, x, stride, scratch, q);
    for (int s = 0; s < p.nstages; ++s)
      for (int b = 0, nb = stage_butterflies(p, s); b < nb; ++b)
        fft_butterfly(p, s, b, scratch, false);
    for (int k = 0; k <= p.m; ++k) dct2_unpack(p, scratch, x, stride, k);
  } else {
    double* tmp = reinterpret_cast<double*>(scratch);
    for (int j = 0; j < p.n; ++j) tmp[j] = x[static_cast<long>(j) * stride];
    for (int k = 0; k < p.n; ++k) x[static_cast<long>(k) * stride] = dct2_naive(p, tmp, 1, k);
  }
}

inline void dct3_line_cpu(const LinePlan& p, double* x, long stride, cplx* scratch) {
  if (p.kind == kFft) {
    for (int k = 0; k < p.m; ++k) dct3_pre(p, x, stride, scratch, k);
    for (int s = 0; s < p.nstages; ++s)
      for (int b = 0, nb = stage_butterflies(p, s); b < nb; ++b)
        fft_butterfly(p, s, b, scratch, true);
    for (int q = 0; q < p.m; ++q) dct3_post(p, scratch, x, stride, q);
  } else {
    double* tmp = reinterpret_cast<double*>(scratch);
    for (int j = 0; j < p.n; ++j) tmp[j] = x[static_cast<long>(j) * stride];
    for (int k = 0; k < p.n; ++k) x[static_cast<long>(k) * stride] = dct3_naive(p, tmp, 1, k);
  }
}

}  // namespace bfmdct
