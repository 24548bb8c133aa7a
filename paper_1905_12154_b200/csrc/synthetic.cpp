// Seeded synthetic densities of BASELINE.json configs C1-C4 (SURVEY §8(d)
// "Synthetic inputs (shared generator)"). Host-only input generation, not part
// of the solve path: it lives in the library so that the Python bench, the
// C++ drivers and the oracle-side golden scripts all regenerate the identical
// float64 arrays from (config, n, seed).
//
// Generator contract:
//  * RNG std::mt19937_64(seed); a uniform on [a, b) is a + (b - a) * u with
//    u = (rng() >> 11) * 2^-53 (no libstdc++ distribution objects);
//  * draws object by object in index order, fields in the order listed below;
//  * samples at cell centres (i + 0.5) * fl(1/n) (grid.hpp:27,69);
//  * "Gaussian" = unit-peak exp(-d2 / (2 s^2)) with d2 = sum_a (x_a - c_a)^2
//    in axis order, summed over the objects in index order from 0.0;
//  * indicators use the reference's closed cell-centre membership
//    (bfm_builtin_density, io.hpp:407-420);
//  * every density is normalised with the reference's Kahan mass
//    (bfm_normalize, grid.hpp:151-164).
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bfm_b200.h"

namespace {

struct Uniform {
  std::mt19937_64 rng;
  explicit Uniform(uint64_t seed) : rng(seed) {}
  double u() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
  double operator()(double a, double b) { return a + (b - a) * u(); }
};

struct Gauss {
  double c[3];
  double s;
};

double coord(int i, int n) { return (i + 0.5) * (1.0 / n); }

// Parallel over axis-0 planes; each node's value depends on that node only, so
// the result does not depend on the thread count.
template <class F>
void for_planes(int n0, F f) {
  unsigned t = std::thread::hardware_concurrency();
  if (t == 0) t = 1;
  if (t > 32) t = 32;
  if (static_cast<int>(t) > n0) t = n0;
  std::vector<std::thread> pool;
  for (unsigned k = 0; k < t; ++k)
    pool.emplace_back([=] {
      for (int i0 = static_cast<int>(k); i0 < n0; i0 += static_cast<int>(t)) f(i0);
    });
  for (auto& th : pool) th.join();
}

void gauss_sum(int d, int n, const std::vector<Gauss>& gs, double* out) {
  const long plane = d == 3 ? static_cast<long>(n) * n : n;
  for_planes(n, [&](int i0) {
    double* row = out + i0 * plane;
    const int n2 = d == 3 ? n : 1;
    long lin = 0;
    for (int i1 = 0; i1 < n; ++i1)
      for (int i2 = 0; i2 < n2; ++i2, ++lin) {
        const double x[3] = {coord(i0, n), coord(i1, n), d == 3 ? coord(i2, n) : 0.0};
        double v = 0.0;
        for (const Gauss& g : gs) {
          double d2 = 0.0;
          for (int a = 0; a < d; ++a) {
            const double dl = x[a] - g.c[a];
            d2 += dl * dl;
          }
          v += std::exp(-d2 / (2.0 * g.s * g.s));
        }
        row[lin] = v;
      }
  });
}

std::vector<Gauss> draw_gauss(Uniform& U, int d, int k, double c_lo, double c_hi, double s_lo,
                              double s_hi) {
  std::vector<Gauss> gs(k);
  for (Gauss& g : gs) {
    for (int a = 0; a < d; ++a) g.c[a] = U(c_lo, c_hi);
    for (int a = d; a < 3; ++a) g.c[a] = 0.0;
    g.s = U(s_lo, s_hi);
  }
  return gs;
}

struct Failed {  // a library call failed; its status and message are kept
  int code;
  std::string msg;
};

void check(int rc) {
  if (rc != BFM_OK) throw Failed{rc, bfm_last_error()};
}

void normalize_into(int d, int n, const std::vector<double>& raw, double* out) {
  const int ext[3] = {n, n, n};
  check(bfm_normalize(d, ext, raw.data(), out));
}

// C3 recipe for one density: 16 Gaussians (centre ~U[0,1]^2, s ~U[0.01,0.1]),
// then a Bernoulli(0.5) mask over 64x64 blocks of (n/64)^2 cells each, drawn
// block by block in row-major order (block zeroed when u < 0.5).
void masked_gauss(Uniform& U, int n, double* out) {
  const std::vector<Gauss> gs = draw_gauss(U, 2, 16, 0.0, 1.0, 0.01, 0.1);
  const int nb = n >= 64 ? 64 : 1;
  std::vector<char> zero(static_cast<size_t>(nb) * nb);
  for (auto& z : zero) z = U.u() < 0.5;
  std::vector<double> raw(static_cast<size_t>(n) * n);
  gauss_sum(2, n, gs, raw.data());
  const int bs = n / nb;
  for (int i0 = 0; i0 < n; ++i0)
    for (int i1 = 0; i1 < n; ++i1)
      if (zero[static_cast<size_t>(i0 / bs) * nb + i1 / bs]) raw[static_cast<size_t>(i0) * n + i1] = 0.0;
  normalize_into(2, n, raw, out);
}

void make(int config, int n, uint64_t seed, double* mu, double* nu) {
  Uniform U(seed);
  const int ext[3] = {n, n, n};
  switch (config) {
    case 1: {  // 3 Gaussians (centre ~U[0.2,0.8]^2, s ~U[0.05,0.15]) vs disc
      const auto gs = draw_gauss(U, 2, 3, 0.2, 0.8, 0.05, 0.15);
      std::vector<double> raw(static_cast<size_t>(n) * n);
      gauss_sum(2, n, gs, raw.data());
      normalize_into(2, n, raw, mu);
      check(bfm_builtin_density(2, ext, "disc:0.5,0.5,0.3", raw.data()));
      normalize_into(2, n, raw, nu);
      return;
    }
    case 2: {
      // mu: union of 5 rectangles; per rectangle w, h ~U[0.1,0.4], then the
      // lower-left corner x0 ~U[0,1-w], y0 ~U[0,1-h]; closed membership
      // x0 <= x <= x0+w on axis 0 and y0 <= y <= y0+h on axis 1.
      std::vector<double> raw(static_cast<size_t>(n) * n, 0.0);
      for (int r = 0; r < 5; ++r) {
        const double w = U(0.1, 0.4), h = U(0.1, 0.4);
        const double x0 = U(0.0, 1.0 - w), y0 = U(0.0, 1.0 - h);
        for (int i0 = 0; i0 < n; ++i0) {
          const double x = coord(i0, n);
          if (!(x >= x0 && x <= x0 + w)) continue;
          for (int i1 = 0; i1 < n; ++i1) {
            const double y = coord(i1, n);
            if (y >= y0 && y <= y0 + h) raw[static_cast<size_t>(i0) * n + i1] = 1.0;
          }
        }
      }
      normalize_into(2, n, raw, mu);
      // nu: 8 Gaussians (centre ~U[0.1,0.9]^2, s ~U[0.02,0.1]), then the annulus
      // centre c ~U[0.45,0.55]^2; zero where sqrt(d2) < 0.15 or > 0.45.
      const auto gs = draw_gauss(U, 2, 8, 0.1, 0.9, 0.02, 0.1);
      const double ca0 = U(0.45, 0.55), ca1 = U(0.45, 0.55);
      gauss_sum(2, n, gs, raw.data());
      for (int i0 = 0; i0 < n; ++i0)
        for (int i1 = 0; i1 < n; ++i1) {
          const double d0 = coord(i0, n) - ca0, d1 = coord(i1, n) - ca1;
          const double r = std::sqrt(d0 * d0 + d1 * d1);
          if (r < 0.15 || r > 0.45) raw[static_cast<size_t>(i0) * n + i1] = 0.0;
        }
      normalize_into(2, n, raw, nu);
      return;
    }
    case 3:
      masked_gauss(U, n, mu);
      masked_gauss(U, n, nu);
      return;
    case 4: {  // 6 3-D Gaussians (centre ~U[0,1]^3, s ~U[0.03,0.12]) vs ball
      const auto gs = draw_gauss(U, 3, 6, 0.0, 1.0, 0.03, 0.12);
      std::vector<double> raw(static_cast<size_t>(n) * n * n);
      gauss_sum(3, n, gs, raw.data());
      normalize_into(3, n, raw, mu);
      check(bfm_builtin_density(3, ext, "ball:0.5,0.5,0.5,0.3", raw.data()));
      normalize_into(3, n, raw, nu);
      return;
    }
    default:
      throw std::invalid_argument("synthetic: config must be 1..4");
  }
}

}  // namespace

namespace bfmgpu {
// Called by bfm_synthetic_densities (capi.cu): returns a BFM status and, on
// failure, its message.
int synthetic_densities(int config, int n, uint64_t seed, double* mu, double* nu, std::string& msg) {
  try {
    if (n < 2 || !mu || !nu) throw std::invalid_argument("synthetic: need n >= 2 and output buffers");
    if (config == 3 && n % 64 != 0 && n >= 64)
      throw std::invalid_argument("synthetic: C3 needs n divisible by 64 (64x64 mask blocks)");
    make(config, n, seed, mu, nu);
    return BFM_OK;
  } catch (const Failed& f) {
    msg = f.msg;
    return f.code;
  } catch (const std::invalid_argument& e) {
    msg = e.what();
    return BFM_ERR_INVALID_ARGUMENT;
  }
}
}  // namespace bfmgpu
