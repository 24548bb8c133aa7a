// ORACLE TEST INFRASTRUCTURE — not part of the product.
//
// FFTW-subset shim so the reference's own headers
// (/root/reference/proj/include/bfm/poisson.hpp:3,22-25,45-51,68-77,91,104,
// 170-171) compile and run in this image, where FFTW3 is not installed (it is
// an unpinned find_library dependency, proj/CMakeLists.txt:11-12). Provides the
// nine symbols poisson.hpp uses: fftw_plan, fftw_r2r_kind, FFTW_REDFT10,
// FFTW_REDFT01, FFTW_ESTIMATE, fftw_plan_r2r, fftw_execute_r2r,
// fftw_destroy_plan, fftw_malloc, fftw_free.
//
// Semantics follow FFTW's documented unnormalised r2r kinds:
//   REDFT10 (DCT-II):  Y_k = 2 sum_j x_j cos(pi k (2j+1) / 2n)
//   REDFT01 (DCT-III): Y_k = x_0 + 2 sum_{j>=1} x_j cos(pi j (2k+1) / 2n)
// applied separably along every axis of a row-major rank-d array. The per-line
// arithmetic is the product's shared routine (paper_1905_12154_b200/csrc/
// dct_line.h), so the reference built against this shim and the sm_100a
// Poisson kernels produce bitwise-identical solves. Axis order is fixed:
// REDFT10 plans run axes d-1 .. 0, REDFT01 plans run axes 0 .. d-1 (the device
// path fuses the adjacent axis-0 transforms around the spectral divide).
// FFTW bitwise output is therefore NOT reproduced ("parity unpinned" against
// real FFTW); the reference's Poisson property tests pin the semantics.
#pragma once

#include <cstddef>
#include <cstdlib>
#include <memory>
#include <vector>

#include "../paper_1905_12154_b200/csrc/dct_plan_host.h"

typedef enum { FFTW_REDFT01 = 4, FFTW_REDFT10 = 5 } fftw_r2r_kind;
#define FFTW_ESTIMATE (1U << 6)

struct bfm_shim_fftw_plan {
  int rank = 0;
  int n[3] = {1, 1, 1};
  bool forward = true;  // REDFT10 on every axis
  std::unique_ptr<bfmdct::HostLinePlan> axis[3];
  std::vector<bfmdct::cplx> scratch;
};
typedef bfm_shim_fftw_plan* fftw_plan;

inline void* fftw_malloc(std::size_t bytes) {
  void* p = nullptr;
  if (posix_memalign(&p, 64, bytes == 0 ? 64 : bytes) != 0) return nullptr;
  return p;
}

inline void fftw_free(void* p) { std::free(p); }

inline fftw_plan fftw_plan_r2r(int rank, const int* n, double* /*in*/, double* /*out*/,
                               const fftw_r2r_kind* kind, unsigned /*flags*/) {
  if (rank < 1 || rank > 3) return nullptr;
  for (int a = 1; a < rank; ++a)
    if (kind[a] != kind[0]) return nullptr;  // mixed kinds are never planned
  auto* p = new bfm_shim_fftw_plan;
  p->rank = rank;
  p->forward = kind[0] == FFTW_REDFT10;
  int maxn = 1;
  for (int a = 0; a < rank; ++a) {
    p->n[a] = n[a];
    p->axis[a].reset(new bfmdct::HostLinePlan);
    try {
      p->axis[a]->build(n[a]);
    } catch (...) {
      delete p;
      return nullptr;
    }
    if (n[a] > maxn) maxn = n[a];
  }
  p->scratch.resize(static_cast<std::size_t>(maxn) + 1);
  return p;
}

inline void fftw_execute_r2r(const fftw_plan p, double* in, double* out) {
  const int d = p->rank;
  std::size_t total = 1;
  for (int a = 0; a < d; ++a) total *= static_cast<std::size_t>(p->n[a]);
  if (in != out)
    for (std::size_t i = 0; i < total; ++i) out[i] = in[i];
  long stride[3] = {1, 1, 1};
  for (int a = d - 2; a >= 0; --a) stride[a] = stride[a + 1] * p->n[a + 1];
  for (int step = 0; step < d; ++step) {
    const int a = p->forward ? d - 1 - step : step;
    const bfmdct::LinePlan& lp = p->axis[a]->plan;
    const long s = stride[a];
    const long len = p->n[a];
    // Every line along axis a: base offsets enumerate the other axes.
    const long outer = static_cast<long>(total) / (len * s);
    for (long o = 0; o < outer; ++o)
      for (long i = 0; i < s; ++i) {
        double* line = out + o * len * s + i;
        if (p->forward)
          bfmdct::dct2_line_cpu(lp, line, s, p->scratch.data());
        else
          bfmdct::dct3_line_cpu(lp, line, s, p->scratch.data());
      }
  }
}

inline void fftw_destroy_plan(fftw_plan p) { delete p; }
