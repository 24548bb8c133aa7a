// Exact c-transform for separable power costs c(x, y) = sum_a |y_a - x_a|^p_a / p_a,
// p_a > 1 (reference cost.hpp:24-48, generic path of transforms.hpp:335-427).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace bfmgpu {

struct CtPowAxis {
  int n;
  long stride;
  const double* Tt;  // [n * n] axis cost, transposed: Tt[j * n + k] = axis_cost(y_j - x_k)
  double tmax;       // max |entry|
};

struct CtPowPass {
  int d, a, last;
  long nlines;
  int tpl, lpc, strided;
  CtPowAxis ax[3];
  const double* phi;
  const uint32_t* state_in;  // argmin chain of the previous passes (a > 0)
  uint32_t* state_out;       // non-last passes
  double* out;               // last pass
  int line_bytes;
};

class CtPowerPlan {
 public:
  CtPowerPlan() = default;
  ~CtPowerPlan();
  CtPowerPlan(const CtPowerPlan&) = delete;
  CtPowerPlan& operator=(const CtPowerPlan&) = delete;
  // exponents[a] > 1 per axis (2 allowed: that axis then costs 0.5*d*d, as in
  // cost.hpp:36-40). Axis extents up to 2048 (dense per-axis cost tables).
  void init(const GridDesc& g, const double* exponents);
  // out = phi^c rounded toward -inf, bit for bit the reference's generic path.
  void run(const double* d_phi, double* d_out, cudaStream_t stream, LaunchCounter* lc);

 private:
  GridDesc g_;
  CtPowPass pass_[3] = {};
  double* tables_[3] = {nullptr, nullptr, nullptr};
  uint32_t* state_[2] = {nullptr, nullptr};
};

// cost.hpp:36-40 on the host (std::pow, the reference's own libm call).
double power_axis_cost(double p, double delta);

}  // namespace bfmgpu
