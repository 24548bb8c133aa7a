// Neumann Poisson solve (-Laplacian)^{-1} by batched DCT-II / DCT-III on
// sm_100a (reference poisson.hpp:42-73 plan, :87-106 solve_neumann).
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "common.cuh"
#include "dct_plan_host.h"

namespace bfmgpu {

struct PoisAxisCfg {
  bfmdct::LinePlan plan;  // device table pointers
  int n, tpl, lpc, strided, line_bytes;
  int cslots;  // complex slots per line buffer (m rounded up to 8 for the swizzle)
  long stride, nlines;
};

class PoissonPlan {
 public:
  PoissonPlan() = default;
  ~PoissonPlan();
  PoissonPlan(const PoissonPlan&) = delete;
  PoissonPlan& operator=(const PoissonPlan&) = delete;

  void init(const GridDesc& g);
  // out = (-Lap)^{-1}(rhs - mean) exactly as the reference's FFTW path with
  // the shared DCT (bitwise equal to oracle/_ref). rhs and out may alias.
  void solve(const double* d_rhs, double* d_out, cudaStream_t stream, LaunchCounter* lc);

 private:
  GridDesc g_;
  std::unique_ptr<bfmdct::HostLinePlan> host_[3];
  PoisAxisCfg cfg_[3] = {};
  void* tables_[3] = {nullptr, nullptr, nullptr};
  double* lam_[3] = {nullptr, nullptr, nullptr};
  double* tmp_ = nullptr;
  double scale_ = 1.0;
};

}  // namespace bfmgpu
