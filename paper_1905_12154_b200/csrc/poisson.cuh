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

  // Multi-GPU slab decomposition along axis 0: DCT-II along
  // axes d-1..1 on a row slab, transpose, [DCT-II axis 0, divide, DCT-III
  // axis 0] on a column slab (global columns col0 .. col0+ncols of the
  // flattened non-axis-0 index), transpose back, DCT-III axes 1..d-1.
  void init_slab_rows(const GridDesc& global, int nrows);
  void init_slab_cols(const GridDesc& global, long col0, int ncols);
  void rows_forward(const double* d_in, double* d_out, cudaStream_t stream, LaunchCounter* lc);
  void cols_fused(const double* d_in, double* d_out, cudaStream_t stream, LaunchCounter* lc);
  void rows_inverse(double* d_inout, cudaStream_t stream, LaunchCounter* lc);

 private:
  void setup(const GridDesc& loc, const GridDesc& global, long col0, int ab, int ae);
  void launch(int axis, int mode, const double* in, double* out, cudaStream_t stream,
              LaunchCounter* lc);
  GridDesc g_;   // grid the kernels walk
  GridDesc gg_;  // problem grid
  long col_off_ = 0;
  std::unique_ptr<bfmdct::HostLinePlan> host_[3];
  PoisAxisCfg cfg_[3] = {};
  void* tables_[3] = {nullptr, nullptr, nullptr};
  double* lam_[3] = {nullptr, nullptr, nullptr};
  double* tmp_ = nullptr;
  double scale_ = 1.0;
};

}  // namespace bfmgpu
