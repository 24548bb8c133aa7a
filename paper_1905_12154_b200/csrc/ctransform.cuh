// Exact quadratic c-transform on sm_100a (reference transforms.hpp:396-432).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace bfmgpu {

struct CtAxis {
  int n;
  long stride;
  double h;
  int dyadic;          // 1: g(k,j) = 0.5 (x_k - y_j)^2 is an exact double
  const double4* G;    // else: [n*n] exact limbs (hi, mid, lo, 0) of hs(x_k)+hs(y_j)-x_k*y_j
};

struct CtPass {
  int d;
  int a;      // axis of this pass
  int last;   // 1 on the final pass (writes psi)
  long nlines;
  int tpl, C, lpc;
  int strided;
  CtAxis ax[3];
  const double* phi;
  const uint32_t* state_in;  // argmin chain of previous passes (a > 0)
  uint32_t* state_out;       // non-last passes
  double* out;               // last pass
  // shared-memory carve-up (bytes, per line)
  int off_fv, off_chain, off_hidx, off_H, off_flag, off_list, off_lohi, off_scal, line_bytes;
  // statistics (device counters, may be null): lines that needed exact resolution
  unsigned long long* slow_queries;
  unsigned long long* stats;  // optional diagnostics (env BFM_CT_STATS=1)
};

class CtPlan {
 public:
  CtPlan() = default;
  ~CtPlan();
  CtPlan(const CtPlan&) = delete;
  CtPlan& operator=(const CtPlan&) = delete;

  void init(const GridDesc& g);
  // out = phi^c (exactly rounded toward -inf). phi and out are device pointers
  // (may not alias). Enqueues g.d kernels on stream.
  void run(const double* d_phi, double* d_out, cudaStream_t stream, LaunchCounter* lc);
  unsigned long long slow_query_count();  // diagnostic (synchronous)
  void stats(unsigned long long* out8);     // diagnostic counters (synchronous)
  const GridDesc& grid() const { return g_; }

 private:
  GridDesc g_;
  CtAxis ax_[3] = {};
  double4* tables_[3] = {nullptr, nullptr, nullptr};
  uint32_t* state_[2] = {nullptr, nullptr};
  unsigned long long* slow_ = nullptr;
  unsigned long long* stats_ = nullptr;
  CtPass pass_[3] = {};
  bool ready_ = false;
  bool dyadic_ = false;
};

}  // namespace bfmgpu
