// Transport map + density pushforward on sm_100a (reference pushforward.hpp).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "radix_sort.cuh"

namespace bfmgpu {

class PushforwardPlan {
 public:
  PushforwardPlan() = default;
  ~PushforwardPlan();
  PushforwardPlan(const PushforwardPlan&) = delete;
  PushforwardPlan& operator=(const PushforwardPlan&) = delete;

  void init(const GridDesc& g);

  // out = target - T#source with T = x - grad(u) (map_from_conjugate,
  // pushforward.hpp:70-91) — or, if target == nullptr, out = T#source.
  // disp_out (d*N, may be null) receives the displacement field.
  void from_potential(const double* d_u, const double* d_source, const double* d_target,
                      double* d_out, double* d_disp_out, cudaStream_t stream, LaunchCounter* lc);
  // rho = splat of source at x + scale*disp (pushforward.hpp:141-172).
  void from_displacement(const double* d_disp, double scale, const double* d_source,
                         double* d_rho, cudaStream_t stream, LaunchCounter* lc);
  // Map only (displacements), no splat.
  void map_only(const double* d_u, double* d_disp, cudaStream_t stream, LaunchCounter* lc);

 private:
  void bin_and_gather(const double* d_source, const double* d_target, double* d_out,
                      cudaStream_t stream, LaunchCounter* lc);
  GridDesc g_;
  uint32_t* key_ = nullptr;  // [N] lo-corner cell of each source (N = no mass)
  uint8_t* cmask_ = nullptr; // [N] axes on which the source is clamped (lo == hi)
  double* w_ = nullptr;      // [d*N] upper-node weight per axis
  int* off_ = nullptr;       // [N+1] first sorted position of each cell
  int* end_ = nullptr;       // [N+1] one past the last
  int* heavy_ = nullptr;     // [N] targets with long deposit lists
  unsigned long long* nheavy_ = nullptr;  // [0] heavy count, [1] buffer fill
  double* hbuf_ = nullptr;   // [2^d * N] merged heavy deposits
  RadixSorter sorter_;
  int key_bits_ = 0;
  int med_blocks_ = 1;       // medium-gather CTAs (each warp owns a kMedium slice of hbuf_)
};

}  // namespace bfmgpu
