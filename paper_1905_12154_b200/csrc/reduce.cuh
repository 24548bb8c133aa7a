// Deterministic fp64 reductions and elementwise kernels (reference
// grid.hpp:124-133,171-183 Kahan integrals, solver.hpp:240,255-258,282-284,
// :341-343, pushforward.hpp:181-196).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace bfmgpu {

constexpr int kRedSlots = 64;
// results[kBoundSlot + slot]: error bound of results[slot] against the
// reference's sequential Kahan evaluation (dot / sum only).
constexpr int kBoundSlot = 32;

class Reducer {
 public:
  Reducer() = default;
  ~Reducer();
  Reducer(const Reducer&) = delete;
  Reducer& operator=(const Reducer&) = delete;
  void init();
  // results[slot] = (sum_i fl(a1_i*b1_i)) * vol [+ (sum_i fl(a2_i*b2_i)) * vol]
  // (a2 may be null). Sums are double-double accurate (one final rounding).
  void dot(const double* a1, const double* b1, const double* a2, const double* b2, long n,
           double vol, int slot, cudaStream_t s, LaunchCounter* lc);
  // Unscaled double-double partial sums for a multi-GPU rank:
  // results[slot..slot+3] = (hi1, lo1, hi2, lo2) of sum fl(a1*b1), sum fl(a2*b2).
  void dot_raw(const double* a1, const double* b1, const double* a2, const double* b2, long n,
               int slot, cudaStream_t s, LaunchCounter* lc);
  // results[slot..slot+1] = (hi, lo) of sum_{m != 0} fl(c * m) (see primal).
  void primal_raw(const double* disp, const double* mu, int d, long n, int slot, cudaStream_t s,
                  LaunchCounter* lc);
  // results[slot] = (sum_i a_i) * vol
  void sum(const double* a, long n, double vol, int slot, cudaStream_t s, LaunchCounter* lc);
  // results[slot] = max_i a_i (a_i >= 0 expected); results[slot+1] = 1 if any
  // non-finite, results[slot+2] = 1 if any negative.
  void scan_density(const double* a, long n, int slot, cudaStream_t s, LaunchCounter* lc);
  // results[slot] = vol * sum_{m != 0} fl(c * m), c = sum_a 0.5*d_a*d_a
  // exponents (optional): a power cost's p_a per axis (cost.hpp:36-40)
  void primal(const double* disp, const double* mu, int d, long n, double vol, int slot,
              cudaStream_t s, LaunchCounter* lc, const double* exponents = nullptr);
  double* device_results() { return results_; }
  // Copies slots [0, count) to host (synchronises the stream).
  void fetch(double* host, int count, cudaStream_t s);

 private:
  double* partials_ = nullptr;
  double* results_ = nullptr;
  double* pinned_ = nullptr;
  int blocks_ = 0;
};

void axpy(double* u, double s, const double* dir, long n, cudaStream_t st, LaunchCounter* lc);
// u[i] += (*d_s) * dir[i], the step size read from device memory (graph replays)
void axpy_dev(double* u, const double* d_s, const double* dir, long n, cudaStream_t st,
              LaunchCounter* lc);
// u[i] += delta
void add_scalar(double* u, double delta, long n, cudaStream_t st, LaunchCounter* lc);

}  // namespace bfmgpu
