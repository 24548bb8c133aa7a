// Shared device/host definitions for the sm_100a BFM kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "dct_line.h"

namespace bfmgpu {

// Thrown by host launchers; the C ABI maps it to BFM_ERR_CUDA.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define BFM_CUDA(call) ::bfmgpu::cuda_check((call), #call)
#define BFM_LAUNCH_CHECK(what) ::bfmgpu::cuda_check(cudaGetLastError(), what)

// Geometry of a cell-centred grid on [0,1]^d, row-major, last axis fastest
// (reference grid.hpp:17-84). Coordinates are (i + 0.5) * h with h = 1.0/n
// evaluated exactly as grid.hpp:27,69.
struct GridDesc {
  int d = 0;
  int n[3] = {1, 1, 1};
  long stride[3] = {0, 0, 0};
  long size = 0;
  double h[3] = {1.0, 1.0, 1.0};
  double vol = 1.0;  // cell volume, product of h in axis order (grid.hpp:71)
};

inline GridDesc make_grid(int d, const int* ext) {
  GridDesc g;
  g.d = d;
  g.size = 1;
  g.vol = 1.0;
  for (int a = 0; a < d; ++a) {
    g.n[a] = ext[a];
    g.h[a] = 1.0 / ext[a];
    g.size *= ext[a];
    g.vol *= g.h[a];
  }
  g.stride[d - 1] = 1;
  for (int a = d - 2; a >= 0; --a) g.stride[a] = g.stride[a + 1] * g.n[a + 1];
  return g;
}

BFM_HD double coord(double h, int i) { return (static_cast<double>(i) + 0.5) * h; }

// Device allocations come from the device's stream-ordered pool with an
// unbounded release threshold: creating and destroying solvers/workspaces
// (hundreds of MB of fields, sort and gather buffers) reuses reserved memory
// instead of paying cudaMalloc/cudaFree page mapping each time.
cudaError_t dev_malloc_bytes(void** p, size_t n);
void dev_free(void* p);
template <class T>
inline cudaError_t dmalloc(T** p, size_t n) {
  return dev_malloc_bytes(reinterpret_cast<void**>(p), n);
}
inline void dfree(const void* p) { dev_free(const_cast<void*>(p)); }

// Kernel-launch counter for the "gpu_launches" evidence in bench.py.
struct LaunchCounter {
  long count = 0;
  void add(long k = 1) { count += k; }
};

}  // namespace bfmgpu
