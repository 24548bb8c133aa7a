// Pooled device allocations (see common.cuh dmalloc / dfree).
#include <cstdint>
#include <mutex>

#include "common.cuh"

namespace bfmgpu {

namespace {
std::mutex g_pool_mu;
bool g_pool_ready[64] = {};

void ensure_pool(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 0 || dev >= 64 || g_pool_ready[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  g_pool_ready[dev] = true;
}
}  // namespace

cudaError_t dev_malloc_bytes(void** p, size_t n) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  ensure_pool(dev);
  if (n == 0) n = 16;
  // ordered on the legacy stream, then completed: the block is usable from
  // any stream afterwards
  e = cudaMallocAsync(p, n, static_cast<cudaStream_t>(0));
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(static_cast<cudaStream_t>(0));
}

void dev_free(void* p) {
  if (!p) return;
  // work on non-blocking streams may still read the block: finish it first
  cudaDeviceSynchronize();
  cudaFreeAsync(p, static_cast<cudaStream_t>(0));
  cudaGetLastError();
}

}  // namespace bfmgpu
