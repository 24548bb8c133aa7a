// Prototype (not product): one thread per grid line, sequential fp64 lower
// hull + monotone query sweep, to size the one-thread-per-line design on C4
// (384^3) lines. Approximate (no exactness); timing only.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

template <int NMAX>
__global__ void seq_hull(const double* __restrict__ phi, int n, long nlines, long lstride_outer,
                         long inner_count, long estride, double h, int* __restrict__ out) {
  const long L = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (L >= nlines) return;
  const long inner = L % inner_count, outer = L / inner_count;
  const long base = outer * lstride_outer + inner;
  short stk[NMAX];
  double sy[NMAX], sf[NMAX];
  int sz = 0;
  for (int j = 0; j < n; ++j) {
    const double y = (j + 0.5) * h;
    const double f = 0.5 * y * y - __ldg(phi + base + j * estride);
    while (sz >= 2) {
      const double d = (sf[sz - 1] - sf[sz - 2]) * (y - sy[sz - 1]) - (f - sf[sz - 1]) * (sy[sz - 1] - sy[sz - 2]);
      if (d < 0.0) break;  // strict corner
      --sz;
    }
    stk[sz] = (short)j;
    sy[sz] = y;
    sf[sz] = f;
    ++sz;
  }
  int i = 0;
  for (int k = 0; k < n; ++k) {
    const double x = (k + 0.5) * h;
    while (i + 1 < sz && sf[i + 1] - x * sy[i + 1] <= sf[i] - x * sy[i]) ++i;
    out[base + k * estride] = stk[i];
  }
}

int main(int argc, char** argv) {
  const int n = 384;
  const long N = (long)n * n * n;
  std::vector<double> h(N);
  for (long i = 0; i < N; ++i) {
    const long a = i / ((long)n * n), b = (i / n) % n, c = i % n;
    const double x = (a + 0.5) / n, y = (b + 0.5) / n, z = (c + 0.5) / n;
    h[i] = 0.5 * (x * x + y * y + z * z) + 0.05 * std::cos(6.0 * x + 2.0 * y) * std::sin(5.0 * z + 1.0) + 0.02 * std::sin(37.0 * x * y);
  }
  double* dphi; int* dout;
  cudaMalloc(&dphi, N * 8); cudaMalloc(&dout, N * 4);
  cudaMemcpy(dphi, h.data(), N * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const long nl = (long)n * n;
  // pass along axis 0 (strided: inner = n*n columns), axis 1, axis 2 (contiguous)
  struct P { long lso, inner, es; const char* name; } ps[3] = {
    {N, (long)n * n, (long)n * n, "axis0 (strided n^2)"},
    {(long)n * n, n, n, "axis1 (strided n)"},
    {n, 1, 1, "axis2 (contiguous)"}};
  for (int blk : {64, 128, 256}) {
    for (auto& p : ps) {
      for (int w = 0; w < 2; ++w) seq_hull<384><<<(nl + blk - 1) / blk, blk>>>(dphi, n, nl, p.lso, p.inner, p.es, 1.0 / n, dout);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) seq_hull<384><<<(nl + blk - 1) / blk, blk>>>(dphi, n, nl, p.lso, p.inner, p.es, 1.0 / n, dout);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("block %d %s: %.3f ms per pass (%s)\n", blk, p.name, ms / 5, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
