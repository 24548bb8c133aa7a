// Deterministic two-stage double-double reductions + elementwise kernels.
//
// The reference sums sequentially with Kahan compensation (grid.hpp:124-133).
// These reductions accumulate per thread in double-double (two_sum) and
// combine partials in a fixed tree, so results are run-to-run bitwise
// deterministic and within an ulp of the exact sum; they only feed scalar
// decisions (sigma rule, stopping tests), never a field.
#include <cmath>

#include "exact.cuh"
#include "reduce.cuh"
#include "pow_dd.h"

namespace bfmgpu {
namespace {

constexpr int kRedThreads = 256;
#ifndef BFM_RED_BLOCKS_PER_SM
#define BFM_RED_BLOCKS_PER_SM 4
#endif
#ifndef BFM_RED_UNROLL
#define BFM_RED_UNROLL 8
#endif
constexpr int kRedBlocks = 148 * BFM_RED_BLOCKS_PER_SM;
constexpr int kRedUnroll = BFM_RED_UNROLL;

struct DD {
  double s, c;
};

__device__ __forceinline__ void dd_add(DD& a, double x) {
  double s, e;
  bfmx::two_sum(a.s, x, s, e);
  a.s = s;
  a.c += e;
}
__device__ __forceinline__ DD dd_merge(DD a, DD b) {
  double s, e;
  bfmx::two_sum(a.s, b.s, s, e);
  return DD{s, (a.c + b.c) + e};
}

__device__ DD block_reduce(DD v) {
  __shared__ double ss[kRedThreads / 32], sc[kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    DD u{__shfl_down_sync(0xffffffffu, v.s, o), __shfl_down_sync(0xffffffffu, v.c, o)};
    v = dd_merge(v, u);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    ss[w] = v.s;
    sc[w] = v.c;
  }
  __syncthreads();
  DD r{0.0, 0.0};
  if (threadIdx.x == 0)
    for (int i = 0; i < kRedThreads / 32; ++i) r = dd_merge(r, DD{ss[i], sc[i]});
  __syncthreads();
  return r;
}

// mode 0: sum a*b ; 1: sum a ; 2: primal ; partial layout [pair][block][2]
struct RedArgs {
  const double* a1;
  const double* b1;
  const double* a2;
  const double* b2;
  long n;
  int mode;
  int d;
  double* partials;
  double pexp[3];  // primal: per-axis exponent of a power cost (0: quadratic axis)
};

// One element's terms (mode 2: 0 for massless nodes, which the sums skip;
// adding an exact 0 leaves a double-double unchanged).
template <int MODE>
__device__ __forceinline__ void red_terms(const RedArgs& A, long i, double& t1, double& t2) {
  t2 = 0.0;
  if (MODE == 0) {
    t1 = A.a1[i] * A.b1[i];
    if (A.a2) t2 = A.a2[i] * A.b2[i];
  } else if (MODE == 1) {
    t1 = A.a1[i];
  } else {
    const double m = A.b1[i];
    double c = 0.0;
    for (int a = 0; a < A.d; ++a) {
      const double dl = A.a1[a * A.n + i];
      // axis_cost (cost.hpp:36-40): 0.5 d^2, or |d|^p / p (correctly rounded pow)
      c += A.pexp[a] == 0.0 ? 0.5 * dl * dl : bfmpow::pow_cr(fabs(dl), A.pexp[a]) / A.pexp[a];
    }
    t1 = m == 0.0 ? 0.0 : c * m;
  }
}

__device__ double block_sum_plain(double v) {
  __shared__ double sa[kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sa[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kRedThreads / 32; ++i) r += sa[i];
  __syncthreads();
  return r;
}

// Besides the two double-double sums, every launch accumulates A = sum_i
// (|t1_i| + |t2_i|) in plain fp64 (a nonnegative sum: relative error <= n*u),
// from which the final kernel derives a rigorous bound on |our value - the
// reference's sequential Kahan value| (see red_final_kernel).
// One instantiation per mode (dot / sum / primal): the primal's pow path must
// not inflate the registers of the bandwidth-bound dot (80 regs and spills
// when they shared one kernel; red_partial 62 -> 165 us per C3 launch).
template <int MODE>
__global__ void __launch_bounds__(kRedThreads) red_partial_kernel(RedArgs A) {
  DD acc1{0.0, 0.0}, acc2{0.0, 0.0};
  double absum = 0.0;
  const long stride = static_cast<long>(gridDim.x) * kRedThreads;
  long i = blockIdx.x * static_cast<long>(kRedThreads) + threadIdx.x;
  // kRedUnroll elements per round, their loads in flight together (one per
  // round: ~2 TB/s; 4: C3 0.79 ms of reductions per iteration; 8: 0.74 ms,
  // C4 2.19 -> 1.99 ms); fixed per-thread order
  for (; i + (kRedUnroll - 1) * stride < A.n; i += kRedUnroll * stride) {
    double t1[kRedUnroll], t2[kRedUnroll];
#pragma unroll
    for (int u = 0; u < kRedUnroll; ++u) red_terms<MODE>(A, i + u * stride, t1[u], t2[u]);
#pragma unroll
    for (int u = 0; u < kRedUnroll; ++u) {
      dd_add(acc1, t1[u]);
      dd_add(acc2, t2[u]);
      absum += fabs(t1[u]) + fabs(t2[u]);
    }
  }
  for (; i < A.n; i += stride) {
    double t1, t2;
    red_terms<MODE>(A, i, t1, t2);
    dd_add(acc1, t1);
    dd_add(acc2, t2);
    absum += fabs(t1) + fabs(t2);
  }
  DD r1 = block_reduce(acc1);
  DD r2 = block_reduce(acc2);
  const double ab = block_sum_plain(absum);
  if (threadIdx.x == 0) {
    A.partials[2 * blockIdx.x] = r1.s;
    A.partials[2 * blockIdx.x + 1] = r1.c;
    A.partials[2 * (gridDim.x + blockIdx.x)] = r2.s;
    A.partials[2 * (gridDim.x + blockIdx.x) + 1] = r2.c;
    A.partials[4 * gridDim.x + blockIdx.x] = ab;
  }
}

// results[slot] = value; results[kBoundSlot + slot] = bound with
//   |value - reference value| <= bound,
// the reference value being fl(fl(K1*vol) + fl(K2*vol)) of sequential Kahan
// sums K (grid.hpp:124-133,171-176). Kahan: |K - S| <= (2u + O(n u^2)) A;
// ours: |D - S| <= u|S| + O(n u^2) A with |S| <= A; the scalings/additions add
// <= 2u|v| each side. 4u*vol*A + 4u|v| covers all of it (u = 2^-53, n <= 2^30).
__global__ void __launch_bounds__(kRedThreads) red_final_kernel(const double* partials, int nb,
                                                                int two, double vol,
                                                                double* results, int slot) {
  DD acc1{0.0, 0.0}, acc2{0.0, 0.0};
  double ab = 0.0;
  for (int i = threadIdx.x; i < nb; i += kRedThreads) {
    acc1 = dd_merge(acc1, DD{partials[2 * i], partials[2 * i + 1]});
    acc2 = dd_merge(acc2, DD{partials[2 * (nb + i)], partials[2 * (nb + i) + 1]});
    ab += partials[4 * nb + i];
  }
  DD r1 = block_reduce(acc1);
  DD r2 = block_reduce(acc2);
  ab = block_sum_plain(ab);
  if (threadIdx.x == 0 && two < 0) {  // raw double-double partial sums (multi-GPU ranks)
    results[slot] = r1.s;
    results[slot + 1] = r1.c;
    results[slot + 2] = r2.s;
    results[slot + 3] = r2.c;
    return;
  }
  if (threadIdx.x == 0) {
    const double s1 = r1.s + r1.c;
    double v = s1 * vol;
    if (two) {
      const double s2 = r2.s + r2.c;
      v = v + s2 * vol;
    }
    results[slot] = v;
    const double u4 = 4.0 * 0x1.0p-53;
    results[kBoundSlot + slot] = u4 * vol * ab + u4 * fabs(v);
  }
}

__global__ void __launch_bounds__(kRedThreads) density_scan_kernel(const double* a, long n,
                                                                   double* partials) {
  double mx = 0.0;
  int bad = 0, neg = 0;
  for (long i = blockIdx.x * static_cast<long>(kRedThreads) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * kRedThreads) {
    const double v = a[i];
    if (!isfinite(v)) bad = 1;
    else if (v < 0.0) neg = 1;
    else mx = fmax(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    bad |= __shfl_down_sync(0xffffffffu, bad, o);
    neg |= __shfl_down_sync(0xffffffffu, neg, o);
  }
  __shared__ double smx[kRedThreads / 32];
  __shared__ int sbad[kRedThreads / 32], sneg[kRedThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    smx[w] = mx;
    sbad[w] = bad;
    sneg[w] = neg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kRedThreads / 32; ++i) {
      mx = fmax(mx, smx[i]);
      bad |= sbad[i];
      neg |= sneg[i];
    }
    partials[3 * blockIdx.x] = mx;
    partials[3 * blockIdx.x + 1] = bad;
    partials[3 * blockIdx.x + 2] = neg;
  }
}

__global__ void density_final_kernel(const double* partials, int nb, double* results, int slot) {
  if (threadIdx.x != 0) return;
  double mx = 0.0, bad = 0.0, neg = 0.0;
  for (int i = 0; i < nb; ++i) {
    mx = fmax(mx, partials[3 * i]);
    bad = fmax(bad, partials[3 * i + 1]);
    neg = fmax(neg, partials[3 * i + 2]);
  }
  results[slot] = mx;
  results[slot + 1] = bad;
  results[slot + 2] = neg;
}

__global__ void axpy_kernel(double* u, double s, const double* dir, long n) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    u[i] = u[i] + s * dir[i];  // solver.hpp:283, no contraction (-fmad=false)
}

__global__ void add_scalar_kernel(double* u, double delta, long n) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    u[i] = u[i] + delta;
}

unsigned ew_grid(long n) {
  long b = (n + 255) / 256;
  if (b > 148L * 16) b = 148L * 16;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

Reducer::~Reducer() {
  if (partials_) dfree(partials_);
  if (results_) dfree(results_);
  if (pinned_) cudaFreeHost(pinned_);
}

void Reducer::init() {
  blocks_ = kRedBlocks;
  BFM_CUDA(dmalloc(&partials_, 5 * blocks_ * sizeof(double)));
  BFM_CUDA(dmalloc(&results_, kRedSlots * sizeof(double)));
  BFM_CUDA(cudaMemset(results_, 0, kRedSlots * sizeof(double)));
  BFM_CUDA(cudaMallocHost(&pinned_, kRedSlots * sizeof(double)));
}

void Reducer::dot(const double* a1, const double* b1, const double* a2, const double* b2, long n,
                  double vol, int slot, cudaStream_t s, LaunchCounter* lc) {
  RedArgs A{a1, b1, a2, b2, n, 0, 0, partials_};
  red_partial_kernel<0><<<blocks_, kRedThreads, 0, s>>>(A);
  red_final_kernel<<<1, kRedThreads, 0, s>>>(partials_, blocks_, a2 ? 1 : 0, vol, results_, slot);
  BFM_LAUNCH_CHECK("reduce dot");
  if (lc) lc->add(2);
}

void Reducer::dot_raw(const double* a1, const double* b1, const double* a2, const double* b2,
                      long n, int slot, cudaStream_t s, LaunchCounter* lc) {
  RedArgs A{a1, b1, a2, b2, n, 0, 0, partials_};
  red_partial_kernel<0><<<blocks_, kRedThreads, 0, s>>>(A);
  red_final_kernel<<<1, kRedThreads, 0, s>>>(partials_, blocks_, -1, 1.0, results_, slot);
  BFM_LAUNCH_CHECK("reduce dot_raw");
  if (lc) lc->add(2);
}

void Reducer::primal_raw(const double* disp, const double* mu, int d, long n, int slot,
                         cudaStream_t s, LaunchCounter* lc) {
  RedArgs A{disp, mu, nullptr, nullptr, n, 2, d, partials_};
  red_partial_kernel<2><<<blocks_, kRedThreads, 0, s>>>(A);
  red_final_kernel<<<1, kRedThreads, 0, s>>>(partials_, blocks_, -1, 1.0, results_, slot);
  BFM_LAUNCH_CHECK("reduce primal_raw");
  if (lc) lc->add(2);
}

void Reducer::sum(const double* a, long n, double vol, int slot, cudaStream_t s,
                  LaunchCounter* lc) {
  RedArgs A{a, nullptr, nullptr, nullptr, n, 1, 0, partials_};
  red_partial_kernel<1><<<blocks_, kRedThreads, 0, s>>>(A);
  red_final_kernel<<<1, kRedThreads, 0, s>>>(partials_, blocks_, 0, vol, results_, slot);
  BFM_LAUNCH_CHECK("reduce sum");
  if (lc) lc->add(2);
}

void Reducer::primal(const double* disp, const double* mu, int d, long n, double vol, int slot,
                     cudaStream_t s, LaunchCounter* lc, const double* exponents) {
  RedArgs A{disp, mu, nullptr, nullptr, n, 2, d, partials_, {0.0, 0.0, 0.0}};
  for (int a = 0; a < d && exponents; ++a) A.pexp[a] = exponents[a] == 2.0 ? 0.0 : exponents[a];
  red_partial_kernel<2><<<blocks_, kRedThreads, 0, s>>>(A);
  red_final_kernel<<<1, kRedThreads, 0, s>>>(partials_, blocks_, 0, vol, results_, slot);
  BFM_LAUNCH_CHECK("reduce primal");
  if (lc) lc->add(2);
}

void Reducer::scan_density(const double* a, long n, int slot, cudaStream_t s, LaunchCounter* lc) {
  density_scan_kernel<<<blocks_, kRedThreads, 0, s>>>(a, n, partials_);
  density_final_kernel<<<1, 32, 0, s>>>(partials_, blocks_, results_, slot);
  BFM_LAUNCH_CHECK("density scan");
  if (lc) lc->add(2);
}

void Reducer::fetch(double* host, int count, cudaStream_t s) {
  BFM_CUDA(cudaMemcpyAsync(pinned_, results_, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  BFM_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < count; ++i) host[i] = pinned_[i];
}

__global__ void axpy_dev_kernel(double* u, const double* s_ptr, const double* dir, long n) {
  const double s = *s_ptr;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    u[i] = u[i] + s * dir[i];  // solver.hpp:283, no contraction (-fmad=false)
}

void axpy_dev(double* u, const double* d_s, const double* dir, long n, cudaStream_t st,
              LaunchCounter* lc) {
  axpy_dev_kernel<<<ew_grid(n), 256, 0, st>>>(u, d_s, dir, n);
  BFM_LAUNCH_CHECK("axpy_dev");
  if (lc) lc->add();
}

void axpy(double* u, double s, const double* dir, long n, cudaStream_t st, LaunchCounter* lc) {
  axpy_kernel<<<ew_grid(n), 256, 0, st>>>(u, s, dir, n);
  BFM_LAUNCH_CHECK("axpy");
  if (lc) lc->add();
}

void add_scalar(double* u, double delta, long n, cudaStream_t st, LaunchCounter* lc) {
  add_scalar_kernel<<<ew_grid(n), 256, 0, st>>>(u, delta, n);
  BFM_LAUNCH_CHECK("add_scalar");
  if (lc) lc->add();
}

namespace {
__global__ void debug_pow_kernel(const double* x, const double* y, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = bfmpow::pow_cr(x[i], y[i]);
}
}  // namespace

// test hook (bfm_debug_pow): the device evaluation of pow_dd.h
void debug_pow_device(const double* h_x, const double* h_y, int n, double* h_out) {
  if (n <= 0) return;
  double *dx = nullptr, *dy = nullptr, *dout = nullptr;
  BFM_CUDA(dmalloc(&dx, sizeof(double) * n));
  BFM_CUDA(dmalloc(&dy, sizeof(double) * n));
  BFM_CUDA(dmalloc(&dout, sizeof(double) * n));
  BFM_CUDA(cudaMemcpy(dx, h_x, sizeof(double) * n, cudaMemcpyHostToDevice));
  BFM_CUDA(cudaMemcpy(dy, h_y, sizeof(double) * n, cudaMemcpyHostToDevice));
  debug_pow_kernel<<<(n + 127) / 128, 128>>>(dx, dy, n, dout);
  BFM_LAUNCH_CHECK("debug_pow_kernel");
  BFM_CUDA(cudaMemcpy(h_out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost));
  dfree(dx);
  dfree(dy);
  dfree(dout);
}

}  // namespace bfmgpu
