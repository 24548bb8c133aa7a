// Transport map, density pushforward and residual on sm_100a.
//
// Reference: pushforward.hpp:70-91 (map_from_conjugate), :51-63
// (locate_cell), :141-172 (splat_displaced: a sequential scatter in source
// order), solver.hpp:249-253 (r = target - rho); gradient grid.hpp:186-208;
// inverse cost gradient cost.hpp:59-68 (p = 2, magnitude capped at sqrt(d)).
//
// The scatter is reformulated as a deterministic gather so the result is
// bitwise equal to the reference's sequential `out[node] += w`:
//   1. map: per source, the clamped target, its lo-corner cell, the
//      per-axis upper weights and a clamp mask (same IEEE sequence as the
//      reference, no FMA); count sources per cell;
//   2. exclusive scan of the counts; place source ids into per-cell buckets;
//      sort each bucket by source id (almost all buckets hold 0-2 ids);
//   3. gather: every target merges the sorted buckets of its 2^d
//      neighbouring cells by source id and folds the nonzero corner weights
//      from 0.0 in increasing source order — exactly the order in which the
//      reference adds them — then writes target - rho.
#include <climits>

#include "pushforward.cuh"
#include <cmath>

namespace bfmgpu {
namespace {

constexpr int kScanItems = 8;
constexpr int kScanThreads = 1024;
constexpr int kScanTile = kScanItems * kScanThreads;
constexpr int kLight = 48;
constexpr int kFoldChunk = 8192;
constexpr int kMedium = 4096;

struct MapArgs {
  GridDesc g;
  const double* u;      // potential (mode 0) or nullptr
  const double* disp;   // displacement (mode 1)
  double scale;
  const double* src;    // source density
  uint32_t* key;        // cell of the lo corner; sentinel = N for massless sources
  uint8_t* cmask;
  double* w;
  double* disp_out;     // optional
  int binning;          // 0: map only
  double diam;          // sqrt(d)
};

__device__ __forceinline__ void node_idx(const GridDesc& g, long lin, int* id) {
  for (int a = 0; a < g.d; ++a) {
    id[a] = static_cast<int>(lin / g.stride[a]);
    lin -= static_cast<long>(id[a]) * g.stride[a];
  }
}

// locate_cell (pushforward.hpp:51-63) against the node table c_i = (i+0.5)h.
__device__ __forceinline__ void locate(int n, double h, double x, int& lo, bool& clamped,
                                       double& whi) {
  const double c0 = coord(h, 0);
  const double cl = coord(h, n - 1);
  if (x <= c0) {
    lo = 0;
    clamped = true;
    whi = 0.0;
    return;
  }
  if (x >= cl) {
    lo = n - 1;
    clamped = true;
    whi = 0.0;
    return;
  }
  int i = static_cast<int>(x * static_cast<double>(n) - 0.5);
  if (i < 0) i = 0;
  if (i > n - 2) i = n - 2;
  while (i + 1 < n - 1 && coord(h, i + 1) <= x) ++i;
  while (i > 0 && coord(h, i) > x) --i;
  const double clo = coord(h, i);
  const double chi = coord(h, i + 1);
  lo = i;
  clamped = false;
  whi = (x - clo) / (chi - clo);
}

__global__ void pf_map_kernel(MapArgs A) {
  const GridDesc& g = A.g;
  for (long s = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; s < g.size;
       s += static_cast<long>(gridDim.x) * blockDim.x) {
    int id[3] = {0, 0, 0};
    node_idx(g, s, id);
    double dsp[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < g.d; ++a) {
      const double x = coord(g.h[a], id[a]);
      if (A.u) {
        const long st = g.stride[a];
        const int n = g.n[a];
        const int j = id[a];
        const double inv_h = static_cast<double>(n);
        const double inv_2h = 0.5 * inv_h;
        double gr;
        if (j == 0) gr = (A.u[s + st] - A.u[s]) * inv_h;
        else if (j == n - 1) gr = (A.u[s] - A.u[s - st]) * inv_h;
        else gr = (A.u[s + st] - A.u[s - st]) * inv_2h;
        double mag = fabs(gr);
        if (!(mag < A.diam)) mag = A.diam;
        const double v = gr < 0.0 ? -mag : mag;
        double t = x - v;
        if (t < 0.0) t = 0.0;
        if (t > 1.0) t = 1.0;
        dsp[a] = t - x;
        if (A.disp_out) A.disp_out[a * g.size + s] = dsp[a];
      } else {
        dsp[a] = A.disp[a * g.size + s];
      }
    }
    if (!A.binning) continue;
    const double m = A.src[s];
    if (m == 0.0) {
      A.key[s] = static_cast<uint32_t>(g.size);
      continue;
    }
    long key = 0;
    uint8_t mask = 0;
    for (int a = 0; a < g.d; ++a) {
      const double x = coord(g.h[a], id[a]);
      const double xp = x + A.scale * dsp[a];
      int lo;
      bool cl;
      double whi;
      locate(g.n[a], g.h[a], xp, lo, cl, whi);
      key += static_cast<long>(lo) * g.stride[a];
      if (cl) mask |= static_cast<uint8_t>(1u << a);
      A.w[a * g.size + s] = whi;
    }
    A.key[s] = static_cast<uint32_t>(key);
    A.cmask[s] = mask;
  }
}

// Bucket boundaries of the sorted (cell, source) pairs: off[c] = first, end[c] = one past last.
__global__ void pf_bounds_kernel(const uint32_t* keys, long n, uint32_t sentinel, int* off, int* end) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const uint32_t k = keys[i];
    if (k == sentinel) continue;
    if (i == 0 || keys[i - 1] != k) off[k] = static_cast<int>(i);
    if (i == n - 1 || keys[i + 1] != k) end[k] = static_cast<int>(i + 1);
  }
}

struct GatherArgs {
  GridDesc g;
  const int* end;
  const int* off;
  const int* bucket;
  const uint8_t* cmask;
  const double* w;
  const double* src;
  const double* target;  // may be null: output rho
  double* out;
};

__device__ __forceinline__ double deposit_weight(const GatherArgs& A, int s, int b) {
  double wt = A.src[s];
  for (int a = 0; a < A.g.d; ++a) {
    const double wh = A.w[a * A.g.size + s];
    wt *= ((b >> a) & 1) ? wh : 1.0 - wh;
  }
  return wt;
}

// Light targets: merge the <= 2^d sorted neighbouring buckets by source id
// and fold in place. Targets with more than kLight deposits are deferred to
// pf_gather_heavy_kernel.
__global__ void pf_gather_kernel(GatherArgs A, int* heavy, int* nheavy) {
  const GridDesc& g = A.g;
  const int corners = 1 << g.d;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < g.size;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    int id[3] = {0, 0, 0};
    node_idx(g, t, id);
    int pos[8], end[8];
    int nl = 0;
    int bits[8];
    int total = 0;
    for (int b = 0; b < corners; ++b) {
      long c = t;
      bool ok = true;
      for (int a = 0; a < g.d; ++a)
        if ((b >> a) & 1) {
          if (id[a] == 0) ok = false;
          c -= g.stride[a];
        }
      if (!ok) continue;
      const int k = A.end[c] - A.off[c];
      if (k <= 0) continue;
      pos[nl] = A.off[c];
      end[nl] = pos[nl] + k;
      bits[nl] = b;
      total += k;
      ++nl;
    }
    if (total > kLight) {
      if (total <= kMedium) heavy[atomicAdd(nheavy, 1)] = static_cast<int>(t);
      else heavy[g.size - 1 - atomicAdd(nheavy + 1, 1)] = static_cast<int>(t);  // huge: from the top
      continue;
    }
    double rho = 0.0;
    while (true) {
      int best = -1, bs = INT_MAX;
      for (int q = 0; q < nl; ++q)
        if (pos[q] < end[q]) {
          const int s = A.bucket[pos[q]];
          if (s < bs) {
            bs = s;
            best = q;
          }
        }
      if (best < 0) break;
      ++pos[best];
      const int b = bits[best];
      if (b & A.cmask[bs]) continue;  // clamped axis: upper corner has weight 0
      const double wt = deposit_weight(A, bs, b);
      if (wt != 0.0) rho += wt;
    }
    A.out[t] = A.target ? A.target[t] - rho : rho;
  }
}

// Medium targets (kLight < K <= kMedium): one warp each; lanes rank and weight
// the deposits into the global buffer, then lane 0 folds them in order while
// the warp streams 32 at a time through shuffles.
__global__ void __launch_bounds__(256) pf_gather_medium_kernel(GatherArgs A, const int* heavy,
                                                              const int* nheavy, double* hbuf,
                                                              unsigned long long* hfill) {
  const GridDesc& g = A.g;
  const int corners = 1 << g.d;
  const int nh = nheavy[0];
  const int lane = threadIdx.x & 31;
  const long warp0 = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
  for (long q = warp0; q < nh; q += nwarps) {
    const long t = heavy[q];
    int id[3] = {0, 0, 0};
    node_idx(g, t, id);
    int pos[8], endp[8], bits[8];
    int nl = 0, K = 0;
    for (int b = 0; b < corners; ++b) {
      long c = t;
      bool ok = true;
      for (int a = 0; a < g.d; ++a)
        if ((b >> a) & 1) {
          if (id[a] == 0) ok = false;
          c -= g.stride[a];
        }
      if (!ok) continue;
      const int k = A.end[c] - A.off[c];
      if (k <= 0) continue;
      pos[nl] = A.off[c];
      endp[nl] = A.end[c];
      bits[nl] = b;
      K += k;
      ++nl;
    }
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(hfill, static_cast<unsigned long long>(K));
    base = __shfl_sync(0xffffffffu, base, 0);
    double* buf = hbuf + base;
    for (int qq = 0; qq < nl; ++qq) {
      for (int i = pos[qq] + lane; i < endp[qq]; i += 32) {
        const int src = A.bucket[i];
        int fin = i - pos[qq];
        for (int o = 0; o < nl; ++o) {
          if (o == qq) continue;
          int lo = pos[o], hi = endp[o];
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (A.bucket[mid] < src) lo = mid + 1;
            else hi = mid;
          }
          fin += lo - pos[o];
        }
        buf[fin] = (bits[qq] & A.cmask[src]) ? 0.0 : deposit_weight(A, src, bits[qq]);
      }
    }
    __syncwarp();
    double rho = 0.0;
    for (int c = 0; c < K; c += 32) {
      const double v = c + lane < K ? buf[c + lane] : 0.0;
      const int m = min(32, K - c);
      for (int i = 0; i < m; ++i) {
        const double w = __shfl_sync(0xffffffffu, v, i);
        if (w != 0.0) rho += w;
      }
    }
    if (lane == 0) A.out[t] = A.target ? A.target[t] - rho : rho;
  }
}

// Heavy targets: one CTA each. Every deposit's position in the source-ordered
// merge of the <= 2^d sorted neighbouring buckets is its index in its own
// bucket plus its rank (lower_bound) in each other bucket (a source lives in
// exactly one bucket, so there are no ties). Weights are written to those
// positions in a global buffer in parallel; one thread then folds them in
// order from 0.0 exactly like the reference's sequential +=.
__global__ void __launch_bounds__(512) pf_gather_heavy_kernel(GatherArgs A, const int* heavy,
                                                             const int* nheavy, double* hbuf,
                                                             unsigned long long* hfill) {
  __shared__ int s_pos[8], s_end[8], s_bits[8], s_nl, s_K;
  __shared__ unsigned long long s_base;
  extern __shared__ __align__(16) unsigned char fold_raw[];
  double* fold = reinterpret_cast<double*>(fold_raw);  // [2 * kFoldChunk]
  const GridDesc& g = A.g;
  const int corners = 1 << g.d;
  const int nh = nheavy[1];
  for (int q = blockIdx.x; q < nh; q += gridDim.x) {
    const long t = heavy[g.size - 1 - q];
    if (threadIdx.x == 0) {
      int id[3] = {0, 0, 0};
      node_idx(g, t, id);
      int nl = 0, K = 0;
      for (int b = 0; b < corners; ++b) {
        long c = t;
        bool ok = true;
        for (int a = 0; a < g.d; ++a)
          if ((b >> a) & 1) {
            if (id[a] == 0) ok = false;
            c -= g.stride[a];
          }
        if (!ok) continue;
        const int k = A.end[c] - A.off[c];
        if (k <= 0) continue;
        s_pos[nl] = A.off[c];
        s_end[nl] = A.end[c];
        s_bits[nl] = b;
        K += k;
        ++nl;
      }
      s_nl = nl;
      s_K = K;
      s_base = atomicAdd(hfill, static_cast<unsigned long long>(K));
    }
    __syncthreads();
    const int nl = s_nl;
    double* buf = hbuf + s_base;
    for (int qq = 0; qq < nl; ++qq) {
      const int p0 = s_pos[qq], p1 = s_end[qq], b = s_bits[qq];
      for (int i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
        const int src = A.bucket[i];
        int fin = i - p0;
        for (int o = 0; o < nl; ++o) {
          if (o == qq) continue;
          int lo = s_pos[o], hi = s_end[o];
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (A.bucket[mid] < src) lo = mid + 1;
            else hi = mid;
          }
          fin += lo - s_pos[o];
        }
        buf[fin] = (b & A.cmask[src]) ? 0.0 : deposit_weight(A, src, b);
      }
    }
    __syncthreads();
    // Sequential fold from shared memory, double-buffered: thread 0 folds
    // chunk c while the other threads stage chunk c+1.
    const int K = s_K;
    const int nch = (K + kFoldChunk - 1) / kFoldChunk;
    double rho = 0.0;
    for (int i = threadIdx.x; i < min(K, kFoldChunk); i += blockDim.x) fold[i] = buf[i];
    __syncthreads();
    for (int c = 0; c < nch; ++c) {
      const double* cur = fold + (c & 1) * kFoldChunk;
      double* nxt = fold + ((c + 1) & 1) * kFoldChunk;
      const int len = min(kFoldChunk, K - c * kFoldChunk);
      if (threadIdx.x == 0) {
#pragma unroll 8
        for (int i = 0; i < len; ++i) {
          const double w = cur[i];
          if (w != 0.0) rho += w;
        }
      } else if (c + 1 < nch) {
        const int base = (c + 1) * kFoldChunk;
        const int len2 = min(kFoldChunk, K - base);
        for (int i = threadIdx.x - 1; i < len2; i += blockDim.x - 1) nxt[i] = buf[base + i];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) A.out[t] = A.target ? A.target[t] - rho : rho;
    __syncthreads();
  }
}

unsigned grid_for(long n, int threads) {
  long b = (n + threads - 1) / threads;
  const long cap = 148L * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

}  // namespace

PushforwardPlan::~PushforwardPlan() {
  for (void* p : {static_cast<void*>(key_), static_cast<void*>(cmask_), static_cast<void*>(w_),
                  static_cast<void*>(off_), static_cast<void*>(end_), static_cast<void*>(heavy_),
                  static_cast<void*>(nheavy_), static_cast<void*>(hbuf_)})
    if (p) cudaFree(p);
}

void PushforwardPlan::init(const GridDesc& g) {
  g_ = g;
  const long N = g.size;
  if (N >= (1L << 29)) throw std::invalid_argument("pushforward: grid too large");
  BFM_CUDA(cudaMalloc(&key_, N * sizeof(uint32_t)));
  BFM_CUDA(cudaMalloc(&cmask_, N));
  BFM_CUDA(cudaMalloc(&w_, g.d * N * sizeof(double)));
  BFM_CUDA(cudaMalloc(&off_, (N + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&end_, (N + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&heavy_, (N + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&nheavy_, 4 * sizeof(unsigned long long)));
  BFM_CUDA(cudaMalloc(&hbuf_, (static_cast<long>(1) << g.d) * N * sizeof(double)));
  sorter_.init(N);
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_heavy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                2 * kFoldChunk * static_cast<int>(sizeof(double))));
  key_bits_ = 1;
  while ((1L << key_bits_) <= N) ++key_bits_;  // cells 0..N-1 plus sentinel N
}

void PushforwardPlan::map_only(const double* d_u, double* d_disp, cudaStream_t stream,
                               LaunchCounter* lc) {
  MapArgs A{};
  A.g = g_;
  A.u = d_u;
  A.scale = 1.0;
  A.disp_out = d_disp;
  A.diam = std::sqrt(static_cast<double>(g_.d));
  pf_map_kernel<<<grid_for(g_.size, 256), 256, 0, stream>>>(A);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
}

void PushforwardPlan::bin_and_gather(const double* d_source, const double* d_target,
                                     double* d_out, cudaStream_t stream, LaunchCounter* lc) {
  const long N = g_.size;
  const uint32_t* skeys = nullptr;
  const int* svals = nullptr;
  sorter_.sort(key_, nullptr, N, key_bits_, stream, lc, &skeys, &svals);
  BFM_CUDA(cudaMemsetAsync(off_, 0, (N + 1) * sizeof(int), stream));
  BFM_CUDA(cudaMemsetAsync(end_, 0, (N + 1) * sizeof(int), stream));
  BFM_CUDA(cudaMemsetAsync(nheavy_, 0, 4 * sizeof(unsigned long long), stream));
  pf_bounds_kernel<<<grid_for(N, 256), 256, 0, stream>>>(skeys, N, static_cast<uint32_t>(N), off_,
                                                         end_);
  GatherArgs G{};
  G.g = g_;
  G.end = end_;
  G.off = off_;
  G.bucket = svals;
  G.cmask = cmask_;
  G.w = w_;
  G.src = d_source;
  G.target = d_target;
  G.out = d_out;
  int* nheavy = reinterpret_cast<int*>(nheavy_);
  pf_gather_kernel<<<grid_for(N, 256), 256, 0, stream>>>(G, heavy_, nheavy);
  BFM_LAUNCH_CHECK("pf_gather_kernel");
  pf_gather_medium_kernel<<<148 * 8, 256, 0, stream>>>(G, heavy_, nheavy, hbuf_, nheavy_ + 1);
  BFM_LAUNCH_CHECK("pf_gather_medium_kernel");
  pf_gather_heavy_kernel<<<148, 512, 2 * kFoldChunk * sizeof(double), stream>>>(G, heavy_, nheavy, hbuf_, nheavy_ + 1);
  BFM_LAUNCH_CHECK("pf_gather_heavy_kernel");
  if (lc) lc->add(4);
}

void PushforwardPlan::from_potential(const double* d_u, const double* d_source,
                                     const double* d_target, double* d_out, double* d_disp_out,
                                     cudaStream_t stream, LaunchCounter* lc) {
  MapArgs A{};
  A.g = g_;
  A.u = d_u;
  A.scale = 1.0;
  A.src = d_source;
  A.key = key_;
  A.cmask = cmask_;
  A.w = w_;
  A.disp_out = d_disp_out;
  A.binning = 1;
  A.diam = std::sqrt(static_cast<double>(g_.d));
  pf_map_kernel<<<grid_for(g_.size, 256), 256, 0, stream>>>(A);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
  bin_and_gather(d_source, d_target, d_out, stream, lc);
}

void PushforwardPlan::from_displacement(const double* d_disp, double scale,
                                        const double* d_source, double* d_rho,
                                        cudaStream_t stream, LaunchCounter* lc) {
  MapArgs A{};
  A.g = g_;
  A.disp = d_disp;
  A.scale = scale;
  A.src = d_source;
  A.key = key_;
  A.cmask = cmask_;
  A.w = w_;
  A.binning = 1;
  A.diam = std::sqrt(static_cast<double>(g_.d));
  pf_map_kernel<<<grid_for(g_.size, 256), 256, 0, stream>>>(A);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
  bin_and_gather(d_source, nullptr, d_rho, stream, lc);
}

}  // namespace bfmgpu
