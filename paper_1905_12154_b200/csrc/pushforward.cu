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

namespace bfmgpu {
namespace {

constexpr int kScanItems = 8;
constexpr int kScanThreads = 1024;
constexpr int kScanTile = kScanItems * kScanThreads;
constexpr int kSmallBucket = 64;
constexpr int kLight = 48;
constexpr int kChunk = 8192;

struct MapArgs {
  GridDesc g;
  const double* u;      // potential (mode 0) or nullptr
  const double* disp;   // displacement (mode 1)
  double scale;
  const double* src;    // source density
  int* key;
  uint8_t* cmask;
  double* w;
  double* disp_out;     // optional
  int* cnt;             // optional (null: map only)
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
    if (!A.cnt) continue;
    const double m = A.src[s];
    if (m == 0.0) {
      A.key[s] = -1;
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
    A.key[s] = static_cast<int>(key);
    A.cmask[s] = mask;
    atomicAdd(&A.cnt[key], 1);
  }
}

// ---- exclusive scan of int counts (3 kernels) ----
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int* in, long n, int* bsum) {
  __shared__ int warp_tot[32];
  const long base = static_cast<long>(blockIdx.x) * kScanTile;
  int v = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const long idx = base + static_cast<long>(i) * kScanThreads + threadIdx.x;
    if (idx < n) v += in[idx];
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    int w = warp_tot[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (threadIdx.x == 0) bsum[blockIdx.x] = w;
  }
}

__device__ int block_exclusive_scan(int v, int* total) {
  __shared__ int warp_tot[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += u;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
    int ti = t;
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, ti, d);
      if (lane >= d) ti += u;
    }
    warp_tot[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  const int r = warp_tot[w] + incl - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_blocks_kernel(int* bsum, long nb) {
  __shared__ int carry_s;
  __shared__ int tot_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (long base = 0; base < nb; base += kScanThreads) {
    const long idx = base + threadIdx.x;
    const int v = idx < nb ? bsum[idx] : 0;
    const int ex = block_exclusive_scan(v, &tot_s);
    if (idx < nb) bsum[idx] = carry_s + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry_s += tot_s;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const int* in, int* out, long n,
                                                                  const int* bsum) {
  __shared__ int tot_s;
  const long base = static_cast<long>(blockIdx.x) * kScanTile;
  int carry = bsum[blockIdx.x];
  // each thread owns kScanItems consecutive elements
  const long mine = base + static_cast<long>(threadIdx.x) * kScanItems;
  int vals[kScanItems];
  int sum = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const long idx = mine + i;
    vals[i] = idx < n ? in[idx] : 0;
    sum += vals[i];
  }
  int ex = block_exclusive_scan(sum, &tot_s) + carry;
  for (int i = 0; i < kScanItems; ++i) {
    const long idx = mine + i;
    if (idx < n) out[idx] = ex;
    ex += vals[i];
  }
}

__global__ void pf_place_kernel(long N, const int* key, const int* off, int* fill, int* bucket) {
  for (long s = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; s < N;
       s += static_cast<long>(gridDim.x) * blockDim.x) {
    const int k = key[s];
    if (k < 0) continue;
    const int slot = off[k] + atomicAdd(&fill[k], 1);
    bucket[slot] = static_cast<int>(s);
  }
}

__global__ void pf_sort_small_kernel(long N, const int* cnt, const int* off, int* bucket,
                                     int* big, int* nbig) {
  for (long c = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; c < N;
       c += static_cast<long>(gridDim.x) * blockDim.x) {
    const int k = cnt[c];
    if (k < 2) continue;
    if (k > kSmallBucket) {
      big[atomicAdd(nbig, 1)] = static_cast<int>(c);
      continue;
    }
    int* b = bucket + off[c];
    for (int i = 1; i < k; ++i) {
      const int v = b[i];
      int j = i - 1;
      while (j >= 0 && b[j] > v) {
        b[j + 1] = b[j];
        --j;
      }
      b[j + 1] = v;
    }
  }
}

// One CTA per large bucket: bitonic sort in shared memory (capacity 32768).
__global__ void __launch_bounds__(1024) pf_sort_big_kernel(const int* cnt, const int* off,
                                                           int* bucket, const int* big,
                                                           const int* nbig, int* scratch) {
  extern __shared__ int sb[];
  const int nb = *nbig;
  for (int q = blockIdx.x; q < nb; q += gridDim.x) {
    const int c = big[q];
    const int k = cnt[c];
    if (k > 32768) {
      // Huge bucket: bitonic sort in a global scratch window [2*off, 2*off + p2).
      int p2 = 1;
      while (p2 < k) p2 <<= 1;
      int* b = bucket + off[c];
      int* sc = scratch + 2L * off[c];
      for (int i = threadIdx.x; i < p2; i += blockDim.x) sc[i] = i < k ? b[i] : INT_MAX;
      __syncthreads();
      for (int size = 2; size <= p2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int i = threadIdx.x; i < p2; i += blockDim.x) {
            const int j = i ^ stride;
            if (j > i) {
              const bool up = (i & size) == 0;
              const int x = sc[i], y = sc[j];
              if ((x > y) == up) {
                sc[i] = y;
                sc[j] = x;
              }
            }
          }
          __syncthreads();
        }
      for (int i = threadIdx.x; i < k; i += blockDim.x) b[i] = sc[i];
      __syncthreads();
      continue;
    }
    int p2 = 1;
    while (p2 < k) p2 <<= 1;
    int* b = bucket + off[c];
    for (int i = threadIdx.x; i < p2; i += blockDim.x) sb[i] = i < k ? b[i] : INT_MAX;
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const int x = sb[i], y = sb[j];
            if ((x > y) == up) {
              sb[i] = y;
              sb[j] = x;
            }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < k; i += blockDim.x) b[i] = sb[i];
    __syncthreads();
  }
}

struct GatherArgs {
  GridDesc g;
  const int* cnt;
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
      const int k = A.cnt[c];
      if (k == 0) continue;
      pos[nl] = A.off[c];
      end[nl] = pos[nl] + k;
      bits[nl] = b;
      total += k;
      ++nl;
    }
    if (total > kLight) {
      heavy[atomicAdd(nheavy, 1)] = static_cast<int>(t);
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

// Heavy targets: one CTA each. The merged source order is produced chunk by
// chunk (source-id ranges holding <= kChunk deposits), sorted in shared
// memory, weighted in parallel, then folded by one thread in order.
__global__ void __launch_bounds__(512) pf_gather_heavy_kernel(GatherArgs A, const int* heavy,
                                                             const int* nheavy) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* key = reinterpret_cast<unsigned*>(sm);                 // [kChunk]
  double* wv = reinterpret_cast<double*>(sm + 4 * kChunk);           // [kChunk]
  __shared__ int s_pos[8], s_end[8], s_bits[8], s_take[8], s_nl, s_cnt;
  __shared__ long s_lim;
  __shared__ double s_rho;
  const GridDesc& g = A.g;
  const int corners = 1 << g.d;
  const int nh = *nheavy;
  for (int q = blockIdx.x; q < nh; q += gridDim.x) {
    const long t = heavy[q];
    if (threadIdx.x == 0) {
      int id[3] = {0, 0, 0};
      node_idx(g, t, id);
      int nl = 0;
      for (int b = 0; b < corners; ++b) {
        long c = t;
        bool ok = true;
        for (int a = 0; a < g.d; ++a)
          if ((b >> a) & 1) {
            if (id[a] == 0) ok = false;
            c -= g.stride[a];
          }
        if (!ok) continue;
        const int k = A.cnt[c];
        if (k == 0) continue;
        s_pos[nl] = A.off[c];
        s_end[nl] = s_pos[nl] + k;
        s_bits[nl] = b;
        ++nl;
      }
      s_nl = nl;
      s_rho = 0.0;
    }
    __syncthreads();
    while (true) {
      if (threadIdx.x == 0) {
        // largest source-id bound lim with <= kChunk pending deposits below it
        long lo = -1, hi = g.size;  // invariant: count(<= lo) <= kChunk
        int remaining = 0;
        for (int b = 0; b < s_nl; ++b) remaining += s_end[b] - s_pos[b];
        if (remaining <= kChunk) {
          lo = g.size;
        } else {
          while (hi - lo > 1) {
            const long mid = (lo + hi) / 2;
            int c = 0;
            for (int b = 0; b < s_nl; ++b) {
              int l2 = s_pos[b], h2 = s_end[b];  // upper_bound of mid
              while (l2 < h2) {
                const int m2 = (l2 + h2) >> 1;
                if (A.bucket[m2] <= mid) l2 = m2 + 1;
                else h2 = m2;
              }
              c += l2 - s_pos[b];
            }
            if (c <= kChunk) lo = mid;
            else hi = mid;
          }
        }
        s_lim = lo;
        int c = 0;
        for (int b = 0; b < s_nl; ++b) {
          int l2 = s_pos[b], h2 = s_end[b];
          while (l2 < h2) {
            const int m2 = (l2 + h2) >> 1;
            if (A.bucket[m2] <= lo) l2 = m2 + 1;
            else h2 = m2;
          }
          s_take[b] = c;
          c += l2 - s_pos[b];
        }
        s_cnt = c;
      }
      __syncthreads();
      const int cnt = s_cnt;
      if (cnt == 0) break;
      int p2 = 1;
      while (p2 < cnt) p2 <<= 1;
      // gather (source << 3 | corner) keys of this chunk
      for (int b = 0; b < s_nl; ++b) {
        const int nb = (b + 1 < s_nl ? s_take[b + 1] : cnt) - s_take[b];
        for (int i = threadIdx.x; i < nb; i += blockDim.x)
          key[s_take[b] + i] = (static_cast<unsigned>(A.bucket[s_pos[b] + i]) << 3) |
                               static_cast<unsigned>(s_bits[b]);
      }
      for (int i = cnt + threadIdx.x; i < p2; i += blockDim.x) key[i] = 0xffffffffu;
      __syncthreads();
      for (int size = 2; size <= p2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int i = threadIdx.x; i < p2; i += blockDim.x) {
            const int j = i ^ stride;
            if (j > i) {
              const bool up = (i & size) == 0;
              const unsigned x = key[i], y = key[j];
              if ((x > y) == up) {
                key[i] = y;
                key[j] = x;
              }
            }
          }
          __syncthreads();
        }
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int src = static_cast<int>(key[i] >> 3);
        const int b = static_cast<int>(key[i] & 7u);
        wv[i] = (b & A.cmask[src]) ? 0.0 : deposit_weight(A, src, b);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double rho = s_rho;
        for (int i = 0; i < cnt; ++i) {
          const double w = wv[i];
          if (w != 0.0) rho += w;
        }
        s_rho = rho;
        for (int b = 0; b < s_nl; ++b)
          s_pos[b] += (b + 1 < s_nl ? s_take[b + 1] : cnt) - s_take[b];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) A.out[t] = A.target ? A.target[t] - s_rho : s_rho;
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
                  static_cast<void*>(cnt_), static_cast<void*>(off_), static_cast<void*>(fill_),
                  static_cast<void*>(bucket_), static_cast<void*>(blocksum_),
                  static_cast<void*>(big_), static_cast<void*>(nbig_),
                  static_cast<void*>(scratch_)})
    if (p) cudaFree(p);
}

void PushforwardPlan::init(const GridDesc& g) {
  g_ = g;
  const long N = g.size;
  if (N >= INT_MAX) throw std::invalid_argument("pushforward: grid too large");
  BFM_CUDA(cudaMalloc(&key_, N * sizeof(int)));
  BFM_CUDA(cudaMalloc(&cmask_, N));
  BFM_CUDA(cudaMalloc(&w_, g.d * N * sizeof(double)));
  BFM_CUDA(cudaMalloc(&cnt_, (N + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&off_, (N + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&fill_, N * sizeof(int)));
  BFM_CUDA(cudaMalloc(&bucket_, N * sizeof(int)));
  scan_blocks_ = (N + kScanTile - 1) / kScanTile;
  BFM_CUDA(cudaMalloc(&blocksum_, (scan_blocks_ + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&big_, N * sizeof(int)));
  BFM_CUDA(cudaMalloc(&scratch_, 2 * (N + 1) * sizeof(int)));
  BFM_CUDA(cudaMalloc(&nbig_, 4 * sizeof(int)));
  BFM_CUDA(cudaFuncSetAttribute(pf_sort_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                32768 * 4));
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_heavy_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kChunk * 12));
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
  scan_reduce_kernel<<<static_cast<unsigned>(scan_blocks_), kScanThreads, 0, stream>>>(cnt_, N,
                                                                                      blocksum_);
  scan_blocks_kernel<<<1, kScanThreads, 0, stream>>>(blocksum_, scan_blocks_);
  scan_apply_kernel<<<static_cast<unsigned>(scan_blocks_), kScanThreads, 0, stream>>>(
      cnt_, off_, N, blocksum_);
  BFM_LAUNCH_CHECK("scan");
  pf_place_kernel<<<grid_for(N, 256), 256, 0, stream>>>(N, key_, off_, fill_, bucket_);
  pf_sort_small_kernel<<<grid_for(N, 256), 256, 0, stream>>>(N, cnt_, off_, bucket_, big_, nbig_);
  pf_sort_big_kernel<<<148, 1024, 32768 * 4, stream>>>(cnt_, off_, bucket_, big_, nbig_,
                                                       scratch_);
  GatherArgs G{};
  G.g = g_;
  G.cnt = cnt_;
  G.off = off_;
  G.bucket = bucket_;
  G.cmask = cmask_;
  G.w = w_;
  G.src = d_source;
  G.target = d_target;
  G.out = d_out;
  pf_gather_kernel<<<grid_for(N, 256), 256, 0, stream>>>(G, big_, nbig_ + 2);
  BFM_LAUNCH_CHECK("pf_gather_kernel");
  pf_gather_heavy_kernel<<<148 * 2, 512, kChunk * 12, stream>>>(G, big_, nbig_ + 2);
  BFM_LAUNCH_CHECK("pf_gather_heavy_kernel");
  if (lc) lc->add(8);
}

void PushforwardPlan::from_potential(const double* d_u, const double* d_source,
                                     const double* d_target, double* d_out, double* d_disp_out,
                                     cudaStream_t stream, LaunchCounter* lc) {
  const long N = g_.size;
  BFM_CUDA(cudaMemsetAsync(cnt_, 0, (N + 1) * sizeof(int), stream));
  BFM_CUDA(cudaMemsetAsync(fill_, 0, N * sizeof(int), stream));
  BFM_CUDA(cudaMemsetAsync(nbig_, 0, 4 * sizeof(int), stream));
  MapArgs A{};
  A.g = g_;
  A.u = d_u;
  A.scale = 1.0;
  A.src = d_source;
  A.key = key_;
  A.cmask = cmask_;
  A.w = w_;
  A.disp_out = d_disp_out;
  A.cnt = cnt_;
  A.diam = std::sqrt(static_cast<double>(g_.d));
  pf_map_kernel<<<grid_for(N, 256), 256, 0, stream>>>(A);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
  bin_and_gather(d_source, d_target, d_out, stream, lc);
}

void PushforwardPlan::from_displacement(const double* d_disp, double scale,
                                        const double* d_source, double* d_rho,
                                        cudaStream_t stream, LaunchCounter* lc) {
  const long N = g_.size;
  BFM_CUDA(cudaMemsetAsync(cnt_, 0, (N + 1) * sizeof(int), stream));
  BFM_CUDA(cudaMemsetAsync(fill_, 0, N * sizeof(int), stream));
  BFM_CUDA(cudaMemsetAsync(nbig_, 0, 4 * sizeof(int), stream));
  MapArgs A{};
  A.g = g_;
  A.disp = d_disp;
  A.scale = scale;
  A.src = d_source;
  A.key = key_;
  A.cmask = cmask_;
  A.w = w_;
  A.cnt = cnt_;
  A.diam = std::sqrt(static_cast<double>(g_.d));
  pf_map_kernel<<<grid_for(N, 256), 256, 0, stream>>>(A);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
  bin_and_gather(d_source, nullptr, d_rho, stream, lc);
}

}  // namespace bfmgpu
