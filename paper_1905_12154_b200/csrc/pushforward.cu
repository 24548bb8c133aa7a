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
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <cmath>
#include <vector>

#include "exact_fold.cuh"
#include "pushforward.cuh"
#include "pow_dd.h"

namespace bfmgpu {
namespace {

constexpr int kLight = 48;
constexpr int kSeqFold = 16384;  // heavy tier: warp-sequential fold up to this many deposits
constexpr int kMedium = 512;   // warp-per-target tier: kLight < K <= kMedium
constexpr int kLarge = 4096;   // CTA-per-target tier with a sequential fold: K <= kLarge
constexpr int kLargeThreads = 128;
constexpr int kLargeBlocks = 148 * 8;  // each CTA owns kLarge doubles of hbuf
constexpr int kLargeSmem = kLarge * 2 * (4 + 2);  // ids + payloads, ping-pong
constexpr int kLargeA = 2048;                      // the smaller CTA-tier instantiation
constexpr int kLargeSmemA = kLargeA * 2 * (4 + 2);
constexpr int kMedWarps = 8;
constexpr int kHeavyIds = 24576;
constexpr int kMedSmem = kMedWarps * 2 * kMedium * (4 + 2);  // ids + payloads, ping-pong
constexpr int kMedBlocks = 148 * 8;  // each warp owns kMedium doubles of hbuf
constexpr int kHeavySmem = kHeavyIds * 4;

struct MapArgs {
  GridDesc g;           // the nodes this launch maps (whole grid or a row slab)
  GridDesc gg;          // the problem grid (coordinates, boundaries, cell keys)
  int row_off;          // global row of local row 0 (row slab), else 0
  long u_shift;         // u index of local node 0 (one halo row above a slab)
  const double* u;      // potential (mode 0) or nullptr
  const double* disp;   // displacement (mode 1)
  double scale;
  const double* src;    // source density
  uint32_t* key;        // global cell of the lo corner; sentinel = N (global) for massless sources
  uint8_t* cmask;
  double* w;
  double* disp_out;     // optional
  int binning;          // 0: map only
  double diam;          // sqrt(d)
  double iexp[3];       // power costs: 1/(p_a - 1) per axis (0: quadratic axis)
};

// Node coordinates of a linear index (grids here have < 2^31 nodes: 32-bit
// divisions, far cheaper than 64-bit ones on the SM).
__device__ __forceinline__ void node_idx(const GridDesc& g, long lin, int* id) {
  const unsigned r = static_cast<unsigned>(lin);
  if (g.d == 1) {
    id[0] = static_cast<int>(r);
    return;
  }
  const unsigned s0 = static_cast<unsigned>(g.stride[0]);
  const unsigned i0 = r / s0;
  const unsigned r0 = r - i0 * s0;
  id[0] = static_cast<int>(i0);
  if (g.d == 2) {
    id[1] = static_cast<int>(r0);
    return;
  }
  const unsigned s1 = static_cast<unsigned>(g.stride[1]);
  const unsigned i1 = r0 / s1;
  id[1] = static_cast<int>(i1);
  id[2] = static_cast<int>(r0 - i1 * s1);
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

// POWER: a power cost's pow inverse gradient (separate instantiation: the
// pow code would double the quadratic map's registers, 32 -> 62)
template <bool POWER>
__global__ void pf_map_kernel(MapArgs A) {
  const GridDesc& g = A.g;
  const GridDesc& gg = A.gg;
  for (long s = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; s < g.size;
       s += static_cast<long>(gridDim.x) * blockDim.x) {
    int id[3] = {0, 0, 0};
    node_idx(g, s, id);
    id[0] += A.row_off;  // global indices from here on
    double dsp[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < g.d; ++a) {
      const double x = coord(gg.h[a], id[a]);
      if (A.u) {
        const long st = g.stride[a];
        const int n = gg.n[a];
        const int j = id[a];
        const long su = s + A.u_shift;
        const double inv_h = static_cast<double>(n);
        const double inv_2h = 0.5 * inv_h;
        double gr;
        if (j == 0) gr = (__ldg(A.u + su + st) - __ldg(A.u + su)) * inv_h;
        else if (j == n - 1) gr = (__ldg(A.u + su) - __ldg(A.u + su - st)) * inv_h;
        else gr = (__ldg(A.u + su + st) - __ldg(A.u + su - st)) * inv_2h;
        // inverse gradient (cost.hpp:59-68): |v| (p = 2) or |v|^(1/(p-1)),
        // correctly rounded (pow_dd.h), capped at sqrt(d)
        double mag = fabs(gr);
        if (POWER && A.iexp[a] > 0.0) mag = bfmpow::pow_cr(mag, A.iexp[a]);
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
      A.key[s] = static_cast<uint32_t>(gg.size);
      continue;
    }
    long key = 0;
    uint8_t mask = 0;
    for (int a = 0; a < g.d; ++a) {
      const double x = coord(gg.h[a], id[a]);
      const double xp = x + A.scale * dsp[a];
      int lo;
      bool cl;
      double whi;
      locate(gg.n[a], gg.h[a], xp, lo, cl, whi);
      key += static_cast<long>(lo) * gg.stride[a];
      if (cl) mask |= static_cast<uint8_t>(1u << a);
      A.w[a * g.size + s] = whi;
    }
    A.key[s] = static_cast<uint32_t>(key);
    A.cmask[s] = mask;
  }
}

struct GatherArgs {
  GridDesc g;        // target nodes (whole grid or a row slab)
  int row_off;       // global row of local target row 0
  long cell_shift;   // cell index of target t's own cell is t + cell_shift
  long nrec;         // deposit records (sources): stride of w
  const int* end;
  const int* off;
  const int* bucket;  // record ids sorted by (cell, record id)
  const uint8_t* cmask;
  const double* w;
  const double* src;  // record mass
  const double* target;  // may be null: output rho
  double* out;
  // every deposit's weight for each of its 2^d corners, in sorted (bucket)
  // order and corner-major (pf_pack_kernel): wts[b * nrec + position]
  const double* wts;
};

// Weight of the deposit at sorted position pos into the corner-b target
// (0 on a clamped axis's upper corner): the same IEEE sequence as
// the reference's weight (pushforward.hpp:161-166: m times each axis's upper
// or lower barycentric weight, in axis order), from the packed record.
__device__ __forceinline__ double pos_weight(const GatherArgs& A, int pos, int b) {
  // packed per corner by pf_pack_kernel: corner-major, so a bucket's deposits
  // are consecutive doubles for the corner that reads them
  return A.wts[static_cast<long>(b) * A.nrec + pos];
}

// bucket bounds and per-corner weights in sorted order (one pass after the sort)
__global__ void pf_pack_kernel(const uint32_t* keys, uint32_t sentinel, int* off, int* end, const int* bucket,
                               long nrec, const int* d_n, const double* src, const double* w,
                               const uint8_t* cmask, int d, double* wts) {
  // the weight of every deposit for each of its 2^d corners (the reference's
  // expression, pushforward.hpp:161-166: m times each axis's upper or lower
  // barycentric weight, in axis order; 0 on a clamped axis's upper corner),
  // corner-major: wts[b * nrec + sorted position]
  const long n = d_n ? *d_n : nrec;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    // bucket boundaries of the sorted (cell, source) pairs: off[c] = first,
    // end[c] = one past the last
    const uint32_t k = keys[i];
    if (k != sentinel) {
      if (i == 0 || keys[i - 1] != k) off[k] = static_cast<int>(i);
      if (i == n - 1 || keys[i + 1] != k) end[k] = static_cast<int>(i + 1);
    }
    const int s = bucket[i];
    const double m = src[s];
    double wa[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < d; ++a) wa[a] = w[a * nrec + s];
    const int mask = cmask[s];
    for (int b = 0; b < (1 << d); ++b) {
      double wt = m;
      for (int a = 0; a < d; ++a) wt *= ((b >> a) & 1) ? wa[a] : 1.0 - wa[a];
      if (b & mask) wt = 0.0;
      wts[static_cast<long>(b) * nrec + i] = wt;
    }
  }
}

// Light targets: merge the <= 2^d sorted neighbouring buckets by source id
// and fold in place. Targets with more than kLight deposits are deferred to
// pf_gather_heavy_kernel.
template <int D>
__global__ void __launch_bounds__(256, D < 3 ? 8 : 6) pf_gather_kernel(GatherArgs A, int* heavy, int* large,
                                                        int* nheavy) {
  constexpr int NC = 1 << D;  // corner b = bit a set: the target is the upper node on axis a
  const GridDesc& g = A.g;
  for (long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; t < g.size;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    int id[3] = {0, 0, 0};
    node_idx(g, t, id);
    id[0] += A.row_off;
    // fixed-size, fully unrolled per-corner state stays in registers
    int pos[NC], end[NC], head[NC];
    int total = 0;
#pragma unroll
    for (int b = 0; b < NC; ++b) {
      long c = t + A.cell_shift;
      bool ok = true;
#pragma unroll
      for (int a = 0; a < D; ++a)
        if ((b >> a) & 1) {
          if (id[a] == 0) ok = false;
          c -= g.stride[a];
        }
      pos[b] = ok ? A.off[c] : 0;
      end[b] = ok ? A.end[c] : 0;
      total += end[b] - pos[b];
    }
    if (total > kLight) {
      if (total <= kMedium) heavy[atomicAdd(nheavy, 1)] = static_cast<int>(t);
      else if (total <= kLargeA) large[atomicAdd(nheavy + 4, 1)] = static_cast<int>(t);
      else if (total <= kLarge) large[g.size - 1 - atomicAdd(nheavy + 7, 1)] = static_cast<int>(t);
      else heavy[g.size - 1 - atomicAdd(nheavy + 1, 1)] = static_cast<int>(t);  // huge: from the top
      continue;
    }
#pragma unroll
    for (int b = 0; b < NC; ++b) head[b] = pos[b] < end[b] ? A.bucket[pos[b]] : INT_MAX;
    double rho = 0.0;
    for (int it = 0; it < total; ++it) {
      // next deposit in source order: the smallest bucket head
      int best = 0, bs = head[0];
#pragma unroll
      for (int b = 1; b < NC; ++b)
        if (head[b] < bs) {
          bs = head[b];
          best = b;
        }
      int bp = 0;
#pragma unroll
      for (int b = 0; b < NC; ++b)
        if (b == best) {
          bp = pos[b];
          ++pos[b];
          head[b] = pos[b] < end[b] ? A.bucket[pos[b]] : INT_MAX;
        }
      const double wt = pos_weight(A, bp, best);  // 0 on a clamped axis's upper corner
      if (wt != 0.0) rho += wt;
    }
    A.out[t] = A.target ? A.target[t] - rho : rho;
  }
}

// The <= 2^d neighbouring cells of target t whose buckets are non-empty.
struct TargetBuckets {
  int pos[8], end[8], bits[8];
  int nl, K;
};
__device__ __forceinline__ void target_buckets(const GatherArgs& A, long t, TargetBuckets& tb) {
  const GridDesc& g = A.g;
  int id[3] = {0, 0, 0};
  node_idx(g, t, id);
  id[0] += A.row_off;
  tb.nl = 0;
  tb.K = 0;
  for (int b = 0; b < (1 << g.d); ++b) {
    long c = t + A.cell_shift;
    bool ok = true;
    for (int a = 0; a < g.d; ++a)
      if ((b >> a) & 1) {
        if (id[a] == 0) ok = false;
        c -= g.stride[a];
      }
    if (!ok) continue;
    const int k = A.end[c] - A.off[c];
    if (k <= 0) continue;
    tb.pos[tb.nl] = A.off[c];
    tb.end[tb.nl] = A.end[c];
    tb.bits[tb.nl] = b;
    tb.K += k;
    ++tb.nl;
  }
}

// target_buckets with the 2^d bucket-bound loads issued by the lanes of one
// warp in parallel (lane b: corner b), compacted in corner order by ballot.
// Call from all 32 lanes; every lane returns the same nl, K and, for
// slot < nl, pos/len/bits of the slot-th non-empty bucket in lane `slot`.
struct LaneBucket {
  int nl, K, pos, len, bits;
};
__device__ __forceinline__ LaneBucket target_buckets_warp(const GatherArgs& A, long t) {
  const GridDesc& g = A.g;
  const int lane = threadIdx.x & 31;
  int id[3] = {0, 0, 0};
  node_idx(g, t, id);
  id[0] += A.row_off;
  int pos = 0, len = 0;
  bool ok = lane < (1 << g.d);
  if (ok) {
    long c = t + A.cell_shift;
    for (int a = 0; a < g.d; ++a)
      if ((lane >> a) & 1) {
        if (id[a] == 0) ok = false;
        c -= g.stride[a];
      }
    if (ok) {
      pos = A.off[c];
      len = A.end[c] - pos;
      ok = len > 0;
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, ok);
  LaneBucket r;
  r.nl = __popc(m);
  int K = ok ? len : 0;
  for (int o = 16; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
  r.K = K;
  // the slot-th set bit of m, for slot = lane
  int src = 0;
  {
    unsigned mm = m;
    for (int i = 0; i < lane && mm; ++i) mm &= mm - 1;
    src = mm ? __ffs(mm) - 1 : 0;
  }
  r.pos = __shfl_sync(0xffffffffu, pos, src);
  r.len = __shfl_sync(0xffffffffu, len, src);
  r.bits = src;
  return r;
}

__device__ __forceinline__ int lower_bound_ids(const int* v, int len, int key) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Sequential fold of w[0..K) from +0.0 by one warp, bit for bit the
// reference's loop (zero weights leave rho unchanged: see the medium tier):
// the lanes load 32 consecutive weights per round (coalesced, one round
// ahead of the chain) and every lane runs the same chain of adds fed by
// shuffles. Call from all 32 lanes of the warp.
__device__ __forceinline__ double warp_seq_fold(const double* w, int K) {
  const int lane = threadIdx.x & 31;
  double rho = 0.0;
  double nxt = lane < K ? w[lane] : 0.0;
  for (int c = 0; c < K; c += 32) {
    const double v = nxt;
    nxt = c + 32 + lane < K ? w[c + 32 + lane] : 0.0;
    const int cnt = min(32, K - c);
    if (cnt == 32) {
#pragma unroll
      for (int i0 = 0; i0 < 32; i0 += 8) {
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __shfl_sync(0xffffffffu, v, i0 + i);
#pragma unroll
        for (int i = 0; i < 8; ++i) rho += x[i];
      }
    } else {
      for (int i = 0; i < cnt; ++i) rho += __shfl_sync(0xffffffffu, v, i);
    }
  }
  return rho;
}

// Group-wide merge (threads gt of ng) of the sorted runs A = x[a0, a0 + la)
// and B = x[a0 + la, a0 + la + lb) (source ids, unique) with their 16-bit
// payloads into y/py[a0, ...): merge path, each thread emits a contiguous
// output range after one binary search for its split.
__device__ __forceinline__ void group_merge2(const int* x, const uint16_t* px, int* y, uint16_t* py, int a0,
                                            int la, int lb, int gt, int ng) {
  const int tot = la + lb;
  const int per = (tot + ng - 1) / ng;
  const int d0 = min(tot, gt * per), d1 = min(tot, d0 + per);
  if (d0 >= d1) return;
  const int* A = x + a0;
  const int* B = A + la;
  // split: i elements from A and d0 - i from B precede output d0
  int lo = max(0, d0 - lb), hi = min(d0, la);
  while (lo < hi) {
    const int i = (lo + hi) >> 1;
    if (A[i] < B[d0 - i - 1]) lo = i + 1;
    else hi = i;
  }
  int i = lo, j = d0 - lo;
  for (int d = d0; d < d1; ++d) {
    const bool takeA = j >= lb || (i < la && A[i] < B[j]);
    if (takeA) {
      y[a0 + d] = A[i];
      py[a0 + d] = px[a0 + i];
      ++i;
    } else {
      y[a0 + d] = B[j];
      py[a0 + d] = px[a0 + la + j];
      ++j;
    }
  }
}

// Merge tree over the runs listed in tab (tab[r]: start, tab[8 + r]: length;
// adjacent in x/px) by the group (threads gt of ng, `bar` synchronises it).
// Returns in x/px the buffer holding the merged sequence.
template <class Sync>
__device__ __forceinline__ void group_merge_runs(int*& x, uint16_t*& px, int*& y, uint16_t*& py, int* tab,
                                                int runs, int gt, int ng, Sync bar) {
  while (runs > 1) {
    for (int r = 0; r + 1 < runs; r += 2) group_merge2(x, px, y, py, tab[r], tab[8 + r], tab[8 + r + 1], gt, ng);
    if (runs & 1) {  // the odd run is copied across
      const int a0 = tab[runs - 1], l0 = tab[8 + runs - 1];
      for (int i = gt; i < l0; i += ng) {
        y[a0 + i] = x[a0 + i];
        py[a0 + i] = px[a0 + i];
      }
    }
    bar();
    const int nr = (runs + 1) >> 1;
    if (gt == 0)
      for (int r = 0; r < nr; ++r) {
        const int l0 = tab[8 + 2 * r] + (2 * r + 1 < runs ? tab[8 + 2 * r + 1] : 0);
        tab[r] = tab[2 * r];
        tab[8 + r] = l0;
      }
    bar();
    runs = nr;
    int* ti = x;
    x = y;
    y = ti;
    uint16_t* tp = px;
    px = py;
    py = tp;
  }
}

// Medium targets (kLight < K <= kMedium): one warp each. The <= 2^d sorted
// buckets (source ids) are staged in shared memory with a 16-bit payload
// (corner bit, index in the bucket) and merged by a log2(buckets)-level tree
// of merge-path merges; the merged order is the source order, the order in
// which the reference adds the deposits. Weights are then written in that
// order to the warp's slice of a global buffer and folded sequentially.
template <int D>
__global__ void __launch_bounds__(kMedWarps * 32) pf_gather_medium_kernel(GatherArgs A,
                                                                         const int* heavy,
                                                                         const int* nheavy,
                                                                         double* hbuf) {
  constexpr int NC = 1 << D;
  extern __shared__ __align__(16) unsigned char med_smem[];
  __shared__ int med_tab[kMedWarps][2 * 8 + 8];  // run starts, run lengths, bucket start per corner
  const GridDesc& g = A.g;
  const int nh = nheavy[0];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int* idsA = reinterpret_cast<int*>(med_smem) + wib * (2 * kMedium);
  int* idsB = idsA + kMedium;
  uint16_t* payA = reinterpret_cast<uint16_t*>(reinterpret_cast<int*>(med_smem) + kMedWarps * 2 * kMedium) +
                   wib * (2 * kMedium);
  uint16_t* payB = payA + kMedium;
  int* tab = med_tab[wib];
  const long warp0 = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
  double* buf = hbuf + warp0 * kMedium;  // the warp's private slice (K <= kMedium)
  for (long q = warp0; q < nh; q += nwarps) {
    const long t = heavy[q];
    int id[3] = {0, 0, 0};
    node_idx(g, t, id);
    id[0] += A.row_off;
    int pos[NC], len[NC];
    int K = 0, nl = 0;
#pragma unroll
    for (int b = 0; b < NC; ++b) {
      long c = t + A.cell_shift;
      bool ok = true;
#pragma unroll
      for (int a = 0; a < D; ++a)
        if ((b >> a) & 1) {
          if (id[a] == 0) ok = false;
          c -= g.stride[a];
        }
      pos[b] = ok ? A.off[c] : 0;
      len[b] = ok ? A.end[c] - pos[b] : 0;
      if (lane == 0) {
        tab[16 + b] = pos[b];
        if (len[b] > 0) {
          tab[nl] = K;
          tab[8 + nl] = len[b];
        }
      }
      if (len[b] > 0) ++nl;
      K += len[b];
    }
    // stage the runs: ids and (corner << 9 | index) payloads (len <= 512)
#pragma unroll
    for (int b = 0, o = 0; b < NC; ++b) {
      for (int i = lane; i < len[b]; i += 32) {
        idsA[o + i] = A.bucket[pos[b] + i];
        payA[o + i] = static_cast<uint16_t>((b << 9) | i);
      }
      o += len[b];
    }
    __syncwarp();
    // merge tree: runs r and r+1 are adjacent; each level halves the runs
    int* xs = idsA;
    int* ys = idsB;
    uint16_t* px = payA;
    uint16_t* py = payB;
    group_merge_runs(xs, px, ys, py, tab, nl, lane, 32, [] { __syncwarp(); });
    // weights in source order
    for (int r = lane; r < K; r += 32) {
      const int pl = px[r];
      const int b = pl >> 9;
      buf[r] = pos_weight(A, tab[16 + b] + (pl & 511), b);
    }
    __syncwarp();
    // Starting from +0.0, rho can never become -0.0, so adding a zero weight
    // leaves it unchanged: folding every weight equals the reference's skip
    // of zero weights bit for bit.
    const double rho = warp_seq_fold(buf, K);
    if (lane == 0) A.out[t] = A.target ? A.target[t] - rho : rho;
    __syncwarp();
  }
}

// Large targets (kMedium < K <= kLarge): one CTA of kLargeThreads each, ids
// staged in shared memory, ranks and weights as above into the CTA's slice of
// the global buffer, then one thread folds them in order (unrolled loads
// ahead of the chain of adds).
// Two instantiations: LK = 2048 (24 KB of shared memory, twice the CTAs per
// SM) for kMedium < K <= 2048 and LK = kLarge for 2048 < K <= kLarge; the
// second list is stored from the back of `large` / `lmeta` (list = 1).
template <int LK>
__global__ void __launch_bounds__(kLargeThreads) pf_gather_large_kernel(GatherArgs A,
                                                                       const int* large,
                                                                       int* nheavy,
                                                                       double* hbuf,
                                                                       unsigned long long* hfill,
                                                                       long long* lmeta, long lcap,
                                                                       int list) {
  // the target's buckets (source ids) are merged by a merge-path tree in
  // shared memory, as in the warp tier, with 16-bit (run << 12 | index)
  // payloads; the weights then go to the CTA's buffer slice in source order
  extern __shared__ __align__(16) unsigned char large_smem[];
  __shared__ int tab[24];  // run starts, run lengths (merge tree)
  __shared__ int s_pos[8], s_bits[8], s_nl, s_K, s_q;
  int* idsA = reinterpret_cast<int*>(large_smem);
  int* idsB = idsA + LK;
  uint16_t* payA = reinterpret_cast<uint16_t*>(idsB + LK);
  uint16_t* payB = payA + LK;
  const int nl_total = nheavy[list ? 7 : 4];
  __shared__ unsigned long long s_base;
  for (;;) {  // targets claimed from a counter (nheavy[6] / [8], zeroed per call)
    if (threadIdx.x == 0) s_q = atomicAdd(nheavy + (list ? 8 : 6), 1);
    __syncthreads();
    const int q = s_q;
    if (q >= nl_total) break;
    const long t = list ? large[A.g.size - 1 - q] : large[q];
    const long mq = list ? lcap - 1 - q : q;
    if (threadIdx.x < 32) {  // bucket bounds: one lane per corner, loads in parallel
      const LaneBucket lb = target_buckets_warp(A, t);
      int start = lb.len;  // exclusive prefix of the slot lengths (slots < nl)
      if (threadIdx.x >= lb.nl) start = 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, start, o);
        if (static_cast<int>(threadIdx.x) >= o) start += v;
      }
      if (static_cast<int>(threadIdx.x) < lb.nl) {
        tab[threadIdx.x] = start - lb.len;
        tab[8 + threadIdx.x] = lb.len;
        s_pos[threadIdx.x] = lb.pos;
        s_bits[threadIdx.x] = lb.bits;
      }
      if (threadIdx.x == 0) {
        s_nl = lb.nl;
        s_K = lb.K;
        // the target's slice of hbuf (shared counter with the heavy tier)
        s_base = atomicAdd(hfill, static_cast<unsigned long long>(lb.K));
        lmeta[mq] = static_cast<long long>((s_base << 13) | static_cast<unsigned long long>(lb.K));
      }
    }
    __syncthreads();
    const int nl = s_nl;
    const int K = s_K;
    double* buf = hbuf + s_base;
    for (int qq = 0; qq < nl; ++qq) {
      const int o = tab[qq], len = tab[8 + qq], p0 = s_pos[qq];
      for (int i = threadIdx.x; i < len; i += blockDim.x) {
        idsA[o + i] = A.bucket[p0 + i];
        payA[o + i] = static_cast<uint16_t>((qq << 12) | i);
      }
    }
    __syncthreads();
    int* xs = idsA;
    int* ys = idsB;
    uint16_t* px = payA;
    uint16_t* py = payB;
    group_merge_runs(xs, px, ys, py, tab, nl, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    for (int r = threadIdx.x; r < K; r += blockDim.x) {
      const int pl = px[r];
      const int qq = pl >> 12;
      buf[r] = pos_weight(A, s_pos[qq] + (pl & 4095), s_bits[qq]);
    }
    __syncthreads();
    // the sequential fold runs in pf_fold_large_kernel (one warp per target,
    // many targets in flight per SM) instead of one warp of this CTA
  }
}

// Folds of the large tier's weight lists (written in source order by
// pf_gather_large_kernel): one warp per target, bit for bit the reference's
// sequential scatter sum (warp_seq_fold).
__global__ void __launch_bounds__(256) pf_fold_large_kernel(GatherArgs A, const int* large, const int* nheavy,
                                                          const double* hbuf, const long long* lmeta, long lcap) {
  const int na = nheavy[4], nb = nheavy[7];
  const int nt = static_cast<int>(gridDim.x * blockDim.x);
  if (na + nb < nt) {
    // few targets (C3): one warp per target, coalesced loads a round ahead of
    // the chain (a lone thread would wait on every sector)
    const int lane = threadIdx.x & 31;
    const int nw = nt >> 5;
    for (int q = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5); q < na + nb; q += nw) {
      const bool b = q >= na;
      const unsigned long long m = static_cast<unsigned long long>(lmeta[b ? lcap - 1 - (q - na) : q]);
      const double rho = warp_seq_fold(hbuf + (m >> 13), static_cast<int>(m & 8191ull));
      if (lane == 0) {
        const long t = b ? large[A.g.size - 1 - (q - na)] : large[q];
        A.out[t] = A.target ? A.target[t] - rho : rho;
      }
    }
    return;
  }
  // many targets (C4: ~10^5 per call): one target per THREAD, 32 independent
  // add chains per warp (the chains, not the loads, bound the warp version)
  for (int q = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); q < na + nb; q += nt) {
    const bool b = q >= na;
    const unsigned long long m = static_cast<unsigned long long>(lmeta[b ? lcap - 1 - (q - na) : q]);
    const int K = static_cast<int>(m & 8191ull);
    const double* w = hbuf + (m >> 13);
    double rho = 0.0;
    int i = 0;
    for (; i + 8 <= K; i += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = w[i + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) rho += v[u];
    }
    for (; i < K; ++i) rho += w[i];
    const long t = b ? large[A.g.size - 1 - (q - na)] : large[q];
    A.out[t] = A.target ? A.target[t] - rho : rho;
  }
}

// Heavy targets (K > kLarge): one CTA each, same merge-rank scheme with the
// ids in shared memory when they fit (else ranked against global memory),
// weights to the global buffer, then the CTA folds them (exact_fold.cuh).
__global__ void __launch_bounds__(512, 2) pf_gather_heavy_kernel(GatherArgs A, const int* heavy,
                                                             int* nheavy, double* hbuf,
                                                             unsigned long long* hfill) {
  __shared__ int s_pos[8], s_end[8], s_bits[8], s_cat[8], s_nl, s_K;
  __shared__ unsigned long long s_base;
  __shared__ int s_q;
  __shared__ FoldTr fold_scr[512 / 32 + 1];
  __shared__ int fold_iscr[512 / 32];
  extern __shared__ int ids[];  // [kHeavyIds]
  const GridDesc& g = A.g;
  const int nh = nheavy[1];
  // targets are claimed from a counter (nheavy[5], zeroed per call): their
  // costs differ by orders of magnitude, so a static stride leaves CTAs idle
  for (;;) {
    if (threadIdx.x == 0) s_q = atomicAdd(nheavy + 5, 1);
    __syncthreads();
    const int q = s_q;
    if (q >= nh) break;
    const long t = heavy[g.size - 1 - q];
    if (threadIdx.x == 0) {
      TargetBuckets tb;
      target_buckets(A, t, tb);
      for (int qq = 0, o = 0; qq < tb.nl; ++qq) {
        s_pos[qq] = tb.pos[qq];
        s_end[qq] = tb.end[qq];
        s_bits[qq] = tb.bits[qq];
        s_cat[qq] = o;
        o += tb.end[qq] - tb.pos[qq];
      }
      s_nl = tb.nl;
      s_K = tb.K;
      s_base = atomicAdd(hfill, static_cast<unsigned long long>(tb.K));
    }
    __syncthreads();
    const int nl = s_nl;
    const int K = s_K;
    const bool staged = K <= kHeavyIds;
    if (staged)
      for (int qq = 0; qq < nl; ++qq)
        for (int i = threadIdx.x; i < s_end[qq] - s_pos[qq]; i += blockDim.x)
          ids[s_cat[qq] + i] = A.bucket[s_pos[qq] + i];
    __syncthreads();
    double* buf = hbuf + s_base;
    for (int qq = 0; qq < nl; ++qq) {
      const int p0 = s_pos[qq], len = s_end[qq] - p0, b = s_bits[qq];
      for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const int src = staged ? ids[s_cat[qq] + i] : A.bucket[p0 + i];
        int fin = i;
        for (int o = 0; o < nl; ++o) {
          if (o == qq) continue;
          fin += staged ? lower_bound_ids(ids + s_cat[o], s_end[o] - s_pos[o], src)
                        : lower_bound_ids(A.bucket + s_pos[o], s_end[o] - s_pos[o], src);
        }
        buf[fin] = pos_weight(A, p0 + i, b);
      }
    }
    __syncthreads();
    // up to kSeqFold deposits a warp's sequential chain is cheaper than the
    // parallel fold's transducer scans and binade restarts
    if (K <= kSeqFold) {
      if (threadIdx.x < 32) {
        const double rho = warp_seq_fold(buf, K);
        if (threadIdx.x == 0) A.out[t] = A.target ? A.target[t] - rho : rho;
      }
    } else {
      const double rho = exact_fold<512, 8>(buf, K, fold_scr, fold_iscr, [] { __syncthreads(); });
      if (threadIdx.x == 0) A.out[t] = A.target ? A.target[t] - rho : rho;
    }
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

// ---- multi-GPU deposit-record routing (dist.py route_records) --------------
// Every source with mass becomes a record for the owner of its lo-corner row
// i0 and, unless clamped on axis 0, for the owner of row i0 + 1 when that is
// another rank. Records are packed (3 + d doubles: key relative to the
// destination's cells as raw bits, mass, d weights, clamp mask) grouped by
// destination and, within a destination, in source order (stable block
// ranks; same scheme as the radix scatter).
constexpr int kRouteThreads = 256;
constexpr int kRouteItems = 8;
constexpr int kRouteTile = kRouteThreads * kRouteItems;
constexpr int kMaxRanks = 64;

struct RouteArgs {
  const uint32_t* key;
  const uint8_t* cmask;
  const double* w;
  const double* mass;
  long nloc;
  long N;       // global sentinel
  long M;       // nodes per row
  int n0;
  int d;
  int P;
  const int* row0;  // [P + 1] row starts (row0[P] = n0)
  int* bcount;      // [P * nblocks] per-destination counts (dest-major)
  double* packed;
};

__device__ __forceinline__ int route_owner(const RouteArgs& A, long row) {
  int lo = 0, hi = A.P - 1;  // largest q with row0[q] <= row
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (A.row0[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void route_dests(const RouteArgs& A, long s, int& d1, int& d2) {
  d1 = d2 = -1;
  if (s >= A.nloc) return;
  const long k = A.key[s];
  if (k == A.N) return;
  const long i0 = k / A.M;
  d1 = route_owner(A, i0);
  if (!(A.cmask[s] & 1u) && i0 + 1 < A.n0) {
    const int q = route_owner(A, i0 + 1);
    if (q != d1) d2 = q;
  }
}

__global__ void __launch_bounds__(kRouteThreads) route_count_kernel(RouteArgs A, long nblocks) {
  __shared__ int cnt[kMaxRanks];
  for (int q = threadIdx.x; q < A.P; q += blockDim.x) cnt[q] = 0;
  __syncthreads();
  const long base = static_cast<long>(blockIdx.x) * kRouteTile;
  for (int r = 0; r < kRouteItems; ++r) {
    int d1, d2;
    route_dests(A, base + static_cast<long>(r) * kRouteThreads + threadIdx.x, d1, d2);
    if (d1 >= 0) atomicAdd(&cnt[d1], 1);
    if (d2 >= 0) atomicAdd(&cnt[d2], 1);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < A.P; q += blockDim.x) A.bcount[static_cast<long>(q) * nblocks + blockIdx.x] = cnt[q];
}

// exclusive scan of m ints in place, one CTA (m = P * nblocks, small)
__global__ void __launch_bounds__(1024) route_scan_kernel(int* a, long m, int* total) {
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long b0 = 0; b0 < m; b0 += 1024) {
    const long i = b0 + threadIdx.x;
    const int v = i < m ? a[i] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      int t = wsum[lane];
      int ti = t;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      wsum[lane] = ti - t;
    }
    __syncthreads();
    if (i < m) a[i] = carry + wsum[w] + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += wsum[31] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kRouteThreads) route_scatter_kernel(RouteArgs A, long nblocks) {
  constexpr int kW = kRouteThreads / 32;
  __shared__ int base[kMaxRanks];
  __shared__ int wcnt[kW][kMaxRanks];
  for (int q = threadIdx.x; q < A.P; q += blockDim.x)
    base[q] = A.bcount[static_cast<long>(q) * nblocks + blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int rec = 3 + A.d;
  const long b0 = static_cast<long>(blockIdx.x) * kRouteTile;
  for (int r = 0; r < kRouteItems; ++r) {
    const long s = b0 + static_cast<long>(r) * kRouteThreads + threadIdx.x;
    int d1, d2;
    route_dests(A, s, d1, d2);
    int pos1 = 0, pos2 = 0;
    for (int q = 0; q < A.P; ++q) {
      const unsigned m = __ballot_sync(0xffffffffu, d1 == q || d2 == q);
      if (lane == 0) wcnt[warp][q] = __popc(m);
      if (d1 == q) pos1 = __popc(m & lt);
      if (d2 == q) pos2 = __popc(m & lt);
    }
    __syncthreads();
    if (d1 >= 0 || d2 >= 0) {
      for (int h = 0; h < 2; ++h) {
        const int q = h == 0 ? d1 : d2;
        if (q < 0) continue;
        int pre = 0;
        for (int ww = 0; ww < warp; ++ww) pre += wcnt[ww][q];
        const long pos = static_cast<long>(base[q]) + pre + (h == 0 ? pos1 : pos2);
        double* out = A.packed + pos * rec;
        const long rel = static_cast<long>(A.key[s]) - (static_cast<long>(A.row0[q]) - 1) * A.M;
        out[0] = __longlong_as_double(rel);
        out[1] = A.mass[s];
        for (int a = 0; a < A.d; ++a) out[2 + a] = A.w[a * A.nloc + s];
        out[2 + A.d] = static_cast<double>(A.cmask[s]);
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < A.P; q += blockDim.x) {
      int tot = 0;
      for (int ww = 0; ww < kW; ++ww) tot += wcnt[ww][q];
      base[q] += tot;
    }
    __syncthreads();
  }
}

// packed records (received, in sender order) -> the gather's SoA inputs
__global__ void route_unpack_kernel(const double* packed, long nrec, int d, uint32_t* keys,
                                    double* mass, double* w, uint8_t* cmask) {
  const int rec = 3 + d;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < nrec;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double* in = packed + i * rec;
    keys[i] = static_cast<uint32_t>(__double_as_longlong(in[0]));
    mass[i] = in[1];
    for (int a = 0; a < d; ++a) w[a * nrec + i] = in[2 + a];
    cmask[i] = static_cast<uint8_t>(in[2 + d]);
  }
}

}  // namespace

PushforwardPlan::~PushforwardPlan() {
  for (void* p : {static_cast<void*>(key_), static_cast<void*>(cmask_), static_cast<void*>(w_),
                  static_cast<void*>(heavy_), static_cast<void*>(nheavy_) /* with off_, end_ */,
                  static_cast<void*>(hbuf_),
                  static_cast<void*>(row0_), static_cast<void*>(bcount_),
                  static_cast<void*>(large_), static_cast<void*>(wts_),
                  static_cast<void*>(lmeta_)})
    if (p) dfree(p);
  if (hcounts_) cudaFreeHost(hcounts_);
}

void PushforwardPlan::init(const GridDesc& g) { setup(g, g, 0, false); }

void PushforwardPlan::init_slab(const GridDesc& global, int row0, int nrows) {
  if (global.d < 2) throw std::invalid_argument("pushforward: slabs need d >= 2");
  int ext[3] = {nrows, global.n[1], global.d > 2 ? global.n[2] : 1};
  setup(make_grid(global.d, ext), global, row0, true);
}

// loc: target/source nodes of this plan (the grid, or rows [row0, row0 +
// nrows) of it); global: the problem grid. A slab's cells start one row above
// its first row (deposits from the cell row above reach its first row).
void PushforwardPlan::setup(const GridDesc& loc, const GridDesc& global, int row0, bool slab) {
  g_ = loc;
  gg_ = global;
  row_off_ = row0;
  cell_shift_ = slab ? loc.stride[0] : 0;
  ncells_ = slab ? loc.size + loc.stride[0] : loc.size;
  if (global.size >= (1L << 29)) throw std::invalid_argument("pushforward: grid too large");
  const long N = loc.size;
  BFM_CUDA(dmalloc(&key_, N * sizeof(uint32_t)));
  BFM_CUDA(dmalloc(&cmask_, N));
  BFM_CUDA(dmalloc(&w_, g_.d * N * sizeof(double)));
  // the per-call counters and the bucket bounds share one allocation so one
  // memset clears them: [64 bytes of counters][off][end]
  {
    unsigned char* pool = nullptr;
    BFM_CUDA(dmalloc(&pool, 64 + 2 * (ncells_ + 1) * sizeof(int)));
    nheavy_ = reinterpret_cast<unsigned long long*>(pool);
    off_ = reinterpret_cast<int*>(pool + 64);
    end_ = off_ + ncells_ + 1;
  }
  BFM_CUDA(dmalloc(&heavy_, (N + 1) * sizeof(int)));
  BFM_CUDA(dmalloc(&large_, (N + 1) * sizeof(int)));
  // large-tier fold list: fewer than 2^d N / (kMedium + 1) targets
  lmeta_cap_ = (8 * N) / (kMedium + 1) + 2;
  BFM_CUDA(dmalloc(&lmeta_, lmeta_cap_ * sizeof(long long)));
  // per-call counters, zeroed by gather(); as ints: [0] warp-tier targets,
  // [1] heavy targets, [2..3] heavy buffer fill (one u64), [4] CTA-tier
  // targets, [5] / [6] heavy / CTA-tier work claims, [7] unused
  ensure_records(N);
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_large_kernel<kLarge>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kLargeSmem));
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_large_kernel<kLargeA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kLargeSmemA));
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_heavy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kHeavySmem));
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_medium_kernel<1>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kMedSmem));
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_medium_kernel<2>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kMedSmem));
  BFM_CUDA(cudaFuncSetAttribute(pf_gather_medium_kernel<3>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, kMedSmem));
  key_bits_ = 1;
  while ((1L << key_bits_) <= ncells_) ++key_bits_;  // cells 0..ncells-1 plus the sentinel
}

void PushforwardPlan::ensure_records(long nrec) {
  if (nrec <= rec_cap_ && hbuf_) return;
  const long cap = std::max<long>(nrec, 1);
  if (hbuf_) {
    dfree(hbuf_);
    hbuf_ = nullptr;
  }
  const long deposits = (static_cast<long>(1) << g_.d) * cap;
  med_blocks_ = static_cast<int>(std::max<long>(1, std::min<long>(kMedBlocks, deposits / (kMedWarps * kMedium))));
  large_blocks_ = static_cast<int>(std::max<long>(1, std::min<long>(kLargeBlocks, deposits / kLarge)));
  const long hcap = std::max<long>(deposits, std::max<long>(static_cast<long>(med_blocks_) * kMedWarps * kMedium,
                                                            static_cast<long>(large_blocks_) * kLarge));
  BFM_CUDA(dmalloc(&hbuf_, hcap * sizeof(double)));
  if (wts_) dfree(wts_);
  BFM_CUDA(dmalloc(&wts_, cap * sizeof(double) * (1L << g_.d)));  // 2^d corner weights per record
  sorter_.init(cap);
  rec_cap_ = cap;
}

void PushforwardPlan::set_cost(const double* exponents) {
  for (int a = 0; a < 3; ++a) {
    iexp_[a] = 0.0;
    if (exponents && a < g_.d && exponents[a] != 2.0) {
      if (!(exponents[a] > 1.0)) throw std::invalid_argument("cost exponents must satisfy p > 1");
      iexp_[a] = 1.0 / (exponents[a] - 1.0);  // cost.hpp:65, the same IEEE expression
    }
  }
}

namespace {
void launch_map(const MapArgs& A, cudaStream_t stream) {
  const bool power = A.iexp[0] > 0.0 || A.iexp[1] > 0.0 || A.iexp[2] > 0.0;
  if (power) pf_map_kernel<true><<<grid_for(A.g.size, 256), 256, 0, stream>>>(A);
  else pf_map_kernel<false><<<grid_for(A.g.size, 256), 256, 0, stream>>>(A);
}

MapArgs map_args(const GridDesc& g, const GridDesc& gg, int row_off, long cell_shift, const double* iexp) {
  MapArgs A{};
  A.g = g;
  A.gg = gg;
  A.row_off = row_off;
  A.u_shift = cell_shift;  // a slab's u carries one halo row on each side
  A.scale = 1.0;
  A.diam = std::sqrt(static_cast<double>(g.d));
  for (int a = 0; a < 3; ++a) A.iexp[a] = iexp[a];
  return A;
}
}  // namespace

void PushforwardPlan::map_only(const double* d_u, double* d_disp, cudaStream_t stream,
                               LaunchCounter* lc) {
  MapArgs A = map_args(g_, gg_, row_off_, cell_shift_, iexp_);
  A.u = d_u;
  A.disp_out = d_disp;
  launch_map(A, stream);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
}

void PushforwardPlan::map_records(const double* d_u_ext, const double* d_source, uint32_t* d_key,
                                  double* d_w, uint8_t* d_cmask, double* d_disp_out,
                                  cudaStream_t stream, LaunchCounter* lc) {
  MapArgs A = map_args(g_, gg_, row_off_, cell_shift_, iexp_);
  A.u = d_u_ext;
  A.src = d_source;
  A.key = d_key;
  A.cmask = d_cmask;
  A.w = d_w;
  A.disp_out = d_disp_out;
  A.binning = 1;
  launch_map(A, stream);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
}

void PushforwardPlan::gather(long nrec, const uint32_t* d_keys, const double* d_mass,
                             const double* d_w, const uint8_t* d_cmask, const double* d_target,
                             double* d_out, cudaStream_t stream, LaunchCounter* lc) {
  ensure_records(nrec);
  const long N = g_.size;
  BFM_CUDA(cudaMemsetAsync(nheavy_, 0, 64 + 2 * (ncells_ + 1) * sizeof(int), stream));  // counters, off, end
  const int* svals = nullptr;
  if (nrec > 0) {
    const uint32_t* skeys = nullptr;
    // massless sources (sentinel keys) deposit nothing: a stable compaction
    // drops them before the sort (their count stays on the device)
    const uint32_t sentinel = static_cast<uint32_t>(ncells_);
    // One-sweep up to 2^24 records (C1: pushforward 0.33 -> 0.25 ms per
    // iteration, C2 0.56 -> 0.48, C3 3.83 -> 3.70); above that the look-back
    // chain over the many tiles makes it a wash (C4: 24.43 vs 24.46 ms), so
    // the multi-kernel passes stay. BFM_PF_SORT=legacy|onesweep overrides (A/B).
    static const char* sort_mode = getenv("BFM_PF_SORT");
    const bool onesweep = sort_mode ? sort_mode[0] == 'o' : nrec <= (1L << 24);
    if (onesweep) {
      // one-sweep: digit histograms in one read of the keys, one scatter
      // kernel per digit (decoupled look-back), sentinels dropped by the
      // first pass, the packed records written by the last
      // (the records are packed after the sort: in sorted order the source
      // ids of neighbouring positions are close, so the gathers coalesce;
      // fused into the last scatter they cost 4x the separate kernel)
      const int* d_n = sorter_.sort_onesweep(d_keys, nrec, sentinel, key_bits_, stream, lc, &skeys, &svals);
      pf_pack_kernel<<<grid_for(nrec, 256), 256, 0, stream>>>(skeys, sentinel, off_, end_, svals, nrec, d_n, d_mass,
                                                               d_w, d_cmask, g_.d, wts_);
      BFM_LAUNCH_CHECK("pf_pack_kernel");
    } else {
      const uint32_t* ckeys = nullptr;
      const int* cvals = nullptr;
      const int* d_n = sorter_.compact(d_keys, nrec, sentinel, stream, lc, &ckeys, &cvals);
      sorter_.sort(ckeys, cvals, nrec, key_bits_, stream, lc, &skeys, &svals, d_n);
      pf_pack_kernel<<<grid_for(nrec, 256), 256, 0, stream>>>(skeys, sentinel, off_, end_, svals, nrec, d_n, d_mass,
                                                               d_w, d_cmask, g_.d, wts_);
      BFM_LAUNCH_CHECK("pf_pack_kernel");
    }
  }
  GatherArgs G{};
  G.g = g_;
  G.row_off = row_off_;
  G.cell_shift = cell_shift_;
  G.nrec = nrec;
  G.end = end_;
  G.off = off_;
  G.bucket = svals;
  G.cmask = d_cmask;
  G.w = d_w;
  G.src = d_mass;
  G.target = d_target;
  G.out = d_out;
  G.wts = wts_;
  int* nheavy = reinterpret_cast<int*>(nheavy_);
  if (g_.d == 1) pf_gather_kernel<1><<<grid_for(N, 256), 256, 0, stream>>>(G, heavy_, large_, nheavy);
  else if (g_.d == 2) pf_gather_kernel<2><<<grid_for(N, 256), 256, 0, stream>>>(G, heavy_, large_, nheavy);
  else pf_gather_kernel<3><<<grid_for(N, 256), 256, 0, stream>>>(G, heavy_, large_, nheavy);
  BFM_LAUNCH_CHECK("pf_gather_kernel");
  if (g_.d == 1)
    pf_gather_medium_kernel<1><<<med_blocks_, kMedWarps * 32, kMedSmem, stream>>>(G, heavy_, nheavy, hbuf_);
  else if (g_.d == 2)
    pf_gather_medium_kernel<2><<<med_blocks_, kMedWarps * 32, kMedSmem, stream>>>(G, heavy_, nheavy, hbuf_);
  else
    pf_gather_medium_kernel<3><<<med_blocks_, kMedWarps * 32, kMedSmem, stream>>>(G, heavy_, nheavy, hbuf_);
  BFM_LAUNCH_CHECK("pf_gather_medium_kernel");
  const long lcap = lmeta_cap_;
  pf_gather_large_kernel<kLargeA><<<2 * large_blocks_, kLargeThreads, kLargeSmemA, stream>>>(
      G, large_, nheavy, hbuf_, nheavy_ + 1, lmeta_, lcap, 0);
  BFM_LAUNCH_CHECK("pf_gather_large_kernel<2048>");
  pf_gather_large_kernel<kLarge><<<large_blocks_, kLargeThreads, kLargeSmem, stream>>>(
      G, large_, nheavy, hbuf_, nheavy_ + 1, lmeta_, lcap, 1);
  BFM_LAUNCH_CHECK("pf_gather_large_kernel<4096>");
  pf_fold_large_kernel<<<148 * 4, 128, 0, stream>>>(G, large_, nheavy, hbuf_, lmeta_, lcap);
  BFM_LAUNCH_CHECK("pf_fold_large_kernel");
  pf_gather_heavy_kernel<<<2 * 148, 512, kHeavySmem, stream>>>(G, heavy_, nheavy, hbuf_, nheavy_ + 1);
  BFM_LAUNCH_CHECK("pf_gather_heavy_kernel");
  if (lc) lc->add(nrec > 0 ? 7 : 6);
}

void PushforwardPlan::set_partition(int P, const int* row_starts) {
  if (P < 1 || P > kMaxRanks) throw std::invalid_argument("pushforward: 1..64 ranks supported");
  nranks_ = P;
  if (!row0_) BFM_CUDA(dmalloc(&row0_, (kMaxRanks + 1) * sizeof(int)));
  BFM_CUDA(cudaMemcpy(row0_, row_starts, (P + 1) * sizeof(int), cudaMemcpyHostToDevice));
  const long nblocks = (g_.size + kRouteTile - 1) / kRouteTile;
  if (bcount_) dfree(bcount_);
  BFM_CUDA(dmalloc(&bcount_, (static_cast<long>(P) * nblocks + 1) * sizeof(int)));
  if (!hcounts_) BFM_CUDA(cudaMallocHost(&hcounts_, (kMaxRanks + 1) * sizeof(int)));
}

void PushforwardPlan::route(const uint32_t* d_key, const double* d_w, const uint8_t* d_cmask,
                            const double* d_mass, double* d_packed, long* counts,
                            cudaStream_t stream, LaunchCounter* lc) {
  if (!nranks_) throw std::invalid_argument("pushforward: route needs set_partition");
  RouteArgs A{};
  A.key = d_key;
  A.cmask = d_cmask;
  A.w = d_w;
  A.mass = d_mass;
  A.nloc = g_.size;
  A.N = gg_.size;
  A.M = g_.stride[0];
  A.n0 = gg_.n[0];
  A.d = g_.d;
  A.P = nranks_;
  A.row0 = row0_;
  A.bcount = bcount_;
  A.packed = d_packed;
  const long nblocks = (g_.size + kRouteTile - 1) / kRouteTile;
  const long m = static_cast<long>(nranks_) * nblocks;
  route_count_kernel<<<static_cast<unsigned>(nblocks), kRouteThreads, 0, stream>>>(A, nblocks);
  // per-destination totals (before the scan turns counts into offsets)
  int* totals = bcount_ + m;  // one spare int
  route_scan_kernel<<<1, 1024, 0, stream>>>(bcount_, m, totals);
  route_scatter_kernel<<<static_cast<unsigned>(nblocks), kRouteThreads, 0, stream>>>(A, nblocks);
  BFM_LAUNCH_CHECK("pf route");
  if (lc) lc->add(3);
  // destination q's records are [offset(q, block 0), offset(q + 1, block 0))
  std::vector<int> first(nranks_ + 1);
  for (int q = 0; q < nranks_; ++q)
    BFM_CUDA(cudaMemcpyAsync(hcounts_ + q, bcount_ + static_cast<long>(q) * nblocks, sizeof(int),
                             cudaMemcpyDeviceToHost, stream));
  BFM_CUDA(cudaMemcpyAsync(hcounts_ + nranks_, totals, sizeof(int), cudaMemcpyDeviceToHost, stream));
  BFM_CUDA(cudaStreamSynchronize(stream));
  for (int q = 0; q < nranks_; ++q) counts[q] = static_cast<long>(hcounts_[q + 1]) - hcounts_[q];
}

void PushforwardPlan::unpack(const double* d_packed, long nrec, uint32_t* d_keys, double* d_mass,
                             double* d_w, uint8_t* d_cmask, cudaStream_t stream, LaunchCounter* lc) {
  if (nrec <= 0) return;
  route_unpack_kernel<<<grid_for(nrec, 256), 256, 0, stream>>>(d_packed, nrec, g_.d, d_keys, d_mass,
                                                                d_w, d_cmask);
  BFM_LAUNCH_CHECK("pf unpack");
  if (lc) lc->add();
}

void PushforwardPlan::from_potential(const double* d_u, const double* d_source,
                                     const double* d_target, double* d_out, double* d_disp_out,
                                     cudaStream_t stream, LaunchCounter* lc) {
  map_records(d_u, d_source, key_, w_, cmask_, d_disp_out, stream, lc);
  gather(g_.size, key_, d_source, w_, cmask_, d_target, d_out, stream, lc);
}

void PushforwardPlan::from_displacement(const double* d_disp, double scale,
                                        const double* d_source, double* d_rho,
                                        cudaStream_t stream, LaunchCounter* lc) {
  MapArgs A = map_args(g_, gg_, row_off_, cell_shift_, iexp_);
  A.disp = d_disp;
  A.scale = scale;
  A.src = d_source;
  A.key = key_;
  A.cmask = cmask_;
  A.w = w_;
  A.binning = 1;
  launch_map(A, stream);
  BFM_LAUNCH_CHECK("pf_map_kernel");
  if (lc) lc->add();
  gather(g_.size, key_, d_source, w_, cmask_, nullptr, d_rho, stream, lc);
}

}  // namespace bfmgpu

// ---- test hook: the parallel sequential-fold on given sequences ------------
namespace bfmgpu {
namespace {
__global__ void __launch_bounds__(512) debug_fold_kernel(const double* w, const long* off, int mode,
                                                        double* out) {
  __shared__ FoldTr scr[2 * 16 + 2];
  __shared__ int iscr[16];
  const long b = off[blockIdx.x];
  const int K = static_cast<int>(off[blockIdx.x + 1] - b);
  double r;
  if (mode == 0) {
    r = exact_fold<512, 8>(w + b, K, scr, iscr, [] { __syncthreads(); });
  } else {
    if (threadIdx.x >= 32) return;
    r = exact_fold<32, 8>(w + b, K, scr, iscr, [] { __syncwarp(); });
  }
  if (threadIdx.x == 0) out[blockIdx.x] = r;
}
}  // namespace

void debug_fold(const double* h_w, const long* h_off, int nseq, int mode, double* h_out) {
  if (nseq == 0) return;
  const long total = h_off[nseq];
  double *dw = nullptr, *dout = nullptr;
  long* doff = nullptr;
  BFM_CUDA(dmalloc(&dw, sizeof(double) * (total + 1)));
  BFM_CUDA(dmalloc(&doff, sizeof(long) * (nseq + 1)));
  BFM_CUDA(dmalloc(&dout, sizeof(double) * nseq));
  BFM_CUDA(cudaMemcpy(dw, h_w, sizeof(double) * total, cudaMemcpyHostToDevice));
  BFM_CUDA(cudaMemcpy(doff, h_off, sizeof(long) * (nseq + 1), cudaMemcpyHostToDevice));
  debug_fold_kernel<<<nseq, mode == 0 ? 512 : 32>>>(dw, doff, mode, dout);
  BFM_LAUNCH_CHECK("debug_fold_kernel");
  BFM_CUDA(cudaMemcpy(h_out, dout, sizeof(double) * nseq, cudaMemcpyDeviceToHost));
  dfree(dw);
  dfree(doff);
  dfree(dout);
}
}  // namespace bfmgpu
