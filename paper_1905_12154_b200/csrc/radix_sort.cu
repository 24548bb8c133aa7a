// Stable LSD radix sort (9-bit digits: three passes cover the 25-27-bit cell
// keys of the pushforward) of (key, value) pairs.
//
// Per pass: (1) per-tile digit histograms (digit-major), (2) exclusive scan
// of the histograms, (3) stable scatter: each tile walks its elements in
// input order in rounds of 256; within a round the rank of an element among
// equal digits is (warp-local rank via __match_any_sync) + (counts of the same
// digit in lower warps) + (running per-tile digit count), so equal keys keep
// their input order. Deterministic by construction.
#include <algorithm>
#include <stdexcept>

#include "radix_sort.cuh"

namespace bfmgpu {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kBits = 9;
constexpr int kBins = 1 << kBits;
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads) rs_hist_kernel(const uint32_t* keys, long n_max, const int* d_n,
                                                         int shift, long nblocks, int* hist) {
  const long n = d_n ? *d_n : n_max;
  __shared__ int h[kBins];
  for (int q = threadIdx.x; q < kBins; q += kThreads) h[q] = 0;
  __syncthreads();
  const long base = static_cast<long>(blockIdx.x) * kTile;
  const unsigned lane = threadIdx.x & 31u;
  uint32_t kr[kItems];  // all of the tile's loads in flight before the first use
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    kr[r] = i < n ? keys[i] : 0u;
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    const bool ok = i < n;
    const unsigned d = ok ? (kr[r] >> shift) & (kBins - 1u) : static_cast<unsigned>(kBins);
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const unsigned m = __match_any_sync(act, d);
      if ((__ffs(m) - 1) == static_cast<int>(lane)) atomicAdd(&h[d], __popc(m));
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kBins; q += kThreads) hist[static_cast<long>(q) * nblocks + blockIdx.x] = h[q];
}

__device__ int block_exscan(int v, int* total) {
  __shared__ int wt[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += u;
  }
  if (lane == 31) wt[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int t = lane < static_cast<int>(blockDim.x >> 5) ? wt[lane] : 0;
    int ti = t;
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, ti, d);
      if (lane >= d) ti += u;
    }
    wt[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  const int r = wt[w] + incl - v;
  __syncthreads();
  return r;
}

// In-place exclusive scan of m ints (m up to a few million), two levels.
constexpr int kScanTile = 1024 * 8;
__global__ void __launch_bounds__(1024) rs_scan_reduce(const int* a, long m, int* bsum) {
  __shared__ int tot;
  const long base = static_cast<long>(blockIdx.x) * kScanTile + threadIdx.x * 8;
  int s = 0;
  for (int i = 0; i < 8; ++i)
    if (base + i < m) s += a[base + i];
  block_exscan(s, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) rs_scan_top(int* bsum, long nb) {
  __shared__ int carry, tot;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long b0 = 0; b0 < nb; b0 += 1024) {
    const long i = b0 + threadIdx.x;
    const int v = i < nb ? bsum[i] : 0;
    const int ex = block_exscan(v, &tot);
    if (i < nb) bsum[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(1024) rs_scan_apply(int* a, long m, const int* bsum) {
  __shared__ int tot;
  const long base = static_cast<long>(blockIdx.x) * kScanTile + threadIdx.x * 8;
  int v[8];
  int s = 0;
  for (int i = 0; i < 8; ++i) {
    v[i] = base + i < m ? a[base + i] : 0;
    s += v[i];
  }
  int ex = block_exscan(s, &tot) + bsum[blockIdx.x];
  for (int i = 0; i < 8; ++i) {
    if (base + i < m) a[base + i] = ex;
    ex += v[i];
  }
}

__global__ void __launch_bounds__(kThreads, 6) rs_scatter_kernel(const uint32_t* kin, const int* vin,
                                                            long n_max, const int* d_n, int shift,
                                                            long nblocks, const int* hist, uint32_t* kout,
                                                            int* vout) {
  const long n = d_n ? *d_n : n_max;
  __shared__ int gbase[kBins];
  __shared__ int run[kBins];
  __shared__ int wcnt[kWarps][kBins];
  for (int q = threadIdx.x; q < kBins; q += kThreads) {
    gbase[q] = hist[static_cast<long>(q) * nblocks + blockIdx.x];
    run[q] = 0;
    for (int w = 0; w < kWarps; ++w) wcnt[w][q] = 0;
  }
  __syncthreads();
  const long base = static_cast<long>(blockIdx.x) * kTile;
  const unsigned lane = threadIdx.x & 31u;
  const int warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t kr[kItems];  // the tile's key loads in flight before the first use
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    kr[r] = i < n ? kin[i] : 0u;
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    const bool ok = i < n;
    uint32_t k = 0;
    int v = 0;
    unsigned d = kBins, m = 0u;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      k = kr[r];
      v = vin ? vin[i] : static_cast<int>(i);
      d = (k >> shift) & (kBins - 1u);
      m = __match_any_sync(act, d);
      if ((__ffs(m) - 1) == static_cast<int>(lane)) wcnt[warp][d] = __popc(m);
    }
    __syncthreads();
    if (ok) {
      int pre = 0;
      for (int w = 0; w < warp; ++w) pre += wcnt[w][d];
      const long pos = static_cast<long>(gbase[d]) + run[d] + pre + __popc(m & lt);
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    if (ok && (__ffs(m) - 1) == static_cast<int>(lane)) {
      atomicAdd(&run[d], __popc(m));
      wcnt[warp][d] = 0;
    }
    __syncthreads();
  }
}

// Stable compaction of the (key, index) pairs whose key differs from the
// sentinel: per-tile counts, an exclusive scan (the total lands in entry nb),
// then each tile writes its kept pairs in input order.
__global__ void __launch_bounds__(kThreads) rs_count_kernel(const uint32_t* keys, long n, uint32_t sentinel,
                                                          int* cnt) {
  const long base = static_cast<long>(blockIdx.x) * kTile;
  int c = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    c += (i < n && keys[i] != sentinel) ? 1 : 0;
  }
  __shared__ int tot;
  block_exscan(c, &tot);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kThreads) rs_compact_kernel(const uint32_t* keys, long n, uint32_t sentinel,
                                                            const int* off, uint32_t* kout, int* vout) {
  const long base = static_cast<long>(blockIdx.x) * kTile;
  __shared__ int tot;
  int run = off[blockIdx.x];
  uint32_t kr[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    kr[r] = i < n ? keys[i] : sentinel;
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
    const bool keep = kr[r] != sentinel;
    const int pre = block_exscan(keep ? 1 : 0, &tot);
    if (keep) {
      kout[run + pre] = kr[r];
      vout[run + pre] = static_cast<int>(i);
    }
    run += tot;
  }
}


// ---- one-sweep sort ----------------------------------------------------------
// aux_ layout (32-bit words): [0, kMaxPass * kBins) global digit counts per
// pass; [kOsCounter, +kMaxPass) dynamic tile counters; [kOsCount] number of
// valid pairs; [kOsState, ...) look-back words of the running pass, kBins per tile.
constexpr int kMaxPass = 4;
constexpr int kOsCounter = kMaxPass * kBins;
constexpr int kOsCount = kOsCounter + kMaxPass;
constexpr int kOsState = kOsCounter + 64;
constexpr unsigned kFlagAgg = 1u << 30;   // the tile's own digit count
constexpr unsigned kFlagIncl = 2u << 30;  // inclusive prefix over tiles 0..t
constexpr unsigned kValMask = (1u << 30) - 1u;
constexpr int kLook = 8;  // predecessors read per look-back round trip

// Digit counts of every pass in one read of the raw keys (sentinels skipped).
__global__ void __launch_bounds__(kThreads) os_hist_kernel(const uint32_t* keys, long n, uint32_t sentinel,
                                                         int npass, unsigned* aux) {
  __shared__ int h[kMaxPass][kBins];
  for (int q = threadIdx.x; q < kMaxPass * kBins; q += kThreads) (&h[0][0])[q] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u;
  const long ntiles = (n + kTile - 1) / kTile;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long base = tile * kTile;
    uint32_t kr[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const long i = base + static_cast<long>(r) * kThreads + threadIdx.x;
      kr[r] = i < n ? keys[i] : sentinel;
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const bool ok = kr[r] != sentinel;
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      if (!ok) continue;
      for (int p = 0; p < npass; ++p) {
        const unsigned d = (kr[r] >> (p * kBits)) & (kBins - 1u);
        const unsigned m = __match_any_sync(act, d);
        if ((__ffs(m) - 1) == static_cast<int>(lane)) atomicAdd(&h[p][d], __popc(m));
      }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < npass * kBins; q += kThreads) {
    const int v = (&h[0][0])[q];
    if (v) atomicAdd(&aux[q], static_cast<unsigned>(v));
  }
}

struct OsArgs {
  const uint32_t* kin;
  const int* vin;   // pass 0: null (value = element index)
  long n_max;       // launch-time bound on the number of inputs
  uint32_t sentinel;
  int pass;
  unsigned* aux;
  uint32_t* kout;
  int* vout;
};

// One digit pass. Tiles take their ids from a counter in launch order, so a
// tile only ever waits for tiles that are already running. Within a tile the
// elements are ordered (warp, round, lane); equal digits keep that order:
// rank = (the digit's count in the warp's earlier rounds) + (lower lanes of
// the round, __match_any_sync) + (the digit's count in lower warps) + (the
// tiles before, by look-back) + (the digit's global base). (Packing the
// pushforward's records here was measured 4x slower than a separate pass.)
template <bool FIRST>
__global__ void __launch_bounds__(kThreads, 4) os_scatter_kernel(OsArgs A) {
  __shared__ int s_tile, s_tot;
  __shared__ int gbase[kBins];
  __shared__ int wcnt[kWarps][kBins];
  const unsigned lane = threadIdx.x & 31u;
  const int warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(&A.aux[kOsCounter + A.pass], 1u));
  for (int q = threadIdx.x; q < kWarps * kBins; q += kThreads) (&wcnt[0][0])[q] = 0;
  // global digit bases: exclusive scan of the pass's digit counts (two bins per thread)
  {
    const unsigned* gh = A.aux + A.pass * kBins;
    const int h0 = static_cast<int>(gh[2 * threadIdx.x]), h1 = static_cast<int>(gh[2 * threadIdx.x + 1]);
    const int ex = block_exscan(h0 + h1, &s_tot);
    gbase[2 * threadIdx.x] = ex;
    gbase[2 * threadIdx.x + 1] = ex + h0;
  }
  __syncthreads();
  const int tile = s_tile;
  const long n = FIRST ? A.n_max : static_cast<long>(s_tot);
  const long base = static_cast<long>(tile) * kTile;
  if (FIRST && tile == 0 && threadIdx.x == 0) A.aux[kOsCount] = static_cast<unsigned>(s_tot);
  if (base >= n) return;
  const long wbase = base + static_cast<long>(warp) * (kItems * 32) + lane;
  uint32_t kr[kItems];
  int vr[kItems];  // the values travel with the keys: both loads in flight together
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = wbase + r * 32;
    kr[r] = i < n ? A.kin[i] : A.sentinel;
    vr[r] = FIRST ? static_cast<int>(i) : (i < n ? A.vin[i] : 0);
  }
  // ranks inside the warp (rounds in order; the per-warp digit counters are
  // only touched by their own warp)
  unsigned short rk[kItems];
  unsigned okmask = 0;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const long i = wbase + r * 32;
    const bool ok = i < n && (!FIRST || kr[r] != A.sentinel);
    const unsigned d = (kr[r] >> (A.pass * kBits)) & (kBins - 1u);
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    unsigned m = 0;
    rk[r] = 0;
    if (ok) {
      okmask |= 1u << r;
      m = __match_any_sync(act, d);
      rk[r] = static_cast<unsigned short>(wcnt[warp][d] + __popc(m & lt));
    }
    __syncwarp();
    if (ok && (__ffs(m) - 1) == static_cast<int>(lane)) wcnt[warp][d] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  // per digit (two per thread: d and d + kThreads): exclusive prefix over the
  // warps and the tile's count, published for BOTH digits before either
  // look-back starts (a successor's look-back waits for them); then the
  // look-back over the earlier tiles, both digits' loads in flight together
  unsigned* state = A.aux + kOsState;
  constexpr int kDig = kBins / kThreads;
  int cnt[kDig];
#pragma unroll
  for (int q = 0; q < kDig; ++q) {
    const int d = threadIdx.x + q * kThreads;
    int c = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int v = wcnt[w][d];
      wcnt[w][d] = c;
      c += v;
    }
    cnt[q] = c;
    *reinterpret_cast<volatile unsigned*>(state + static_cast<long>(tile) * kBins + d) =
        static_cast<unsigned>(c) | (tile == 0 ? kFlagIncl : kFlagAgg);
  }
  // look-back: kLook predecessors per digit are read per round trip
  // (independent loads), then consumed in order up to the first unpublished
  // one (measured: 8 per round beats 16 or 32, and beats polling the
  // unpublished entry alone)
  unsigned excl[kDig];
  int pt[kDig];
#pragma unroll
  for (int q = 0; q < kDig; ++q) {
    excl[q] = 0;
    pt[q] = tile - 1;
  }
  while (true) {
    bool any = false;
#pragma unroll
    for (int q = 0; q < kDig; ++q) any = any || pt[q] >= 0;
    if (!any) break;
    unsigned v[kDig][kLook];
#pragma unroll
    for (int q = 0; q < kDig; ++q)
#pragma unroll
      for (int u = 0; u < kLook; ++u)
        v[q][u] = pt[q] - u >= 0
                      ? *reinterpret_cast<volatile unsigned*>(state + static_cast<long>(pt[q] - u) * kBins +
                                                               threadIdx.x + q * kThreads)
                      : (2u << 30);  // (kFlagIncl: nothing before tile 0; also a finished digit)
#pragma unroll
    for (int q = 0; q < kDig; ++q) {
      if (pt[q] < 0) continue;
      bool done = false;
#pragma unroll
      for (int u = 0; u < kLook; ++u) {
        if (done) continue;
        const unsigned f = v[q][u] >> 30;
        if (f == 0) {  // not published yet: retry from here
          done = true;
          continue;
        }
        excl[q] += v[q][u] & kValMask;
        --pt[q];
        if (f == 2) {
          pt[q] = -1;
          done = true;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kDig; ++q) {
    const int d = threadIdx.x + q * kThreads;
    if (tile > 0)
      *reinterpret_cast<volatile unsigned*>(state + static_cast<long>(tile) * kBins + d) =
          (excl[q] + static_cast<unsigned>(cnt[q])) | kFlagIncl;
    gbase[d] += static_cast<int>(excl[q]);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    if (!((okmask >> r) & 1u)) continue;
    const uint32_t k = kr[r];
    const unsigned d = (k >> (A.pass * kBits)) & (kBins - 1u);
    const int v = vr[r];
    const long pos = static_cast<long>(gbase[d]) + wcnt[warp][d] + rk[r];
    A.kout[pos] = k;
    A.vout[pos] = v;
  }
}

}  // namespace

RadixSorter::~RadixSorter() {
  for (int i = 0; i < 2; ++i) {
    if (kbuf_[i]) dfree(kbuf_[i]);
    if (vbuf_[i]) dfree(vbuf_[i]);
  }
  if (hist_) dfree(hist_);
  if (bsum_) dfree(bsum_);
  if (cnt_) dfree(cnt_);
  if (aux_) dfree(aux_);
}

void RadixSorter::init(long n) {
  for (int i = 0; i < 2; ++i) {  // re-init (capacity growth) releases the old buffers
    if (kbuf_[i]) dfree(kbuf_[i]);
    if (vbuf_[i]) dfree(vbuf_[i]);
    kbuf_[i] = nullptr;
    vbuf_[i] = nullptr;
  }
  if (hist_) dfree(hist_);
  if (bsum_) dfree(bsum_);
  if (cnt_) dfree(cnt_);
  hist_ = nullptr;
  bsum_ = nullptr;
  cnt_ = nullptr;
  cap_ = n;
  blocks_ = (n + kTile - 1) / kTile;
  for (int i = 0; i < 2; ++i) {
    BFM_CUDA(dmalloc(&kbuf_[i], (n + 1) * sizeof(uint32_t)));
    BFM_CUDA(dmalloc(&vbuf_[i], (n + 1) * sizeof(int)));
  }
  const long m = static_cast<long>(kBins) * blocks_;
  BFM_CUDA(dmalloc(&hist_, (m + 1) * sizeof(int)));
  BFM_CUDA(dmalloc(&bsum_, ((m + kScanTile - 1) / kScanTile + 1) * sizeof(int)));
  BFM_CUDA(dmalloc(&cnt_, (blocks_ + 2) * sizeof(int)));
  if (aux_) dfree(aux_);
  aux_ = nullptr;
  aux_words_ = kOsState + blocks_ * kBins;  // one look-back region, cleared before every pass
  BFM_CUDA(dmalloc(&aux_, aux_words_ * sizeof(unsigned)));
}

void RadixSorter::sort(const uint32_t* keys_in, const int* vals_in, long n, int bits, cudaStream_t s,
                       LaunchCounter* lc, const uint32_t** keys_out, const int** vals_out, const int* d_n) {
  const long nb = (n + kTile - 1) / kTile;
  const long m = static_cast<long>(kBins) * nb;
  const long sb = (m + kScanTile - 1) / kScanTile;
  const uint32_t* kin = keys_in;
  const int* vin = vals_in;
  int cur = 0;
  for (int shift = 0; shift < bits; shift += kBits) {
    rs_hist_kernel<<<static_cast<unsigned>(nb), kThreads, 0, s>>>(kin, n, d_n, shift, nb, hist_);
    rs_scan_reduce<<<static_cast<unsigned>(sb), 1024, 0, s>>>(hist_, m, bsum_);
    rs_scan_top<<<1, 1024, 0, s>>>(bsum_, sb);
    rs_scan_apply<<<static_cast<unsigned>(sb), 1024, 0, s>>>(hist_, m, bsum_);
    rs_scatter_kernel<<<static_cast<unsigned>(nb), kThreads, 0, s>>>(kin, vin, n, d_n, shift, nb, hist_,
                                                                     kbuf_[cur], vbuf_[cur]);
    BFM_LAUNCH_CHECK("radix sort pass");
    if (lc) lc->add(5);
    kin = kbuf_[cur];
    vin = vbuf_[cur];
    cur ^= 1;
  }
  *keys_out = kin;
  *vals_out = vin;
}


const int* RadixSorter::sort_onesweep(const uint32_t* keys_in, long n, uint32_t sentinel, int bits,
                                      cudaStream_t s, LaunchCounter* lc, const uint32_t** keys_out,
                                      const int** vals_out) {
  const int npass = (bits + kBits - 1) / kBits;
  if (npass < 1 || npass > kMaxPass) throw std::invalid_argument("radix sort: 1..36 key bits supported");
  const long nb = (n + kTile - 1) / kTile;
  // one look-back region (nb * kBins words) is reused by every pass: the
  // passes run back to back on the stream and each clears it first
  BFM_CUDA(cudaMemsetAsync(aux_, 0, kOsState * sizeof(unsigned), s));
  os_hist_kernel<<<static_cast<unsigned>(std::min<long>(nb, 148 * 8)), kThreads, 0, s>>>(keys_in, n, sentinel,
                                                                                        npass, aux_);
  const uint32_t* kin = keys_in;
  const int* vin = nullptr;
  int cur = 0;
  for (int p = 0; p < npass; ++p) {
    BFM_CUDA(cudaMemsetAsync(aux_ + kOsState, 0, static_cast<size_t>(nb) * kBins * sizeof(unsigned), s));
    OsArgs A{};
    A.kin = kin;
    A.vin = vin;
    A.n_max = n;
    A.sentinel = sentinel;
    A.pass = p;
    A.aux = aux_;
    A.kout = kbuf_[cur];
    A.vout = vbuf_[cur];
    if (p == 0) os_scatter_kernel<true><<<static_cast<unsigned>(nb), kThreads, 0, s>>>(A);
    else os_scatter_kernel<false><<<static_cast<unsigned>(nb), kThreads, 0, s>>>(A);
    BFM_LAUNCH_CHECK("one-sweep scatter");
    kin = kbuf_[cur];
    vin = vbuf_[cur];
    cur ^= 1;
  }
  if (lc) lc->add(1 + npass);
  *keys_out = kin;
  *vals_out = vin;
  return reinterpret_cast<const int*>(aux_ + kOsCount);
}

}  // namespace bfmgpu

namespace bfmgpu {

const int* RadixSorter::compact(const uint32_t* keys_in, long n, uint32_t sentinel, cudaStream_t s,
                                LaunchCounter* lc, const uint32_t** keys_out, const int** vals_out) {
  const long nb = (n + kTile - 1) / kTile;
  const long m = nb + 1;  // entry nb receives the total
  const long sb = (m + kScanTile - 1) / kScanTile;
  BFM_CUDA(cudaMemsetAsync(cnt_ + nb, 0, sizeof(int), s));
  rs_count_kernel<<<static_cast<unsigned>(nb), kThreads, 0, s>>>(keys_in, n, sentinel, cnt_);
  rs_scan_reduce<<<static_cast<unsigned>(sb), 1024, 0, s>>>(cnt_, m, bsum_);
  rs_scan_top<<<1, 1024, 0, s>>>(bsum_, sb);
  rs_scan_apply<<<static_cast<unsigned>(sb), 1024, 0, s>>>(cnt_, m, bsum_);
  // kbuf_/vbuf_[1]: the first sort pass reads them and writes buffer 0
  rs_compact_kernel<<<static_cast<unsigned>(nb), kThreads, 0, s>>>(keys_in, n, sentinel, cnt_, kbuf_[1],
                                                                   vbuf_[1]);
  BFM_LAUNCH_CHECK("radix compact");
  if (lc) lc->add(5);
  *keys_out = kbuf_[1];
  *vals_out = vbuf_[1];
  return cnt_ + nb;
}

}  // namespace bfmgpu
