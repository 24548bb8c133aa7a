// Neumann Poisson solve on sm_100a: batched DCT-II (REDFT10) along axes
// d-1..1, one fused kernel for [DCT-II axis 0 -> spectral divide -> DCT-III
// axis 0], then DCT-III along axes 1..d-1 (reference poisson.hpp:87-106).
// 2d-1 HBM passes of read+write per solve.
//
// Each CTA owns `lpc` grid lines (consecutive along the fastest other axis
// for strided axes, so global loads/stores are coalesced), stages each line
// in shared memory, and runs the shared line algorithm of dct_line.h with the
// butterflies of a stage spread over the line's threads. Every value goes
// through the same IEEE operations as the CPU shim (bitwise-equal results).
#include <cstdlib>
#include <cstring>
#include <vector>

#include "poisson.cuh"

namespace bfmgpu {
namespace {

using bfmdct::cplx;

enum { kFwd = 0, kInv = 1, kFused = 2 };

struct PoisArgs {
  PoisAxisCfg ax;
  int mode;
  int d;
  int n1, n2;  // extents of axes 1, 2 (fused divide)
  const double* in;
  double* out;
  const double* lam0;
  const double* lam1;
  const double* lam2;
  double scale;
  long col_off;  // multi-GPU column slab: global index of local column 0
  int npass;
  int pstage[bfmdct::kMaxStages];
  int pfused[bfmdct::kMaxStages];
  unsigned pmagic[bfmdct::kMaxStages];  // division by q1 (fused) or q (single)
};

// Shared-memory layout of a line: complex slot i lives at sw(i), an XOR
// swizzle of the low three bits (8 complex = 128 B = all 32 banks) with
// higher index bits. It makes the strided butterfly groups of the late FFT
// stages and the digit-reversed gathers of the unpack/post phases (nearly)
// conflict-free for 2^a 3^b line lengths. The double view of the same
// buffer keeps the two halves of a complex slot adjacent.
__device__ __forceinline__ int sw(int i) { return i ^ (((i >> 4) ^ (i >> 5) ^ (i >> 8)) & 7); }
__device__ __forceinline__ double& dref(double* zd, int j) { return zd[2 * sw(j >> 1) + (j & 1)]; }
__device__ __forceinline__ cplx& cref(cplx* z, int i) { return z[sw(i)]; }

__device__ __forceinline__ void gsync(int tpl, int l) {
  if (tpl <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(l + 1), "r"(tpl) : "memory");
  }
}

__device__ __forceinline__ long line_base(const PoisAxisCfg& ax, long L) {
  const long inner = L % ax.stride, outer = L / ax.stride;
  return outer * static_cast<long>(ax.n) * ax.stride + inner;
}

// Spectral divide for axis-0 wavenumber k of the line with other wavenumbers
// (k1, k2): poisson.hpp:93-103 (lam summed as (l0 + l1) + l2).
__device__ __forceinline__ double divide(const PoisArgs& a, double v, int k, double l1v,
                                         double l2v) {
  const double l01 = a.lam0[k] + l1v;
  const double lam = l01 + l2v;
  return lam == 0.0 ? 0.0 : v / (lam * a.scale);
}

// FFT passes: pairs of consecutive DIF stages are fused so a thread keeps
// R0*R1 points in registers across both stages (one shared-memory round trip
// per pass instead of per stage). Each butterfly is butterfly_regs, the same
// arithmetic the CPU shim runs stage by stage.
template <int R0, int R1>
__device__ __forceinline__ void fused_pass(const PoisArgs& a, cplx* z, int s, int pi, bool inverse,
                                           int t, int tpl) {
  const bfmdct::LinePlan& P = a.ax.plan;
  const int L0 = P.span[s];
  const int q0 = L0 / R0, q1 = q0 / R1;
  const int twm0 = P.m / L0, twm1 = P.m / q0;
  const int ng = P.m / (R0 * R1);
  const unsigned magic = a.pmagic[pi];
  for (int g = t; g < ng; g += tpl) {
    const int blk = magic ? static_cast<int>(__umulhi(static_cast<unsigned>(g), magic)) : g;
    const int jpp = g - blk * q1;
    const int base = blk * L0 + jpp;
    cplx x[R0 * R1];
#pragma unroll
    for (int aa = 0; aa < R0; ++aa)
#pragma unroll
      for (int bb = 0; bb < R1; ++bb) x[aa * R1 + bb] = cref(z, base + aa * q0 + bb * q1);
#pragma unroll
    for (int bb = 0; bb < R1; ++bb) {
      cplx col[R0];
#pragma unroll
      for (int aa = 0; aa < R0; ++aa) col[aa] = x[aa * R1 + bb];
      bfmdct::butterfly_regs(P, R0, col, twm0 * (jpp + bb * q1), inverse);
#pragma unroll
      for (int aa = 0; aa < R0; ++aa) x[aa * R1 + bb] = col[aa];
    }
#pragma unroll
    for (int aa = 0; aa < R0; ++aa) bfmdct::butterfly_regs(P, R1, x + aa * R1, twm1 * jpp, inverse);
#pragma unroll
    for (int aa = 0; aa < R0; ++aa)
#pragma unroll
      for (int bb = 0; bb < R1; ++bb) cref(z, base + aa * q0 + bb * q1) = x[aa * R1 + bb];
  }
}

template <int R>
__device__ __forceinline__ void single_pass(const PoisArgs& a, cplx* z, int s, int pi, bool inverse,
                                            int t, int tpl) {
  const bfmdct::LinePlan& P = a.ax.plan;
  const int L = P.span[s];
  const int q = L / R;
  const int twm = P.m / L;
  const int nb = P.m / R;
  const unsigned magic = a.pmagic[pi];
  for (int b = t; b < nb; b += tpl) {
    const int blk = magic ? static_cast<int>(__umulhi(static_cast<unsigned>(b), magic)) : b;
    const int j = b - blk * q;
    const int base = blk * L + j;
    cplx x[R];
#pragma unroll
    for (int u = 0; u < R; ++u) x[u] = cref(z, base + u * q);
    bfmdct::butterfly_regs(P, R, x, twm * j, inverse);
#pragma unroll
    for (int u = 0; u < R; ++u) cref(z, base + u * q) = x[u];
  }
}

__device__ __forceinline__ void fft_stages(const PoisArgs& a, cplx* z, bool inverse, int t,
                                           int tpl, int l) {
  const bfmdct::LinePlan& P = a.ax.plan;
  for (int pi = 0; pi < a.npass; ++pi) {
    const int s = a.pstage[pi];
    const int r0 = P.radix[s];
    if (a.pfused[pi]) {
      const int r1 = P.radix[s + 1];
      if (r0 == 4 && r1 == 4) fused_pass<4, 4>(a, z, s, pi, inverse, t, tpl);
      else if (r0 == 4 && r1 == 2) fused_pass<4, 2>(a, z, s, pi, inverse, t, tpl);
      else if (r0 == 4 && r1 == 3) fused_pass<4, 3>(a, z, s, pi, inverse, t, tpl);
      else if (r0 == 2 && r1 == 3) fused_pass<2, 3>(a, z, s, pi, inverse, t, tpl);
      else fused_pass<3, 3>(a, z, s, pi, inverse, t, tpl);
    } else {
      if (r0 == 4) single_pass<4>(a, z, s, pi, inverse, t, tpl);
      else if (r0 == 2) single_pass<2>(a, z, s, pi, inverse, t, tpl);
      else single_pass<3>(a, z, s, pi, inverse, t, tpl);
    }
    gsync(tpl, l);
  }
}

// Two shared buffers per line (zA, zB): phases read one and write the other,
// so no register staging is needed; butterflies run in place.
__global__ void __launch_bounds__(512) pois_fft_kernel(PoisArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PoisAxisCfg& ax = a.ax;
  const bfmdct::LinePlan& P = ax.plan;
  const int tpl = ax.tpl, lpc = ax.lpc, n = ax.n, m = P.m;
  const int l = threadIdx.x / tpl;
  const int t = threadIdx.x - l * tpl;
  const long L0 = static_cast<long>(blockIdx.x) * lpc;
  __shared__ long s_base[32];  // lpc <= 32
  if (threadIdx.x < lpc) {
    const long L = L0 + threadIdx.x;
    s_base[threadIdx.x] = L < ax.nlines ? line_base(ax, L) : -1;
  }
  __syncthreads();
  // load (coalesced): thread's line is fixed, no per-element division
  const int ml = ax.strided ? static_cast<int>(threadIdx.x % lpc) : l;
  const int step = ax.strided ? blockDim.x / lpc : tpl;
  const int first = ax.strided ? static_cast<int>(threadIdx.x / lpc) : t;
  {
    const long base = s_base[ml];
    double* zA = reinterpret_cast<double*>(smem + static_cast<long>(ml) * ax.line_bytes);
    // batches of kLoadBatch independent loads per thread keep enough bytes in
    // flight to cover HBM latency with one CTA per SM
    constexpr int kLoadBatch = 8;
    if (base >= 0)
      for (int j0 = first; j0 < n; j0 += kLoadBatch * step) {
        double v[kLoadBatch];
#pragma unroll
        for (int u = 0; u < kLoadBatch; ++u) {
          const int j = j0 + u * step;
          v[u] = j < n ? a.in[base + static_cast<long>(j) * ax.stride] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kLoadBatch; ++u) {
          const int j = j0 + u * step;
          if (j < n) {
            if (a.mode == kInv) dref(zA, j) = v[u];
            else dref(zA, bfmdct::dct2_vpos(P, j)) = v[u];
          }
        }
      }
  }
  __syncthreads();
  const long lbase = s_base[l];
  const bool active = lbase >= 0;
  double* zAd = reinterpret_cast<double*>(smem + static_cast<long>(l) * ax.line_bytes);
  double* zBd = zAd + 2 * ax.cslots;
  cplx* zA = reinterpret_cast<cplx*>(zAd);
  cplx* zB = reinterpret_cast<cplx*>(zBd);
  double l1v = 0.0, l2v = 0.0;
  if (a.mode == kFused && active) {
    const long c = lbase + a.col_off;
    if (a.d == 2) {
      l1v = a.lam1[c];
    } else if (a.d == 3) {
      l1v = a.lam1[c / a.n2];
      l2v = a.lam2[c % a.n2];
    }
  }
  double* outbuf = zAd;  // where the line's final values end up
  if (a.mode == kInv) {
    if (active)
      for (int k = t; k < m; k += tpl) {
        const cplx A = bfmdct::dct3_V_vals(P, dref(zAd, k), k == 0 ? 0.0 : dref(zAd, n - k), k);
        const int km = m - k;
        const cplx B = bfmdct::dct3_V_vals(P, dref(zAd, km), dref(zAd, n - km), km);
        cref(zB, k) = bfmdct::dct3_pre_vals(P, A, B, k);
      }
    gsync(tpl, l);
    if (active) fft_stages(a, zB, true, t, tpl, l);
    else for (int s = 0; s < a.npass; ++s) gsync(tpl, l);
    if (active)
      for (int q = t; q < m; q += tpl) {
        const cplx v = cref(zB, bfmdct::tab_i(P.rev, q));
        dref(zAd, bfmdct::dct3_ypos(P, 2 * q)) = v.re;
        dref(zAd, bfmdct::dct3_ypos(P, 2 * q + 1)) = v.im;
      }
    outbuf = zAd;
  } else {
    if (active) fft_stages(a, zA, false, t, tpl, l);
    else for (int s = 0; s < a.npass; ++s) gsync(tpl, l);
    if (a.mode == kFwd) {
      if (active)
        for (int k = t; k <= m; k += tpl) {
          double yk, ynk;
          bfmdct::dct2_unpack_vals(P, cref(zA, bfmdct::tab_i(P.rev, k == m ? 0 : k)),
                                   cref(zA, bfmdct::tab_i(P.rev, k == 0 ? 0 : m - k)), k, yk, ynk);
          dref(zBd, k) = yk;
          if (k > 0 && k < m) dref(zBd, n - k) = ynk;
        }
      outbuf = zBd;
    } else {
      const int half = m / 2;
      if (active)
        for (int k = t; k <= half; k += tpl) {
          const int km = m - k;
          double yk, ynk, ykm, ynkm;
          bfmdct::dct2_unpack_vals(P, cref(zA, bfmdct::tab_i(P.rev, k == m ? 0 : k)),
                                   cref(zA, bfmdct::tab_i(P.rev, k == 0 ? 0 : m - k)), k, yk, ynk);
          bfmdct::dct2_unpack_vals(P, cref(zA, bfmdct::tab_i(P.rev, km == m ? 0 : km)),
                                   cref(zA, bfmdct::tab_i(P.rev, km == 0 ? 0 : m - km)), km, ykm, ynkm);
          const double xk = divide(a, yk, k, l1v, l2v);
          const double xnk = (k > 0 && k < m) ? divide(a, ynk, n - k, l1v, l2v) : 0.0;
          const double xkm = divide(a, ykm, km, l1v, l2v);
          const double xnkm = (km > 0 && km < m) ? divide(a, ynkm, n - km, l1v, l2v) : 0.0;
          const double b_k = k == 0 ? 0.0 : xnk;
          const double b_km = km == m ? xkm : xnkm;
          const cplx Vk = bfmdct::dct3_V_vals(P, xk, b_k, k);
          const cplx Vkm = bfmdct::dct3_V_vals(P, xkm, b_km, km);
          cref(zB, k) = bfmdct::dct3_pre_vals(P, Vk, Vkm, k);
          if (km < m && km != k) cref(zB, km) = bfmdct::dct3_pre_vals(P, Vkm, Vk, km);
        }
      gsync(tpl, l);
      if (active) fft_stages(a, zB, true, t, tpl, l);
      else for (int s = 0; s < a.npass; ++s) gsync(tpl, l);
      if (active)
        for (int q = t; q < m; q += tpl) {
          const cplx v = cref(zB, bfmdct::tab_i(P.rev, q));
          dref(zAd, bfmdct::dct3_ypos(P, 2 * q)) = v.re;
          dref(zAd, bfmdct::dct3_ypos(P, 2 * q + 1)) = v.im;
        }
      outbuf = zAd;
    }
  }
  __syncthreads();
  // store (coalesced)
  {
    const long base = s_base[ml];
    double* src = reinterpret_cast<double*>(smem + static_cast<long>(ml) * ax.line_bytes) +
                  (outbuf == zAd ? 0 : 2 * ax.cslots);
    if (base >= 0)
      for (int j = first; j < n; j += step) a.out[base + static_cast<long>(j) * ax.stride] = dref(src, j);
  }
}

// Direct O(n^2) form for extents that are not 2 * 2^a 3^b.
__global__ void __launch_bounds__(512) pois_naive_kernel(PoisArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const PoisAxisCfg& ax = a.ax;
  const bfmdct::LinePlan& P = ax.plan;
  const int tpl = ax.tpl, lpc = ax.lpc, n = ax.n;
  const int l = threadIdx.x / tpl;
  const int t = threadIdx.x - l * tpl;
  const long L0 = static_cast<long>(blockIdx.x) * lpc;
  for (int idx = threadIdx.x; idx < n * lpc; idx += blockDim.x) {
    int ll, j;
    if (ax.strided) {
      ll = idx % lpc;
      j = idx / lpc;
    } else {
      ll = idx / n;
      j = idx - ll * n;
    }
    const long L = L0 + ll;
    if (L >= ax.nlines) continue;
    double* xa = reinterpret_cast<double*>(smem + static_cast<long>(ll) * ax.line_bytes);
    xa[j] = a.in[line_base(ax, L) + static_cast<long>(j) * ax.stride];
  }
  __syncthreads();
  const long L = L0 + l;
  const bool active = L < ax.nlines;
  double* xa = reinterpret_cast<double*>(smem + static_cast<long>(l) * ax.line_bytes);
  double* yb = xa + n;
  double l1v = 0.0, l2v = 0.0;
  if (a.mode == kFused && active) {
    const long inner = line_base(ax, L) + a.col_off;
    if (a.d == 2) {
      l1v = a.lam1[inner];
    } else if (a.d == 3) {
      l1v = a.lam1[inner / a.n2];
      l2v = a.lam2[inner % a.n2];
    }
  }
  if (active) {
    for (int k = t; k < n; k += tpl) {
      double v = a.mode == kInv ? bfmdct::dct3_naive(P, xa, 1, k) : bfmdct::dct2_naive(P, xa, 1, k);
      if (a.mode == kFused) v = divide(a, v, k, l1v, l2v);
      yb[k] = v;
    }
  }
  gsync(tpl, l);
  if (a.mode == kFused && active) {
    for (int k = t; k < n; k += tpl) xa[k] = bfmdct::dct3_naive(P, yb, 1, k);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * lpc; idx += blockDim.x) {
    int ll, j;
    if (ax.strided) {
      ll = idx % lpc;
      j = idx / lpc;
    } else {
      ll = idx / n;
      j = idx - ll * n;
    }
    const long LL = L0 + ll;
    if (LL >= ax.nlines) continue;
    const double* xl = reinterpret_cast<const double*>(smem + static_cast<long>(ll) * ax.line_bytes);
    const double* src = a.mode == kFused ? xl : xl + n;
    a.out[line_base(ax, LL) + static_cast<long>(j) * ax.stride] = src[j];
  }
}

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>& keep) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  BFM_CUDA(dmalloc(&d, v.size() * sizeof(T)));
  BFM_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  keep.push_back(d);
  return d;
}

}  // namespace

PoissonPlan::~PoissonPlan() {
  for (int a = 0; a < 3; ++a) {
    if (tables_[a]) {
      auto* v = static_cast<std::vector<void*>*>(tables_[a]);
      for (void* p : *v) dfree(p);
      delete v;
    }
    if (lam_[a]) dfree(lam_[a]);
  }
  if (tmp_) dfree(tmp_);
}

void PoissonPlan::init(const GridDesc& g) { setup(g, g, 0, 0, g.d); }

void PoissonPlan::init_slab_rows(const GridDesc& global, int nrows) {
  if (global.d < 2) throw std::invalid_argument("solve_neumann: slabs need d >= 2");
  int ext[3] = {nrows, global.n[1], global.d > 2 ? global.n[2] : 1};
  setup(make_grid(global.d, ext), global, 0, 1, global.d);
}

void PoissonPlan::init_slab_cols(const GridDesc& global, long col0, int ncols) {
  if (global.d < 2) throw std::invalid_argument("solve_neumann: slabs need d >= 2");
  int ext[2] = {global.n[0], ncols};
  setup(make_grid(2, ext), global, col0, 0, 1);
}

// loc: the grid the kernels walk; global: the problem grid (spectrum,
// normalisation). A column slab is (n0 x ncols) with a virtual second axis.
void PoissonPlan::setup(const GridDesc& loc, const GridDesc& global, long col0, int ab, int ae) {
  constexpr double kPi = 3.14159265358979323846;
  g_ = loc;
  gg_ = global;
  col_off_ = col0;
  scale_ = 1.0;
  for (int a = 0; a < global.d; ++a) scale_ *= 2.0 * global.n[a];
  for (int a = 0; a < global.d; ++a) {
    const int n = global.n[a];
    std::vector<double> lam(n);
    const double na = n;
    for (int k = 0; k < n; ++k) lam[k] = (2.0 - 2.0 * std::cos(kPi * k / na)) * na * na;
    BFM_CUDA(dmalloc(&lam_[a], n * sizeof(double)));
    BFM_CUDA(cudaMemcpy(lam_[a], lam.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  }
  const GridDesc& g = loc;
  int dev = 0;
  BFM_CUDA(cudaGetDevice(&dev));
  int max_optin = 0;
  BFM_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int budget = max_optin - 1024;
  for (int a = ab; a < ae; ++a) {  // axes whose line transforms this plan runs
    const int n = g.n[a];
    host_[a].reset(new bfmdct::HostLinePlan);
    host_[a]->build(n);
    const bfmdct::HostLinePlan& H = *host_[a];
    auto* keep = new std::vector<void*>;
    tables_[a] = keep;
    PoisAxisCfg& c = cfg_[a];
    c.plan = H.plan;
    c.plan.wm = upload(H.wm, *keep);
    c.plan.rev = upload(H.rev, *keep);
    c.plan.cs = upload(H.cs, *keep);
    c.plan.wn = upload(H.wn, *keep);
    c.plan.cosmat = upload(H.cosmat, *keep);
    c.n = n;
    c.stride = g.stride[a];
    c.nlines = g.size / n;
    c.strided = a != g.d - 1;
    if (H.plan.kind == bfmdct::kFft) {
      const int m = H.plan.m;
      // about 16 points per thread in the fused radix passes; short lines
      // (m <= 256, e.g. C4's 384-point lines) of large grids get a half warp
      // each (two lines per warp, synchronised together by __syncwarp), so
      // the passes' 12-16 butterfly groups keep most lanes busy and twice as
      // many lines fit the register file (C4 Poisson 11.5 -> 9.1 ms per
      // iteration); small grids keep a full warp per line (more CTAs)
      int tpl = (m + 15) / 16;
      const bool many = g.size / n >= 16384;  // enough lines to fill the SMs twice over
      tpl = (tpl <= 16 && many) ? 16 : std::max(32, ((tpl + 31) / 32) * 32);
      if (tpl > 256) tpl = 256;
      c.tpl = tpl;
      c.cslots = (m + 7) & ~7;
      c.line_bytes = 2 * 16 * c.cslots;
    } else {
      c.tpl = n >= 256 ? 256 : 32 * ((n + 31) / 32);
      c.line_bytes = ((16 * n) + 15) & ~15;
    }
    if (c.line_bytes > budget) throw std::invalid_argument("solve_neumann: line exceeds shared memory");
    int lpc = std::min(budget / c.line_bytes, 512 / c.tpl);
    // strided axes: 8 lines per CTA (64 B row segments) keeps several CTAs
    // per SM so one CTA's loads overlap another's butterflies (C4: 32 lines,
    // one 196 KB CTA per SM, 9.4 ms of Poisson per iteration; 16: 8.9; 8:
    // 7.8; 4: 9.7)
    lpc = std::min(lpc, c.strided ? 8 : std::max(4, 128 / c.tpl));
    if (c.tpl > 32) lpc = std::min(lpc, 15);
    // long contiguous lines (C3: 64 KB each): one line per CTA, three CTAs
    // per SM that drift out of phase (C3 Poisson 2.20 -> 2.09 ms per iteration)
    if (!c.strided && c.line_bytes >= 32768) lpc = 1;
    if (const char* e = getenv(c.strided ? "BFM_POIS_LPC_S" : "BFM_POIS_LPC_C"))  // tuning experiments
      lpc = std::max(1, std::min(atoi(e), std::min(budget / c.line_bytes, 512 / c.tpl)));
    lpc = static_cast<int>(std::min<long>(lpc, c.nlines));
    c.lpc = std::max(1, lpc);
  }
  BFM_CUDA(cudaFuncSetAttribute(pois_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
  BFM_CUDA(cudaFuncSetAttribute(pois_naive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
}

void PoissonPlan::launch(int axis, int mode, const double* in, double* out, cudaStream_t stream,
                         LaunchCounter* lc) {
  {
    const int d = gg_.d;
    PoisArgs A;
    std::memset(&A, 0, sizeof(A));
    A.ax = cfg_[axis];
    A.mode = mode;
    A.d = d;
    A.n1 = d > 1 ? gg_.n[1] : 1;
    A.n2 = d > 2 ? gg_.n[2] : 1;
    A.in = in;
    A.out = out;
    A.lam0 = lam_[0];
    A.lam1 = d > 1 ? lam_[1] : nullptr;
    A.lam2 = d > 2 ? lam_[2] : nullptr;
    A.scale = scale_;
    A.col_off = col_off_;
    const PoisAxisCfg& c = cfg_[axis];
    A.npass = 0;
    for (int st = 0; st < c.plan.nstages;) {
      const bool fuse = st + 1 < c.plan.nstages;
      const int q0 = c.plan.span[st] / c.plan.radix[st];
      const unsigned q = static_cast<unsigned>(fuse ? q0 / c.plan.radix[st + 1] : q0);
      A.pstage[A.npass] = st;
      A.pfused[A.npass] = fuse ? 1 : 0;
      A.pmagic[A.npass] = q == 1 ? 0u : static_cast<unsigned>((0x100000000ULL + q - 1) / q);
      ++A.npass;
      st += fuse ? 2 : 1;
    }
    const long blocks = (c.nlines + c.lpc - 1) / c.lpc;
    const size_t sm = static_cast<size_t>(c.lpc) * c.line_bytes;
    if (c.plan.kind == bfmdct::kFft)
      pois_fft_kernel<<<static_cast<unsigned>(blocks), c.lpc * c.tpl, sm, stream>>>(A);
    else
      pois_naive_kernel<<<static_cast<unsigned>(blocks), c.lpc * c.tpl, sm, stream>>>(A);
    BFM_LAUNCH_CHECK("pois kernel");
    if (lc) lc->add();
  }
}

void PoissonPlan::solve(const double* d_rhs, double* d_out, cudaStream_t stream,
                        LaunchCounter* lc) {
  const int d = g_.d;
  const double* cur = d_rhs;
  for (int a = d - 1; a >= 1; --a) {
    launch(a, kFwd, cur, d_out, stream, lc);
    cur = d_out;
  }
  launch(0, kFused, cur, d_out, stream, lc);
  for (int a = 1; a < d; ++a) launch(a, kInv, d_out, d_out, stream, lc);
}

void PoissonPlan::rows_forward(const double* d_in, double* d_out, cudaStream_t stream,
                               LaunchCounter* lc) {
  const double* cur = d_in;
  for (int a = g_.d - 1; a >= 1; --a) {
    launch(a, kFwd, cur, d_out, stream, lc);
    cur = d_out;
  }
}

void PoissonPlan::cols_fused(const double* d_in, double* d_out, cudaStream_t stream,
                             LaunchCounter* lc) {
  launch(0, kFused, d_in, d_out, stream, lc);
}

void PoissonPlan::rows_inverse(double* d_inout, cudaStream_t stream, LaunchCounter* lc) {
  for (int a = 1; a < g_.d; ++a) launch(a, kInv, d_inout, d_inout, stream, lc);
}

}  // namespace bfmgpu
