// Exact quadratic c-transform, B200 (sm_100a).
//
// Reference semantics (transforms.hpp:396-432, :340-391, exact.hpp:167-179):
//   psi(x) = RD( min_y  sum_a [hs(x_a) + hs(y_a) - x_a*y_a] - phi(y) )
// with hs(c) = fl(0.5*c*c), exact products and sums, and a single rounding
// toward -inf (-0 -> +0). The minimum is unique, so any exact algorithm gives
// the reference's bits (checked against oracle/_ref in tests/).
//
// One kernel launch per axis pass, reference axis order 0..d-1. Inter-pass
// state is the argmin INDEX chain (uint32: j0 | j1<<16) plus phi at the chain
// (q): the exact candidate value is recomputed from the chain and the per-axis
// terms g_a(k,j) = hs(x_k)+hs(y_j)-x_k*y_j. Two kernels:
//  * ct_dy_kernel (every extent a power of two; see the section header
//    below): an EXACT lower hull with strict corners, every exact decision
//    made on shared-memory-resident exact data.
//  * ct_pass_kernel (other extents, e.g. C4's 384^3): g from exact 3-limb host
//    tables; per grid line (staged in shared memory, tpl threads per line) the
//    lower hull is built with fp64 orientation tests that only keep CERTIFIED
//    strict corners (monotone chains + a log2(tpl)-level bridge-merge tree),
//    every non-corner point within the rounding bound of its hull edge is
//    flagged "suspect" (log-coded per-edge slack), each query walks to its
//    tangent corner, and queries whose neighbourhood is not certified are
//    resolved exactly among the corners and suspects within a rigorous
//    margin (exact.cuh expansions). The last pass rounds the winner's exact
//    value down once.
#include <cassert>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctransform.cuh"
#include "exact.cuh"

namespace bfmgpu {
namespace {

constexpr double kU = 1.1102230246251565e-16;  // 2^-53

#if defined(BFM_DEBUG_BOUNDS)
#define BFM_DASSERT(c) assert(c)
#else
#define BFM_DASSERT(c) ((void)0)
#endif

__device__ __forceinline__ int padj(int j) { return j + (j >> 5); }

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---- TMA bulk copies (cp.async.bulk, sm_90+) with an mbarrier ---------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned;
// completion is signalled on bar as transaction bytes
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void group_sync(int tpl, int l) {
  if (tpl <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(l + 1), "r"(tpl) : "memory");
  }
}

__device__ __forceinline__ unsigned long long dbits(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(v));
}
__device__ __forceinline__ double bitsd(unsigned long long v) {
  return __longlong_as_double(static_cast<long long>(v));
}

struct LineGeo {
  long base;
  long phi_other;
  int k[3];  // coordinate indices (k[0] global: local + p.k0_off)
  int valid;
};

__device__ __forceinline__ double g_approx(const CtAxis& A, int k, int j) {
  if (A.dyadic) {
    const double dl = coord(A.h, k) - coord(A.h, j);
    return 0.5 * dl * dl;
  }
  BFM_DASSERT(k >= 0 && k < A.n && j >= 0 && j < A.n);
  return __ldg(&A.G[static_cast<long>(k) * A.n + j].x);
}

__device__ __forceinline__ int g_terms(const CtAxis& A, int k, int j, double* t) {
  if (A.dyadic) {
    const double dl = coord(A.h, k) - coord(A.h, j);
    t[0] = 0.5 * dl * dl;
    return 1;
  }
  BFM_DASSERT(k >= 0 && k < A.n && j >= 0 && j < A.n);
  // read-only for the whole launch: the non-coherent path lets the compiler
  // issue the loads of several candidates ahead of earlier result stores
  const double2* row = reinterpret_cast<const double2*>(&A.G[static_cast<long>(k) * A.n + j]);
  const double2 v01 = __ldg(row), v23 = __ldg(row + 1);
  const double4 v = make_double4(v01.x, v01.y, v23.x, v23.y);
  int m = 0;
  t[m++] = v.x;
  if (v.y != 0.0) t[m++] = v.y;
  if (v.z != 0.0) t[m++] = v.z;
  return m;
}

__device__ __forceinline__ long phi_index(const CtPass& p, const LineGeo& g, uint32_t chain,
                                          int j) {
  BFM_DASSERT(j >= 0 && j < p.ax[p.a].n);
  BFM_DASSERT(p.a < 1 || (chain & 0xFFFFu) < static_cast<uint32_t>(p.ax[0].n));
  BFM_DASSERT(p.a < 2 || (chain >> 16) < static_cast<uint32_t>(p.ax[1].n));
  // pregathered: the previous pass already stored phi(chain*, y) at every
  // node y (its q output), so candidate j reads its own node — a coalesced
  // line read instead of a gather along the chain
  if (p.pregathered) return g.base + static_cast<long>(j) * p.ax[p.a].stride;
  long idx = g.phi_other + static_cast<long>(j) * p.ax[p.a].stride;
  if (p.a >= 1) idx += static_cast<long>(chain & 0xFFFFu) * p.ax[0].stride;
  if (p.a >= 2) idx += static_cast<long>(chain >> 16) * p.ax[1].stride;
  return idx;
}

// Exact terms of V(k, j) = -phi(chain, j) + sum_{b<a} g_b(k_b, j_b*) + g_a(k, j).
__device__ int cand_terms(const CtPass& p, const LineGeo& g, uint32_t chain, int j, int k,
                          double* t) {
  int m = 0;
  t[m++] = -__ldg(&p.phi[phi_index(p, g, chain, j)]);
  if (p.a >= 1) m += g_terms(p.ax[0], g.k[0], static_cast<int>(chain & 0xFFFFu), t + m);
  if (p.a >= 2) m += g_terms(p.ax[1], g.k[1], static_cast<int>(chain >> 16), t + m);
  m += g_terms(p.ax[p.a], k, j, t + m);
  return m;
}

// ---- exact fixed-point candidates (non-dyadic grids with n <= 512) --------
// Every coordinate y = fl((j+1/2) fl(1/n)) >= 2^-10 is a multiple of 2^-62,
// hs(y) >= 2^-21 a multiple of 2^-74 and x*y of 2^-124, so g * 2^124 is an
// exact integer below 2^124. A candidate V = sum_b g_b - phi is then an exact
// signed 128-bit integer whenever phi is a multiple of 2^-124 below 4 in
// magnitude (checked per value; otherwise the expansion path is used).
__device__ __forceinline__ bool to_fixed124(double v, __int128& out) {
  const long long b = __double_as_longlong(v);
  const int ex = static_cast<int>((b >> 52) & 0x7ff);
  long long m = b & 0xFFFFFFFFFFFFFll;
  if (ex == 0) {
    if (m == 0) {
      out = 0;
      return true;
    }
    return false;  // subnormal: far below 2^-124
  }
  if (ex == 0x7ff) return false;
  m |= 1ll << 52;
  const int sh = ex - 1075 + 124;  // v = m 2^(ex - 1075)
  if (sh > 73) return false;       // |v| >= 4
  __int128 r;
  if (sh >= 0) {
    r = static_cast<__int128>(m) << sh;
  } else {
    if (sh < -52 || (m & ((1ll << -sh) - 1)) != 0) return false;  // not a multiple of 2^-124
    r = m >> -sh;
  }
  out = b < 0 ? -r : r;
  return true;
}
// RD(V * 2^-124) (round toward -inf; V != 0 gives a normal double)
__device__ __forceinline__ double rd_fixed124(__int128 V) {
  if (V == 0) return 0.0;
  const bool neg = V < 0;
  unsigned __int128 w = neg ? static_cast<unsigned __int128>(-V) : static_cast<unsigned __int128>(V);
  const unsigned long long hi = static_cast<unsigned long long>(w >> 64);
  const unsigned long long lo = static_cast<unsigned long long>(w);
  const int msb = hi ? 127 - __clzll(static_cast<long long>(hi)) : 63 - __clzll(static_cast<long long>(lo));
  int e2 = -124;  // value = mant * 2^e2
  unsigned long long mant;
  if (msb <= 52) {
    mant = lo;
  } else {
    const int drop = msb - 52;
    mant = static_cast<unsigned long long>(w >> drop);
    const unsigned __int128 rest = w - (static_cast<unsigned __int128>(mant) << drop);
    e2 += drop;
    if (neg && rest != 0) {  // magnitude rounds up for a negative value
      ++mant;
      if (mant == (1ull << 53)) {
        mant >>= 1;
        ++e2;
      }
    }
  }
  const double p2 = __longlong_as_double(static_cast<long long>(e2 + 1023) << 52);  // exact power of two
  const double r = static_cast<double>(mant) * p2;
  return neg ? -r : r;
}
__device__ __forceinline__ bool g_fixed(const CtAxis& A, int k, int j, __int128& out) {
  if (A.dyadic) return to_fixed124(g_approx(A, k, j), out);  // exact double on dyadic axes
  out = A.GF[static_cast<long>(k) * A.n + j];
  return true;
}
// Exact candidate value V(k, j) * 2^124, when representable.
__device__ __forceinline__ bool cand_fixed(const CtPass& p, const LineGeo& g, uint32_t chain, int j, int k,
                                           __int128& V) {
  __int128 f;
  if (!to_fixed124(__ldg(&p.phi[phi_index(p, g, chain, j)]), f)) return false;
  V = -f;
  __int128 t;
  if (p.a >= 1) {
    if (!g_fixed(p.ax[0], g.k[0], static_cast<int>(chain & 0xFFFFu), t)) return false;
    V += t;
  }
  if (p.a >= 2) {
    if (!g_fixed(p.ax[1], g.k[1], static_cast<int>(chain >> 16), t)) return false;
    V += t;
  }
  if (!g_fixed(p.ax[p.a], k, j, t)) return false;
  V += t;
  return true;
}

__device__ __forceinline__ bool g_fixed_dyadic(const CtAxis& A, int k, int j, __int128& out) {
  return to_fixed124(g_approx(A, k, j), out);  // exact double on dyadic axes
}
// Exact fixed-point values of two candidates (ka, ja), (kb, jb) at once (jb < 0: only the first). Every
// global load of both candidates (phi at the chain, the table entries of the
// chain's axes and of the pass axis) is issued before the first conversion,
// so a flagged query pays one memory round trip instead of one per load.
__device__ __forceinline__ bool cand_fixed2(const CtPass& p, const LineGeo& g, const uint32_t* chain_s,
                                            int ka, int ja, int kb, int jb, __int128& Va, __int128& Vb) {
  const int jb2 = jb >= 0 ? jb : ja;
  const uint32_t cha = p.a > 0 ? chain_s[ja] : 0u;
  const uint32_t chb = p.a > 0 ? chain_s[jb2] : 0u;
  const double pha = __ldg(&p.phi[phi_index(p, g, cha, ja)]);
  const double phb = __ldg(&p.phi[phi_index(p, g, chb, jb2)]);
  __int128 ta[3] = {0, 0, 0}, tb[3] = {0, 0, 0};
  bool ok = true;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const bool chain_axis = b < 2;
    if (chain_axis && p.a <= b) continue;
    const CtAxis& A = chain_axis ? p.ax[b] : p.ax[p.a];
    const int kk = chain_axis ? g.k[b] : ka;
    const int kk2 = chain_axis ? g.k[b] : kb;
    const int j0 = !chain_axis ? ja : (b == 0 ? static_cast<int>(cha & 0xFFFFu) : static_cast<int>(cha >> 16));
    const int j1 = !chain_axis ? jb2 : (b == 0 ? static_cast<int>(chb & 0xFFFFu) : static_cast<int>(chb >> 16));
    if (A.dyadic) {  // (mixed grids only: rare, kept out of line)
      ok = g_fixed_dyadic(A, kk, j0, ta[b]) && ok;
      ok = g_fixed_dyadic(A, kk2, j1, tb[b]) && ok;
    } else {
      ta[b] = A.GF[static_cast<long>(kk) * A.n + j0];
      tb[b] = A.GF[static_cast<long>(kk2) * A.n + j1];
    }
  }
  __int128 fa, fb;
  ok = to_fixed124(pha, fa) && ok;
  ok = to_fixed124(phb, fb) && ok;
  Va = ((ta[0] + ta[1]) + ta[2]) - fa;
  Vb = ((tb[0] + tb[1]) + tb[2]) - fb;
  return ok;
}

// Certified strict convexity of the middle point (fp64 orientation with a
// rounding bound; near-collinear counts as NOT convex).
__device__ __forceinline__ bool convex3(double ya, double fa, double yb, double fb, double yc,
                                        double fc) {
  const double t1 = (fb - fa) * (yc - yb);
  const double t2 = (fc - fb) * (yb - ya);
  const double bound = 8.0 * kU * (fabs(t1) + fabs(t2));
  return (t1 - t2) < -bound;
}

struct Smem {
  double* fh;          // f~_j
  uint32_t* chain;     // argmin chain of element j
  uint16_t* hidx;      // chunk hull stacks, later per-query winners
  uint16_t* H;         // compacted hull corners
  uint8_t* dlt;        // per-edge slack code (0: no suspects)
  uint16_t* flist;     // compacted list of flagged queries
  int* lo;
  int* hi;
  int* off;
  unsigned long long* scal;  // 0 A, 1 Smax, 2 Dmax, 3 hull size, 4 #non-convex, 5 #flagged
  LineGeo* geo;
};

__device__ __forceinline__ Smem carve(const CtPass& p, unsigned char* base, int l) {
  Smem s;
  unsigned char* b = base + static_cast<long>(l) * p.line_bytes;
  s.fh = reinterpret_cast<double*>(b + p.off_fv);
  s.chain = reinterpret_cast<uint32_t*>(b + p.off_chain);
  s.hidx = reinterpret_cast<uint16_t*>(b + p.off_hidx);
  s.H = reinterpret_cast<uint16_t*>(b + p.off_H);
  s.dlt = reinterpret_cast<uint8_t*>(b + p.off_flag);
  s.flist = reinterpret_cast<uint16_t*>(b + p.off_list);
  s.lo = reinterpret_cast<int*>(b + p.off_lohi);
  s.hi = s.lo + p.tpl;
  s.off = s.hi + p.tpl;
  s.scal = reinterpret_cast<unsigned long long*>(b + p.off_scal);
  s.geo = reinterpret_cast<LineGeo*>(b + p.off_scal + 64);
  return s;
}

struct DdBest {
  int j;
  double h, l;
};

// Slack codes: Delta <= 2^(code - 128) * sref, code in [1, 255] (conservative).
__device__ __forceinline__ uint8_t slack_code(double D, double sref) {
  if (!(D > 0.0)) return 1;
  int e;
  frexp(D / sref, &e);  // D/sref < 2^e
  e += 128;
  if (e < 1) e = 1;
  if (e > 255) e = 255;
  return static_cast<uint8_t>(e);
}
__device__ __forceinline__ double slack_value(uint8_t c, double sref) {
  // sref * 2^(c - 128): the power of two is built from its bits (c - 128 is in
  // [-127, 127], always a normal double) — exact, like ldexp, without its
  // range handling
  const double p2 = __longlong_as_double(static_cast<long long>(static_cast<int>(c) - 128 + 1023) << 52);
  return sref * p2;
}
__device__ __forceinline__ void slack_max(uint8_t* dlt, int e, uint8_t c) {
  unsigned* w = reinterpret_cast<unsigned*>(dlt + (e & ~3));
  const int sh = 8 * (e & 3);
  unsigned old = *w;
  while (true) {
    const unsigned cur = (old >> sh) & 0xffu;
    if (cur >= c) return;
    const unsigned nv = (old & ~(0xffu << sh)) | (static_cast<unsigned>(c) << sh);
    const unsigned prev = atomicCAS(w, old, nv);
    if (prev == old) return;
    old = prev;
  }
}

// Threads per CTA (lpc * tpl) at most for the non-dyadic kernel (its exact
// path lives in local memory anyway; 1024 measured fastest).
constexpr int kNdThreads = 768;

__global__ void __launch_bounds__(kNdThreads) ct_pass_kernel(CtPass p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tpl = p.tpl;
  const int l = threadIdx.x / tpl;
  const int t = threadIdx.x - l * tpl;
  const int lpc = p.lpc;
  const CtAxis& A = p.ax[p.a];
  const int n = A.n;
  const double h = A.h;
  const int C = p.C;
  Smem s = carve(p, smem, l);

  // ---- per-line geometry + scalar reset
  if (t == 0) {
    const long L = static_cast<long>(blockIdx.x) * lpc + l;
    LineGeo g;
    g.valid = L < p.nlines;
    g.base = 0;
    g.phi_other = 0;
    g.k[0] = g.k[1] = g.k[2] = 0;
    if (g.valid) {
      const long inner = L % A.stride, outer = L / A.stride;
      g.base = outer * static_cast<long>(n) * A.stride + inner;
      long rem = g.base;
      for (int b = 0; b < p.d; ++b) {
        const int c = static_cast<int>(rem / p.ax[b].stride);
        rem -= static_cast<long>(c) * p.ax[b].stride;
        g.k[b] = c;
        if (b > p.a) g.phi_other += static_cast<long>(c) * p.ax[b].stride;
      }
    }
    g.k[0] += p.k0_off;
    *s.geo = g;
    for (int q = 0; q < 8; ++q) s.scal[q] = 0ull;
  }
  __syncthreads();

  long long tph = clock64();
  auto PH = [&](int i) {
    if (p.stats && t == 0) {
      const long long now = clock64();
      atomicAdd(p.stats + 8 + i, static_cast<unsigned long long>(now - tph));
      tph = now;
    }
  };
  // ---- load: phi at the chain (cp.async) into fh, the chain into chain ---
  {
    const int ml = p.strided ? static_cast<int>(threadIdx.x % lpc) : l;
    const Smem sm = carve(p, smem, ml);
    const LineGeo g = *sm.geo;
    const int step = p.strided ? blockDim.x / lpc : tpl;
    const int first = p.strided ? static_cast<int>(threadIdx.x / lpc) : t;
    for (int j = first; j < n + 4; j += step) sm.dlt[j] = 0;
    if (g.valid) {
      {
        constexpr int kBatch = 8;
        for (int j0 = first; j0 < n; j0 += kBatch * step) {
          uint32_t ch[kBatch];
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int j = j0 + u * step;
            ch[u] = (p.a > 0 && j < n) ? p.state_in[g.base + static_cast<long>(j) * A.stride] : 0u;
          }
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int j = j0 + u * step;
            if (j >= n) continue;
            cp_async8(&sm.fh[padj(j)], &p.phi[phi_index(p, g, ch[u], j)]);
            if (p.a > 0) sm.chain[j] = ch[u];
          }
        }
      }
    }
    cp_async_wait_all();
  }
  __syncthreads();
  // line maxima for the rounding bounds (A = max |f~|, Smax = max |phi| + G + hs)
  {
    double amax = 0.0, smax = 0.0;
    const LineGeo g = *s.geo;
    if (g.valid) {
      for (int j = t; j < n; j += tpl) {
        const double y = coord(h, j);
        const double hy = 0.5 * y * y;
        // f~_j = fl(fl(-phi_j + G~_j) + hs(y_j)) in place of phi_j
        const double ph = s.fh[padj(j)];
        const uint32_t ch = p.a > 0 ? s.chain[j] : 0u;
        double G = 0.0;
        if (p.a >= 1) G += g_approx(p.ax[0], g.k[0], static_cast<int>(ch & 0xFFFFu));
        if (p.a >= 2) G += g_approx(p.ax[1], g.k[1], static_cast<int>(ch >> 16));
        const double f = (-ph + G) + hy;
        s.fh[padj(j)] = f;
        const double S = fabs(ph) + G + hy;
        amax = fmax(amax, fabs(f));
        smax = fmax(smax, S);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&s.scal[0], dbits(amax));
      atomicMax(&s.scal[1], dbits(smax));
    }
  }
  __syncthreads();

  const LineGeo geo = *s.geo;
  const bool active = geo.valid;
  const double Aabs = bitsd(s.scal[0]);
  const double Smax = bitsd(s.scal[1]);
  const double e_f = 8.0 * kU * Smax;          // |f_j - f~_j|
  const double e_r = 4.0 * kU * (Aabs + 1.0);  // |F^ - (f~ - x y)|
  const double e_F = e_f + e_r;
  const double e_d = 32.0 * kU * Aabs;                  // chord slack error
  const double tau = 2.0 * e_f + e_d;
  const double Mc = 4.0 * e_F;
  const double sref = fmax(Smax, 1e-300);
  const int j0 = t * C;
  const int j1 = min(n, j0 + C);
  uint16_t* st = s.hidx + t * (C + 2);
  auto P_y = [&](int idx) { return coord(h, idx); };
  auto P_f = [&](int idx) { return s.fh[padj(idx)]; };

  PH(0);  // load + maxima
  // ---- 0. convex fast path: every interior point a certified strict corner?
  {
    int bad = 0;
    if (active) {
      const int a0 = max(j0, 1), a1 = min(j1, n - 1);
      for (int j = a0; j < a1; ++j)
        if (!convex3(P_y(j - 1), P_f(j - 1), P_y(j), P_f(j), P_y(j + 1), P_f(j + 1))) ++bad;
    }
    if (bad) atomicAdd(reinterpret_cast<unsigned int*>(&s.scal[4]), static_cast<unsigned>(bad));
  }
  group_sync(tpl, l);
  const bool convex_line = s.scal[4] == 0ull;

  if (!convex_line) {
    PH(1);  // convexity test
    // ---- 1. chunk hulls (Andrew's monotone chain) -----------------------
    if (active) {
      int sz = 0;
      double ya = 0, fa = 0, yb = 0, fb = 0;  // top two stack points
      for (int j = j0; j < j1; ++j) {
        const double yj = P_y(j), fj = P_f(j);
        while (sz >= 2) {
          if (convex3(ya, fa, yb, fb, yj, fj)) break;
          --sz;
          yb = ya;
          fb = fa;
          if (sz >= 2) {
            const int ia = st[sz - 2];
            ya = P_y(ia);
            fa = P_f(ia);
          }
        }
        st[sz++] = static_cast<uint16_t>(j);
        ya = yb;
        fa = fb;
        yb = yj;
        fb = fj;
      }
      s.lo[t] = 0;
      s.hi[t] = sz;
    }
    PH(2);  // chunk hulls
    // ---- 2. tree merge by bridge walks ----------------------------------
    for (int lvl = 1; lvl < tpl; lvl <<= 1) {
      // a level-lvl merge reads chunks [t, t + 2 lvl): inside one warp up to
      // lvl = 16 (tpl is a multiple of 32)
      if (2 * lvl <= 32) __syncwarp();
      else group_sync(tpl, l);
      if (active && (t % (2 * lvl)) == 0 && t + lvl < tpl) {
        const int gA = t, gB = t + lvl, gE = min(t + 2 * lvl, tpl);
        int ca = gB - 1;
        while (ca >= gA && s.lo[ca] >= s.hi[ca]) --ca;
        int cb = gB;
        while (cb < gE && s.lo[cb] >= s.hi[cb]) ++cb;
        if (ca >= gA && cb < gE) {
          int pa = s.hi[ca] - 1, pb = s.lo[cb];
          auto ptidx = [&](int c, int q) { return static_cast<int>(s.hidx[c * (C + 2) + q]); };
          while (true) {
            bool moved = false;
            while (true) {  // retreat a
              int cp = ca, pp = pa - 1;
              if (pp < s.lo[cp]) {
                cp = ca - 1;
                while (cp >= gA && s.lo[cp] >= s.hi[cp]) --cp;
                if (cp < gA) break;
                pp = s.hi[cp] - 1;
              }
              const int ip = ptidx(cp, pp), ia = ptidx(ca, pa), ib = ptidx(cb, pb);
              if (convex3(P_y(ip), P_f(ip), P_y(ia), P_f(ia), P_y(ib), P_f(ib))) break;
              s.hi[ca] = pa;
              ca = cp;
              pa = pp;
              moved = true;
            }
            while (true) {  // advance b
              int cq = cb, pq = pb + 1;
              if (pq >= s.hi[cq]) {
                cq = cb + 1;
                while (cq < gE && s.lo[cq] >= s.hi[cq]) ++cq;
                if (cq >= gE) break;
                pq = s.lo[cq];
              }
              const int ia = ptidx(ca, pa), ib = ptidx(cb, pb), iq = ptidx(cq, pq);
              if (convex3(P_y(ia), P_f(ia), P_y(ib), P_f(ib), P_y(iq), P_f(iq))) break;
              s.lo[cb] = pb + 1;
              cb = cq;
              pb = pq;
              moved = true;
            }
            if (!moved) break;
          }
        }
      }
    }
    group_sync(tpl, l);
    PH(3);  // merges
    // ---- 3. compaction into H -------------------------------------------
    {
      const int cnt = active ? max(0, s.hi[t] - s.lo[t]) : 0;
      const int lane = t & 31, w = t >> 5;
      int v = cnt;
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
      }
      if (lane == 31) s.off[w] = v;
      group_sync(tpl, l);
      int pre = 0;
      for (int ww = 0; ww < w; ++ww) pre += s.off[ww];
      const int o = pre + v - cnt;
      for (int i = 0; i < cnt; ++i) s.H[o + i] = st[s.lo[t] + i];
      if (t == tpl - 1) s.scal[3] = static_cast<unsigned long long>(o + cnt);
    }
    group_sync(tpl, l);
    PH(4);  // compaction
    // ---- 4. suspects: per-edge max slack (log-coded, conservative) --------
    const int hsz0 = static_cast<int>(s.scal[3]);
    if (active && j0 < j1) {
      int lo_e = 0, hi_e = hsz0 - 1;  // largest e with H[e] <= j0
      while (lo_e < hi_e) {
        const int mid = (lo_e + hi_e + 1) >> 1;
        if (s.H[mid] <= j0) lo_e = mid;
        else hi_e = mid - 1;
      }
      int e = lo_e;
      double dloc = 0.0;
      int ecur = -1;
      double emax = -1.0;
      for (int j = j0; j < j1; ++j) {
        while (e + 1 < hsz0 && s.H[e + 1] <= j) ++e;
        const int ca = s.H[e];
        if (ca == j || e + 1 >= hsz0) continue;
        const int cb = s.H[e + 1];
        const double ya = P_y(ca), yb = P_y(cb), fa = P_f(ca), fb = P_f(cb);
        const double tt = (P_y(j) - ya) / (yb - ya);
        const double Lc = fa + (fb - fa) * tt;
        const double dt = P_f(j) - Lc;
        if (dt <= tau) {
          const double D = tau - dt;
          dloc = fmax(dloc, D);
          if (e != ecur) {
            if (ecur >= 0) slack_max(s.dlt, ecur, slack_code(emax, sref));
            ecur = e;
            emax = D;
          } else {
            emax = fmax(emax, D);
          }
        }
      }
      if (ecur >= 0) slack_max(s.dlt, ecur, slack_code(emax, sref));
      if (dloc > 0.0) atomicMax(&s.scal[2], dbits(dloc));
    }
    group_sync(tpl, l);
  }
  const int hsz = convex_line ? n : static_cast<int>(s.scal[3]);
  BFM_DASSERT(!active || (hsz >= 1 && hsz <= n));
  const double Dmax = convex_line ? 0.0 : bitsd(s.scal[2]);
  const double Mw = Mc + Dmax;
  uint16_t* res = s.hidx;  // hidx is dead after compaction
  auto HH = [&](int i) { return convex_line ? i : static_cast<int>(s.H[i]); };
  group_sync(tpl, l);

  PH(5);  // suspects (or convexity test on convex lines)
  // ---- 5. queries ---------------------------------------------------------
  if (active) {
    auto Fhat = [&](int idx, double xk) { return P_f(idx) - xk * P_y(idx); };
    auto slope_ge = [&](int i, double xk) {
      const int a = HH(i), b = HH(i + 1);
      return (P_f(b) - P_f(a)) >= xk * (P_y(b) - P_y(a));
    };
    // ---- 5a. tangent corner of every query: balanced merge path of the
    //          query slopes x_k against the hull-edge slopes (ties: query first)
    {
      const int E = hsz - 1;
      const int total = n + E;
      const int per = (total + tpl - 1) / tpl;
      const int d0 = min(total, t * per), d1 = min(total, d0 + per);
      if (d0 < d1) {
        int lo = max(0, d0 - E), hi = min(d0, n);
        while (lo < hi) {
          const int q = (lo + hi) >> 1;
          if (slope_ge(d0 - q - 1, coord(h, q))) lo = q + 1;
          else hi = q;
        }
        int k = lo, i = d0 - lo;
        for (int d = d0; d < d1; ++d) {
          if (k < n && (i >= E || slope_ge(i, coord(h, k)))) {
            res[k] = static_cast<uint16_t>(i);
            ++k;
          } else {
            ++i;
          }
        }
      }
    }
  }
  group_sync(tpl, l);
  PH(6);  // merge-path tangents
  // ---- 5b. uniform certification: the tangent corner is the only candidate
  //          if both neighbours are beyond the walk margin and neither
  //          adjacent edge holds suspects. Others are flagged (bit 15).
  if (active) {
    auto Fhat = [&](int idx, double xk) { return P_f(idx) - xk * P_y(idx); };
    unsigned* nflag = reinterpret_cast<unsigned*>(&s.scal[5]);
    const unsigned lane = threadIdx.x & 31u;
    // tpl is a multiple of 32: every warp belongs to one line and runs the
    // same number of iterations (needed by the ballot below)
    for (int kb = t - static_cast<int>(lane); kb < n; kb += tpl) {
      const int k = kb + static_cast<int>(lane);
      const bool in = k < n;
      bool lone = true;
      if (in) {
        const int i = res[k];
        const double xk = coord(h, k);
        const double F0 = Fhat(HH(i), xk);
        const double Fl = i > 0 ? Fhat(HH(i - 1), xk) : INFINITY;
        const double Fr = i < hsz - 1 ? Fhat(HH(i + 1), xk) : INFINITY;
        // an adjacent edge's suspects cannot win unless the edge passes the same
        // relevance tests the full resolution applies (see visit below)
        auto edge_quiet = [&](int e, double Fa, double Fb) {
          const uint8_t code = s.dlt[e];
          if (code == 0) return true;
          const double slack = slack_value(code, sref) + Mc;
          if (fmin(Fa, Fb) > F0 + slack) return true;
          const int a = HH(e), b = HH(e + 1);
          return fabs(Fa - Fb) > slack * (1.000001 * (b - a)) + Mc;
        };
        lone = Fl > F0 + Mw && Fr > F0 + Mw &&
               (convex_line || ((i == 0 || edge_quiet(i - 1, Fl, F0)) &&
                                (i >= hsz - 1 || edge_quiet(i, F0, Fr))));
        if (p.stats) {
          atomicAdd(p.stats + 0, 1ull);
          if (!lone) atomicAdd(p.stats + 1, 1ull);
          // why: a neighbouring corner within the margin, or an adjacent edge
          if (!(Fl > F0 + Mw && Fr > F0 + Mw)) atomicAdd(p.stats + 6, 1ull);
          if (!(Fl > F0 + Mw && Fr > F0 + Mw) && !((Fl > F0 + Mc) && (Fr > F0 + Mc)))
            atomicAdd(p.stats + 7, 1ull);  // ... even within the corner-only margin Mc
        }
        res[k] = lone ? static_cast<uint16_t>(HH(i)) : static_cast<uint16_t>(i | 0x8000);
      }
      // flagged queries are appended to the line's list (warp-aggregated)
      const unsigned fm = __ballot_sync(0xffffffffu, in && !lone);
      if (fm) {
        unsigned b0 = 0;
        if (lane == static_cast<unsigned>(__ffs(fm) - 1)) b0 = atomicAdd(nflag, __popc(fm));
        b0 = __shfl_sync(0xffffffffu, b0, __ffs(fm) - 1);
        if (in && !lone) s.flist[b0 + __popc(fm & ((1u << lane) - 1u))] = static_cast<uint16_t>(k);
      }
    }
  }
  group_sync(tpl, l);
  PH(7);  // certification
  // ---- 5c. flagged queries: full resolution from their tangent corner. The
  //          lists of all the CTA's lines are shared by all its threads, so a
  //          line with many flagged queries does not hold its CTA alone.
  // (sharing pays off with many short lines per CTA; with few long lines
  // each line keeps its own list)
  const bool share = lpc >= 4;
  if (share) __syncthreads();
  else group_sync(tpl, l);
  {
    auto nflagged = [&](int q) {
      return static_cast<int>(*reinterpret_cast<const unsigned*>(&carve(p, smem, q).scal[5]));
    };
    int total = 0;
    if (share)
      for (int q = 0; q < lpc; ++q) total += nflagged(q);
    else
      total = nflagged(l);
    const int first = share ? static_cast<int>(threadIdx.x) : t;
    const int stride = share ? static_cast<int>(blockDim.x) : tpl;
    for (int gi = first; gi < total; gi += stride) {
      int lq = share ? 0 : l, fi = gi;
      while (share) {
        const int c = nflagged(lq);
        if (fi < c) break;
        fi -= c;
        ++lq;
      }
      // the query's line: its shared memory and constants (as computed above
      // by that line's own threads)
      const Smem s = carve(p, smem, lq);
      const LineGeo geo = *s.geo;
      const double Aabs = bitsd(s.scal[0]);
      const double Smax = bitsd(s.scal[1]);
      const double e_f = 8.0 * kU * Smax;
      const double e_r = 4.0 * kU * (Aabs + 1.0);
      const double Mc = 4.0 * (e_f + e_r);
      const double sref = fmax(Smax, 1e-300);
      const bool convex_line = s.scal[4] == 0ull;
      const int hsz = convex_line ? n : static_cast<int>(s.scal[3]);
      const double Mw = Mc + (convex_line ? 0.0 : bitsd(s.scal[2]));
      uint16_t* res = s.hidx;
      auto P_f = [&](int idx) { return s.fh[padj(idx)]; };
      auto HH = [&](int i) { return convex_line ? i : static_cast<int>(s.H[i]); };
      auto Fhat = [&](int idx, double xk) { return P_f(idx) - xk * P_y(idx); };
      const int k = s.flist[fi];
      const int rv = res[k];
      const int i = rv & 0x7fff;
      const double xk = coord(h, k);
      int L = i;
      double Fmin = Fhat(HH(L), xk);
      while (L > 0) {
        const double Fl = Fhat(HH(L - 1), xk);
        if (Fl < Fmin) { --L; Fmin = Fl; } else break;
      }
      int R = L;
      if (L == i) {
        while (R < hsz - 1) {
          const double Fr = Fhat(HH(R + 1), xk);
          if (Fr < Fmin) { ++R; Fmin = Fr; } else break;
        }
        L = R;
      }
      while (L > 0) {
        const double Fl = Fhat(HH(L - 1), xk);
        if (Fl <= Fmin + Mw) { --L; Fmin = fmin(Fmin, Fl); } else break;
      }
      while (R < hsz - 1) {
        const double Fr = Fhat(HH(R + 1), xk);
        if (Fr <= Fmin + Mw) { ++R; Fmin = fmin(Fmin, Fr); } else break;
      }
      int win = HH(L);
      double outv = 0.0;
      bool have_out = false;
      const bool lone = L == R && (convex_line || ((L == 0 || s.dlt[L - 1] == 0) &&
                                                   (R >= hsz - 1 || s.dlt[R] == 0)));
      if (!lone) {
        const int e0 = L > 0 ? L - 1 : 0;
        const int e1 = R < hsz - 1 ? R : hsz - 2;
        // One traversal of the candidates: the corners L..R, then the
        // suspects of the adjacent edges that pass the relevance tests. A
        // candidate is evaluated exactly when its F^ is within the margin of
        // the running minimum (a superset of those within the margin of the
        // final minimum, which contain the exact argmin). Fixed-point grids
        // (mode 0) evaluate candidates in pairs with all their loads in
        // flight together; a value outside the fixed-point range restarts
        // the traversal on the expansion path (mode 1). The loop body exists
        // once: this path is instruction-cache bound.
        for (int mode = p.fixed ? 0 : 1;; mode = 1) {
          double Fbest = Fmin;  // min over the corners L..R
          int bestj = -1;
          __int128 bv = 0;      // mode 0: exact best value
          double bt[12];        // mode 1: exact best terms / best round-down
          int bm = 0;
          double brd = INFINITY;
          bool fail = false;
          int pend = -1;  // mode 0: first candidate of an unfinished pair
          int c = L, e = e0 - 1, js = 0, jend = 0;
          while (true) {
            int j = -1;
            bool flush = false;
            if (c <= R) {
              j = HH(c++);
            } else if (js < jend) {
              j = js++;
            } else if (!convex_line && e < e1) {
              ++e;
              const uint8_t code = s.dlt[e];
              if (p.stats) atomicAdd(p.stats + 3, 1ull);
              if (code == 0) continue;
              const int a = HH(e), b = HH(e + 1);
              const double Fa = Fhat(a, xk), Fb = Fhat(b, xk);
              const double slack = slack_value(code, sref) + Mc;
              if (fmin(Fa, Fb) > Fmin + slack) continue;
              if (fabs(Fa - Fb) > slack * (1.000001 * (b - a)) + Mc) continue;
              js = a + 1;
              jend = b;
              continue;
            } else {
              if (pend < 0) break;
              flush = true;  // an odd candidate is left
            }
            if (!flush) {
              const double F = Fhat(j, xk);
              const bool in = F <= Fbest + Mc;
              Fbest = fmin(Fbest, F);
              if (!in) continue;
            }
            if (mode == 0) {
              if (!flush && pend < 0) {
                pend = j;
                continue;
              }
              __int128 Va, Vb;
              if (!cand_fixed2(p, geo, s.chain, k, pend, k, j, Va, Vb)) {
                fail = true;
                break;
              }
              if (bestj < 0 || Va < bv) {
                bestj = pend;
                bv = Va;
              }
              if (j >= 0 && Vb < bv) {
                bestj = j;
                bv = Vb;
              }
              pend = -1;
              if (flush) break;
            } else {
              double ct[12];
              const uint32_t ch = p.a > 0 ? s.chain[j] : 0u;
              const int cm = cand_terms(p, geo, ch, j, k, ct);
              if (p.last) {
                // RD is monotone: RD(min_j V_j) = min_j RD(V_j)
                brd = fmin(brd, bfmx::round_down_sum(ct, cm));
                bestj = j;
              } else {
                if (bestj >= 0) {
                  if (p.slow_queries) atomicAdd(p.slow_queries, 1ull);
                  if (bfmx::sign_diff(ct, cm, bt, bm) >= 0) continue;
                }
                bestj = j;
                for (int q = 0; q < cm; ++q) bt[q] = ct[q];
                bm = cm;
              }
            }
          }
          if (fail) continue;  // (mode 0 only)
          win = bestj;
          if (p.last) {
            outv = mode == 0 ? rd_fixed124(bv) : brd;
            have_out = true;
          }
          break;
        }
      }
      BFM_DASSERT(win >= 0 && win < n);
      if (p.last && have_out) {
        p.out[geo.base + static_cast<long>(k) * A.stride] = outv;
        res[k] = 0xffffu;  // done
      } else {
        // (last pass: the final round-down loop below evaluates the winner)
        res[k] = static_cast<uint16_t>(win);
      }
    }
  }
  if (share) __syncthreads();
  else group_sync(tpl, l);
  PH(8);  // flagged queries
  if (p.last && active) {
    // final round-downs of the queries not written by the flagged path: two
    // queries per round (their loads in flight together); the body is kept
    // rolled, the kernel is instruction-cache bound
    for (int kk = t; kk < n; kk += 2 * tpl) {
      const int k2 = kk + tpl;
      const int w1 = res[kk];
      const int w2 = k2 < n ? static_cast<int>(res[k2]) : 0xffff;
      const bool v1 = w1 != 0xffff, v2 = w2 != 0xffff;
      if (!v1 && !v2) continue;
      const int ka = v1 ? kk : k2, ja = v1 ? w1 : w2;
      const int jb = (v1 && v2) ? w2 : -1;
      __int128 Va, Vb;
      const bool fx = p.fixed && cand_fixed2(p, geo, s.chain, ka, ja, k2, jb, Va, Vb);
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && jb < 0) break;
        const int k = u == 0 ? ka : k2, j = u == 0 ? ja : jb;
        double v;
        if (fx) {
          v = rd_fixed124(u == 0 ? Va : Vb);
        } else {
          double tv[12];
          const int m = cand_terms(p, geo, p.a > 0 ? s.chain[j] : 0u, j, k, tv);
          v = bfmx::round_down_sum(tv, m);
        }
        p.out[geo.base + static_cast<long>(k) * A.stride] = v;
      }
    }
  }
  PH(9);  // final round-downs
  if (p.last) return;
  __syncthreads();

  // ---- 6. intermediate passes: coalesced write of the argmin chain ---------
  // (same fixed thread -> line mapping as the load: no per-element division)
  {
    const int ml = p.strided ? static_cast<int>(threadIdx.x % lpc) : l;
    const int step = p.strided ? blockDim.x / lpc : tpl;
    const int first = p.strided ? static_cast<int>(threadIdx.x / lpc) : t;
    const Smem sm = carve(p, smem, ml);
    const LineGeo g = *sm.geo;
    if (g.valid)
      for (int k = first; k < n; k += step) {
        const long node = g.base + static_cast<long>(k) * A.stride;
        const int win = sm.hidx[k];
        uint32_t packed;
        uint32_t ch = 0u;
        if (p.a == 0) {
          packed = static_cast<uint32_t>(win);
        } else {
          ch = sm.chain[win];
          packed = ch | (static_cast<uint32_t>(win) << 16);
        }
        p.state_out[node] = packed;
        // phi at the winner's full chain, for the next pass (or the row owner)
        if (p.q_out) p.q_out[node] = p.phi[phi_index(p, g, ch, win)];
      }
  }
}

// ============================================================================
// Dyadic grids (every n_a a power of two): exact-hull kernel.
//
// On a dyadic grid every candidate of pass a is
//   V(k, j) = s_j - x_k y_j - q_j (+ hs(x_k)),   s_j = G_j + hs(y_j),
// where G_j = sum_{b<a} g_b(k_b, j_b*) (from the argmin chain) and s_j are
// exact doubles (multiples of 2^-(2L+3), far below 2^53 units) and q_j = phi
// at the chain. Each line keeps f~_j = fl(s_j - q_j), q_j and the chain in
// shared memory, so every decision is made on-chip:
//  * f~ drives the fp64 filters; the exact f_j = s_j - q_j (s_j recomputed
//    from the chain) is used only where a filter cannot decide.
//  * The lower hull is the EXACT hull of (y_j, f_j) with strict corners only:
//    orientation tests use a rigorous fp64 filter and fall back to an exact
//    sign (sum_i w_i s_i is exact in fp64; the w_i q_i are summed in 127-bit
//    integers when their exponents are close, else by error-free cascades).
//    C-concave potentials (phi = psi^c, every other c-transform of an
//    iteration) have exactly collinear runs on ~40% of their nodes; the exact
//    hull drops those runs' interior points, which can never be strictly
//    better than the run's end corners.
//  * Hulls are built per thread chunk (monotone chain) and merged in a
//    log2(threads) tree; each merged group's hull is contiguous, so a bridge
//    is found by galloping searches on the two monotone predicates of the
//    classic bridge walk, and B's surviving corners are moved next to A's.
//  * Over strict corners F(i) = f_{H_i} - x y_{H_i} is exactly unimodal, so a
//    query is decided by its tangent corner when both neighbours are beyond
//    the fp64 margin; otherwise the corners within the margin (usually two,
//    exactly tied on c-concave input) are compared exactly as
//    two_sum(s_j - x_k y_j, -q_j) — exact because s_j - x_k y_j is.
//  * The last pass writes RD((s_w - hs(y_w)) + 0.5 (x_k - y_w)^2 - q_w), the
//    reference's single round-down (exact.hpp:167-179).
// Non-dyadic grids keep ct_pass_kernel<false> (3-limb g tables).
// ============================================================================
constexpr int kDyThreads = 768;

// Lines are stored unpadded: setup picks an odd number of points per thread,
// so the per-thread chunk walks (stride C doubles) are bank-conflict free.
__device__ __forceinline__ int dyi(int j) { return j; }
// Exact node coordinate on a dyadic grid: (2j + 1) * (h / 2) == (j + 0.5) * h.
__device__ __forceinline__ double dy_coord(double hh, int j) { return static_cast<double>(2 * j + 1) * hh; }
constexpr int kDyStage = 6;  // corners staged per thread and round of a merge move

struct DySmem {
  double* f;       // f~_j (padded index)
  double* q;       // exact q_j (padded index)
  uint32_t* ch;    // argmin chain of element j (passes a >= 1)
  uint16_t* H;     // hull: the hull of the chunk group led by chunk g is
                   //   stored contiguously from g * C
  uint16_t* res;   // per-query tangent corner, then winner
  int* gsz;        // hull size of the group led by chunk t
  int* bA;         // bridge of the merge led by chunk t: keep A[0..bA], B[bB..)
  int* bB;
  unsigned long long* scal;  // 0 A (max |f~|), 3 hull size, 4 #uncertified interior points
  LineGeo* geo;
};

__device__ __forceinline__ DySmem dy_carve(const CtPass& p, unsigned char* base, int l) {
  DySmem s;
  unsigned char* b = base + static_cast<long>(l) * p.line_bytes;
  s.f = reinterpret_cast<double*>(b + p.off_fv);
  s.q = reinterpret_cast<double*>(b + p.off_chain);
  s.ch = reinterpret_cast<uint32_t*>(b + p.off_flag);
  s.H = reinterpret_cast<uint16_t*>(b + p.off_hidx);
  s.res = reinterpret_cast<uint16_t*>(b + p.off_H);
  s.gsz = reinterpret_cast<int*>(b + p.off_lohi);
  s.bA = s.gsz + p.tpl;
  s.bB = s.bA + p.tpl;
  s.scal = reinterpret_cast<unsigned long long*>(b + p.off_scal);
  s.geo = reinterpret_cast<LineGeo*>(b + p.off_scal + 64);
  return s;
}

// Exact s_j = G_j + hs(y_j) of element j (G from the chain; exact on dyadic grids).
__device__ __forceinline__ double dy_s_c(const CtPass& p, const LineGeo& g, uint32_t c, int j) {
  const double y = dy_coord(0.5 * p.ax[p.a].h, j);
  double G = 0.0;
  if (p.a >= 1) {
    G = g_approx(p.ax[0], g.k[0], static_cast<int>(c & 0xFFFFu));
    if (p.a >= 2) G += g_approx(p.ax[1], g.k[1], static_cast<int>(c >> 16));
  }
  return G + 0.5 * y * y;
}
__device__ __forceinline__ double dy_s(const CtPass& p, const LineGeo& g, const uint32_t* ch, int j) {
  const double y = dy_coord(0.5 * p.ax[p.a].h, j);
  double G = 0.0;
  if (p.a >= 1) {
    const uint32_t c = ch[j];
    G = g_approx(p.ax[0], g.k[0], static_cast<int>(c & 0xFFFFu));
    if (p.a >= 2) G += g_approx(p.ax[1], g.k[1], static_cast<int>(c >> 16));
  }
  return G + 0.5 * y * y;
}

// Integer path for the sign of sum_i coef_i v_i: the four doubles as m 2^e
// with 53-bit m; when their exponents lie within 56 of each other the signed
// sum of coef_i m_i 2^(e_i - emin) fits in 127 bits (|coef m| < 2^69).
__device__ __forceinline__ bool dy_sign_int(const double* v, const int* coef, int& sgn) {
  int e[4];
  int emin = 4096, emax = -4096;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long b = __double_as_longlong(v[i]);
    const int ex = static_cast<int>((b >> 52) & 0x7ff);
    e[i] = ex ? ex : 1;
    if ((b & 0x7FFFFFFFFFFFFFFFll) != 0) {
      emin = min(emin, e[i]);
      emax = max(emax, e[i]);
    }
  }
  if (emax < emin) {
    sgn = 0;
    return true;
  }
  if (emax - emin > 56) return false;
  __int128 acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long b = __double_as_longlong(v[i]);
    long long mm = b & 0xFFFFFFFFFFFFFll;
    if (((b >> 52) & 0x7ff) != 0) mm |= 1ll << 52;
    if (mm == 0) continue;
    __int128 t = static_cast<__int128>(mm) * coef[i];
    t <<= (e[i] - emin);
    acc += b < 0 ? -t : t;
  }
  sgn = acc > 0 ? 1 : (acc < 0 ? -1 : 0);
  return true;
}

__device__ __noinline__ int dy_sign_slow(const double* x) {
  bfmx::Exp<8> e;
  e.clear();
  for (int i = 0; i < 7; ++i) e.grow(x[i]);
  return e.sign();
}

// Exact sign of x0 + x1 + x2 + x3: error-free cascades (usually one pass decides).
__device__ __forceinline__ int dy_sign_sum4(double x0, double x1, double x2, double x3) {
  for (int pass = 0; pass < 16; ++pass) {
    double sm, er;
    bfmx::two_sum(x1, x0, sm, er);
    x1 = sm;
    x0 = er;
    bfmx::two_sum(x2, x1, sm, er);
    x2 = sm;
    x1 = er;
    bfmx::two_sum(x3, x2, sm, er);
    x3 = sm;
    x2 = er;
    const double rest = (fabs(x0) + fabs(x1)) + fabs(x2);
    if (rest == 0.0) return x3 > 0.0 ? 1 : (x3 < 0.0 ? -1 : 0);
    if (fabs(x3) > 1.01 * rest) return x3 > 0.0 ? 1 : -1;
  }
  bfmx::Exp<8> e;
  e.clear();
  e.grow(x0);
  e.grow(x1);
  e.grow(x2);
  e.grow(x3);
  return e.sign();
}

// Exact sign of (c-a) f_b - (c-b) f_a - (b-a) f_c with f = s - q (a < b < c):
// negative iff b is a strict lower-hull corner of (a, b, c).
// Exact sign of 2 f_b - f_a - f_c for consecutive a = b-1, c = b+1 (the
// local-corner test): (2 s_b - s_a - s_c) is exact in fp64 and 2 q_b is
// exact, so the value is an exact sum of four doubles, distilled by
// error-free cascades (usually one pass decides).
__device__ __forceinline__ int dy_orient_local(const CtPass& p, const LineGeo& g, const uint32_t* ch,
                                               const double* Q, int b) {
  const double sa = dy_s(p, g, ch, b - 1), sb = dy_s(p, g, ch, b), sc = dy_s(p, g, ch, b + 1);
  return dy_sign_sum4((2.0 * sb - sa) - sc, -2.0 * Q[dyi(b)], Q[dyi(b - 1)], Q[dyi(b + 1)]);
}

__device__ __noinline__ int dy_orient_exact(const CtPass& p, const LineGeo& g, const uint32_t* ch,
                                            const double* Q, int a, int b, int c) {
  const double sa = dy_s(p, g, ch, a), sb = dy_s(p, g, ch, b), sc = dy_s(p, g, ch, c);
  const double qa = Q[dyi(a)], qb = Q[dyi(b)], qc = Q[dyi(c)];
  const double w1 = static_cast<double>(c - a), w2 = static_cast<double>(c - b),
               w3 = static_cast<double>(b - a);
  // exact: integers below 2^16 times multiples of 2^-(2L+3) bounded by 1.5
  const double S = (w1 * sb - w2 * sa) - w3 * sc;
  {
    const double v[4] = {S, qb, qa, qc};
    const int coef[4] = {1, -(c - a), c - b, b - a};
    int sg;
    if (dy_sign_int(v, coef, sg)) return sg;
  }
  // error-free cascades (VecSum) until the leading term dominates
  double x[7];
  double pr, r;
  x[0] = S;
  bfmx::two_prod(w1, qb, pr, r);
  x[1] = -r;
  x[4] = -pr;
  bfmx::two_prod(w2, qa, pr, r);
  x[2] = r;
  x[5] = pr;
  bfmx::two_prod(w3, qc, pr, r);
  x[3] = r;
  x[6] = pr;
  for (int pass = 0; pass < 12; ++pass) {
#pragma unroll
    for (int i = 1; i < 7; ++i) {
      double sm, er;
      bfmx::two_sum(x[i], x[i - 1], sm, er);
      x[i] = sm;
      x[i - 1] = er;
    }
    double rest = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) rest += fabs(x[i]);
    if (rest == 0.0) return x[6] > 0.0 ? 1 : (x[6] < 0.0 ? -1 : 0);
    if (fabs(x[6]) > 1.01 * rest) return x[6] > 0.0 ? 1 : -1;
  }
  return dy_sign_slow(x);
}

// QG: the small-state form (p.qglobal): contiguous lines only; q and the chain
// are not staged in shared memory but read from global memory (L1/L2: the
// line's rows were just streamed) by the f~ phase, the rare exact tests, the
// flagged queries and the output gather.
template <bool QG>
__global__ void __launch_bounds__(kDyThreads) ct_dy_kernel(CtPass p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tpl = p.tpl;
  const int l = threadIdx.x / tpl;
  const int t = threadIdx.x - l * tpl;
  const int lpc = p.lpc;
  const CtAxis& A = p.ax[p.a];
  const int n = A.n;
  const double h = A.h;
  const int C = p.C;
  DySmem s = dy_carve(p, smem, l);

  if (t == 0) {
    const long L = static_cast<long>(blockIdx.x) * lpc + l;
    LineGeo g;
    g.valid = L < p.nlines;
    g.base = 0;
    g.phi_other = 0;
    g.k[0] = g.k[1] = g.k[2] = 0;
    if (g.valid) {
      const long inner = L % A.stride, outer = L / A.stride;
      g.base = outer * static_cast<long>(n) * A.stride + inner;
      long rem = g.base;
      for (int b = 0; b < p.d; ++b) {
        const int c = static_cast<int>(rem / p.ax[b].stride);
        rem -= static_cast<long>(c) * p.ax[b].stride;
        g.k[b] = c;
        if (b > p.a) g.phi_other += static_cast<long>(c) * p.ax[b].stride;
      }
    }
    g.k[0] += p.k0_off;
    if (p.t0) g.phi_other = g.base;  // transposed pass 0: line L is row L of phi^T
    *s.geo = g;
    for (int q = 0; q < 8; ++q) s.scal[q] = 0ull;
  }
  __syncthreads();

  // diagnostics (p.stats): per-thread counters flushed once at the end, and
  // per-phase clocks of each line's thread 0
  long long tph = clock64();
  unsigned c_flag = 0, c_walk = 0, c_xchunk = 0, c_xmerge = 0, c_merge = 0;
  int in_merge = 0;
  auto PH = [&](int i) {
    if (p.stats && t == 0) {
      const long long now = clock64();
      atomicAdd(p.stats + 8 + i, static_cast<unsigned long long>(now - tph));
      tph = now;
    }
  };

  // ---- load: q_j (cp.async), chain_j; then f~_j = fl(s_j - q_j) ----------
  // Contiguous pregathered passes (a >= 1 along the last axis) take the TMA
  // bulk path: per line two cp.async.bulk copies (q: 8n bytes, chain: 4n
  // bytes) completing on one mbarrier.
  if (!QG) {
  __shared__ __align__(8) uint64_t tma_bar;
  const bool tma = (p.pregathered || p.t0) && !p.strided && A.stride == 1 && (n & 3) == 0;
  if (tma) {
    if (threadIdx.x == 0) {
      mbar_init(&tma_bar, 1);
      unsigned bytes = 0;
      for (int ll = 0; ll < lpc; ++ll)
        if (dy_carve(p, smem, ll).geo->valid) bytes += (p.a > 0 ? 12u : 8u) * static_cast<unsigned>(n);
      mbar_expect_tx(&tma_bar, bytes);
      for (int ll = 0; ll < lpc; ++ll) {
        const DySmem sm = dy_carve(p, smem, ll);
        const LineGeo g = *sm.geo;
        if (!g.valid) continue;
        bulk_g2s(sm.q, &p.phi[g.base], 8u * n, &tma_bar);
        if (p.a > 0) bulk_g2s(sm.ch, &p.state_in[g.base], 4u * n, &tma_bar);
      }
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(&tma_bar, 0);
  }
  {
    const int ml = p.strided ? static_cast<int>(threadIdx.x % lpc) : l;
    const DySmem sm = dy_carve(p, smem, ml);
    const LineGeo g = *sm.geo;
    const int step = p.strided ? blockDim.x / lpc : tpl;
    const int first = p.strided ? static_cast<int>(threadIdx.x / lpc) : t;
    if (g.valid) {
      if (tma) {
        // contiguous line: q (and the chain) are whole rows, moved by the
        // TMA bulk copies issued above (one thread for the CTA)
      } else if (p.a == 0) {
        for (int j = first; j < n; j += step)
          cp_async8(&sm.q[dyi(j)], &p.phi[g.phi_other + static_cast<long>(j) * A.stride]);
      } else if (p.pregathered && tma) {
        // contiguous line: chain and q are whole rows, moved by TMA bulk
        // copies issued below (one thread for the CTA)
      } else if (p.pregathered) {
        // q sits at the candidate's own node: chain and q both go straight
        // to shared memory, every load of the line in flight at once
        for (int j = first; j < n; j += step) {
          const long node = g.base + static_cast<long>(j) * A.stride;
          cp_async4(&sm.ch[j], &p.state_in[node]);
          cp_async8(&sm.q[dyi(j)], &p.phi[node]);
        }
      } else {
        constexpr int kBatch = 8;
        for (int j0 = first; j0 < n; j0 += kBatch * step) {
          uint32_t chv[kBatch];
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int j = j0 + u * step;
            chv[u] = j < n ? p.state_in[g.base + static_cast<long>(j) * A.stride] : 0u;
          }
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int j = j0 + u * step;
            if (j >= n) continue;
            cp_async8(&sm.q[dyi(j)], &p.phi[phi_index(p, g, chv[u], j)]);
            sm.ch[j] = chv[u];
          }
        }
      }
    }
    cp_async_wait_all();
  }
  __syncthreads();
  }

  const LineGeo geo = *s.geo;
  const bool active = geo.valid;
  const double* F = s.f;
  // QG: the line's own rows in global memory (contiguous: element j at [j])
  const double* Q = QG ? p.phi + (p.a == 0 ? geo.phi_other : geo.base) : s.q;
  const uint32_t* CH = QG ? (p.a > 0 ? p.state_in + geo.base : nullptr) : s.ch;
  auto P_f = [&](int j) { return F[dyi(j)]; };
  const double hh = 0.5 * h;
  auto P_y = [&](int j) { return dy_coord(hh, j); };
  // ---- f~ and the line maximum of |f~| (rounding bounds) -------------------
  {
    double amax = 0.0;
    if (active)
      if (QG) {
        // q and the chain straight from global memory, eight coalesced loads
        // of each in flight per thread. The small-state form also remembers
        // which f~ are exact (no rounding in s - q): three exact neighbours
        // decide a local corner from shared memory alone, without reading q
        // and the chain back from L2.
        constexpr int kB = 8;
        // (flags in the second half of the res buffer, free until the hull is compacted)
        uint8_t* fx = reinterpret_cast<uint8_t*>(s.res) + n;
        for (int jb = t; jb < n; jb += kB * tpl) {
          double qv[kB];
          uint32_t cv[kB];
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const int j = jb + u * tpl;
            qv[u] = j < n ? __ldg(Q + j) : 0.0;
            cv[u] = (p.a > 0 && j < n) ? __ldg(CH + j) : 0u;
          }
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const int j = jb + u * tpl;
            if (j >= n) continue;
            double f, er;
            bfmx::two_sum(dy_s_c(p, geo, cv[u], j), -qv[u], f, er);
            fx[j] = er == 0.0 ? 1 : 0;
            s.f[dyi(j)] = f;
            amax = fmax(amax, fabs(f));
          }
        }
      } else {
        for (int j = t; j < n; j += tpl) {
          const double f = dy_s(p, geo, CH, j) - Q[dyi(j)];
          s.f[dyi(j)] = f;
          amax = fmax(amax, fabs(f));
        }
      }
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s.scal[0], dbits(amax));
  }
  group_sync(tpl, l);
  PH(0);
  const double Aabs = bitsd(s.scal[0]);
  // (the 1e-290 floors cover gradual underflow of tiny values)
  const double e_f = kU * Aabs + 1e-290;             // |f_j - f~_j|
  const double ef2 = 2.0000001 * e_f;                // filter slack per unit index span
  const double e_F = e_f + 4.0 * kU * (Aabs + 1.0);  // |F^_j - (f_j - x y_j)|
  const double Mc = 4.0 * e_F;                       // > 2 e_F: margin on F^ differences
  // Orientation filter on index differences (the common factor h dropped):
  // D = (f_b - f_a)(c - b) - (f_c - f_b)(b - a) with f~; certified when
  // |D| exceeds the rounding of the products plus 2 e_f (c - a).
  auto filt = [&](int a, double fa, int b, double fb, int c, double fc, int& und) {
    const double t1 = (fb - fa) * static_cast<double>(c - b);
    const double t2 = (fc - fb) * static_cast<double>(b - a);
    const double bound = 8.0 * kU * (fabs(t1) + fabs(t2)) + ef2 * static_cast<double>(c - a) + 1e-290;
    const double D = t1 - t2;
    und = !(D < -bound) && !(D > bound);
    return D < -bound;
  };
  auto convex_x = [&](int a, double fa, int b, double fb, int c, double fc) {
    int und;
    const bool cv = filt(a, fa, b, fb, c, fc, und);
    if (p.stats) c_merge += in_merge;
    if (!und) return cv;
    if (p.stats) {
      if (in_merge) ++c_xmerge;
      else ++c_xchunk;
    }
    return dy_orient_exact(p, geo, CH, Q, a, b, c) < 0;
  };
  const int j0 = t * C;
  const int j1 = min(n, j0 + C);
  // ---- 0. local corners: a point that is not a strict corner of (j-1, j, j+1)
  //         lies on or above that chord and can never be a strict hull
  //         corner, so it is dropped here (exactly: the filter, then the exact
  //         sign). This removes the interiors of exactly collinear runs before
  //         any merge. A line without drops is convex: its hull is the line.
  uint8_t* keep = reinterpret_cast<uint8_t*>(s.res);  // res is free until phase 4
  {
    int bad = 0;
    if (active && j0 < j1) {
      double fa = j0 > 0 ? P_f(j0 - 1) : 0.0, fb = P_f(j0);
      for (int j = j0; j < j1; ++j) {
        const double fc = j + 1 < n ? P_f(j + 1) : 0.0;
        int k = 1;
        if (j > 0 && j + 1 < n) {
          int und;
          k = filt(j - 1, fa, j, fb, j + 1, fc, und);
          if (und) {
            if (p.stats) ++c_xchunk;
            if (QG && keep[n + j - 1] && keep[n + j] && keep[n + j + 1]) {
              // 2 f_b - f_a - f_c from exact f~ values
              double h1, l1, h2, l2;
              bfmx::two_sum(fb, -fa, h1, l1);
              bfmx::two_sum(fb, -fc, h2, l2);
              k = dy_sign_sum4(l1, l2, h1, h2) < 0;
            } else {
              k = dy_orient_local(p, geo, CH, Q, j) < 0;
            }
          }
        }
        keep[j] = static_cast<uint8_t>(k);
        bad += !k;
        fa = fb;
        fb = fc;
      }
    }
    if (bad) atomicAdd(reinterpret_cast<unsigned int*>(&s.scal[4]), static_cast<unsigned>(bad));
  }
  group_sync(tpl, l);
  PH(1);
  const bool convex_line = s.scal[4] == 0ull;

  // kept_convex: every chunk's monotone chain ran without a pop and every
  // join between consecutive chunks is a strict corner, so the kept points
  // are a convex sequence and are the hull (phase 1b); the hull then lives in
  // the res buffer and the per-query results in H (line flag: scal[7])
  bool kept_convex = false;
  if (!convex_line) {
    // ---- 1. chunk hulls (monotone chain, exact strict corners) at H[t*C..)
    uint16_t* st = s.H + t * C;
    bool popped = false;
    if (active) {
      int sz = 0;
      double fa = 0, fb = 0;
      int ia = 0, ib = 0;
      for (int j = j0; j < j1; ++j) {
        if (!keep[j]) continue;
        const double fj = P_f(j);
        while (sz >= 2) {
          if (convex_x(ia, fa, ib, fb, j, fj)) break;
          popped = true;
          --sz;
          ib = ia;
          fb = fa;
          if (sz >= 2) {
            ia = st[sz - 2];
            fa = P_f(ia);
          }
        }
        st[sz++] = static_cast<uint16_t>(j);
        ia = ib;
        fa = fb;
        ib = j;
        fb = fj;
      }
      s.gsz[t] = sz;
    }
    if (popped) atomicOr(reinterpret_cast<unsigned int*>(&s.scal[5]), 1u);
    group_sync(tpl, l);
    PH(2);
    auto cvx3 = [&](int i0, int i1, int i2) { return convex_x(i0, P_f(i0), i1, P_f(i1), i2, P_f(i2)); };
    // ---- 1b. no pops anywhere (typical of c-concave input on the first
    //          pass): check the chunk joins, then compact the chunk hulls
    if (active && s.scal[5] == 0ull) {
      const int m = s.gsz[t];
      bool bad = false;
      if (m > 0) {
        int tp = t - 1;
        while (tp >= 0 && s.gsz[tp] == 0) --tp;
        int tn = t + 1;
        while (tn < tpl && s.gsz[tn] == 0) ++tn;
        if (tp >= 0) {  // (last kept before, first, second or next chunk's first)
          const int c = m >= 2 ? st[1] : (tn < tpl ? s.H[tn * C] : -1);
          if (c >= 0 && !cvx3(s.H[tp * C + s.gsz[tp] - 1], st[0], c)) bad = true;
        }
        if (!bad && m >= 2 && tn < tpl && !cvx3(st[m - 2], st[m - 1], s.H[tn * C])) bad = true;
      }
      if (bad) atomicOr(reinterpret_cast<unsigned int*>(&s.scal[6]), 1u);
      group_sync(tpl, l);
      if (s.scal[6] == 0ull) {
        kept_convex = true;
        // exclusive prefix of the chunk sizes (warps never straddle lines:
        // tpl is a multiple of 32), then every chunk moves to res
        const int lane = threadIdx.x & 31;
        int inc = m;
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += u;
        }
        if (lane == 31) s.bA[t >> 5] = inc;
        group_sync(tpl, l);
        int base = 0;
        for (int w = 0; w < (t >> 5); ++w) base += s.bA[w];
        uint16_t* R = s.res;
        for (int i = 0, o = base + inc - m; i < m; ++i) R[o + i] = st[i];
        if (t == tpl - 1) {
          s.scal[3] = static_cast<unsigned long long>(base + inc);
          s.scal[7] = 1ull;
          if (p.stats) atomicAdd(p.stats + 28, 1ull);  // lines on the kept-convex path
        }
      }
    }
    if (!kept_convex) {
      if (p.stats && t == 0 && active) atomicAdd(p.stats + 29, 1ull);  // lines merged
      in_merge = 1;
      // ---- 2. tree merge: bridge by galloping searches, then B's surviving
      //         corners are moved next to A's (register-staged, in place)
      uint16_t* Hh = s.H;
      for (int lvl = 1, li = 0; lvl < tpl; lvl <<= 1, ++li) {
        if (2 * lvl <= 32) __syncwarp();
        else group_sync(tpl, l);
        if (p.stats && t == 0) {  // per-level clocks of thread 0 (diagnostics)
          const long long now = clock64();
          if (li > 0) atomicAdd(p.stats + 18 + li - 1, static_cast<unsigned long long>(now - tph));
          tph = now;
        }
        if (active && (t % (2 * lvl)) == 0) {
          const int gB = t + lvl;
          const int szA = s.gsz[t];
          const int szB = gB < tpl ? s.gsz[gB] : 0;
          const uint16_t* HA = Hh + t * C;
          const uint16_t* HB = Hh + gB * C;
          int ia = szA - 1, ib = 0;
          if (szA > 0 && szB > 0) {
            while (true) {
              bool moved = false;
              // retreat: P(a) = (a == 0 || cvx(A[a-1], A[a], B[ib])) holds up to
              // the tangent from B[ib] and fails after it
              const int qb = HB[ib];
              if (ia > 0 && !cvx3(HA[ia - 1], HA[ia], qb)) {
                int bad = ia, good = 0, step = 1;
                while (true) {
                  const int c = bad - step;
                  if (c <= 0) break;
                  if (cvx3(HA[c - 1], HA[c], qb)) {
                    good = c;
                    break;
                  }
                  bad = c;
                  step <<= 1;
                }
                while (bad - good > 1) {
                  const int mid = (bad + good) >> 1;
                  if (cvx3(HA[mid - 1], HA[mid], qb)) good = mid;
                  else bad = mid;
                }
                ia = good;
                moved = true;
              }
              // advance: Q(b) = (b == last || cvx(A[ia], B[b], B[b+1])) fails
              // before the tangent from A[ia] and holds from it on
              const int pa = HA[ia];
              if (ib < szB - 1 && !cvx3(pa, HB[ib], HB[ib + 1])) {
                int bad = ib, good = szB - 1, step = 1;
                while (true) {
                  const int c = bad + step;
                  if (c >= szB - 1) break;
                  if (cvx3(pa, HB[c], HB[c + 1])) {
                    good = c;
                    break;
                  }
                  bad = c;
                  step <<= 1;
                }
                while (good - bad > 1) {
                  const int mid = (bad + good) >> 1;
                  if (cvx3(pa, HB[mid], HB[mid + 1])) good = mid;
                  else bad = mid;
                }
                ib = good;
                moved = true;
              }
              if (!moved) break;
            }
          }
          s.bA[t] = ia;
          s.bB[t] = ib;
          s.gsz[t] = (ia + 1) + (szB - ib);
        }
        if (2 * lvl <= 32) __syncwarp();
        else group_sync(tpl, l);
        // move B[ib..szB) to A's end (a left move): each round reads its corners
        // before any is written; at most lvl*C corners over 2*lvl threads, so
        // ceil(C / (2 kDyStage)) rounds (uniform over the line) suffice
        const int g = t & ~(2 * lvl - 1);
        const int gthreads = min(2 * lvl, tpl - g);
        int nmv = 0, dst0 = 0;
        const uint16_t* src = Hh;
        if (active && g + lvl < tpl) {
          const int ia = s.bA[g], ib = s.bB[g];
          nmv = s.gsz[g] - (ia + 1);
          src = Hh + (g + lvl) * C + ib;
          dst0 = g * C + ia + 1;
        }
        const int rounds = (C + 2 * kDyStage - 1) / (2 * kDyStage);
        for (int rd = 0; rd < rounds; ++rd) {
          const int base = rd * kDyStage * gthreads + (t - g);
          uint16_t v[kDyStage];
  #pragma unroll
          for (int r = 0; r < kDyStage; ++r) {
            const int i = base + r * gthreads;
            if (i < nmv) v[r] = src[i];
          }
          if (2 * lvl <= 32) __syncwarp();
          else group_sync(tpl, l);
  #pragma unroll
          for (int r = 0; r < kDyStage; ++r) {
            const int i = base + r * gthreads;
            if (i < nmv) Hh[dst0 + i] = v[r];
          }
        }
      }
      group_sync(tpl, l);
      if (p.stats && t == 0) atomicAdd(p.stats + 27, static_cast<unsigned long long>(clock64() - tph));
      if (t == 0) s.scal[3] = static_cast<unsigned long long>(s.gsz[0]);
    }  // !kept_convex
    PH(3);
  }
  group_sync(tpl, l);
  const int hsz = convex_line ? n : static_cast<int>(s.scal[3]);
  BFM_DASSERT(!active || (hsz >= 1 && hsz <= n));
  const uint16_t* Hf = kept_convex ? s.res : s.H;
  uint16_t* res = kept_convex ? s.H : s.res;
  auto HH = [&](int i) { return convex_line ? i : static_cast<int>(Hf[i]); };

  // ---- 4. tangent corner of every query: balanced merge path of the query
  //         slopes x_k against the hull-edge slopes (ties: query first)
  if (active) {
    auto slope_ge = [&](int i, double xh) {  // xh = x_k h
      const int a = HH(i), b = HH(i + 1);
      return (P_f(b) - P_f(a)) >= xh * static_cast<double>(b - a);
    };
    const int E = hsz - 1;
    const int total = n + E;
    const int per = (total + tpl - 1) / tpl;
    const int d0 = min(total, t * per), d1 = min(total, d0 + per);
    if (d0 < d1) {
      int lo = max(0, d0 - E), hi = min(d0, n);
      while (lo < hi) {
        const int qm = (lo + hi) >> 1;
        if (slope_ge(d0 - qm - 1, P_y(qm) * h)) lo = qm + 1;
        else hi = qm;
      }
      int k = lo, i = d0 - lo;
      double xh = P_y(k) * h;
      for (int d = d0; d < d1; ++d) {
        if (k < n && (i >= E || slope_ge(i, xh))) {
          res[k] = static_cast<uint16_t>(i);
          ++k;
          xh = P_y(k) * h;
        } else {
          ++i;
        }
      }
    }
  }
  group_sync(tpl, l);
  PH(4);

  // ---- 5. certification and exact resolution, per query --------------------
  if (active) {
    for (int k = t; k < n; k += tpl) {
      const int i = res[k];
      const double xk = P_y(k);
      auto Fh = [&](int c) {
        const int j = HH(c);
        return P_f(j) - xk * P_y(j);
      };
      const double F0 = Fh(i);
      bool lone = true;
      if (i > 0) lone = Fh(i - 1) > F0 + Mc;
      if (lone && i < hsz - 1) lone = Fh(i + 1) > F0 + Mc;
      int win = HH(i);
      if (!lone) {
        if (p.stats) ++c_flag;
        // descend to the local minimum of F^, then take every corner within
        // the margin: the exact minimum over (unimodal) corners lies inside
        int L = i;
        double Fmin = F0;
        while (L > 0) {
          const double Fl = Fh(L - 1);
          if (Fl < Fmin) { --L; Fmin = Fl; } else break;
        }
        int R = L;
        if (L == i) {
          while (R < hsz - 1) {
            const double Fr = Fh(R + 1);
            if (Fr < Fmin) { ++R; Fmin = Fr; } else break;
          }
          L = R;
        }
        while (L > 0) {
          const double Fl = Fh(L - 1);
          if (Fl <= Fmin + Mc) { --L; Fmin = fmin(Fmin, Fl); } else break;
        }
        while (R < hsz - 1) {
          const double Fr = Fh(R + 1);
          if (Fr <= Fmin + Mc) { ++R; Fmin = fmin(Fmin, Fr); } else break;
        }
        if (p.stats) c_walk += R - L + 1;
        // exact: V_j - hs(x_k) = two_sum(s_j - x_k y_j, -q_j), lexicographic
        double bh = 0.0, bl = 0.0;
        for (int c = L; c <= R; ++c) {
          const int j = HH(c);
          double vh, vl;
          bfmx::two_sum(dy_s(p, geo, CH, j) - xk * P_y(j), -Q[dyi(j)], vh, vl);
          if (c == L || vh < bh || (vh == bh && vl < bl)) {
            win = j;
            bh = vh;
            bl = vl;
          }
        }
      }
      if (p.last) {
        const double yw = P_y(win);
        const double dl = xk - yw;
        const double G = dy_s(p, geo, CH, win) - 0.5 * yw * yw;  // exact
        p.out[geo.base + static_cast<long>(k) * A.stride] =
            bfmx::round_down2(G + 0.5 * dl * dl, -Q[dyi(win)]);
      } else {
        res[k] = static_cast<uint16_t>(win);
      }
    }
  }
  PH(5);
  if (p.stats) {
    unsigned vv[5] = {c_flag, c_walk, c_xchunk, c_xmerge, c_merge};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      unsigned x = vv[i];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) == 0 && x) atomicAdd(p.stats + 1 + i, static_cast<unsigned long long>(x));
    }
    if (t == 0 && active) atomicAdd(p.stats + 0, static_cast<unsigned long long>(n));
  }
  if (p.last) return;
  __syncthreads();

  // ---- 6. intermediate passes: argmin chain and q at the winner ------------
  {
    const int ml = p.strided ? static_cast<int>(threadIdx.x % lpc) : l;
    const int step = p.strided ? blockDim.x / lpc : tpl;
    const int first = p.strided ? static_cast<int>(threadIdx.x / lpc) : t;
    const DySmem sm = dy_carve(p, smem, ml);
    const LineGeo g = *sm.geo;
    if (g.valid)
      for (int k = first; k < n; k += step) {
        const long node = g.base + static_cast<long>(k) * A.stride;
        const int win = (sm.scal[7] ? sm.H : sm.res)[k];
        const uint32_t* chp = QG ? CH : sm.ch;  // (QG: one line per thread group, ml == l)
        const double* qp = QG ? Q : sm.q;
        const uint32_t packed = p.a == 0 ? static_cast<uint32_t>(win)
                                         : (chp[win] | (static_cast<uint32_t>(win) << 16));
        p.state_out[node] = packed;
        if (p.q_out) p.q_out[node] = qp[dyi(win)];
      }
  }
}

// Tiled transposes for the transposed pass 0: in (rows x cols) -> out (cols x
// rows), 32 x 32 tiles through padded shared memory, both sides coalesced.
template <class T>
__device__ __forceinline__ void transpose_tile(const T* in, T* out, int rows, int cols, T (*tile)[33]) {
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8)
    if (r0 + i < rows && c0 + tx < cols) tile[i][tx] = in[static_cast<long>(r0 + i) * cols + c0 + tx];
  __syncthreads();
  for (int i = ty; i < 32; i += 8)
    if (c0 + i < cols && r0 + tx < rows) out[static_cast<long>(c0 + i) * rows + r0 + tx] = tile[tx][i];
}
__global__ void __launch_bounds__(256) ct_transpose_f64(const double* in, double* out, int rows, int cols) {
  __shared__ double tile[32][33];
  transpose_tile(in, out, rows, cols, tile);
}
__global__ void __launch_bounds__(256) ct_transpose_state(const uint32_t* sin, const double* qin, uint32_t* sout,
                                                          double* qout, int rows, int cols) {
  __shared__ double tq[32][33];
  __shared__ uint32_t ts[32][33];
  transpose_tile(qin, qout, rows, cols, tq);
  transpose_tile(sin, sout, rows, cols, ts);
}

int align16(int v) { return (v + 15) & ~15; }

bool is_dyadic(int n) { return n > 0 && (n & (n - 1)) == 0 && n <= (1 << 25); }

}  // namespace

CtPlan::~CtPlan() {
  for (int a = 0; a < 3; ++a)
    if (tables_[a]) {
      bool shared = false;
      for (int b = 0; b < a; ++b) shared |= tables_[b] == tables_[a];
      if (!shared) {
        dfree(tables_[a]);
        if (ftables_[a]) dfree(ftables_[a]);
      }
    }
  for (auto* p : state_)
    if (p) dfree(p);
  for (auto* p : qbuf_)
    if (p) dfree(p);
  if (slow_) dfree(slow_);
  if (stats_) dfree(stats_);
  if (phit_) dfree(phit_);
  if (statet_) dfree(statet_);
  if (qt_) dfree(qt_);
}

void CtPlan::init(const GridDesc& g) { setup(g, g, 0, g.d, 0, false, false); }

void CtPlan::init_slab_rows(const GridDesc& global, int row0, int nrows) {
  if (global.d < 2) throw std::invalid_argument("ctransform: slabs need d >= 2");
  int ext[3] = {nrows, global.n[1], global.d > 2 ? global.n[2] : 1};
  setup(make_grid(global.d, ext), global, 1, global.d, row0, true, false);
}

void CtPlan::init_slab_cols(const GridDesc& global, int ncols) {
  if (global.d < 2) throw std::invalid_argument("ctransform: slabs need d >= 2");
  int ext[2] = {global.n[0], ncols};
  setup(make_grid(2, ext), global, 0, 1, 0, false, true);
}

// loc: the grid the kernels walk (the whole grid, a row slab, or the
// (n0 x ncols) column slab whose second axis is virtual); global: the
// problem's grid (coordinates, dyadic tables). Passes [pb, pe) of loc.
void CtPlan::setup(const GridDesc& loc, const GridDesc& global, int pb, int pe, int k0_off,
                   bool pregathered, bool virtual_cols) {
  g_ = loc;
  pb_ = pb;
  pe_ = pe;
  k0_off_ = k0_off;
  // real axes share the global grid's extent and coordinates; the column
  // slab's second axis is virtual (a flattened block of columns)
  const int nreal = virtual_cols ? 1 : loc.d;
  for (int a = 0; a < loc.d; ++a) {
    CtAxis& A = ax_[a];
    A.stride = loc.stride[a];
    A.G = nullptr;
    if (a >= nreal) {  // virtual column axis
      A.n = loc.n[a];
      A.h = 1.0;
      A.dyadic = 1;
      continue;
    }
    if (global.n[a] > 65535) throw std::invalid_argument("ctransform: extent above 65535");
    A.n = global.n[a];
    A.h = global.h[a];
    A.dyadic = is_dyadic(global.n[a]) ? 1 : 0;
    if (!A.dyadic) {
      for (int b = 0; b < a; ++b)
        if (!ax_[b].dyadic && global.n[b] == global.n[a]) tables_[a] = tables_[b];
      if (!tables_[a]) {
        if (global.n[a] > 4096) throw std::invalid_argument("ctransform: non-dyadic extent above 4096");
        const int n = global.n[a];
        std::vector<double4> host(static_cast<size_t>(n) * n);
        for (int k = 0; k < n; ++k) {
          const double x = coord(global.h[a], k);
          for (int j = 0; j < n; ++j) {
            const double y = coord(global.h[a], j);
            double pr, pe2;
            bfmx::two_prod(x, y, pr, pe2);
            bfmx::Exp<8> e;
            e.clear();
            e.grow(0.5 * x * x);
            e.grow(0.5 * y * y);
            e.grow(-pe2);
            e.grow(-pr);
            // peel off up to three limbs, largest first; the remainder must vanish
            double limb[3] = {0.0, 0.0, 0.0};
            for (int q = 0; q < 3; ++q) {
              limb[q] = e.approx();
              e.grow(-limb[q]);
            }
            if (e.n != 0) throw std::runtime_error("ctransform: g table entry needs > 3 limbs");
            host[static_cast<size_t>(k) * n + j] = make_double4(limb[0], limb[1], limb[2], 0.0);
          }
        }
        BFM_CUDA(dmalloc(&tables_[a], host.size() * sizeof(double4)));
        BFM_CUDA(cudaMemcpy(tables_[a], host.data(), host.size() * sizeof(double4),
                            cudaMemcpyHostToDevice));
        // the same values as exact integers g * 2^124 when every coordinate
        // is a multiple of 2^-62 (coord(h, 0) >= 2^-10, i.e. n <= 512)
        if (coord(global.h[a], 0) >= 0x1p-10) {
          std::vector<__int128> fx(host.size());
          bool ok = true;
          auto fixed = [&](double v, int scale) -> __int128 {  // v * 2^scale, must be an integer
            if (v == 0.0) return 0;
            int E = 0;
            const double f = std::frexp(std::fabs(v), &E);  // |v| = f 2^E, f in [0.5, 1)
            const long long m = static_cast<long long>(std::ldexp(f, 53));  // exact
            const int sh = E - 53 + scale;
            __int128 r;
            if (sh >= 0) {
              if (sh > 126 - 53) ok = false;
              r = static_cast<__int128>(m) << (sh > 70 ? 70 : sh);
            } else {
              if (sh < -53 || (m & ((1ll << -sh) - 1)) != 0) ok = false;
              r = sh < -53 ? 0 : (m >> -sh);
            }
            return v < 0 ? -r : r;
          };
          for (int k = 0; k < n && ok; ++k) {
            const double x = coord(global.h[a], k);
            for (int j = 0; j < n; ++j) {
              const double y = coord(global.h[a], j);
              const __int128 X = fixed(x, 62), Y = fixed(y, 62);
              const __int128 g = fixed(0.5 * x * x, 124) + fixed(0.5 * y * y, 124) - X * Y;
              // must equal the limbs of the expansion table
              const double4 L = host[static_cast<size_t>(k) * n + j];
              if (g != fixed(L.x, 124) + fixed(L.y, 124) + fixed(L.z, 124)) ok = false;
              fx[static_cast<size_t>(k) * n + j] = g;
            }
          }
          if (ok) {
            BFM_CUDA(dmalloc(&ftables_[a], fx.size() * sizeof(__int128)));
            BFM_CUDA(cudaMemcpy(ftables_[a], fx.data(), fx.size() * sizeof(__int128), cudaMemcpyHostToDevice));
          }
        }
      }
      A.G = tables_[a];
      for (int b = 0; b < a; ++b)
        if (tables_[b] == tables_[a]) ftables_[a] = ftables_[b];
      A.GF = ftables_[a];
    }
  }
  dyadic_ = true;
  for (int a = 0; a < global.d; ++a) dyadic_ = dyadic_ && is_dyadic(global.n[a]);
  if (loc.d > 1 && pe - pb > 1) {
    BFM_CUDA(dmalloc(&state_[0], loc.size * sizeof(uint32_t)));
    BFM_CUDA(dmalloc(&qbuf_[0], loc.size * sizeof(double)));
    if (pe - pb > 2) {
      BFM_CUDA(dmalloc(&state_[1], loc.size * sizeof(uint32_t)));
      BFM_CUDA(dmalloc(&qbuf_[1], loc.size * sizeof(double)));
    }
  }
  BFM_CUDA(dmalloc(&slow_, sizeof(unsigned long long)));
  BFM_CUDA(cudaMemset(slow_, 0, sizeof(unsigned long long)));
  if (getenv("BFM_CT_STATS")) {
    BFM_CUDA(dmalloc(&stats_, 32 * sizeof(unsigned long long)));
    BFM_CUDA(cudaMemset(stats_, 0, 32 * sizeof(unsigned long long)));
  }

  int dev = 0;
  BFM_CUDA(cudaGetDevice(&dev));
  int max_optin = 0;
  BFM_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int budget = max_optin - 1024;

  // shared-memory layout, threads and lines per CTA of a dyadic pass (qg: the small-state form)
    auto dy_layout = [&](CtPass& P, int a, int n, bool qg) {
      // exact-hull kernel: (s, q) per point in shared memory; about 11 points
      // per thread, up to kDyThreads threads per line
      // about cpt points per thread, and an ODD count C (the unpadded
      // per-thread chunk walks are then bank-conflict free)
      int cpt = 11;
      // tiny grids (C1: 256 lines of 256 points, one line per CTA): three points
      // per thread shorten the per-thread loops of a latency-bound line (C1
      // c-transform 55 -> 45 us per call); with many lines (128^3) or longer
      // ones (512^2) eleven stay better
      if (n <= 256 && P.nlines < 1024) cpt = 3;
      if (const char* e = getenv("BFM_CT_C")) cpt = std::max(2, atoi(e));  // tuning experiments
      // Small-state form (qg) for long contiguous lines: q and the chain stay
      // in global memory, so four 4096-lines of 192 threads fit one SM
      // instead of two of 384. On a generic potential that is 24-29 % faster
      // (C5 4096^2: 1.91 -> 1.44 ms per call, 8192^2: 8.44 -> 6.00); on a
      // c-concave input it is 1-7 % slower (its exactly collinear runs send
      // 16 % of the points through the exact local test, which then reads q
      // and the chain from L2), so the caller's hint picks the form per call.
      if (qg) cpt = 22;
      if (const char* e = getenv("BFM_CT_QG_C")) { if (qg) cpt = std::max(2, atoi(e)); }
      int best_tpl = 32, best_err = 1 << 30;
      for (int tp = 32; tp <= kDyThreads; tp += 32) {
        const int c = (n + tp - 1) / tp;
        const int err = std::abs(c - cpt) + ((c & 1) || qg ? 0 : 3) + (tp > n ? 2000 : 0);
        if (err < best_err) {
          best_err = err;
          best_tpl = tp;
        }
      }
      P.tpl = best_tpl;
      P.C = (n + P.tpl - 1) / P.tpl;
      int o = 0;
      P.off_fv = o;
      o = align16(o + 8 * n);
      P.qglobal = qg ? 1 : 0;
      P.off_chain = o;
      if (!qg) o = align16(o + 8 * n);
      P.off_flag = o;  // chain (uint32, passes a >= 1)
      if (a > 0 && !qg) o = align16(o + 4 * n);
      P.off_hidx = o;  // hull
      o = align16(o + 2 * P.tpl * P.C);
      P.off_H = o;  // per-query tangent / winner
      o = align16(o + 2 * n);
      P.off_list = o;  // unused
      P.off_lohi = o;  // gsz, bA, bB
      o = align16(o + 12 * P.tpl);
      P.off_scal = o;
      o = align16(o + 64 + static_cast<int>(sizeof(LineGeo)));
      P.line_bytes = o;
      if (o > budget) throw std::invalid_argument("ctransform: grid line too long for shared memory");
      // two CTAs per SM: a CTA's loads overlap the other's hull work
      int lpc = std::min<long>(budget / (2 * o), kDyThreads / (2 * P.tpl));
      if (qg) lpc = 1;  // independent CTAs, as many as fit
      // strided passes: two adjacent columns per CTA (one CTA per SM) rather
      // than two one-column CTAs — the column pair shares every 32-byte
      // sector of its loads and stores (C3 c-transform 1.774 -> 1.697 ms per
      // call; the contiguous passes are better at one line per CTA)
      if (P.strided && budget / o >= 2) lpc = std::max(lpc, std::min(2, kDyThreads / P.tpl));
      if (const char* e = getenv(P.strided ? "BFM_DY_LPC_S" : "BFM_DY_LPC_C"))  // tuning experiments
        lpc = std::max(1, std::min<int>(std::min<long>(atoi(e), budget / o), kDyThreads / P.tpl));
      lpc = std::min(lpc, P.strided ? 16 : 8);
      // tiny grids (C1, 256 lines per pass): one line per CTA spreads the
      // latency-bound passes over the SMs (C1 c-transform 62.6 -> 55.5 us per
      // call); at 1024 lines (C2) the packed CTAs were faster (119 vs 150 us)
      if (P.nlines < 1024) lpc = static_cast<int>(std::min<long>(lpc, std::max<long>(1, P.nlines / (2 * 148))));
      lpc = static_cast<int>(std::min<long>(lpc, P.nlines));
      P.lpc = std::max(lpc, 1);
      P.slow_queries = slow_;
      P.stats = stats_;
    };
  for (int a = pb; a < pe; ++a) {
    CtPass& P = pass_[a];
    std::memset(&P, 0, sizeof(P));
    P.d = loc.d;
    P.a = a;
    P.last = a == global.d - 1;
    P.k0_off = k0_off;
    P.pregathered = pregathered ? 1 : 0;
    for (int b = 0; b < loc.d; ++b) P.ax[b] = ax_[b];
    const int n = loc.n[a];
    P.nlines = loc.size / n;
    P.strided = a != loc.d - 1;
    P.fixed = 1;
    for (int b = 0; b < loc.d; ++b)
      if (!P.ax[b].dyadic && !P.ax[b].GF) P.fixed = 0;
    const bool dy = dyadic_;
    if (dy) {
      // the small-state form of the last (contiguous) pass, for lines of 4096 points and more
      const bool want_q = a == loc.d - 1 && n >= 4096 && !virtual_cols;
      bool staged_ok = true;
      try {
        dy_layout(P, a, n, false);
      } catch (const std::invalid_argument&) {
        // the staged line state (24 bytes per point) does not fit: the last
        // pass can still run in the small-state form alone (12 bytes per
        // point: lines of up to ~17 k points), and so can pass 0 of a 2-D
        // grid on the transposed potential (checked below)
        const bool t0_can = a == 0 && loc.d == 2 && pb == 0 && pe == 2 && !virtual_cols && !pregathered && k0_off == 0;
        if (!want_q && !t0_can) throw;
        staged_ok = false;
        if (t0_can && !want_q) pass0_needs_t0_ = true;
      }
      if (want_q) {
        passq_ = P;
        dy_layout(passq_, a, n, true);
        have_q_ = true;
        if (!staged_ok) {
          P = passq_;
          q_only_ = true;
        }
      }
      continue;
    }
    P.tpl = n <= 512 ? 32 : (n <= 1024 ? 64 : (n <= 2048 ? 128 : 256));
    P.C = (n + P.tpl - 1) / P.tpl;
    int o = 0;
    P.off_fv = o;
    o = align16(o + 8 * (n + n / 32 + 1));
    P.off_chain = o;  // chain (uint32, passes a > 0)
    if (a > 0) o = align16(o + 4 * n);
    P.off_hidx = o;
    o = align16(o + 2 * std::max(P.tpl * (P.C + 2), n));
    P.off_H = o;
    o = align16(o + 2 * n);
    P.off_flag = o;  // per-edge slack code (uint8)
    o = align16(o + n + 4);
    P.off_list = o;  // flagged query list (uint16)
    o = align16(o + 2 * n);
    P.off_lohi = o;
    o = align16(o + 12 * P.tpl);
    P.off_scal = o;
    o = align16(o + 64 + static_cast<int>(sizeof(LineGeo)));
    P.line_bytes = o;
    if (o > budget) throw std::invalid_argument("ctransform: grid line too long for shared memory");
    int lpc = std::min<long>(budget / o, kNdThreads / P.tpl);
    // 12 short lines per CTA: two CTAs per SM on C4's 384-lines (measured
    // best among 4/8/12/16: 49 vs 53 ms of c-transform per C4 iteration at 16)
    int lcap = 12;
    if (const char* e = getenv("BFM_ND_LPC")) lcap = std::max(1, atoi(e));  // tuning experiments
    lpc = std::min(lpc, lcap);
    if (P.tpl > 32) lpc = std::min(lpc, 15);
    lpc = static_cast<int>(std::min<long>(lpc, P.nlines));
    P.lpc = std::max(lpc, 1);
    P.slow_queries = slow_;
    P.stats = stats_;
  }
  // Transposed pass 0 (2-D dyadic grids, whole-grid plans): pass 0's lines are
  // the columns of phi — two per CTA at best, every row a separate sector.
  // On phi^T they are contiguous rows like the last pass's (one line per CTA,
  // coalesced loads and stores); the two tiled transposes (phi in; chain and q
  // out) cost less than the strided pass loses. BFM_CT_T0=0/1 overrides.
  t0_ = dyadic_ && loc.d == 2 && pb == 0 && pe == 2 && !virtual_cols && !pregathered && k0_off == 0 &&
        loc.size >= (1L << 22);
  if (const char* e = getenv("BFM_CT_T0"))
    t0_ = atoi(e) != 0 && dyadic_ && loc.d == 2 && pb == 0 && pe == 2 && !virtual_cols && !pregathered;
  if (pass0_needs_t0_) t0_ = true;
  if (t0_) {
    BFM_CUDA(dmalloc(&phit_, loc.size * sizeof(double)));
    BFM_CUDA(dmalloc(&statet_, loc.size * sizeof(uint32_t)));
    BFM_CUDA(dmalloc(&qt_, loc.size * sizeof(double)));
    CtPass& T = pass0t_;
    T = pass_[0];
    T.t0 = 1;
    T.strided = 0;
    T.ax[0].stride = 1;
    T.ax[1].stride = loc.n[0];
    if (!pass0_needs_t0_) {
      // lines per CTA as for a contiguous pass
      int lpc = std::min<long>(budget / (2 * T.line_bytes), kDyThreads / (2 * T.tpl));
      if (const char* e = getenv("BFM_DY_LPC_C"))
        lpc = std::max(1, std::min<int>(std::min<long>(atoi(e), budget / T.line_bytes), kDyThreads / T.tpl));
      lpc = std::min(lpc, 8);
      lpc = static_cast<int>(std::min<long>(lpc, T.nlines));
      T.lpc = std::max(lpc, 1);
    }
    // the transposed pass 0 is contiguous: with lines of 4096 points and more
    // it has a small-state twin (its only form when the staged state does not fit)
    have_qt_ = loc.n[0] >= 4096;
    if (have_qt_) {
      pass0tq_ = T;
      dy_layout(pass0tq_, 0, loc.n[0], true);
    } else if (pass0_needs_t0_) {
      throw std::invalid_argument("ctransform: grid line too long for shared memory");
    }
  }
  qg_mode_ = 2;  // 0: never, 1: whenever available, 2: by the caller's hint (default)
  if (const char* e = getenv("BFM_CT_QG")) qg_mode_ = atoi(e);
  if (const char* e = getenv("BFM_CT_QG_MIX")) qg_mix_ = atoi(e);
  BFM_CUDA(cudaFuncSetAttribute(ct_dy_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
  BFM_CUDA(cudaFuncSetAttribute(ct_dy_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
  BFM_CUDA(cudaFuncSetAttribute(ct_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
  ready_ = true;
}

void CtPlan::launch(const CtPass& P, cudaStream_t stream, LaunchCounter* lc) {
  const long blocks = (P.nlines + P.lpc - 1) / P.lpc;
  if (dyadic_)
    if (P.qglobal)
      ct_dy_kernel<true><<<static_cast<unsigned>(blocks), P.lpc * P.tpl, P.lpc * P.line_bytes, stream>>>(P);
    else
      ct_dy_kernel<false><<<static_cast<unsigned>(blocks), P.lpc * P.tpl, P.lpc * P.line_bytes, stream>>>(P);
  else
    ct_pass_kernel<<<static_cast<unsigned>(blocks), P.lpc * P.tpl, P.lpc * P.line_bytes, stream>>>(P);
  BFM_LAUNCH_CHECK("ct_pass_kernel");
  if (lc) lc->add();
}

void CtPlan::run_cols(const double* d_phi_cols, uint32_t* d_chain, double* d_q, cudaStream_t stream,
                      LaunchCounter* lc) {
  CtPass P = pass_[0];
  P.phi = d_phi_cols;
  P.state_out = d_chain;
  P.q_out = d_q;
  launch(P, stream, lc);
}

void CtPlan::run_rows(const uint32_t* d_chain0, const double* d_q, double* d_out,
                      cudaStream_t stream, LaunchCounter* lc) {
  for (int a = 1; a < g_.d; ++a) {
    CtPass P = pass_[a];
    P.phi = a == 1 ? d_q : qbuf_[0];
    P.pregathered = 1;
    P.state_in = a == 1 ? d_chain0 : state_[0];
    P.state_out = P.last ? nullptr : state_[0];
    P.q_out = P.last ? nullptr : qbuf_[0];
    P.out = d_out;
    launch(P, stream, lc);
  }
}

// Pass a >= 1 reads phi(chain*, y) at its own nodes from the previous pass's
// q output (written next to the argmin chain) instead of gathering phi.
void CtPlan::run(const double* d_phi, double* d_out, cudaStream_t stream, LaunchCounter* lc,
                 cudaEvent_t before_last, bool concave_input) {
  const bool qg = qg_mode_ == 1 || (qg_mode_ == 2 && !concave_input);
  // hinted calls: per-pass choice of the form (bit 0: transposed pass 0, bit 1: last pass)
  const bool qg_first = qg || (qg_mode_ == 2 && concave_input && (qg_mix_ & 1));
  const bool qg_last = qg || (qg_mode_ == 2 && concave_input && (qg_mix_ & 2));
  for (int a = 0; a < g_.d; ++a) {
    if (a == 0 && t0_) {
      const int n0 = g_.n[0], n1 = g_.n[1];
      const dim3 gin((n1 + 31) / 32, (n0 + 31) / 32), gout((n0 + 31) / 32, (n1 + 31) / 32);
      ct_transpose_f64<<<gin, 256, 0, stream>>>(d_phi, phit_, n0, n1);
      CtPass P = ((qg_first || pass0_needs_t0_) && have_qt_) ? pass0tq_ : pass0t_;
      P.phi = phit_;
      P.pregathered = 0;
      P.state_in = nullptr;
      P.state_out = statet_;
      P.q_out = qt_;
      P.out = d_out;
      launch(P, stream, lc);
      ct_transpose_state<<<gout, 256, 0, stream>>>(statet_, qt_, state_[0], qbuf_[0], n1, n0);
      BFM_LAUNCH_CHECK("ct transposes");
      if (lc) lc->add(2);
      continue;
    }
    CtPass P = ((qg_last || q_only_) && have_q_ && a == g_.d - 1) ? passq_ : pass_[a];
    if (P.last && before_last) BFM_CUDA(cudaStreamWaitEvent(stream, before_last, 0));
    P.phi = a == 0 ? d_phi : qbuf_[(a - 1) & 1];
    P.pregathered = a > 0 ? 1 : 0;
    P.state_in = a > 0 ? state_[(a - 1) & 1] : nullptr;
    P.state_out = P.last ? nullptr : state_[a & 1];
    P.q_out = P.last ? nullptr : qbuf_[a & 1];
    P.out = d_out;
    launch(P, stream, lc);
  }
}

void CtPlan::stats(unsigned long long* out8) {
  for (int i = 0; i < 32; ++i) out8[i] = 0;
  if (stats_) BFM_CUDA(cudaMemcpy(out8, stats_, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
}

unsigned long long CtPlan::slow_query_count() {
  unsigned long long v = 0;
  BFM_CUDA(cudaMemcpy(&v, slow_, sizeof(v), cudaMemcpyDeviceToHost));
  return v;
}

}  // namespace bfmgpu

// ---- diagnostics (exported through the C ABI for tests) --------------------
namespace bfmgpu {
namespace {
__global__ void debug_rd_kernel(const double* t, int m, int count, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = bfmx::round_down_sum(t + static_cast<long>(i) * m, m);
}
}  // namespace

void debug_round_down(const double* h_terms, int m, int count, double* h_out) {
  double *dt = nullptr, *dout = nullptr;
  BFM_CUDA(dmalloc(&dt, sizeof(double) * m * count));
  BFM_CUDA(dmalloc(&dout, sizeof(double) * count));
  BFM_CUDA(cudaMemcpy(dt, h_terms, sizeof(double) * m * count, cudaMemcpyHostToDevice));
  debug_rd_kernel<<<(count + 127) / 128, 128>>>(dt, m, count, dout);
  BFM_LAUNCH_CHECK("debug_rd_kernel");
  BFM_CUDA(cudaMemcpy(h_out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost));
  dfree(dt);
  dfree(dout);
}
}  // namespace bfmgpu
