// Exact quadratic c-transform, B200 (sm_100a).
//
// Reference semantics (transforms.hpp:396-432, :340-391, exact.hpp:167-179):
//   psi(x) = RD( min_y  sum_a [hs(x_a) + hs(y_a) - x_a*y_a] - phi(y) )
// with hs(c) = fl(0.5*c*c), exact products and sums, and a single rounding
// toward -inf (-0 -> +0). The minimum is unique, so any exact algorithm gives
// the reference's bits (checked against oracle/_ref in tests/).
//
// Design (one kernel per axis pass, reference axis order 0..d-1):
//  * Inter-pass state is the argmin INDEX chain (uint32: j0 | j1<<16), not an
//    expansion: the exact candidate value is recomputed from the chain, one
//    phi gather and the per-axis g_a(k,j) = hs(x_k)+hs(y_j)-x_k*y_j terms
//    (an exact double 0.5*(x-y)^2 on dyadic grids, an exact double-double
//    table otherwise). Traffic per pass: read phi or (chain + gathered phi),
//    write chain or psi — the 16*d B/node algorithmic figure of SURVEY §8(d).
//  * Per grid line (staged in shared memory, TPL threads per line): the
//    minimisation min_j f_j - x_k*y_j is a discrete Legendre transform. Each
//    thread builds the lower hull of its chunk (monotone chain, fp64
//    orientation that pops anything not CERTIFIED strictly convex), a
//    log2(TPL)-level tree merges neighbouring hulls by bridge walks, the hull
//    is compacted, and every non-corner point is checked against its hull
//    edge: a point above the edge by more than the rounding bound can never
//    be a minimiser; closer points are flagged "suspect" with their slack.
//  * Each query walks to its tangent corner, expands to every corner within
//    a rigorous margin of the approximate minimum, and adds the suspects of
//    the adjacent edges. One candidate (the normal case) is the exact
//    argmin with no exact arithmetic at all; otherwise candidates are
//    compared with exact expansion arithmetic (exact.cuh).
//  * The last pass rounds the winner's exact value down once.
#include <cassert>
#include <cmath>
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
  int k[3];
  int valid;
};

__device__ __forceinline__ double g_approx(const CtAxis& A, int k, int j) {
  if (A.dyadic) {
    const double dl = coord(A.h, k) - coord(A.h, j);
    return 0.5 * dl * dl;
  }
  BFM_DASSERT(k >= 0 && k < A.n && j >= 0 && j < A.n);
  return A.G[static_cast<long>(k) * A.n + j].x;
}

__device__ __forceinline__ int g_terms(const CtAxis& A, int k, int j, double* t) {
  if (A.dyadic) {
    const double dl = coord(A.h, k) - coord(A.h, j);
    t[0] = 0.5 * dl * dl;
    return 1;
  }
  BFM_DASSERT(k >= 0 && k < A.n && j >= 0 && j < A.n);
  const double4 v = A.G[static_cast<long>(k) * A.n + j];
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
  long idx = g.phi_other + static_cast<long>(j) * p.ax[p.a].stride;
  if (p.a >= 1) idx += static_cast<long>(chain & 0xFFFFu) * p.ax[0].stride;
  if (p.a >= 2) idx += static_cast<long>(chain >> 16) * p.ax[1].stride;
  return idx;
}

// Exact terms of V(k, j) = -phi(chain, j) + sum_{b<a} g_b(k_b, j_b*) + g_a(k, j).
__device__ int cand_terms(const CtPass& p, const LineGeo& g, uint32_t chain, int j, int k,
                          double* t) {
  int m = 0;
  t[m++] = -p.phi[phi_index(p, g, chain, j)];
  if (p.a >= 1) m += g_terms(p.ax[0], g.k[0], static_cast<int>(chain & 0xFFFFu), t + m);
  if (p.a >= 2) m += g_terms(p.ax[1], g.k[1], static_cast<int>(chain >> 16), t + m);
  m += g_terms(p.ax[p.a], k, j, t + m);
  return m;
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
  double* fv;
  uint32_t* chain;
  uint16_t* hidx;
  uint16_t* H;
  uint8_t* flag;
  int* lo;
  int* hi;
  int* off;
  unsigned long long* scal;  // 0: A bits, 1: Smax bits, 2: dmax bits, 3: hull size
  LineGeo* geo;
};

__device__ __forceinline__ Smem carve(const CtPass& p, unsigned char* base, int l) {
  Smem s;
  unsigned char* b = base + static_cast<long>(l) * p.line_bytes;
  s.fv = reinterpret_cast<double*>(b + p.off_fv);
  s.chain = reinterpret_cast<uint32_t*>(b + p.off_chain);
  s.hidx = reinterpret_cast<uint16_t*>(b + p.off_hidx);
  s.H = reinterpret_cast<uint16_t*>(b + p.off_H);
  s.flag = reinterpret_cast<uint8_t*>(b + p.off_flag);
  s.lo = reinterpret_cast<int*>(b + p.off_lohi);
  s.hi = s.lo + p.tpl;
  s.off = s.hi + p.tpl;
  s.scal = reinterpret_cast<unsigned long long*>(b + p.off_scal);
  s.geo = reinterpret_cast<LineGeo*>(b + p.off_scal + 64);
  return s;
}

__global__ void __launch_bounds__(1024) ct_pass_kernel(CtPass p) {
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
    *s.geo = g;
    s.scal[0] = 0ull;
    s.scal[1] = 0ull;
    s.scal[2] = 0ull;
    s.scal[3] = 0ull;
  }
  __syncthreads();

  // ---- load: f~_j = fl(-phi + sum_{b<a} g_b + hs(y_j)) -----------------
  {
    double amax = 0.0, smax = 0.0;
    int ml;  // the line this thread loads for (fixed per thread)
    if (p.strided) {
      ml = threadIdx.x % lpc;
      const Smem sm = carve(p, smem, ml);
      const LineGeo g = *sm.geo;
      for (int idx = threadIdx.x; idx < n * lpc; idx += blockDim.x) {
        const int j = idx / lpc;
        sm.flag[j] = 0;
        if (!g.valid) continue;
        const long node = g.base + static_cast<long>(j) * A.stride;
        uint32_t ch = 0;
        if (p.a > 0) ch = p.state_in[node];
        const double ph = p.phi[phi_index(p, g, ch, j)];
        const double y = coord(h, j);
        const double hy = 0.5 * y * y;
        double f = -ph;
        double S = fabs(ph) + hy;
        if (p.a >= 1) {
          const double g0 = g_approx(p.ax[0], g.k[0], static_cast<int>(ch & 0xFFFFu));
          f += g0;
          S += g0;
        }
        if (p.a >= 2) {
          const double g1 = g_approx(p.ax[1], g.k[1], static_cast<int>(ch >> 16));
          f += g1;
          S += g1;
        }
        f += hy;
        sm.fv[padj(j)] = f;
        if (p.a > 0) sm.chain[j] = ch;
        amax = fmax(amax, fabs(f));
        smax = fmax(smax, S);
      }
    } else {
      ml = l;
      const LineGeo g = *s.geo;
      for (int j = t; j < n; j += tpl) {
        s.flag[j] = 0;
        if (!g.valid) continue;
        const long node = g.base + j;
        uint32_t ch = 0;
        if (p.a > 0) ch = p.state_in[node];
        const double ph = p.phi[phi_index(p, g, ch, j)];
        const double y = coord(h, j);
        const double hy = 0.5 * y * y;
        double f = -ph;
        double S = fabs(ph) + hy;
        if (p.a >= 1) {
          const double g0 = g_approx(p.ax[0], g.k[0], static_cast<int>(ch & 0xFFFFu));
          f += g0;
          S += g0;
        }
        if (p.a >= 2) {
          const double g1 = g_approx(p.ax[1], g.k[1], static_cast<int>(ch >> 16));
          f += g1;
          S += g1;
        }
        f += hy;
        s.fv[padj(j)] = f;
        if (p.a > 0) s.chain[j] = ch;
        amax = fmax(amax, fabs(f));
        smax = fmax(smax, S);
      }
    }
    const Smem sm = carve(p, smem, ml);
    atomicMax(&sm.scal[0], dbits(amax));
    atomicMax(&sm.scal[1], dbits(smax));
  }
  __syncthreads();

  const LineGeo geo = *s.geo;
  const bool active = geo.valid;
  const double Aabs = bitsd(s.scal[0]);
  const double Smax = bitsd(s.scal[1]);
  const double e_f = 8.0 * kU * Smax;
  const double e_r = 4.0 * kU * (Aabs + 1.0);
  const double e_F = e_f + e_r;
  const double e_d = 32.0 * kU * Aabs;
  const double tau = 2.0 * e_f + e_d;
  const int j0 = t * C;
  const int j1 = min(n, j0 + C);
  uint16_t* st = s.hidx + t * (C + 2);
  auto P_y = [&](int idx) { return coord(h, idx); };
  auto P_f = [&](int idx) { return s.fv[padj(idx)]; };

  // ---- 1. chunk hulls (Andrew's monotone chain) -------------------------
  if (active) {
    int sz = 0;
    for (int j = j0; j < j1; ++j) {
      const double yj = P_y(j), fj = P_f(j);
      while (sz >= 2) {
        const int ia = st[sz - 2], ib = st[sz - 1];
        if (convex3(P_y(ia), P_f(ia), P_y(ib), P_f(ib), yj, fj)) break;
        --sz;
      }
      st[sz++] = static_cast<uint16_t>(j);
    }
    s.lo[t] = 0;
    s.hi[t] = sz;
  }

  // ---- 2. tree merge by bridge walks -------------------------------------
  for (int lvl = 1; lvl < tpl; lvl <<= 1) {
    group_sync(tpl, l);
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

  // ---- 3. compaction into H ---------------------------------------------
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
  const int hsz = static_cast<int>(s.scal[3]);
  BFM_DASSERT(!active || (hsz >= 1 && hsz <= n));

  // ---- 4. suspects: non-corners within tau of their hull edge -----------
  if (active && j0 < j1) {
    int lo_e = 0, hi_e = hsz - 1;  // largest e with H[e] <= j0
    while (lo_e < hi_e) {
      const int mid = (lo_e + hi_e + 1) >> 1;
      if (s.H[mid] <= j0) lo_e = mid;
      else hi_e = mid - 1;
    }
    int e = lo_e;
    double dloc = 0.0;
    for (int j = j0; j < j1; ++j) {
      while (e + 1 < hsz && s.H[e + 1] <= j) ++e;
      const int ca = s.H[e];
      if (ca == j || e + 1 >= hsz) continue;
      const int cb = s.H[e + 1];
      const double ya = P_y(ca), yb = P_y(cb), fa = P_f(ca), fb = P_f(cb);
      const double tt = (P_y(j) - ya) / (yb - ya);
      const double Lc = fa + (fb - fa) * tt;
      const double dt = P_f(j) - Lc;
      if (dt <= tau) {
        s.flag[e] = 1;
        dloc = fmax(dloc, tau - dt);
      }
    }
    if (dloc > 0.0) atomicMax(&s.scal[2], dbits(dloc));
  }
  group_sync(tpl, l);
  const double dmax = bitsd(s.scal[2]);
  const double Ms = 4.0 * e_F + dmax + 4.0 * e_r;
  const double cmp_margin = 4.0 * e_F;
  uint16_t* res = s.hidx;  // hidx is dead after compaction
  group_sync(tpl, l);

  // ---- 5. queries ---------------------------------------------------------
  if (active && j0 < j1) {
    auto Fhat = [&](int idx, double xk) { return P_f(idx) - xk * P_y(idx); };
    auto slope_ge = [&](int i, double xk) {
      const int a = s.H[i], b = s.H[i + 1];
      return (P_f(b) - P_f(a)) >= xk * (P_y(b) - P_y(a));
    };
    double xk = coord(h, j0);
    int lo_i = 0, hi_i = hsz - 1;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i) >> 1;
      if (slope_ge(mid, xk)) hi_i = mid;
      else lo_i = mid + 1;
    }
    int i = lo_i;
    for (int k = j0; k < j1; ++k) {
      xk = coord(h, k);
      while (i < hsz - 1 && !slope_ge(i, xk)) ++i;
      // descend to a local minimum of F^ over corners
      int L = i;
      double Fmin = Fhat(s.H[L], xk);
      while (L > 0) {
        const double Fl = Fhat(s.H[L - 1], xk);
        if (Fl < Fmin) { --L; Fmin = Fl; } else break;
      }
      int R = L;
      if (L == i) {
        while (R < hsz - 1) {
          const double Fr = Fhat(s.H[R + 1], xk);
          if (Fr < Fmin) { ++R; Fmin = Fr; } else break;
        }
        L = R;
      }
      // expand within the certified margin
      while (L > 0) {
        const double Fl = Fhat(s.H[L - 1], xk);
        if (Fl <= Fmin + Ms) { --L; Fmin = fmin(Fmin, Fl); } else break;
      }
      while (R < hsz - 1) {
        const double Fr = Fhat(s.H[R + 1], xk);
        if (Fr <= Fmin + Ms) { ++R; Fmin = fmin(Fmin, Fr); } else break;
      }
      const bool sus = (L > 0 && s.flag[L - 1]) || (R < hsz - 1 && s.flag[R]) ||
                       (L < R);  // interior flags only matter with several corners
      int win;
      if (!sus) {
        win = s.H[L];
      } else {
        // exact resolution over corners [L,R] + suspects of edges [L-1, R]
        if (p.slow_queries) atomicAdd(p.slow_queries, 1ull);
        const int e0 = L > 0 ? L - 1 : 0;
        const int e1 = R < hsz - 1 ? R + 1 : hsz - 1;
        int best = -1;
        double bestF = 0.0;
        double bt[12];
        int bm = 0;
        auto consider = [&](int j) {
          const double Fj = Fhat(j, xk);
          if (best >= 0 && Fj - bestF > cmp_margin) return;
          double ct[12];
          const uint32_t ch = p.a > 0 ? s.chain[j] : 0u;
          const int cm = cand_terms(p, geo, ch, j, k, ct);
          if (best >= 0 && bfmx::sign_diff(ct, cm, bt, bm) >= 0) return;
          best = j;
          bestF = Fj;
          for (int q = 0; q < cm; ++q) bt[q] = ct[q];
          bm = cm;
        };
        for (int e = e0; e <= e1; ++e) {
          const int c = s.H[e];
          if (e >= L && e <= R) consider(c);
          if (e < e1 && s.flag[e]) {
            const int cb = s.H[e + 1];
            const double ya = P_y(c), yb = P_y(cb), fa = P_f(c), fb = P_f(cb);
            for (int j = c + 1; j < cb; ++j) {
              const double tt = (P_y(j) - ya) / (yb - ya);
              const double dt = P_f(j) - (fa + (fb - fa) * tt);
              if (dt <= tau) consider(j);
            }
          }
        }
        win = best;
      }
      BFM_DASSERT(win >= 0 && win < n);
      res[k] = static_cast<uint16_t>(win);
    }
  }
  __syncthreads();

  // ---- 6. write-out (coalesced) -------------------------------------------
  const bool all_dyadic = p.ax[0].dyadic && (p.d < 2 || p.ax[1].dyadic) &&
                          (p.d < 3 || p.ax[2].dyadic);
  for (int idx = threadIdx.x; idx < n * lpc; idx += blockDim.x) {
    int ll, k;
    if (p.strided) {
      ll = idx % lpc;
      k = idx / lpc;
    } else {
      ll = idx / n;
      k = idx - ll * n;
    }
    const Smem sm = carve(p, smem, ll);
    const LineGeo g = *sm.geo;
    if (!g.valid) continue;
    const long node = g.base + static_cast<long>(k) * A.stride;
    const int win = sm.hidx[k];
    const uint32_t ch = p.a > 0 ? sm.chain[win] : 0u;
    if (!p.last) {
      p.state_out[node] = p.a == 0 ? static_cast<uint32_t>(win)
                                   : (ch | (static_cast<uint32_t>(win) << 16));
    } else {
      double tv[12];
      const int m = cand_terms(p, g, ch, win, k, tv);
      double r;
      if (all_dyadic) {
        double G = 0.0;
        for (int q = 1; q < m; ++q) G += tv[q];  // exact on dyadic grids
        r = bfmx::round_down2(G, tv[0]);
      } else {
        r = bfmx::round_down_sum(tv, m);
      }
      p.out[node] = r;
    }
  }
}

int align16(int v) { return (v + 15) & ~15; }

bool is_dyadic(int n) { return n > 0 && (n & (n - 1)) == 0 && n <= (1 << 25); }

}  // namespace

CtPlan::~CtPlan() {
  for (int a = 0; a < 3; ++a)
    if (tables_[a]) {
      bool shared = false;
      for (int b = 0; b < a; ++b) shared |= tables_[b] == tables_[a];
      if (!shared) cudaFree(tables_[a]);
    }
  for (auto* p : state_)
    if (p) cudaFree(p);
  if (slow_) cudaFree(slow_);
}

void CtPlan::init(const GridDesc& g) {
  g_ = g;
  for (int a = 0; a < g.d; ++a) {
    if (g.n[a] > 65535) throw std::invalid_argument("ctransform: extent above 65535");
    CtAxis& A = ax_[a];
    A.n = g.n[a];
    A.stride = g.stride[a];
    A.h = g.h[a];
    A.dyadic = is_dyadic(g.n[a]) ? 1 : 0;
    A.G = nullptr;
    if (!A.dyadic) {
      for (int b = 0; b < a; ++b)
        if (!ax_[b].dyadic && g.n[b] == g.n[a]) tables_[a] = tables_[b];
      if (!tables_[a]) {
        if (g.n[a] > 4096) throw std::invalid_argument("ctransform: non-dyadic extent above 4096");
        const int n = g.n[a];
        std::vector<double4> host(static_cast<size_t>(n) * n);
        for (int k = 0; k < n; ++k) {
          const double x = coord(g.h[a], k);
          for (int j = 0; j < n; ++j) {
            const double y = coord(g.h[a], j);
            double pr, pe;
            bfmx::two_prod(x, y, pr, pe);
            bfmx::Exp<8> e;
            e.clear();
            e.grow(0.5 * x * x);
            e.grow(0.5 * y * y);
            e.grow(-pe);
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
        BFM_CUDA(cudaMalloc(&tables_[a], host.size() * sizeof(double4)));
        BFM_CUDA(cudaMemcpy(tables_[a], host.data(), host.size() * sizeof(double4),
                            cudaMemcpyHostToDevice));
      }
      A.G = tables_[a];
    }
  }
  if (g.d > 1) {
    BFM_CUDA(cudaMalloc(&state_[0], g.size * sizeof(uint32_t)));
    if (g.d > 2) BFM_CUDA(cudaMalloc(&state_[1], g.size * sizeof(uint32_t)));
  }
  BFM_CUDA(cudaMalloc(&slow_, sizeof(unsigned long long)));
  BFM_CUDA(cudaMemset(slow_, 0, sizeof(unsigned long long)));

  int dev = 0;
  BFM_CUDA(cudaGetDevice(&dev));
  int max_optin = 0;
  BFM_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int budget = max_optin - 1024;

  for (int a = 0; a < g.d; ++a) {
    CtPass& P = pass_[a];
    std::memset(&P, 0, sizeof(P));
    P.d = g.d;
    P.a = a;
    P.last = a == g.d - 1;
    for (int b = 0; b < g.d; ++b) P.ax[b] = ax_[b];
    const int n = g.n[a];
    P.nlines = g.size / n;
    P.tpl = n <= 1024 ? 32 : (n <= 2048 ? 64 : 128);
    P.C = (n + P.tpl - 1) / P.tpl;
    P.strided = a != g.d - 1;
    int o = 0;
    P.off_fv = o;
    o = align16(o + 8 * (n + n / 32 + 1));
    P.off_chain = o;
    if (a > 0) o = align16(o + 4 * n);
    P.off_hidx = o;
    o = align16(o + 2 * std::max(P.tpl * (P.C + 2), n));
    P.off_H = o;
    o = align16(o + 2 * n);
    P.off_flag = o;
    o = align16(o + n);
    P.off_lohi = o;
    o = align16(o + 12 * P.tpl);
    P.off_scal = o;
    o = align16(o + 64 + static_cast<int>(sizeof(LineGeo)));
    P.line_bytes = o;
    if (o > budget) throw std::invalid_argument("ctransform: grid line too long for shared memory");
    int lpc = std::min<long>(budget / o, 1024 / P.tpl);
    lpc = std::min(lpc, P.strided ? 16 : 8);
    if (P.tpl > 32) lpc = std::min(lpc, 15);
    lpc = static_cast<int>(std::min<long>(lpc, P.nlines));
    P.lpc = std::max(lpc, 1);
    P.slow_queries = slow_;
  }
  BFM_CUDA(cudaFuncSetAttribute(ct_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                budget));
  ready_ = true;
}

void CtPlan::run(const double* d_phi, double* d_out, cudaStream_t stream, LaunchCounter* lc) {
  for (int a = 0; a < g_.d; ++a) {
    CtPass P = pass_[a];
    P.phi = d_phi;
    P.state_in = a > 0 ? state_[(a - 1) & 1] : nullptr;
    P.state_out = P.last ? nullptr : state_[a & 1];
    P.out = d_out;
    const long blocks = (P.nlines + P.lpc - 1) / P.lpc;
    ct_pass_kernel<<<static_cast<unsigned>(blocks), P.lpc * P.tpl, P.lpc * P.line_bytes,
                     stream>>>(P);
    BFM_LAUNCH_CHECK("ct_pass_kernel");
    if (lc) lc->add();
  }
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
  BFM_CUDA(cudaMalloc(&dt, sizeof(double) * m * count));
  BFM_CUDA(cudaMalloc(&dout, sizeof(double) * count));
  BFM_CUDA(cudaMemcpy(dt, h_terms, sizeof(double) * m * count, cudaMemcpyHostToDevice));
  debug_rd_kernel<<<(count + 127) / 128, 128>>>(dt, m, count, dout);
  BFM_LAUNCH_CHECK("debug_rd_kernel");
  BFM_CUDA(cudaMemcpy(h_out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost));
  cudaFree(dt);
  cudaFree(dout);
}
}  // namespace bfmgpu
