// Exact c-transform for separable power costs on sm_100a.
//
// Reference semantics (transforms.hpp:335-427 generic path, cost.hpp:36-40):
//   phi^c(x) = RD( min_y  sum_a axis_cost_a(y_a - x_a) - phi(y) ),
// axis_cost_a(d) = |d|^p_a / p_a (0.5*d*d when p_a == 2), evaluated as a
// double on the node coordinates, every sum exact, one rounding toward -inf.
//
// Design: the Legendre/hull shortcut of the quadratic kernel does not apply,
// so each axis pass is a dense min-plus product per grid line against the
// per-axis cost table (host-evaluated with std::pow, uploaded transposed so
// the queries of a warp read consecutive entries). As in ctransform.cu the
// inter-pass state is the argmin chain; candidate values are recomputed from
// it exactly. A double pass finds the approximate minimum; every candidate
// within a rigorous rounding margin of it is then compared exactly
// (expansion sign), and the last pass takes the minimum of the candidates'
// exact round-downs (RD is monotone).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "ctransform_power.cuh"
#include "exact.cuh"

namespace bfmgpu {
namespace {

constexpr double kU = 1.1102230246251565e-16;  // 2^-53

struct PowGeo {
  long base;
  long phi_other;
  int k[3];
  int valid;
};

__device__ __forceinline__ long pow_phi_index(const CtPowPass& p, const PowGeo& g, uint32_t chain,
                                              int j) {
  long idx = g.phi_other + static_cast<long>(j) * p.ax[p.a].stride;
  if (p.a >= 1) idx += static_cast<long>(chain & 0xFFFFu) * p.ax[0].stride;
  if (p.a >= 2) idx += static_cast<long>(chain >> 16) * p.ax[1].stride;
  return idx;
}

// Exact terms of V(k, j): -phi(chain, j), axis_cost_b(k_b, j_b*) (b < a),
// axis_cost_a(k, j). Returns the count (<= 4).
__device__ __forceinline__ int pow_terms(const CtPowPass& p, const PowGeo& g, uint32_t chain, int j,
                                         int k, double* t) {
  int m = 0;
  t[m++] = -p.phi[pow_phi_index(p, g, chain, j)];
  if (p.a >= 1) {
    const CtPowAxis& B = p.ax[0];
    t[m++] = B.Tt[static_cast<long>(chain & 0xFFFFu) * B.n + g.k[0]];
  }
  if (p.a >= 2) {
    const CtPowAxis& B = p.ax[1];
    t[m++] = B.Tt[static_cast<long>(chain >> 16) * B.n + g.k[1]];
  }
  const CtPowAxis& A = p.ax[p.a];
  t[m++] = A.Tt[static_cast<long>(j) * A.n + k];
  return m;
}

__global__ void __launch_bounds__(512) ct_pow_kernel(CtPowPass p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tpl = p.tpl, lpc = p.lpc;
  const int l = threadIdx.x / tpl;
  const int t = threadIdx.x - l * tpl;
  const CtPowAxis& A = p.ax[p.a];
  const int n = A.n;
  auto line_smem = [&](int q) { return smem + static_cast<long>(q) * p.line_bytes; };
  auto f_of = [&](int q) { return reinterpret_cast<double*>(line_smem(q)); };
  auto ch_of = [&](int q) { return reinterpret_cast<uint32_t*>(line_smem(q) + 8L * n); };
  auto res_of = [&](int q) { return reinterpret_cast<uint16_t*>(line_smem(q) + 12L * n); };
  auto smax_of = [&](int q) {
    return reinterpret_cast<unsigned long long*>(line_smem(q) + ((14L * n + 15) & ~15L));
  };
  auto geo_of = [&](int q) { return reinterpret_cast<PowGeo*>(smax_of(q) + 2); };

  if (t == 0) {
    const long L = static_cast<long>(blockIdx.x) * lpc + l;
    PowGeo g;
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
    *geo_of(l) = g;
    *smax_of(l) = 0ull;
  }
  __syncthreads();

  // load (coalesced for strided lines): f~_j = fl(-phi + costs of the chain)
  {
    const int ml = p.strided ? static_cast<int>(threadIdx.x % lpc) : l;
    const int step = p.strided ? blockDim.x / lpc : tpl;
    const int first = p.strided ? static_cast<int>(threadIdx.x / lpc) : t;
    const PowGeo g = *geo_of(ml);
    double* f = f_of(ml);
    uint32_t* ch = ch_of(ml);
    double smax = 0.0;
    if (g.valid)
      for (int j = first; j < n; j += step) {
        const uint32_t c = p.a > 0 ? p.state_in[g.base + static_cast<long>(j) * A.stride] : 0u;
        double tv[4];
        const int m = pow_terms(p, g, c, j, 0, tv) - 1;  // without the current axis' cost
        double s = tv[0], S = fabs(tv[0]);
        for (int i = 1; i < m; ++i) {
          s += tv[i];
          S += fabs(tv[i]);
        }
        f[j] = s;
        ch[j] = c;
        smax = fmax(smax, S);
      }
    atomicMax(smax_of(ml), static_cast<unsigned long long>(__double_as_longlong(smax)));
  }
  __syncthreads();

  const PowGeo geo = *geo_of(l);
  if (geo.valid) {
    const double* f = f_of(l);
    const uint32_t* ch = ch_of(l);
    uint16_t* res = res_of(l);
    const double Smax = __longlong_as_double(static_cast<long long>(*smax_of(l)));
    // |v~_j - V_j| <= u |v~_j| + 2.0001 u S_j with |v~_j| <= Smax + tmax (1 + u):
    // candidates within 2E of the approximate minimum, E = 4 u (Smax + tmax)
    const double E = 4.0 * kU * (Smax + A.tmax);
    for (int k = t; k < n; k += tpl) {
      double vmin = INFINITY;
      for (int j = 0; j < n; ++j) vmin = fmin(vmin, f[j] + A.Tt[static_cast<long>(j) * n + k]);
      const double thr = vmin + 2.0 * E;
      if (p.last) {
        double best = INFINITY;
        for (int j = 0; j < n; ++j) {
          if (!(f[j] + A.Tt[static_cast<long>(j) * n + k] <= thr)) continue;
          double tv[4];
          const int m = pow_terms(p, geo, ch[j], j, k, tv);
          best = fmin(best, bfmx::round_down_sum(tv, m));
        }
        p.out[geo.base + static_cast<long>(k) * A.stride] = best;
      } else {
        int bestj = -1;
        double bt[4];
        int bm = 0;
        for (int j = 0; j < n; ++j) {
          if (!(f[j] + A.Tt[static_cast<long>(j) * n + k] <= thr)) continue;
          double tv[4];
          const int m = pow_terms(p, geo, ch[j], j, k, tv);
          if (bestj >= 0 && bfmx::sign_diff(tv, m, bt, bm) >= 0) continue;
          bestj = j;
          for (int i = 0; i < m; ++i) bt[i] = tv[i];
          bm = m;
        }
        res[k] = static_cast<uint16_t>(bestj);
      }
    }
  }
  if (p.last) return;
  __syncthreads();
  // argmin chain of this pass (coalesced mapping)
  {
    const int ml = p.strided ? static_cast<int>(threadIdx.x % lpc) : l;
    const int step = p.strided ? blockDim.x / lpc : tpl;
    const int first = p.strided ? static_cast<int>(threadIdx.x / lpc) : t;
    const PowGeo g = *geo_of(ml);
    if (g.valid)
      for (int k = first; k < n; k += step) {
        const int win = res_of(ml)[k];
        const uint32_t packed =
            p.a == 0 ? static_cast<uint32_t>(win) : (ch_of(ml)[win] | (static_cast<uint32_t>(win) << 16));
        p.state_out[g.base + static_cast<long>(k) * A.stride] = packed;
      }
  }
}

}  // namespace

double power_axis_cost(double p, double delta) {
  if (p == 2.0) return 0.5 * delta * delta;
  return std::pow(std::fabs(delta), p) / p;
}

CtPowerPlan::~CtPowerPlan() {
  for (int a = 0; a < 3; ++a) {
    bool shared = false;
    for (int b = 0; b < a; ++b) shared |= tables_[b] == tables_[a];
    if (tables_[a] && !shared) dfree(tables_[a]);
  }
  for (auto* s : state_)
    if (s) dfree(s);
}

void CtPowerPlan::init(const GridDesc& g, const double* exponents) {
  g_ = g;
  CtPowAxis ax[3] = {};
  for (int a = 0; a < g.d; ++a) {
    const double pa = exponents[a];
    if (!(pa > 1.0)) throw std::invalid_argument("cost exponents must satisfy p > 1");
    const int n = g.n[a];
    if (n > 2048) throw std::invalid_argument("power-cost c-transform: axis extents up to 2048");
    for (int b = 0; b < a; ++b)
      if (g.n[b] == n && exponents[b] == pa) {
        tables_[a] = tables_[b];
        ax[a].tmax = ax[b].tmax;
      }
    if (!tables_[a]) {
      std::vector<double> T(static_cast<size_t>(n) * n);
      double tmax = 0.0;
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j) {
          // transforms.hpp:380-383: axis_cost(axis, y_j - x_k) on the node table
          const double v = power_axis_cost(pa, coord(g.h[a], j) - coord(g.h[a], k));
          T[static_cast<size_t>(j) * n + k] = v;
          tmax = std::fmax(tmax, std::fabs(v));
        }
      BFM_CUDA(dmalloc(&tables_[a], T.size() * sizeof(double)));
      BFM_CUDA(cudaMemcpy(tables_[a], T.data(), T.size() * sizeof(double), cudaMemcpyHostToDevice));
      ax[a].tmax = tmax;
    }
    ax[a].n = n;
    ax[a].stride = g.stride[a];
    ax[a].Tt = tables_[a];
  }
  if (g.d > 1) {
    BFM_CUDA(dmalloc(&state_[0], g.size * sizeof(uint32_t)));
    if (g.d > 2) BFM_CUDA(dmalloc(&state_[1], g.size * sizeof(uint32_t)));
  }
  for (int a = 0; a < g.d; ++a) {
    CtPowPass& P = pass_[a];
    std::memset(&P, 0, sizeof(P));
    P.d = g.d;
    P.a = a;
    P.last = a == g.d - 1;
    for (int b = 0; b < g.d; ++b) P.ax[b] = ax[b];
    const int n = g.n[a];
    P.nlines = g.size / n;
    P.tpl = n >= 256 ? 256 : 32 * ((n + 31) / 32);
    P.strided = a != g.d - 1;
    P.line_bytes = static_cast<int>(((14L * n + 15) & ~15L) + 16 + ((sizeof(PowGeo) + 15) & ~15UL));
    int lpc = 512 / P.tpl;
    lpc = std::min(lpc, P.strided ? 16 : 8);
    lpc = static_cast<int>(std::min<long>(lpc, P.nlines));
    P.lpc = std::max(lpc, 1);
  }
  BFM_CUDA(cudaFuncSetAttribute(ct_pow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
}

void CtPowerPlan::run(const double* d_phi, double* d_out, cudaStream_t stream, LaunchCounter* lc) {
  for (int a = 0; a < g_.d; ++a) {
    CtPowPass P = pass_[a];
    P.phi = d_phi;
    P.state_in = a > 0 ? state_[(a - 1) & 1] : nullptr;
    P.state_out = P.last ? nullptr : state_[a & 1];
    P.out = d_out;
    const long blocks = (P.nlines + P.lpc - 1) / P.lpc;
    ct_pow_kernel<<<static_cast<unsigned>(blocks), P.lpc * P.tpl,
                    static_cast<size_t>(P.lpc) * P.line_bytes, stream>>>(P);
    BFM_LAUNCH_CHECK("ct_pow_kernel");
    if (lc) lc->add();
  }
}

}  // namespace bfmgpu
