// ORACLE TEST INFRASTRUCTURE — not part of the product; never linked into
// paper_1905_12154_b200. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg may load oracle/liboracle.so.
//
// An independent CPU restatement of the reference's BFM hot path, written
// from the reference's documented semantics (file:line cited per function):
//  * c-transform: exact separable minimisation by brute force per grid line
//    with exact floating-point expansions between passes, one exactly-rounded
//    (toward -inf) output per node (transforms.hpp:396-432, exact.hpp:167-179).
//    The reference uses a parity divide-and-conquer instead; the exact minimum
//    is unique, so both must agree bitwise — tests check that.
//  * map / splat / residual / Neumann DCT solve / Kahan integrals / step-size
//    rule / the back-and-forth iterate (solver.hpp, pushforward.hpp,
//    poisson.hpp, grid.hpp).
// The DCT uses the same shared line routine as the product and the FFTW shim
// (paper_1905_12154_b200/csrc/dct_line.h) — FFTW itself is absent.
//
// Pinning: tests/test_oracle.py checks this restatement bitwise against
// oracle/_ref/libbfmref.so (the unmodified reference headers) and against the
// golden fixtures in tests/golden/.
//
// Build: -O3 -ffp-contract=off (no FMA contraction).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "../include/bfm_b200.h"
#include "../paper_1905_12154_b200/csrc/dct_plan_host.h"

namespace {

thread_local std::string g_err;

// ---------------------------------------------------------------- exact sums
// Nonoverlapping expansion, increasing magnitude, zero-free.
struct Expn {
  std::vector<double> c;
  void add(double b) {  // exact: grow with zero elimination (Shewchuk)
    if (b == 0.0) return;
    double q = b;
    size_t o = 0;
    for (size_t i = 0; i < c.size(); ++i) {
      const double s = q + c[i];
      const double bv = s - q;
      const double e = (q - (s - bv)) + (c[i] - bv);
      q = s;
      if (e != 0.0) c[o++] = e;
    }
    c.resize(o);
    if (q != 0.0) c.push_back(q);
  }
  int sign() const { return c.empty() ? 0 : (c.back() > 0.0 ? 1 : -1); }
  double approx() const {
    double s = 0.0;
    for (double v : c) s += v;
    return s;
  }
};

void two_prod(double a, double b, double& p, double& e) {
  p = a * b;
  e = std::fma(a, b, -p);
}

// Sign of (value(e) - d), exact.
int sign_minus(const Expn& e, double d) {
  Expn t = e;
  t.add(-d);
  return t.sign();
}

// Largest double <= exact value; -0 -> +0 (exact.hpp:167-179 semantics).
double round_down(const Expn& e) {
  if (e.sign() == 0) return 0.0;
  double d = e.approx();
  const double inf = std::numeric_limits<double>::infinity();
  while (sign_minus(e, d) < 0) d = std::nextafter(d, -inf);
  while (true) {
    const double up = std::nextafter(d, inf);
    if (sign_minus(e, up) >= 0) d = up;
    else break;
  }
  return d == 0.0 ? 0.0 : d;
}

int compare(const Expn& a, const Expn& b) {
  Expn t = a;
  for (double v : b.c) t.add(-v);
  return t.sign();
}

// --------------------------------------------------------------- grid
struct Grid {
  int d = 0;
  int n[3] = {1, 1, 1};
  long stride[3] = {0, 0, 0};
  long size = 0;
  double h[3] = {1, 1, 1};
  double vol = 1.0;
  // grid.hpp:60-76
  explicit Grid(int dim, const int* ext) {
    d = dim;
    size = 1;
    vol = 1.0;
    for (int a = 0; a < d; ++a) {
      n[a] = ext[a];
      h[a] = 1.0 / ext[a];
      size *= ext[a];
      vol *= h[a];
    }
    stride[d - 1] = 1;
    for (int a = d - 2; a >= 0; --a) stride[a] = stride[a + 1] * n[a + 1];
  }
  double coord(int a, int i) const { return (i + 0.5) * h[a]; }  // grid.hpp:27
  void idx(long lin, int* i) const {
    for (int a = 0; a < d; ++a) {
      i[a] = static_cast<int>(lin / stride[a]);
      lin -= static_cast<long>(i[a]) * stride[a];
    }
  }
};

void check_grid(int dim, const int* ext) {
  if (dim < 1 || dim > 3) throw std::string("grid dimension must be 1, 2, or 3");
  for (int a = 0; a < dim; ++a)
    if (ext[a] < 2) throw std::string("grid extent must be at least 2");
}

double hs(double c) { return 0.5 * c * c; }  // transforms.hpp:253 half square

// ------------------------------------------------------------ c-transform
// transforms.hpp:340-391 semantics with a brute-force line minimum: pass a
// replaces every node's exact state by min_j (state_j + hs(y_j) - x_k*y_j)
// along axis a; finally adds sum_a hs(x_a) and rounds down once.
std::vector<double> ctransform(const Grid& g, const double* phi) {
  std::vector<Expn> cur(g.size), nxt(g.size);
  for (long i = 0; i < g.size; ++i) cur[i].add(-phi[i]);
  for (int a = 0; a < g.d; ++a) {
    const int n = g.n[a];
    const long s = g.stride[a];
    std::vector<double> y(n), hy(n);
    for (int j = 0; j < n; ++j) {
      y[j] = g.coord(a, j);
      hy[j] = hs(y[j]);
    }
    const long lines = g.size / n;
    std::vector<double> approx(n);
    for (long l = 0; l < lines; ++l) {
      // base of line l: enumerate the other axes in row-major order
      const long outer = l / s, inner = l % s;
      const long base = outer * n * s + inner;
      for (int j = 0; j < n; ++j) approx[j] = cur[base + j * s].approx() + hy[j];
      for (int k = 0; k < n; ++k) {
        int best = -1;
        double best_ap = 0.0;
        Expn best_e;
        for (int j = 0; j < n; ++j) {
          const double ap = approx[j] - y[k] * y[j];
          if (best >= 0) {
            const double margin =
                1e-12 * (std::fabs(ap) + std::fabs(best_ap) + std::fabs(approx[j]) + 1.0);
            if (ap - best_ap > margin) continue;
          }
          Expn e = cur[base + j * s];
          double p, pe;
          two_prod(y[k], y[j], p, pe);
          e.add(hy[j]);
          e.add(-pe);
          e.add(-p);
          if (best < 0 || compare(e, best_e) < 0) {
            best = j;
            best_e = e;
            best_ap = ap;
          }
        }
        nxt[base + k * s] = best_e;
      }
    }
    std::swap(cur, nxt);
  }
  std::vector<double> out(g.size);
  for (long i = 0; i < g.size; ++i) {
    int id[3] = {0, 0, 0};
    g.idx(i, id);
    Expn e = cur[i];
    for (int a = 0; a < g.d; ++a) e.add(hs(g.coord(a, id[a])));
    out[i] = round_down(e);
  }
  return out;
}

// ------------------------------------------------------------ map / splat
// grid.hpp:186-208 gradient; cost.hpp:59-68 inverse gradient (p = 2) with the
// sqrt(d) cap; pushforward.hpp:70-91 clamp and displacement.
void map_from_conjugate(const Grid& g, const double* u, double* disp) {
  const double cap = std::sqrt(static_cast<double>(g.d));
  for (int a = 0; a < g.d; ++a) {
    const long s = g.stride[a];
    const int n = g.n[a];
    const double inv_h = static_cast<double>(n);
    const double inv_2h = 0.5 * inv_h;
    for (long lin = 0; lin < g.size; ++lin) {
      int id[3];
      g.idx(lin, id);
      const int j = id[a];
      double gr;
      if (j == 0) gr = (u[lin + s] - u[lin]) * inv_h;
      else if (j == n - 1) gr = (u[lin] - u[lin - s]) * inv_h;
      else gr = (u[lin + s] - u[lin - s]) * inv_2h;
      double mag = std::fabs(gr);
      if (!(mag < cap)) mag = cap;
      const double v = gr < 0.0 ? -mag : mag;
      const double x = g.coord(a, j);
      double t = x - v;
      if (t < 0.0) t = 0.0;
      if (t > 1.0) t = 1.0;
      disp[a * g.size + lin] = t - x;
    }
  }
}

// pushforward.hpp:51-63 locate_cell.
void locate(const std::vector<double>& c, double x, int& lo, int& hi, double& w) {
  const int n = static_cast<int>(c.size());
  if (x <= c[0]) { lo = hi = 0; w = 0.0; return; }
  if (x >= c[n - 1]) { lo = hi = n - 1; w = 0.0; return; }
  int i = static_cast<int>(x * n - 0.5);
  if (i < 0) i = 0;
  if (i > n - 2) i = n - 2;
  while (i + 1 < n - 1 && c[i + 1] <= x) ++i;
  while (i > 0 && c[i] > x) --i;
  lo = i;
  hi = i + 1;
  w = (x - c[i]) / (c[i + 1] - c[i]);
}

// pushforward.hpp:141-172 splat_displaced: sequential scatter in source order.
void splat(const Grid& g, const double* disp, const double* mu, double scale, double* out) {
  std::vector<double> c[3];
  for (int a = 0; a < g.d; ++a) {
    c[a].resize(g.n[a]);
    for (int i = 0; i < g.n[a]; ++i) c[a][i] = g.coord(a, i);
  }
  for (long i = 0; i < g.size; ++i) out[i] = 0.0;
  for (long lin = 0; lin < g.size; ++lin) {
    const double m = mu[lin];
    if (m == 0.0) continue;
    int id[3];
    g.idx(lin, id);
    int lo[3], hi[3];
    double w[3];
    for (int a = 0; a < g.d; ++a) {
      const double x = c[a][id[a]] + scale * disp[a * g.size + lin];
      locate(c[a], x, lo[a], hi[a], w[a]);
    }
    for (int corner = 0; corner < (1 << g.d); ++corner) {
      double wt = m;
      long node = 0;
      for (int a = 0; a < g.d; ++a) {
        const bool up = (corner >> a) & 1;
        wt *= up ? w[a] : 1.0 - w[a];
        node += g.stride[a] * (up ? hi[a] : lo[a]);
      }
      out[node] += wt;
    }
  }
}

// ------------------------------------------------------------ reductions
struct Kahan {  // grid.hpp:124-133
  double sum = 0.0, carry = 0.0;
  void add(double v) {
    const double y = v - carry;
    const double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
};

double integrate(const Grid& g, const double* f, const double* w) {  // grid.hpp:171-183
  Kahan k;
  for (long i = 0; i < g.size; ++i) k.add(w ? f[i] * w[i] : f[i]);
  return k.sum * g.vol;
}

// ------------------------------------------------------------ Poisson
// poisson.hpp:42-73 (eigenvalues) and :87-106 (solve) with the shared DCT,
// axis order d-1..0 forward and 0..d-1 inverse (oracle/fftw3.h).
struct Poisson {
  Grid g;
  std::unique_ptr<bfmdct::HostLinePlan> plan[3];
  std::vector<double> lam[3];
  double scale = 1.0;
  std::vector<bfmdct::cplx> scratch;
  explicit Poisson(const Grid& gg) : g(gg) {
    constexpr double kPi = 3.14159265358979323846;
    int maxn = 1;
    for (int a = 0; a < 3; ++a) {
      if (a < g.d) {
        plan[a].reset(new bfmdct::HostLinePlan);
        plan[a]->build(g.n[a]);
        scale *= 2.0 * g.n[a];
        const double na = g.n[a];
        lam[a].resize(g.n[a]);
        for (int k = 0; k < g.n[a]; ++k) lam[a][k] = (2.0 - 2.0 * std::cos(kPi * k / na)) * na * na;
        maxn = std::max(maxn, g.n[a]);
      } else {
        lam[a] = {0.0};
      }
    }
    scratch.resize(maxn + 1);
  }
  void axis(double* b, int a, bool fwd) {
    const long s = g.stride[a];
    const long len = g.n[a];
    const long outer = g.size / (len * s);
    for (long o = 0; o < outer; ++o)
      for (long i = 0; i < s; ++i) {
        double* line = b + o * len * s + i;
        if (fwd) bfmdct::dct2_line_cpu(plan[a]->plan, line, s, scratch.data());
        else bfmdct::dct3_line_cpu(plan[a]->plan, line, s, scratch.data());
      }
  }
  void solve(const double* rhs, double* out) {
    std::vector<double> b(rhs, rhs + g.size);
    for (int a = g.d - 1; a >= 0; --a) axis(b.data(), a, true);
    long idx = 0;
    for (size_t k0 = 0; k0 < lam[0].size(); ++k0)
      for (size_t k1 = 0; k1 < lam[1].size(); ++k1)
        for (size_t k2 = 0; k2 < lam[2].size(); ++k2, ++idx) {
          const double l = (lam[0][k0] + lam[1][k1]) + lam[2][k2];
          b[idx] = l == 0.0 ? 0.0 : b[idx] / (l * scale);
        }
    for (int a = 0; a < g.d; ++a) axis(b.data(), a, false);
    std::memcpy(out, b.data(), g.size * sizeof(double));
  }
};

// ------------------------------------------------------------ solver
double update_sigma(double sigma, double inc, double gn, const bfm_config& c) {  // solver.hpp:68-76
  const double pred = sigma * gn;
  if (inc < c.beta_1 * pred) sigma *= c.alpha_2;
  else if (inc > c.beta_2 * pred) sigma *= c.alpha_1;
  return std::max(sigma, c.sigma_min);
}

void default_config(bfm_config* c) {  // solver.hpp:46-63
  c->mode = BFM_MODE_BACK_AND_FORTH;
  c->tolerance = 1e-4;
  c->max_iterations = 2000;
  c->threads = 0;
  c->sigma_init = 0.0;
  c->sigma_min = 0.01;
  c->beta_1 = 0.25;
  c->beta_2 = 0.75;
  c->alpha_1 = 1.25;
  c->alpha_2 = 0.8;
  c->has_exact_cost = 0;
  c->exact_cost = 0.0;
  c->exact_tolerance = 0.0;
}

}  // namespace

struct orc_solver {  // solver.hpp:146-368 restated
  Grid g;
  bfm_config cfg;
  std::vector<double> mu, nu, phi, psi, dir;
  Poisson pois;
  double sigma = 0, last_pair = 0, prev_dual = std::numeric_limits<double>::quiet_NaN();
  double probe_dual = 0, probe_gn = 0;
  bool fresh = false;
  int iteration = 0, stall = 0;
  std::vector<bfm_iteration_stats> trace;
  orc_solver(const Grid& gg) : g(gg), pois(gg) {}

  double pair() { return integrate(g, phi.data(), nu.data()) + integrate(g, psi.data(), mu.data()); }

  double ascent(const std::vector<double>& u, const std::vector<double>& src,
                const std::vector<double>& tgt, std::vector<double>& d) {  // :245-260
    std::vector<double> disp(g.d * g.size), rho(g.size), r(g.size);
    map_from_conjugate(g, u.data(), disp.data());
    splat(g, disp.data(), src.data(), 1.0, rho.data());
    for (long i = 0; i < g.size; ++i) r[i] = tgt[i] - rho[i];
    d.resize(g.size);
    pois.solve(r.data(), d.data());
    Kahan k;
    for (long i = 0; i < g.size; ++i) k.add(r[i] * d[i]);
    return k.sum * g.vol;
  }
  void probe() {  // :264-280
    if (fresh) return;
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      psi = ctransform(g, phi.data());
      const double v = pair();
      if (v < last_pair - 1e-10) throw std::string("blowup");
      last_pair = v;
      probe_dual = v;
    } else {
      probe_dual = last_pair;
    }
    probe_gn = ascent(psi, mu, nu, dir);
    fresh = true;
  }
  void axpy(std::vector<double>& u, double s, const std::vector<double>& d) {
    for (long i = 0; i < g.size; ++i) u[i] += s * d[i];
  }
  bfm_iteration_stats step() {  // :189-207, :286-328
    probe();
    bfm_iteration_stats st{};
    st.iteration = iteration + 1;
    st.residual = std::sqrt(std::max(probe_gn, 0.0));
    const double v2 = probe_dual;
    st.sigma_first = sigma;
    st.grad_norm_sq_first = probe_gn;
    axpy(phi, sigma, dir);
    psi = ctransform(g, phi.data());
    const double v3 = pair();
    st.increase_first = v3 - v2;
    sigma = update_sigma(sigma, st.increase_first, probe_gn, cfg);
    phi = ctransform(g, psi.data());
    const double v4 = pair();
    if (v4 < v3 - 1e-10) throw std::string("blowup");
    if (cfg.mode == BFM_MODE_BACK_AND_FORTH) {
      std::vector<double> dir2;
      const double gn2 = ascent(phi, nu, mu, dir2);
      st.sigma_second = sigma;
      st.grad_norm_sq_second = gn2;
      axpy(psi, sigma, dir2);
      phi = ctransform(g, psi.data());
      const double v5 = pair();
      st.increase_second = v5 - v4;
      sigma = update_sigma(sigma, st.increase_second, gn2, cfg);
      st.dual_value = v5;
      last_pair = v5;
    } else {
      st.dual_value = v4;
      last_pair = v4;
    }
    fresh = false;
    ++iteration;
    if (std::fabs(st.dual_value - prev_dual) < 1e-12) ++stall;
    else stall = 0;
    prev_dual = st.dual_value;
    trace.push_back(st);
    return st;
  }
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

#define OGUARD(...)                       \
  try {                                   \
    __VA_ARGS__;                          \
    return BFM_OK;                        \
  } catch (const std::string& e) {        \
    g_err = e;                            \
    return e == "blowup" ? BFM_ERR_NUMERICAL_BLOWUP : BFM_ERR_INVALID_ARGUMENT; \
  } catch (const std::exception& e) {     \
    g_err = e.what();                     \
    return BFM_ERR_ERROR;                 \
  }

double orc_update_sigma(double sigma, double inc, double gn, const bfm_config* c) {
  bfm_config d;
  default_config(&d);
  return update_sigma(sigma, inc, gn, c ? *c : d);
}

int orc_ctransform(int dim, const int* ext, const double* phi, double* out) {
  OGUARD({
    check_grid(dim, ext);
    Grid g(dim, ext);
    const auto r = ctransform(g, phi);
    std::memcpy(out, r.data(), g.size * sizeof(double));
  })
}

int orc_map_from_conjugate(int dim, const int* ext, const double* u, int /*side*/, double* disp) {
  OGUARD({
    check_grid(dim, ext);
    map_from_conjugate(Grid(dim, ext), u, disp);
  })
}

int orc_pushforward_density(int dim, const int* ext, const double* disp, const double* mu,
                            double* rho) {
  OGUARD({
    check_grid(dim, ext);
    splat(Grid(dim, ext), disp, mu, 1.0, rho);
  })
}

int orc_displacement_interpolant(int dim, const int* ext, const double* disp, const double* mu,
                                 double t, double* rho) {
  OGUARD({
    check_grid(dim, ext);
    splat(Grid(dim, ext), disp, mu, t, rho);
  })
}

int orc_solve_neumann(int dim, const int* ext, const double* rhs, double* out) {
  OGUARD({
    check_grid(dim, ext);
    Poisson p(Grid(dim, ext));
    p.solve(rhs, out);
  })
}

// Multi-GPU slab checks (tests/test_dist_cpu.py): one DCT axis of an array,
// and the column-slab axis-0 step [DCT-II, divide, DCT-III] of poisson.hpp
// for global flattened columns col0 .. col0 + ncols (d >= 2).
int orc_dct_axis(int dim, const int* ext, int axis, int inverse, double* data) {
  OGUARD({
    check_grid(dim, ext);
    if (axis < 0 || axis >= dim) throw std::invalid_argument("orc_dct_axis: bad axis");
    Grid g(dim, ext);
    bfmdct::HostLinePlan plan;
    plan.build(g.n[axis]);
    std::vector<bfmdct::cplx> scratch(g.n[axis] + 1);
    const long st = g.stride[axis];
    const long len = g.n[axis];
    const long outer = g.size / (len * st);
    for (long o = 0; o < outer; ++o)
      for (long i = 0; i < st; ++i) {
        double* line = data + o * len * st + i;
        if (inverse) bfmdct::dct3_line_cpu(plan.plan, line, st, scratch.data());
        else bfmdct::dct2_line_cpu(plan.plan, line, st, scratch.data());
      }
  })
}

int orc_poisson_cols(int dim, const int* ext, long col0, int ncols, const double* in,
                     double* out) {
  OGUARD({
    check_grid(dim, ext);
    if (dim < 2) throw std::invalid_argument("orc_poisson_cols: d >= 2");
    Poisson p{Grid(dim, ext)};
    const int n0 = ext[0];
    const int n2 = dim > 2 ? ext[2] : 1;
    std::vector<double> col(n0);
    for (int c = 0; c < ncols; ++c) {
      for (int k = 0; k < n0; ++k) col[k] = in[static_cast<long>(k) * ncols + c];
      bfmdct::dct2_line_cpu(p.plan[0]->plan, col.data(), 1, p.scratch.data());
      const long gc = col0 + c;
      const double l1 = p.lam[1][dim > 2 ? gc / n2 : gc];
      const double l2 = dim > 2 ? p.lam[2][gc % n2] : p.lam[2][0];
      for (int k = 0; k < n0; ++k) {
        const double l = (p.lam[0][k] + l1) + l2;
        col[k] = l == 0.0 ? 0.0 : col[k] / (l * p.scale);
      }
      bfmdct::dct3_line_cpu(p.plan[0]->plan, col.data(), 1, p.scratch.data());
      for (int k = 0; k < n0; ++k) out[static_cast<long>(k) * ncols + c] = col[k];
    }
  })
}

int orc_integrate(int dim, const int* ext, const double* f, const double* w, double* out) {
  OGUARD({
    check_grid(dim, ext);
    *out = integrate(Grid(dim, ext), f, w);
  })
}

// Runs `iters` back-and-forth steps from phi = psi = 0 and returns the final
// phi, psi (not gauge fixed) and the per-iteration dual values.
int orc_run_steps(int dim, const int* ext, const double* mu, const double* nu, int iters,
                  double* phi_out, double* psi_out, double* duals) {
  OGUARD({
    check_grid(dim, ext);
    Grid g(dim, ext);
    orc_solver s(g);
    default_config(&s.cfg);
    s.mu.assign(mu, mu + g.size);
    s.nu.assign(nu, nu + g.size);
    s.phi.assign(g.size, 0.0);
    s.psi.assign(g.size, 0.0);
    double sup = 0.0;
    for (double v : s.mu) sup = std::max(sup, v);
    for (double v : s.nu) sup = std::max(sup, v);
    s.sigma = 8.0 / sup;
    for (int it = 0; it < iters; ++it) {
      const auto st = s.step();
      if (duals) duals[it] = st.dual_value;
    }
    std::memcpy(phi_out, s.phi.data(), g.size * sizeof(double));
    std::memcpy(psi_out, s.psi.data(), g.size * sizeof(double));
  })
}

}  // extern "C"
