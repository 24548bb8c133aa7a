// A driver written purely against the reference's C++ API surface
// (bfm::Solver / bfm::solve / ctransform / SpectralPlan ... as declared in
// /root/reference/proj/include/bfm/*.hpp), compiled against the B200 facade
// include/bfm_b200/bfm.hpp instead of the reference headers. Checks follow the
// reference's own tests (test_solver.cpp:43-124,184-235, test_poisson.cpp:41-79).
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "bfm_b200/bfm.hpp"

using namespace bfm;

static int failures = 0;
static void report(bool ok, const char* what) {
  std::printf("%s  %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

static DensityField disc(const Grid& g, double cx, double cy, double r) {
  std::vector<double> raw(g.size(), 0.0);
  for (int i = 0; i < g.extent(0); ++i)
    for (int j = 0; j < g.extent(1); ++j) {
      const double dx = g.coord(0, i) - cx, dy = g.coord(1, j) - cy;
      if (dx * dx + dy * dy <= r * r) raw[g.linear(i, j)] = 1.0;
    }
  return normalize(g, raw);
}

int main() {
  SolverConfig cfg;
  report(std::fabs(update_sigma(1.0, 0.1, 1.0, cfg) - 0.8) <= 1e-15 &&
             std::fabs(update_sigma(1.0, 0.9, 1.0, cfg) - 1.25) <= 1e-15 &&
             update_sigma(0.012, 0.0, 1.0, cfg) == 0.01,
         "update_sigma KATs (test_solver.cpp:43-55)");

  {
    Grid g({64, 64});
    DensityField mu = disc(g, 0.25, 0.25, 0.125), nu = disc(g, 0.75, 0.75, 0.125);
    SolverConfig c;
    c.tolerance = -1.0;
    c.max_iterations = 40;
    c.exact_cost = 0.25;
    c.exact_tolerance = 1e-4;
    SolveReport rep = solve(CostModel::quadratic(2), mu, nu, c);
    report(rep.termination == Termination::cost_target_met && rep.iterations <= 6 &&
               std::fabs(rep.dual_value - 0.25) <= 1e-4 && std::fabs(rep.primal_cost - 0.25) <= 1e-3,
           "two discs converge in a handful of iterations (test_solver.cpp:98-124)");
    report(std::fabs(integrate(rep.phi)) <= 1e-12, "report potentials are gauge fixed");
  }
  {
    // benchmark.hpp:27-43,84-124: a paper case from the builtin shapes
    Grid g({128, 128});
    DensityField mu = normalize(g, builtin_density(g, "square:0.5,0.5,0.25").values);
    DensityField nu = normalize(
        g, builtin_density(g, "square:0.1875,0.1875,0.125+square:0.8125,0.1875,0.125+"
                              "square:0.1875,0.8125,0.125+square:0.8125,0.8125,0.125")
               .values);
    SolverConfig c;
    c.tolerance = -1.0;
    c.exact_cost = 0.0625;
    c.exact_tolerance = 1e-4;
    c.max_iterations = 1000;
    SolveReport rep = solve(CostModel::quadratic(2), mu, nu, c);
    report(rep.termination == Termination::cost_target_met && rep.iterations >= 1 &&
               rep.iterations <= 5,
           "four_squares reaches the exact cost 1/16 within 3+-2 iterations (benchmark.hpp:56-63)");
  }
  {
    Grid g({32, 32});
    DensityField mu = disc(g, 0.5, 0.5, 0.2);
    SolveReport rep = solve(CostModel::quadratic(2), mu, mu, SolverConfig{});
    report(rep.termination == Termination::tolerance_met && rep.iterations == 0 && rep.dual_value == 0.0,
           "identical marginals terminate immediately (test_solver.cpp:57-70)");
  }
  {
    Grid g({48, 48});
    DensityField mu = disc(g, 0.3, 0.4, 0.15), nu = disc(g, 0.7, 0.6, 0.2);
    SolverConfig c;
    c.tolerance = 1e-5;
    c.max_iterations = 30;
    SolveReport a = solve(CostModel::quadratic(2), mu, nu, c);
    SolveReport b = solve(CostModel::quadratic(2), mu, nu, c);
    report(a.iterations == b.iterations && a.dual_value == b.dual_value &&
               std::memcmp(a.phi.values.data(), b.phi.values.data(), a.phi.values.size() * 8) == 0,
           "solves are deterministic (test_solver.cpp:215-235)");
  }
  {
    Grid g({16, 16});
    DensityField ok = disc(g, 0.5, 0.5, 0.25), heavy = ok;
    for (auto& v : heavy.values) v *= 2.0;
    bool threw = false;
    try {
      solve(CostModel::quadratic(2), heavy, ok, SolverConfig{});
    } catch (const InfeasibleInput&) {
      threw = true;
    }
    report(threw, "mass must be one -> InfeasibleInput (test_solver.cpp:261-266)");
  }
  {
    Grid g({64});
    SpectralPlan plan(g);
    ScalarField rhs(g);
    for (int j = 0; j < 64; ++j) rhs.values[j] = std::cos(3.14159265358979323846 * g.coord(0, j));
    Potential u = plan.solve_neumann(rhs);
    const double lam = (2.0 - 2.0 * std::cos(3.14159265358979323846 / 64)) * 64 * 64;
    double worst = 0.0;
    for (int j = 0; j < 64; ++j) worst = std::fmax(worst, std::fabs(u.values[j] - rhs.values[j] / lam));
    report(worst < 1e-12, "cosine modes are eigenfunctions (test_poisson.cpp:41-62)");
  }
  {
    Grid g({24, 24});
    Potential phi(g);
    for (std::size_t i = 0; i < g.size(); ++i) phi.values[i] = std::sin(0.37 * i);
    const CostModel q = CostModel::quadratic(2);
    Potential c = ctransform(q, phi), cc = ctransform(q, c), ccc = ctransform(q, cc);
    bool ok = std::memcmp(c.values.data(), ccc.values.data(), c.values.size() * 8) == 0;
    for (std::size_t i = 0; i < g.size(); ++i) ok = ok && phi.values[i] <= cc.values[i];
    report(ok, "Galois laws phi <= phi^cc, phi^ccc == phi^c bitwise (test_transforms.cpp:255-283)");
  }
  std::printf("facade: %d failure(s)\n", failures);
  return failures;
}
