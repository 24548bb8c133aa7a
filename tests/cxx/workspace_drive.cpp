// The reference's operator-level API with a reusable workspace
// (transforms.hpp:231-283,396-432: TransformWorkspace, CtransformPath,
// ctransform(model, phi, ws, path); acceptance_main.cpp:176-218 and
// test_transforms.cpp:232-313 drive it this way) against the B200 facade.
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

static bool same_bits(const Potential& a, const Potential& b) {
  return a.values.size() == b.values.size() &&
         std::memcmp(a.values.data(), b.values.data(), a.values.size() * sizeof(double)) == 0;
}

static Potential wavy(const Grid& g, double amp) {
  Potential p(g);
  for (int i = 0; i < g.extent(0); ++i)
    for (int j = 0; j < g.extent(1); ++j) {
      const double x = g.coord(0, i), y = g.coord(1, j);
      p.values[g.linear(i, j)] = 0.5 * (x * x + y * y) + amp * std::cos(7.0 * x + 3.0 * y) * std::sin(5.0 * y);
    }
  return p;
}

int main() {
  const Grid g({64, 48});
  const CostModel quad = CostModel::quadratic(2);
  const Potential phi = wavy(g, 0.05);
  TransformWorkspace ws(g, 4);
  report(ws.grid() == g && ws.threads() == 4, "workspace keeps its grid and thread count");
  const Potential a = ctransform(quad, phi, ws);
  const Potential b = ctransform(quad, phi);
  report(same_bits(a, b), "ctransform with a workspace == without (bitwise)");
  const Potential c = ctransform(quad, phi, ws, CtransformPath::divide_and_conquer);
  report(same_bits(a, c), "divide_and_conquer path == automatic path (bitwise)");
  // workspace reuse: phi^ccc == phi^c (Galois law, test_transforms.cpp:255-283)
  const Potential a3 = ctransform(quad, ctransform(quad, a, ws), ws);
  report(same_bits(a3, a), "phi^ccc == phi^c on one reused workspace");
  bool threw = false;
  try {
    TransformWorkspace other(Grid({32, 48}));
    (void)ctransform(quad, phi, other);
  } catch (const GridMismatch&) {
    threw = true;
  }
  report(threw, "workspace of another grid -> GridMismatch");
  threw = false;
  try {
    (void)ctransform(CostModel::quadratic(3), phi, ws);
  } catch (const GridMismatch&) {
    threw = true;
  }
  report(threw, "cost dimension != grid dimension -> GridMismatch");

  // power costs: the exact c-transform runs on the device; p = 2 exponents
  // reproduce the quadratic transform bit for bit
  const Potential p2 = ctransform(CostModel::power({2.0, 2.0}), phi, ws);
  report(same_bits(p2, a), "power cost (2, 2) == quadratic (bitwise)");
  const Potential p3 = ctransform(CostModel::power({1.5, 3.0}), phi, ws);
  bool finite = true;
  for (double v : p3.values) finite = finite && std::isfinite(v);
  report(finite, "power cost (1.5, 3) c-transform is finite");
  threw = false;
  try {
    (void)CostModel::power({1.0, 2.0});
  } catch (const InvalidArgument&) {
    threw = true;
  }
  report(threw, "exponent p <= 1 -> InvalidArgument (cost.hpp:24-30)");
  {
    // power-cost solve (acceptance_main.cpp:345-370 style, small): mu = nu
    // terminates at once with dual 0; a shifted pair moves and stays finite
    std::vector<double> raw(g.size(), 0.0), raw2(g.size(), 0.0);
    for (int i = 0; i < g.extent(0); ++i)
      for (int j = 0; j < g.extent(1); ++j) {
        const double x = g.coord(0, i), y = g.coord(1, j);
        if ((x - 0.3) * (x - 0.3) + (y - 0.5) * (y - 0.5) <= 0.04) raw[g.linear(i, j)] = 1.0;
        if ((x - 0.7) * (x - 0.7) + (y - 0.5) * (y - 0.5) <= 0.04) raw2[g.linear(i, j)] = 1.0;
      }
    SolverConfig cfg;
    cfg.tolerance = -1.0;
    cfg.max_iterations = 5;
    const SolveReport r = solve(CostModel::power({1.5, 3.0}), normalize(g, raw), normalize(g, raw2), cfg);
    report(r.iterations == 5 && std::isfinite(r.dual_value) && r.dual_value > 0.0,
           "power-cost solve (1.5, 3) runs 5 iterations with a positive dual");
  }

  // SpectralPlan reuse (poisson.hpp:42-113): two solves on one plan agree
  SpectralPlan plan(g);
  ScalarField r(g);
  for (std::size_t i = 0; i < r.values.size(); ++i) r.values[i] = std::sin(0.37 * static_cast<double>(i));
  const Potential u1 = plan.solve_neumann(r);
  const Potential u2 = plan.solve_neumann(r);
  report(same_bits(u1, u2), "SpectralPlan: repeated solves are bitwise identical");
  std::printf("%d failure(s)\n", failures);
  return failures;
}
