// ORACLE TEST INFRASTRUCTURE — not part of the product.
//
// C-ABI wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/bfm/*.hpp) compiled with the FFTW-subset shim
// in oracle/fftw3.h. Built by oracle/Makefile into oracle/_ref/libbfmref.so.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
// --impl reference) load it. Entry points mirror include/bfm_b200.h with a
// ref_ prefix so the same test code drives both sides.
//
// Build flags: -O3 -DNDEBUG -ffp-contract=off (the reference's Release build
// emits separate mul/add).
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "bfm/interpolation.hpp"
#include "bfm/io.hpp"
#include "bfm/pushforward.hpp"
#include "bfm/solver.hpp"
#include "bfm/transforms.hpp"
#include "../include/bfm_b200.h"

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const bfm::InvalidArgument*>(&e)) return BFM_ERR_INVALID_ARGUMENT;
  if (dynamic_cast<const bfm::GridMismatch*>(&e)) return BFM_ERR_GRID_MISMATCH;
  if (dynamic_cast<const bfm::NegativeInput*>(&e)) return BFM_ERR_NEGATIVE_INPUT;
  if (dynamic_cast<const bfm::AllZeroInput*>(&e)) return BFM_ERR_ALL_ZERO_INPUT;
  if (dynamic_cast<const bfm::InfeasibleInput*>(&e)) return BFM_ERR_INFEASIBLE_INPUT;
  if (dynamic_cast<const bfm::NumericalBlowup*>(&e)) return BFM_ERR_NUMERICAL_BLOWUP;
  if (dynamic_cast<const bfm::TOutOfRange*>(&e)) return BFM_ERR_T_OUT_OF_RANGE;
  if (dynamic_cast<const bfm::IoError*>(&e)) return BFM_ERR_IO;
  return BFM_ERR_ERROR;
}

#define GUARD(...)                         \
  try {                                    \
    __VA_ARGS__;                           \
    return BFM_OK;                         \
  } catch (const std::exception& e) {      \
    return code_of(e);                     \
  }

bfm::Grid make_grid(int dim, const int* ext) {
  return bfm::Grid(std::vector<int>(ext, ext + dim));
}

bfm::SolverConfig to_cfg(const bfm_config* c) {
  bfm::SolverConfig r;
  if (!c) return r;
  r.mode = c->mode == BFM_MODE_GRADIENT_ASCENT ? bfm::SolverMode::gradient_ascent
                                               : bfm::SolverMode::back_and_forth;
  r.tolerance = c->tolerance;
  r.max_iterations = c->max_iterations;
  r.threads = c->threads;
  r.sigma_init = c->sigma_init;
  r.sigma_min = c->sigma_min;
  r.beta_1 = c->beta_1;
  r.beta_2 = c->beta_2;
  r.alpha_1 = c->alpha_1;
  r.alpha_2 = c->alpha_2;
  if (c->has_exact_cost) r.exact_cost = c->exact_cost;
  r.exact_tolerance = c->exact_tolerance;
  return r;
}

void to_stats(const bfm::IterationStats& s, bfm_iteration_stats* o) {
  o->iteration = s.iteration;
  o->residual = s.residual;
  o->dual_value = s.dual_value;
  o->sigma_first = s.sigma_first;
  o->sigma_second = s.sigma_second;
  o->grad_norm_sq_first = s.grad_norm_sq_first;
  o->grad_norm_sq_second = s.grad_norm_sq_second;
  o->increase_first = s.increase_first;
  o->increase_second = s.increase_second;
}

bfm::TransportMap make_map(const bfm::Grid& g, const double* disp) {
  bfm::TransportMap m(g);
  for (int a = 0; a < g.dim(); ++a)
    m.displacement[a].assign(disp + a * g.size(), disp + (a + 1) * g.size());
  return m;
}

}  // namespace

struct ref_solver {
  bfm::Grid grid;
  std::unique_ptr<bfm::Solver> solver;
  bfm::SolveReport report;
  bool has_report = false;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_config_default(bfm_config* c) {
  bfm::SolverConfig d;
  c->mode = BFM_MODE_BACK_AND_FORTH;
  c->tolerance = d.tolerance;
  c->max_iterations = d.max_iterations;
  c->threads = d.threads;
  c->sigma_init = d.sigma_init;
  c->sigma_min = d.sigma_min;
  c->beta_1 = d.beta_1;
  c->beta_2 = d.beta_2;
  c->alpha_1 = d.alpha_1;
  c->alpha_2 = d.alpha_2;
  c->has_exact_cost = 0;
  c->exact_cost = 0.0;
  c->exact_tolerance = d.exact_tolerance;
}

double ref_update_sigma(double sigma, double inc, double gn, const bfm_config* c) {
  return bfm::update_sigma(sigma, inc, gn, to_cfg(c));
}

int ref_solver_create(int dim, const int* ext, const double* mu, const double* nu,
                      const bfm_config* cfg, ref_solver** out) {
  GUARD({
    auto s = std::make_unique<ref_solver>();
    s->grid = make_grid(dim, ext);
    bfm::DensityField m(s->grid), n(s->grid);
    std::memcpy(m.values.data(), mu, s->grid.size() * sizeof(double));
    std::memcpy(n.values.data(), nu, s->grid.size() * sizeof(double));
    s->solver = std::make_unique<bfm::Solver>(bfm::CostModel::quadratic(dim), m, n,
                                              to_cfg(cfg));
    *out = s.release();
  })
}

void ref_solver_destroy(ref_solver* s) { delete s; }
int ref_solver_iteration(const ref_solver* s) { return s->solver->iteration(); }
double ref_solver_sigma(const ref_solver* s) { return s->solver->sigma(); }
int ref_solver_dual_value(ref_solver* s, double* out) { GUARD(*out = s->solver->dual_value()) }
int ref_solver_residual(ref_solver* s, double* out) { GUARD(*out = s->solver->residual()) }

int ref_solver_step(ref_solver* s, bfm_iteration_stats* out) {
  GUARD({
    const bfm::IterationStats st = s->solver->step();
    if (out) to_stats(st, out);
  })
}

int ref_solver_run(ref_solver* s, bfm_report* out) {
  GUARD({
    s->report = s->solver->run();
    s->has_report = true;
    out->termination = static_cast<int>(s->report.termination);
    out->iterations = s->report.iterations;
    out->dual_value = s->report.dual_value;
    out->primal_cost = s->report.primal_cost;
    out->residual = s->report.residual;
    out->wall_seconds = s->report.wall_seconds;
  })
}

int ref_solver_trace(const ref_solver* s, bfm_iteration_stats* out, int cap, int* count) {
  const auto& t = s->solver->trace();
  *count = static_cast<int>(t.size());
  for (int i = 0; i < cap && i < static_cast<int>(t.size()); ++i) to_stats(t[i], out + i);
  return BFM_OK;
}

int ref_solver_field(ref_solver* s, int which, double* out) {
  const auto& f = which == BFM_FIELD_PHI ? s->solver->phi() : s->solver->psi();
  std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
  return BFM_OK;
}

int ref_solver_report_field(ref_solver* s, int which, double* out) {
  if (!s->has_report) {
    g_err = "no report";
    return BFM_ERR_ERROR;
  }
  const std::vector<double>* v = nullptr;
  if (which == BFM_FIELD_PHI) v = &s->report.phi.values;
  else if (which == BFM_FIELD_PSI) v = &s->report.psi.values;
  else v = &s->report.map.displacement[which - BFM_FIELD_MAP0];
  std::memcpy(out, v->data(), v->size() * sizeof(double));
  return BFM_OK;
}

int ref_ctransform(int dim, const int* ext, const double* phi, double* out, int threads) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::Potential p(g);
    std::memcpy(p.values.data(), phi, g.size() * sizeof(double));
    bfm::TransformWorkspace ws(g, threads > 0 ? threads : bfm::default_thread_count());
    const bfm::Potential r = bfm::ctransform(bfm::CostModel::quadratic(dim), p, ws);
    std::memcpy(out, r.values.data(), g.size() * sizeof(double));
  })
}

// Power costs c = sum_a |y_a - x_a|^p_a / p_a (cost.hpp:24-31): the generic
// path of transforms.hpp:396-427 and the pow inverse gradient of cost.hpp:59-68.
static bfm::CostModel cost_model(int dim, const double* exponents) {
  if (!exponents) return bfm::CostModel::quadratic(dim);
  return bfm::CostModel::power(std::vector<double>(exponents, exponents + dim));
}

int ref_ctransform_cost(int dim, const int* ext, const double* exponents, const double* phi,
                        double* out, int threads) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::Potential p(g);
    std::memcpy(p.values.data(), phi, g.size() * sizeof(double));
    bfm::TransformWorkspace ws(g, threads > 0 ? threads : bfm::default_thread_count());
    const bfm::Potential r = bfm::ctransform(cost_model(dim, exponents), p, ws);
    std::memcpy(out, r.values.data(), g.size() * sizeof(double));
  })
}

int ref_map_from_conjugate_cost(int dim, const int* ext, const double* exponents, const double* u,
                                int side, double* disp) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::Potential p(g);
    std::memcpy(p.values.data(), u, g.size() * sizeof(double));
    const bfm::TransportMap m = bfm::map_from_conjugate(
        cost_model(dim, exponents), p, side == 0 ? bfm::MapSource::mu_side : bfm::MapSource::nu_side);
    for (int a = 0; a < dim; ++a)
      std::memcpy(disp + static_cast<size_t>(a) * g.size(), m.displacement[a].data(),
                  g.size() * sizeof(double));
  })
}

int ref_solver_create_cost(int dim, const int* ext, const double* exponents, const double* mu,
                           const double* nu, const bfm_config* cfg, ref_solver** out) {
  GUARD({
    auto s = std::make_unique<ref_solver>();
    s->grid = make_grid(dim, ext);
    bfm::DensityField m(s->grid), n(s->grid);
    std::memcpy(m.values.data(), mu, s->grid.size() * sizeof(double));
    std::memcpy(n.values.data(), nu, s->grid.size() * sizeof(double));
    s->solver = std::make_unique<bfm::Solver>(cost_model(dim, exponents), m, n, to_cfg(cfg));
    *out = s.release();
  })
}

int ref_map_from_conjugate(int dim, const int* ext, const double* u, int side, double* disp) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::Potential p(g);
    std::memcpy(p.values.data(), u, g.size() * sizeof(double));
    const bfm::TransportMap m = bfm::map_from_conjugate(
        bfm::CostModel::quadratic(dim), p,
        side == BFM_MAP_NU_SIDE ? bfm::MapSource::nu_side : bfm::MapSource::mu_side);
    for (int a = 0; a < dim; ++a)
      std::memcpy(disp + a * g.size(), m.displacement[a].data(), g.size() * sizeof(double));
  })
}

int ref_pushforward_density(int dim, const int* ext, const double* disp, const double* mu,
                            double* rho) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::DensityField m(g);
    std::memcpy(m.values.data(), mu, g.size() * sizeof(double));
    const bfm::DensityField r = bfm::pushforward_density(make_map(g, disp), m);
    std::memcpy(rho, r.values.data(), g.size() * sizeof(double));
  })
}

int ref_displacement_interpolant(int dim, const int* ext, const double* disp,
                                 const double* mu, double t, double* rho) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::DensityField m(g);
    std::memcpy(m.values.data(), mu, g.size() * sizeof(double));
    const bfm::DensityField r = bfm::displacement_interpolant(make_map(g, disp), m, t);
    std::memcpy(rho, r.values.data(), g.size() * sizeof(double));
  })
}

int ref_solve_neumann(int dim, const int* ext, const double* rhs, double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::SpectralPlan plan(g);
    plan.solve_neumann(rhs, out);
  })
}

int ref_integrate(int dim, const int* ext, const double* f, const double* w, double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::ScalarField ff(g);
    std::memcpy(ff.values.data(), f, g.size() * sizeof(double));
    if (w) {
      bfm::DensityField ww(g);
      std::memcpy(ww.values.data(), w, g.size() * sizeof(double));
      *out = bfm::integrate(ff, ww);
    } else {
      *out = bfm::integrate(ff);
    }
  })
}

int ref_primal_cost(int dim, const int* ext, const double* disp, const double* mu,
                    double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::DensityField m(g);
    std::memcpy(m.values.data(), mu, g.size() * sizeof(double));
    *out = bfm::primal_cost(make_map(g, disp), m, bfm::CostModel::quadratic(dim));
  })
}

int ref_primal_cost_cost(int dim, const int* ext, const double* exponents, const double* disp,
                         const double* mu, double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::DensityField m(g);
    std::memcpy(m.values.data(), mu, g.size() * sizeof(double));
    *out = bfm::primal_cost(make_map(g, disp), m, cost_model(dim, exponents));
  })
}

// Fixture helpers (io.hpp:452-476 builtin_density, grid.hpp:151-164 normalize).
int ref_builtin_density(int dim, const int* ext, const char* spec, double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    const bfm::DensityField f = bfm::builtin_density(g, spec);
    std::memcpy(out, f.values.data(), g.size() * sizeof(double));
  })
}

int ref_normalize(int dim, const int* ext, const double* raw, double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    const bfm::DensityField f =
        bfm::normalize(g, std::vector<double>(raw, raw + g.size()));
    std::memcpy(out, f.values.data(), g.size() * sizeof(double));
  })
}

int ref_hm1dot_norm_sq(int dim, const int* ext, const double* f, double* out) {
  GUARD({
    const bfm::Grid g = make_grid(dim, ext);
    bfm::SpectralPlan plan(g);
    *out = plan.hm1dot_norm_sq(f);
  })
}

}  // extern "C"
