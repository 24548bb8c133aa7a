// Header-only C++ facade over the C ABI (include/bfm_b200.h) that re-exposes
// the reference solver API (/root/reference/proj/include/bfm/*.hpp) with the
// same names, signatures and exception types, so drivers written against the
// reference (e.g. tools/bfm_ot.cpp's run_solver, benchmark.hpp's
// run_benchmark_case) compile unchanged against this header and run on the
// B200. Quadratic costs (the north-star path) and separable power costs
// (CostModel::power): the power-cost map uses a correctly rounded pow where the
// reference calls glibc's (one ulp apart on ~0.1 % of calls). Link with
// -lbfm_b200 (paper_1905_12154_b200/libbfm_b200.so).
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../bfm_b200.h"

namespace bfm {

// ---- errors.hpp:8-42 ---------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : Error { using Error::Error; };
struct GridMismatch : Error { using Error::Error; };
struct NegativeInput : Error { using Error::Error; };
struct AllZeroInput : Error { using Error::Error; };
struct InfeasibleInput : Error { using Error::Error; };
struct NumericalBlowup : Error { using Error::Error; };
struct TOutOfRange : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };

namespace detail {
inline void check(int rc) {
  if (rc == BFM_OK) return;
  const std::string m = bfm_last_error();
  switch (rc) {
    case BFM_ERR_INVALID_ARGUMENT: throw InvalidArgument(m);
    case BFM_ERR_GRID_MISMATCH: throw GridMismatch(m);
    case BFM_ERR_NEGATIVE_INPUT: throw NegativeInput(m);
    case BFM_ERR_ALL_ZERO_INPUT: throw AllZeroInput(m);
    case BFM_ERR_INFEASIBLE_INPUT: throw InfeasibleInput(m);
    case BFM_ERR_NUMERICAL_BLOWUP: throw NumericalBlowup(m);
    case BFM_ERR_T_OUT_OF_RANGE: throw TOutOfRange(m);
    case BFM_ERR_IO: throw IoError(m);
    default: throw Error(m);
  }
}
}  // namespace detail

// ---- grid.hpp:17-115 ---------------------------------------------------------
class Grid {
 public:
  Grid() = default;
  explicit Grid(const std::vector<int>& dims) { init(dims); }
  Grid(std::initializer_list<int> dims) { init(std::vector<int>(dims)); }
  int dim() const { return dim_; }
  int extent(int axis) const { return dims_[axis]; }
  double spacing(int axis) const { return spacing_[axis]; }
  double coord(int axis, int idx) const { return (idx + 0.5) * spacing_[axis]; }
  std::size_t size() const { return size_; }
  double cell_volume() const { return volume_; }
  std::size_t stride(int axis) const { return stride_[axis]; }
  std::size_t linear(std::array<int, 3> idx) const {
    std::size_t lin = 0;
    for (int a = 0; a < dim_; ++a) lin += static_cast<std::size_t>(idx[a]) * stride_[a];
    return lin;
  }
  std::size_t linear(int i0, int i1 = 0, int i2 = 0) const { return linear({i0, i1, i2}); }
  std::vector<double> axis_coords(int axis) const {
    std::vector<double> c(dims_[axis]);
    for (int i = 0; i < dims_[axis]; ++i) c[i] = coord(axis, i);
    return c;
  }
  std::vector<int> extents() const { return std::vector<int>(dims_.begin(), dims_.begin() + dim_); }
  bool operator==(const Grid& o) const {
    if (dim_ != o.dim_) return false;
    for (int a = 0; a < dim_; ++a)
      if (dims_[a] != o.dims_[a]) return false;
    return true;
  }
  bool operator!=(const Grid& o) const { return !(*this == o); }
  const int* extents_ptr() const { return dims_.data(); }

 private:
  void init(const std::vector<int>& dims) {
    if (dims.empty() || dims.size() > 3) throw InvalidArgument("grid dimension must be 1, 2, or 3");
    dim_ = static_cast<int>(dims.size());
    size_ = 1;
    volume_ = 1.0;
    for (int a = 0; a < dim_; ++a) {
      if (dims[a] < 2) throw InvalidArgument("grid extent must be at least 2");
      dims_[a] = dims[a];
      spacing_[a] = 1.0 / dims[a];
      size_ *= static_cast<std::size_t>(dims[a]);
      volume_ *= spacing_[a];
    }
    stride_[dim_ - 1] = 1;
    for (int a = dim_ - 2; a >= 0; --a) stride_[a] = stride_[a + 1] * static_cast<std::size_t>(dims_[a + 1]);
  }
  int dim_ = 0;
  std::array<int, 3> dims_{1, 1, 1};
  std::array<double, 3> spacing_{1.0, 1.0, 1.0};
  std::array<std::size_t, 3> stride_{0, 0, 0};
  std::size_t size_ = 0;
  double volume_ = 1.0;
};

struct ScalarField {
  ScalarField() = default;
  explicit ScalarField(const Grid& g, double fill = 0.0) : grid(g), values(g.size(), fill) {}
  Grid grid;
  std::vector<double> values;
};
struct Potential : ScalarField {
  Potential() = default;
  explicit Potential(const Grid& g, double fill = 0.0) : ScalarField(g, fill) {}
};
struct DensityField : ScalarField {
  DensityField() = default;
  explicit DensityField(const Grid& g, double fill = 0.0) : ScalarField(g, fill) {}
};

// ---- cost.hpp:17-81 ----------------------------------------------------------------
// Separable costs sum_a |y_a - x_a|^p_a / p_a, every operator and the solver
// on the B200 (bfm_*_cost entry points for p != 2).
class CostModel {
 public:
  static CostModel quadratic(int dim) {
    if (dim < 1 || dim > 3) throw InvalidArgument("cost dimension must be 1..3");
    return CostModel(std::vector<double>(dim, 2.0));
  }
  static CostModel power(const std::vector<double>& p) {
    if (p.empty() || p.size() > 3) throw InvalidArgument("cost dimension must be 1..3");
    for (double q : p)
      if (!(q > 1.0)) throw InvalidArgument("cost exponents must satisfy p > 1");
    return CostModel(p);
  }
  int dim() const { return static_cast<int>(p_.size()); }
  bool is_quadratic() const { return quadratic_; }
  double exponent(int axis) const { return p_[axis]; }
  const double* exponents() const { return p_.data(); }
  double axis_cost(int axis, double delta) const {
    const double p = p_[axis];
    if (p == 2.0) return 0.5 * delta * delta;
    return std::pow(std::fabs(delta), p) / p;
  }

 private:
  explicit CostModel(std::vector<double> p) : p_(std::move(p)) {
    quadratic_ = true;
    for (double q : p_)
      if (q != 2.0) quadratic_ = false;
  }
  std::vector<double> p_;
  bool quadratic_ = true;
};

// ---- pushforward.hpp:22-36 ---------------------------------------------------
enum class MapSource { mu_side, nu_side };
struct TransportMap {
  Grid grid;
  std::array<std::vector<double>, 3> displacement;
  MapSource source = MapSource::mu_side;
  TransportMap() = default;
  explicit TransportMap(const Grid& g, MapSource s = MapSource::mu_side) : grid(g), source(s) {
    for (int a = 0; a < g.dim(); ++a) displacement[a].assign(g.size(), 0.0);
  }
};
inline TransportMap identity_map(const Grid& g) { return TransportMap(g); }

namespace detail {
inline void require_same_grid(const Grid& a, const Grid& b, const char* what) {
  if (a != b) throw GridMismatch(std::string("grid mismatch in ") + what);
}
inline std::vector<double> flat_disp(const TransportMap& m) {
  std::vector<double> d(m.grid.dim() * m.grid.size());
  for (int a = 0; a < m.grid.dim(); ++a)
    std::copy(m.displacement[a].begin(), m.displacement[a].end(), d.begin() + a * m.grid.size());
  return d;
}
}  // namespace detail

// ---- operators -----------------------------------------------------------------
namespace detail {
struct WorkspaceDeleter {
  void operator()(bfm_workspace* w) const { bfm_workspace_destroy(w); }
};
}  // namespace detail

// transforms.hpp:231: both paths are exact, so they return the same bits (the
// reference's automatic quadratic shortcut and its generic divide and
// conquer agree bitwise; so do ours).
enum class CtransformPath { automatic, divide_and_conquer };

// transforms.hpp:233-283: a grid's reusable c-transform state. Here it owns a
// device workspace (bfm_workspace): the per-axis plans, tables and inter-pass
// buffers are built once and reused by every ctransform on it. `threads` is
// accepted for API parity (the device ignores it).
class TransformWorkspace {
 public:
  explicit TransformWorkspace(const Grid& grid, int threads = 1)
      : grid_(grid), threads_(threads < 1 ? 1 : threads) {
    bfm_workspace* w = nullptr;
    detail::check(bfm_workspace_create(grid.dim(), grid.extents_ptr(), &w));
    ws_.reset(w);
  }
  const Grid& grid() const { return grid_; }
  int threads() const { return threads_; }
  bfm_workspace* handle() const { return ws_.get(); }

 private:
  Grid grid_;
  int threads_;
  std::unique_ptr<bfm_workspace, detail::WorkspaceDeleter> ws_;
};

inline Potential ctransform(const CostModel& model, const Potential& phi, TransformWorkspace& ws,
                            CtransformPath path = CtransformPath::automatic) {  // transforms.hpp:396-427
  (void)path;
  const Grid& g = phi.grid;
  if (model.dim() != g.dim()) throw GridMismatch("ctransform: cost dimension does not match grid");
  if (ws.grid() != g) throw GridMismatch("ctransform: workspace built for a different grid");
  Potential out(g);
  if (model.is_quadratic())
    detail::check(bfm_workspace_ctransform(ws.handle(), phi.values.data(), out.values.data()));
  else
    detail::check(bfm_ctransform_cost(g.dim(), g.extents_ptr(), model.exponents(), phi.values.data(),
                                      out.values.data()));
  return out;
}

inline Potential ctransform(const CostModel& model, const Potential& phi) {  // transforms.hpp:429-432
  if (model.dim() != phi.grid.dim()) throw GridMismatch("ctransform: cost dimension does not match grid");
  Potential out(phi.grid);
  if (model.is_quadratic())
    detail::check(bfm_ctransform(phi.grid.dim(), phi.grid.extents_ptr(), phi.values.data(), out.values.data()));
  else
    detail::check(bfm_ctransform_cost(phi.grid.dim(), phi.grid.extents_ptr(), model.exponents(),
                                      phi.values.data(), out.values.data()));
  return out;
}

inline TransportMap map_from_conjugate(const CostModel& model, const Potential& psi,
                                       MapSource source = MapSource::mu_side) {  // pushforward.hpp:70-91
  if (model.dim() != psi.grid.dim())
    throw GridMismatch("map_from_conjugate: cost dimension does not match grid");
  TransportMap map(psi.grid, source);
  std::vector<double> d(psi.grid.dim() * psi.grid.size());
  detail::check(bfm_map_from_conjugate_cost(psi.grid.dim(), psi.grid.extents_ptr(),
                                            model.is_quadratic() ? nullptr : model.exponents(),
                                            psi.values.data(),
                                            source == MapSource::nu_side ? BFM_MAP_NU_SIDE : BFM_MAP_MU_SIDE,
                                            d.data()));
  for (int a = 0; a < psi.grid.dim(); ++a)
    map.displacement[a].assign(d.begin() + a * psi.grid.size(), d.begin() + (a + 1) * psi.grid.size());
  return map;
}

inline DensityField pushforward_density(const TransportMap& map, const DensityField& mu) {
  detail::require_same_grid(map.grid, mu.grid, "pushforward_density");
  DensityField out(mu.grid);
  const std::vector<double> d = detail::flat_disp(map);
  detail::check(bfm_pushforward_density(mu.grid.dim(), mu.grid.extents_ptr(), d.data(), mu.values.data(),
                                        out.values.data()));
  return out;
}

inline DensityField displacement_interpolant(const TransportMap& map, const DensityField& mu,
                                             double t) {  // interpolation.hpp:18-22
  detail::require_same_grid(map.grid, mu.grid, "pushforward_density");
  DensityField out(mu.grid);
  const std::vector<double> d = detail::flat_disp(map);
  detail::check(bfm_displacement_interpolant(mu.grid.dim(), mu.grid.extents_ptr(), d.data(),
                                             mu.values.data(), t, out.values.data()));
  return out;
}

inline std::vector<DensityField> frame_sequence(const TransportMap& map, const DensityField& mu,
                                                int count) {  // interpolation.hpp:24-38
  if (count < 2) throw InvalidArgument("frame_sequence: need at least two frames");
  std::vector<DensityField> frames;
  for (int k = 0; k < count; ++k)
    frames.push_back(displacement_interpolant(map, mu, static_cast<double>(k) / (count - 1)));
  return frames;
}

inline double primal_cost(const TransportMap& map, const DensityField& mu, const CostModel& model) {
  detail::require_same_grid(map.grid, mu.grid, "primal_cost");
  if (model.dim() != map.grid.dim()) throw GridMismatch("primal_cost: cost dimension does not match grid");
  const std::vector<double> d = detail::flat_disp(map);
  double v = 0.0;
  detail::check(bfm_primal_cost_cost(mu.grid.dim(), mu.grid.extents_ptr(),
                                     model.is_quadratic() ? nullptr : model.exponents(), d.data(),
                                     mu.values.data(), &v));
  return v;
}

inline double integrate(const ScalarField& f, const DensityField& w) {  // grid.hpp:171-176
  detail::require_same_grid(f.grid, w.grid, "integrate");
  double v = 0.0;
  detail::check(bfm_integrate(f.grid.dim(), f.grid.extents_ptr(), f.values.data(), w.values.data(), &v));
  return v;
}
inline double integrate(const ScalarField& f) {  // grid.hpp:179-183
  double v = 0.0;
  detail::check(bfm_integrate(f.grid.dim(), f.grid.extents_ptr(), f.values.data(), nullptr, &v));
  return v;
}

inline DensityField normalize(const Grid& grid, const std::vector<double>& raw) {  // grid.hpp:151-164
  if (raw.size() != grid.size()) throw GridMismatch("normalize: sample count does not match grid");
  double sum = 0.0, carry = 0.0;
  for (double v : raw) {
    if (v < 0.0) throw NegativeInput("normalize: negative density sample");
    const double y = v - carry;
    const double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
  const double mass = sum * grid.cell_volume();
  if (mass <= 0.0) throw AllZeroInput("normalize: density has zero total mass");
  DensityField out(grid);
  for (std::size_t i = 0; i < raw.size(); ++i) out.values[i] = raw[i] / mass;
  return out;
}

// io.hpp:452-476: indicator of a '+'-union of builtin shapes (not normalised)
inline DensityField builtin_density(const Grid& g, const std::string& spec) {
  DensityField f(g);
  detail::check(bfm_builtin_density(g.dim(), g.extents_ptr(), spec.c_str(), f.values.data()));
  return f;
}

// poisson.hpp:40-113
class SpectralPlan {  // poisson.hpp:42-113; the device plan is built once per SpectralPlan
 public:
  explicit SpectralPlan(const Grid& grid) : grid_(grid) {
    bfm_workspace* w = nullptr;
    detail::check(bfm_workspace_create(grid.dim(), grid.extents_ptr(), &w));
    ws_.reset(w, detail::WorkspaceDeleter());
  }
  const Grid& grid() const { return grid_; }
  void solve_neumann(const double* rhs, double* out) const {
    detail::check(bfm_workspace_solve_neumann(ws_.get(), rhs, out));
  }
  Potential solve_neumann(const ScalarField& rhs) const {
    if (rhs.grid != grid_) throw GridMismatch("field grid does not match plan");
    Potential u(grid_);
    solve_neumann(rhs.values.data(), u.values.data());
    return u;
  }

 private:
  Grid grid_;
  std::shared_ptr<bfm_workspace> ws_;
};

// ---- solver.hpp:32-374 -------------------------------------------------------
enum class SolverMode { back_and_forth, gradient_ascent };
enum class Termination { tolerance_met, max_iterations, dual_stalled, cost_target_met };

inline const char* termination_name(Termination t) {
  switch (t) {
    case Termination::tolerance_met: return "tolerance_met";
    case Termination::max_iterations: return "max_iterations";
    case Termination::dual_stalled: return "dual_stalled";
    case Termination::cost_target_met: return "cost_target_met";
  }
  return "unknown";
}

struct SolverConfig {
  SolverMode mode = SolverMode::back_and_forth;
  double tolerance = 1e-4;
  int max_iterations = 2000;
  int threads = 0;
  double sigma_init = 0.0;
  double sigma_min = 0.01;
  double beta_1 = 0.25;
  double beta_2 = 0.75;
  double alpha_1 = 1.25;
  double alpha_2 = 0.8;
  std::optional<double> exact_cost;
  double exact_tolerance = 0.0;
};

namespace detail {
inline bfm_config to_c(const SolverConfig& c) {
  bfm_config r;
  r.mode = c.mode == SolverMode::gradient_ascent ? BFM_MODE_GRADIENT_ASCENT : BFM_MODE_BACK_AND_FORTH;
  r.tolerance = c.tolerance;
  r.max_iterations = c.max_iterations;
  r.threads = c.threads;
  r.sigma_init = c.sigma_init;
  r.sigma_min = c.sigma_min;
  r.beta_1 = c.beta_1;
  r.beta_2 = c.beta_2;
  r.alpha_1 = c.alpha_1;
  r.alpha_2 = c.alpha_2;
  r.has_exact_cost = c.exact_cost ? 1 : 0;
  r.exact_cost = c.exact_cost ? *c.exact_cost : 0.0;
  r.exact_tolerance = c.exact_tolerance;
  return r;
}
}  // namespace detail

inline double update_sigma(double sigma, double increase, double grad_norm_sq,
                           const SolverConfig& config = {}) {
  const bfm_config c = detail::to_c(config);
  return bfm_update_sigma(sigma, increase, grad_norm_sq, &c);
}

struct IterationStats {
  int iteration = 0;
  double residual = 0.0;
  double dual_value = 0.0;
  double sigma_first = 0.0;
  double sigma_second = 0.0;
  double grad_norm_sq_first = 0.0;
  double grad_norm_sq_second = 0.0;
  double increase_first = 0.0;
  double increase_second = 0.0;
};

struct SolveReport {
  Termination termination = Termination::max_iterations;
  int iterations = 0;
  double dual_value = 0.0;
  double primal_cost = 0.0;
  double residual = 0.0;
  double wall_seconds = 0.0;
  std::vector<IterationStats> trace;
  Potential phi;
  Potential psi;
  TransportMap map;
};

class Solver {
 public:
  Solver(const CostModel& model, const DensityField& mu, const DensityField& nu,
         const SolverConfig& config = {})
      : grid_(mu.grid) {
    detail::require_same_grid(mu.grid, nu.grid, "solve");
    if (model.dim() != mu.grid.dim()) throw GridMismatch("solve: cost dimension does not match grid");
    const bfm_config c = detail::to_c(config);
    detail::check(bfm_solver_create_cost(grid_.dim(), grid_.extents_ptr(),
                                         model.is_quadratic() ? nullptr : model.exponents(),
                                         mu.values.data(), nu.values.data(), &c, &h_));
  }
  ~Solver() {
    if (h_) bfm_solver_destroy(h_);
  }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  int iteration() const { return bfm_solver_iteration(h_); }
  double sigma() const { return bfm_solver_sigma(h_); }
  Potential phi() const { return field(BFM_FIELD_PHI); }
  Potential psi() const { return field(BFM_FIELD_PSI); }
  std::vector<IterationStats> trace() const {
    int n = 0;
    bfm_solver_trace(h_, nullptr, 0, &n);
    std::vector<bfm_iteration_stats> raw(static_cast<std::size_t>(n));
    bfm_solver_trace(h_, raw.data(), n, &n);
    std::vector<IterationStats> t;
    for (const auto& r : raw) t.push_back(convert(r));
    return t;
  }
  double dual_value() {
    double v = 0.0;
    detail::check(bfm_solver_dual_value(h_, &v));
    return v;
  }
  double residual() {
    double v = 0.0;
    detail::check(bfm_solver_residual(h_, &v));
    return v;
  }
  IterationStats step() {
    bfm_iteration_stats st;
    detail::check(bfm_solver_step(h_, &st));
    return convert(st);
  }
  SolveReport run() {
    bfm_report r;
    detail::check(bfm_solver_run(h_, &r));
    SolveReport rep;
    rep.termination = static_cast<Termination>(r.termination);
    rep.iterations = r.iterations;
    rep.dual_value = r.dual_value;
    rep.primal_cost = r.primal_cost;
    rep.residual = r.residual;
    rep.wall_seconds = r.wall_seconds;
    rep.trace = trace();
    rep.phi = report_field(BFM_FIELD_PHI);
    rep.psi = report_field(BFM_FIELD_PSI);
    rep.map = TransportMap(grid_, MapSource::mu_side);
    for (int a = 0; a < grid_.dim(); ++a)
      rep.map.displacement[a] = report_field(BFM_FIELD_MAP0 + a).values;
    return rep;
  }

 private:
  static IterationStats convert(const bfm_iteration_stats& s) {
    return IterationStats{s.iteration, s.residual, s.dual_value, s.sigma_first, s.sigma_second,
                          s.grad_norm_sq_first, s.grad_norm_sq_second, s.increase_first,
                          s.increase_second};
  }
  Potential field(int which) const {
    Potential p(grid_);
    detail::check(bfm_solver_field(h_, which, p.values.data()));
    return p;
  }
  Potential report_field(int which) const {
    Potential p(grid_);
    detail::check(bfm_solver_report_field(h_, which, p.values.data()));
    return p;
  }
  Grid grid_;
  bfm_solver* h_ = nullptr;
};

inline SolveReport solve(const CostModel& model, const DensityField& mu, const DensityField& nu,
                         const SolverConfig& config = {}) {
  Solver solver(model, mu, nu, config);
  return solver.run();
}

}  // namespace bfm
