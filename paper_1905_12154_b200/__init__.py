"""B200-native back-and-forth (BFM) optimal-transport solver.

Python mirror of the reference's C++ solver API
(/root/reference/proj/include/bfm/solver.hpp:32-374, transforms.hpp:396-432,
pushforward.hpp:70-196, poisson.hpp:87-113, grid.hpp:151-183) over the C ABI
in include/bfm_b200.h (libbfm_b200.so, hand-written sm_100a kernels).

There is no CPU fallback: every compute call goes through the CUDA library
and raises if it is missing or no device is present.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BFM_LIB_OVERRIDE") or os.path.join(_HERE, "libbfm_b200.so")

# ---------------------------------------------------------------- errors
class Error(RuntimeError):
    """bfm::Error (errors.hpp:8-10)."""


class InvalidArgument(Error):
    pass


class GridMismatch(Error):
    pass


class NegativeInput(Error):
    pass


class AllZeroInput(Error):
    pass


class InfeasibleInput(Error):
    pass


class NumericalBlowup(Error):
    pass


class TOutOfRange(Error):
    pass


class IoError(Error):
    pass


class DeviceError(Error):
    """CUDA failure or no device (the reference has no equivalent)."""


_ERRORS = {
    1: Error,
    2: InvalidArgument,
    3: GridMismatch,
    4: NegativeInput,
    5: AllZeroInput,
    6: InfeasibleInput,
    7: NumericalBlowup,
    8: TOutOfRange,
    9: IoError,
    10: DeviceError,
}

# ---------------------------------------------------------------- enums
BACK_AND_FORTH, GRADIENT_ASCENT = 0, 1
TERMINATION_NAMES = ["tolerance_met", "max_iterations", "dual_stalled", "cost_target_met"]
MU_SIDE, NU_SIDE = 0, 1
FIELD_PHI, FIELD_PSI, FIELD_MAP0 = 0, 1, 2


class _Config(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("tolerance", C.c_double),
        ("max_iterations", C.c_int),
        ("threads", C.c_int),
        ("sigma_init", C.c_double),
        ("sigma_min", C.c_double),
        ("beta_1", C.c_double),
        ("beta_2", C.c_double),
        ("alpha_1", C.c_double),
        ("alpha_2", C.c_double),
        ("has_exact_cost", C.c_int),
        ("exact_cost", C.c_double),
        ("exact_tolerance", C.c_double),
    ]


class _Stats(C.Structure):
    _fields_ = [
        ("iteration", C.c_int),
        ("residual", C.c_double),
        ("dual_value", C.c_double),
        ("sigma_first", C.c_double),
        ("sigma_second", C.c_double),
        ("grad_norm_sq_first", C.c_double),
        ("grad_norm_sq_second", C.c_double),
        ("increase_first", C.c_double),
        ("increase_second", C.c_double),
    ]


class _Report(C.Structure):
    _fields_ = [
        ("termination", C.c_int),
        ("iterations", C.c_int),
        ("dual_value", C.c_double),
        ("primal_cost", C.c_double),
        ("residual", C.c_double),
        ("wall_seconds", C.c_double),
    ]


_lib = None


def _declare(lib, prefix: str):
    """Declares argtypes for the C ABI (used for both the product library and
    the oracle's ref_-prefixed mirror)."""
    P = C.c_void_p
    I = C.c_int
    D = C.c_double
    sig = {
        "solver_create": (I, [I, P, P, P, P, P]),
        "solver_destroy": (None, [P]),
        "solver_iteration": (I, [P]),
        "solver_sigma": (D, [P]),
        "solver_dual_value": (I, [P, P]),
        "solver_residual": (I, [P, P]),
        "solver_step": (I, [P, P]),
        "solver_run": (I, [P, P]),
        "solver_trace": (I, [P, P, I, P]),
        "solver_field": (I, [P, I, P]),
        "solver_report_field": (I, [P, I, P]),
        "map_from_conjugate": (I, [I, P, P, I, P]),
        "pushforward_density": (I, [I, P, P, P, P]),
        "displacement_interpolant": (I, [I, P, P, P, D, P]),
        "solve_neumann": (I, [I, P, P, P]),
        "integrate": (I, [I, P, P, P, P]),
        "primal_cost": (I, [I, P, P, P, P]),
        "update_sigma": (D, [D, D, D, P]),
        "last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, prefix + name, None)
        if f is None:
            continue
        f.restype = res
        f.argtypes = args


def load_library(path: str = LIB_PATH):
    """Loads libbfm_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(path)
    _declare(lib, "bfm_")
    lib.bfm_ctransform.restype = C.c_int
    lib.bfm_ctransform.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.bfm_device_available.restype = C.c_int
    lib.bfm_config_default.argtypes = [C.c_void_p]
    lib.bfm_workspace_create.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
    lib.bfm_workspace_destroy.argtypes = [C.c_void_p]
    for fn in ("bfm_ctransform_device", "bfm_solve_neumann_device"):
        getattr(lib, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        getattr(lib, fn).restype = C.c_int
    lib.bfm_pushforward_residual_device.argtypes = [C.c_void_p] * 6
    lib.bfm_pushforward_residual_device.restype = C.c_int
    lib.bfm_workspace_last_launches.argtypes = [C.c_void_p]
    lib.bfm_workspace_last_launches.restype = C.c_int
    lib.bfm_solver_launches.argtypes = [C.c_void_p]
    lib.bfm_solver_launches.restype = C.c_long
    lib.bfm_solver_time_steps.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    lib.bfm_solver_time_steps.restype = C.c_int
    lib.bfm_solver_set_timing.argtypes = [C.c_void_p, C.c_int]
    lib.bfm_solver_set_timing.restype = C.c_int
    lib.bfm_solver_op_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.bfm_solver_op_times.restype = C.c_int
    lib.bfm_ctransform_cost.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.bfm_ctransform_cost.restype = C.c_int
    lib.bfm_builtin_density.argtypes = [C.c_int, C.c_void_p, C.c_char_p, C.c_void_p]
    lib.bfm_builtin_density.restype = C.c_int
    lib.bfm_normalize.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.bfm_normalize.restype = C.c_int
    lib.bfm_set_device.argtypes = [C.c_int]
    lib.bfm_set_device.restype = C.c_int
    lib.bfm_solver_set_graphs.argtypes = [C.c_void_p, C.c_int]
    lib.bfm_solver_set_graphs.restype = C.c_int
    lib.bfm_solver_debug_force_exact.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.bfm_solver_debug_force_exact.restype = C.c_int
    lib.bfm_solver_exact_replays.argtypes = [C.c_void_p]
    lib.bfm_solver_exact_replays.restype = C.c_long
    lib.bfm_synthetic_densities.argtypes = [C.c_int, C.c_int, C.c_ulonglong, C.c_void_p, C.c_void_p]
    lib.bfm_synthetic_densities.restype = C.c_int
    _lib = lib
    return lib


def set_device(device: int) -> None:
    lib = load_library()
    _check(lib, lib.bfm_set_device(int(device)))


def device_available() -> bool:
    return bool(load_library().bfm_device_available())


def _check(lib, rc: int, prefix: str = "bfm_"):
    if rc != 0:
        msg = getattr(lib, prefix + "last_error")().decode()
        raise _ERRORS.get(rc, Error)(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _extents(shape: Sequence[int]):
    return (C.c_int * len(shape))(*[int(s) for s in shape])


# ---------------------------------------------------------------- data types
@dataclasses.dataclass
class SolverConfig:
    """solver.hpp:46-63."""

    mode: int = BACK_AND_FORTH
    tolerance: float = 1e-4
    max_iterations: int = 2000
    threads: int = 0
    sigma_init: float = 0.0
    sigma_min: float = 0.01
    beta_1: float = 0.25
    beta_2: float = 0.75
    alpha_1: float = 1.25
    alpha_2: float = 0.8
    exact_cost: Optional[float] = None
    exact_tolerance: float = 0.0

    def _c(self) -> _Config:
        c = _Config()
        c.mode = self.mode
        c.tolerance = self.tolerance
        c.max_iterations = self.max_iterations
        c.threads = self.threads
        c.sigma_init = self.sigma_init
        c.sigma_min = self.sigma_min
        c.beta_1 = self.beta_1
        c.beta_2 = self.beta_2
        c.alpha_1 = self.alpha_1
        c.alpha_2 = self.alpha_2
        c.has_exact_cost = 0 if self.exact_cost is None else 1
        c.exact_cost = 0.0 if self.exact_cost is None else float(self.exact_cost)
        c.exact_tolerance = self.exact_tolerance
        return c


@dataclasses.dataclass
class IterationStats:
    """solver.hpp:78-88."""

    iteration: int = 0
    residual: float = 0.0
    dual_value: float = 0.0
    sigma_first: float = 0.0
    sigma_second: float = 0.0
    grad_norm_sq_first: float = 0.0
    grad_norm_sq_second: float = 0.0
    increase_first: float = 0.0
    increase_second: float = 0.0

    @staticmethod
    def _from(s: _Stats) -> "IterationStats":
        return IterationStats(*[getattr(s, f[0]) for f in _Stats._fields_])


@dataclasses.dataclass
class SolveReport:
    """solver.hpp:90-101 (phi/psi gauge fixed; map = displacement per axis)."""

    termination: str
    iterations: int
    dual_value: float
    primal_cost: float
    residual: float
    wall_seconds: float
    trace: List[IterationStats]
    phi: np.ndarray
    psi: np.ndarray
    map: np.ndarray  # shape (d, *grid)


def update_sigma(sigma: float, increase: float, grad_norm_sq: float,
                 config: Optional[SolverConfig] = None, _lib_override=None, _prefix="bfm_") -> float:
    """solver.hpp:68-76."""
    lib = _lib_override or load_library()
    cfg = (config or SolverConfig())._c()
    return getattr(lib, _prefix + "update_sigma")(sigma, increase, grad_norm_sq, C.byref(cfg))


class Solver:
    """bfm::Solver (solver.hpp:146-368) on the B200. mu, nu: float64 arrays of
    the grid's shape (1-3 dims), each normalised to unit mass."""

    _prefix = "bfm_"

    def __init__(self, mu, nu, config: Optional[SolverConfig] = None, _lib=None,
                 exponents: Optional[Sequence[float]] = None):
        """exponents: CostModel::power (cost.hpp:24-30), one p > 1 per axis;
        None is the quadratic cost."""
        self._lib = _lib or load_library()
        mu = _f64(mu)
        nu = _f64(nu)
        if mu.shape != nu.shape:
            raise GridMismatch("grid mismatch in solve")
        self.shape = mu.shape
        self.config = config or SolverConfig()
        self._cfg = self.config._c()
        h = C.c_void_p()
        self._h = None
        if exponents is None:
            rc = self._fn("solver_create")(len(mu.shape), _extents(mu.shape), _ptr(mu), _ptr(nu),
                                           C.byref(self._cfg), C.byref(h))
        else:
            if len(exponents) != mu.ndim:
                raise GridMismatch("solve: cost dimension does not match grid")
            ex = (C.c_double * 3)(*([float(e) for e in exponents] + [2.0] * (3 - len(exponents))))
            f = self._fn("solver_create_cost")
            f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            f.restype = C.c_int
            rc = f(len(mu.shape), _extents(mu.shape), ex, _ptr(mu), _ptr(nu), C.byref(self._cfg), C.byref(h))
        self._check(rc)
        self._h = h

    def _fn(self, name):
        return getattr(self._lib, self._prefix + name)

    def _check(self, rc):
        _check(self._lib, rc, self._prefix)

    def __del__(self):
        if getattr(self, "_h", None):
            self._fn("solver_destroy")(self._h)
            self._h = None

    def iteration(self) -> int:
        return self._fn("solver_iteration")(self._h)

    def sigma(self) -> float:
        return self._fn("solver_sigma")(self._h)

    def dual_value(self) -> float:
        v = C.c_double()
        self._check(self._fn("solver_dual_value")(self._h, C.byref(v)))
        return v.value

    def residual(self) -> float:
        v = C.c_double()
        self._check(self._fn("solver_residual")(self._h, C.byref(v)))
        return v.value

    def step(self) -> IterationStats:
        st = _Stats()
        self._check(self._fn("solver_step")(self._h, C.byref(st)))
        return IterationStats._from(st)

    def trace(self) -> List[IterationStats]:
        cnt = C.c_int()
        self._fn("solver_trace")(self._h, None, 0, C.byref(cnt))
        buf = (_Stats * max(1, cnt.value))()
        self._fn("solver_trace")(self._h, buf, cnt.value, C.byref(cnt))
        return [IterationStats._from(buf[i]) for i in range(cnt.value)]

    def _field(self, fn, which) -> np.ndarray:
        out = np.empty(self.shape, dtype=np.float64)
        self._check(self._fn(fn)(self._h, which, _ptr(out)))
        return out

    def phi(self) -> np.ndarray:
        return self._field("solver_field", FIELD_PHI)

    def psi(self) -> np.ndarray:
        return self._field("solver_field", FIELD_PSI)

    def run(self) -> SolveReport:
        rep = _Report()
        self._check(self._fn("solver_run")(self._h, C.byref(rep)))
        d = len(self.shape)
        disp = np.stack([self._field("solver_report_field", FIELD_MAP0 + a) for a in range(d)])
        return SolveReport(
            termination=TERMINATION_NAMES[rep.termination],
            iterations=rep.iterations,
            dual_value=rep.dual_value,
            primal_cost=rep.primal_cost,
            residual=rep.residual,
            wall_seconds=rep.wall_seconds,
            trace=self.trace(),
            phi=self._field("solver_report_field", FIELD_PHI),
            psi=self._field("solver_report_field", FIELD_PSI),
            map=disp,
        )

    def launches(self) -> int:
        return int(self._lib.bfm_solver_launches(self._h))

    OPS = ("ctransform", "pushforward", "poisson", "reduce")

    def set_timing(self, on: bool) -> None:
        """Per-operator CUDA-event timing on the solver stream (resets totals)."""
        self._check(self._lib.bfm_solver_set_timing(self._h, 1 if on else 0))

    def op_times(self) -> dict:
        """{op: (total ms, calls)} accumulated since set_timing(True)."""
        ms = (C.c_double * 4)()
        n = (C.c_long * 4)()
        self._check(self._lib.bfm_solver_op_times(self._h, ms, n))
        return {name: (ms[i], n[i]) for i, name in enumerate(self.OPS)}

    def set_graphs(self, on: bool) -> None:
        """CUDA-graph iterations (default) or eager launches (same kernels, same bits)."""
        self._check(self._lib.bfm_solver_set_graphs(self._h, 1 if on else 0))

    def debug_force_exact(self, iteration: int, probe_only: bool = False) -> None:
        """Test hook: replay `iteration` with reference-order (Kahan) scalars."""
        self._check(self._lib.bfm_solver_debug_force_exact(self._h, int(iteration),
                                                           1 if probe_only else 0))

    def exact_replays(self) -> int:
        return int(self._lib.bfm_solver_exact_replays(self._h))

    def time_steps(self, k: int) -> float:
        """Runs k iterations between CUDA events on the solver stream; returns ms."""
        ms = C.c_double()
        self._check(self._lib.bfm_solver_time_steps(self._h, int(k), C.byref(ms)))
        return ms.value


def solve(mu, nu, config: Optional[SolverConfig] = None) -> SolveReport:
    """bfm::solve (solver.hpp:370-374)."""
    return Solver(mu, nu, config).run()


# ---------------------------------------------------------------- operators
def ctransform(phi, exponents: Optional[Sequence[float]] = None) -> np.ndarray:
    """phi^c exactly rounded (transforms.hpp:396-432): quadratic cost, or
    CostModel::power(exponents) (cost.hpp:24-48, p_a > 1 per axis)."""
    lib = load_library()
    phi = _f64(phi)
    out = np.empty_like(phi)
    if exponents is None:
        _check(lib, lib.bfm_ctransform(phi.ndim, _extents(phi.shape), _ptr(phi), _ptr(out)))
    else:
        ex = (C.c_double * 3)(*([float(e) for e in exponents] + [2.0] * (3 - len(exponents))))
        if len(exponents) != phi.ndim:
            raise GridMismatch("ctransform: cost dimension does not match grid")
        _check(lib, lib.bfm_ctransform_cost(phi.ndim, _extents(phi.shape), ex, _ptr(phi), _ptr(out)))
    return out


def _exps(exponents, d):
    if len(exponents) != d:
        raise GridMismatch("cost dimension does not match grid")
    return (C.c_double * 3)(*([float(e) for e in exponents] + [2.0] * (3 - d)))


def map_from_conjugate(u, side: int = MU_SIDE, exponents: Optional[Sequence[float]] = None) -> np.ndarray:
    """pushforward.hpp:70-91: displacement field, shape (d, *grid); exponents:
    a power cost's p per axis (cost.hpp:58-68 inverse gradient)."""
    lib = load_library()
    u = _f64(u)
    disp = np.empty((u.ndim,) + u.shape, dtype=np.float64)
    if exponents is None:
        _check(lib, lib.bfm_map_from_conjugate(u.ndim, _extents(u.shape), _ptr(u), side, _ptr(disp)))
    else:
        f = lib.bfm_map_from_conjugate_cost
        f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        f.restype = C.c_int
        _check(lib, f(u.ndim, _extents(u.shape), _exps(exponents, u.ndim), _ptr(u), side, _ptr(disp)))
    return disp


def debug_pow(x, y, on_device: bool = True) -> np.ndarray:
    """Test hook: the library's correctly rounded x^y (pow_dd.h)."""
    lib = load_library()
    x = _f64(x).reshape(-1)
    y = np.broadcast_to(_f64(y), x.shape).copy()
    out = np.empty_like(x)
    f = lib.bfm_debug_pow
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    f.restype = C.c_int
    _check(lib, f(_ptr(x), _ptr(y), x.size, 1 if on_device else 0, _ptr(out)))
    return out


def _check_disp(disp: np.ndarray, mu: np.ndarray, what: str) -> None:
    """The C ABI reads d*N doubles of disp: reject other shapes as the
    reference's require_same_grid does (pushforward.hpp, GridMismatch)."""
    if disp.shape != (mu.ndim,) + mu.shape:
        raise GridMismatch(f"{what}: displacement shape {disp.shape} does not match the grid "
                           f"{(mu.ndim,) + mu.shape}")


def pushforward_density(disp, mu) -> np.ndarray:
    """pushforward.hpp:176-178."""
    lib = load_library()
    mu = _f64(mu)
    disp = _f64(disp)
    _check_disp(disp, mu, "pushforward_density")
    rho = np.empty_like(mu)
    _check(lib, lib.bfm_pushforward_density(mu.ndim, _extents(mu.shape), _ptr(disp), _ptr(mu),
                                            _ptr(rho)))
    return rho


def displacement_interpolant(disp, mu, t: float) -> np.ndarray:
    """interpolation.hpp:18-22."""
    lib = load_library()
    mu = _f64(mu)
    disp = _f64(disp)
    _check_disp(disp, mu, "displacement_interpolant")
    rho = np.empty_like(mu)
    _check(lib, lib.bfm_displacement_interpolant(mu.ndim, _extents(mu.shape), _ptr(disp),
                                                 _ptr(mu), float(t), _ptr(rho)))
    return rho


def frame_sequence(disp, mu, count: int) -> List[np.ndarray]:
    """interpolation.hpp:24-38."""
    if count < 2:
        raise InvalidArgument("frame_sequence: need at least two frames")
    return [displacement_interpolant(disp, mu, k / (count - 1)) for k in range(count)]


def solve_neumann(rhs) -> np.ndarray:
    """SpectralPlan::solve_neumann (poisson.hpp:87-113)."""
    lib = load_library()
    rhs = _f64(rhs)
    out = np.empty_like(rhs)
    _check(lib, lib.bfm_solve_neumann(rhs.ndim, _extents(rhs.shape), _ptr(rhs), _ptr(out)))
    return out


def integrate(f, w=None) -> float:
    """grid.hpp:171-183 (w=None: Lebesgue)."""
    lib = load_library()
    f = _f64(f)
    v = C.c_double()
    wp = None
    if w is not None:
        w = _f64(w)
        if w.shape != f.shape:
            raise GridMismatch("grid mismatch in integrate")
        wp = _ptr(w)
    _check(lib, lib.bfm_integrate(f.ndim, _extents(f.shape), _ptr(f), wp, C.byref(v)))
    return v.value


def primal_cost(disp, mu, exponents: Optional[Sequence[float]] = None) -> float:
    """pushforward.hpp:181-196 (quadratic, or a power cost's p per axis)."""
    lib = load_library()
    mu = _f64(mu)
    disp = _f64(disp)
    _check_disp(disp, mu, "primal_cost")
    v = C.c_double()
    if exponents is None:
        _check(lib, lib.bfm_primal_cost(mu.ndim, _extents(mu.shape), _ptr(disp), _ptr(mu),
                                        C.byref(v)))
    else:
        f = lib.bfm_primal_cost_cost
        f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        f.restype = C.c_int
        _check(lib, f(mu.ndim, _extents(mu.shape), _exps(exponents, mu.ndim), _ptr(disp), _ptr(mu),
                      C.byref(v)))
    return v.value


# ---------------------------------------------------------------- grid helpers
def axis_coords(n: int) -> np.ndarray:
    """grid.hpp:27,41-45: (i + 0.5) * (1.0 / n)."""
    return (np.arange(n, dtype=np.float64) + 0.5) * (1.0 / n)


def normalize(raw) -> np.ndarray:
    """grid.hpp:151-164: raw / (Kahan sum * cell volume), the reference's own
    summation order (host)."""
    lib = load_library()
    raw = _f64(raw)
    out = np.empty_like(raw)
    _check(lib, lib.bfm_normalize(raw.ndim, _extents(raw.shape), _ptr(raw), _ptr(out)))
    return out


def synthetic_densities(config: int, n: int, seed: int):
    """BASELINE.json configs C1-C4 from the library's shared generator
    (bfm_synthetic_densities: std::mt19937_64); returns (mu, nu)."""
    lib = load_library()
    shape = (n, n, n) if config == 4 else (n, n)
    mu = np.empty(shape, dtype=np.float64)
    nu = np.empty(shape, dtype=np.float64)
    _check(lib, lib.bfm_synthetic_densities(int(config), int(n), int(seed), _ptr(mu), _ptr(nu)))
    return mu, nu


def builtin_density(shape: Sequence[int], spec: str) -> np.ndarray:
    """io.hpp:452-476: indicator of a '+'-union of builtin shapes
    ("disc:x,y,r", "ball:x,y,z,r", "square:x,y,side", "cube:x,y,z,side") at the
    cell centres; not normalised."""
    lib = load_library()
    out = np.empty(tuple(int(n) for n in shape), dtype=np.float64)
    _check(lib, lib.bfm_builtin_density(len(shape), _extents(shape), spec.encode(), _ptr(out)))
    return out
