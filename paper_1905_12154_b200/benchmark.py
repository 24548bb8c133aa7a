"""Paper-case harness (reference benchmark.hpp:19-149).

The reference's four closed-form cases with known exact transport costs, the
published iteration counts they are checked against (±2), and a runner that
iterates until |dual − exact| ≤ tol (the exact-cost stopping rule,
solver.hpp:211-226). The solves run on the GPU solver; densities are the
reference's builtin shapes normalised exactly as the reference does
(bfm_builtin_density / bfm_normalize)."""
from __future__ import annotations

import dataclasses
from typing import IO, List, Optional, Tuple

from . import BACK_AND_FORTH, SolverConfig, builtin_density, normalize, solve


@dataclasses.dataclass
class BenchmarkCase:
    name: str
    dim: int
    mu_spec: str
    nu_spec: str
    exact_cost: float


def standard_benchmark_cases() -> List[BenchmarkCase]:
    """benchmark.hpp:27-43: two discs, two balls, a square to four squares,
    a cube to eight cubes (exact costs 1/4, 3/8, 1/16, 3/32)."""
    corners2 = [(0.1875, 0.1875), (0.8125, 0.1875), (0.1875, 0.8125), (0.8125, 0.8125)]
    corners3 = [(x, y, z) for z in (0.1875, 0.8125) for y in (0.1875, 0.8125) for x in (0.1875, 0.8125)]
    return [
        BenchmarkCase("two_discs", 2, "disc:0.25,0.25,0.125", "disc:0.75,0.75,0.125", 0.25),
        BenchmarkCase("two_balls", 3, "ball:0.25,0.25,0.25,0.125", "ball:0.75,0.75,0.75,0.125", 0.375),
        BenchmarkCase("four_squares", 2, "square:0.5,0.5,0.25",
                      "+".join(f"square:{x},{y},0.125" for x, y in corners2), 0.0625),
        BenchmarkCase("eight_cubes", 3, "cube:0.5,0.5,0.5,0.25",
                      "+".join(f"cube:{x},{y},{z},0.125" for x, y, z in corners3), 0.09375),
    ]


# benchmark.hpp:56-63: reference iteration counts (grid-independent for these
# cases); a run passes within ±2 of them.
_REFERENCE_COUNTS = {
    ("two_discs", 128, 1e-4): 3, ("two_discs", 256, 1e-4): 3, ("two_discs", 512, 1e-4): 3,
    ("two_discs", 128, 1e-8): 5, ("two_discs", 256, 1e-8): 5, ("two_discs", 512, 1e-8): 5,
    ("two_balls", 128, 1e-4): 6, ("four_squares", 256, 1e-4): 3,
    ("four_squares", 512, 1e-4): 3, ("four_squares", 512, 1e-5): 5,
    ("four_squares", 512, 1e-6): 13, ("eight_cubes", 128, 1e-3): 3,
}


def expected_iterations(name: str, n: int, tol: float) -> Optional[Tuple[int, int]]:
    for (cname, cn, ctol), ref in _REFERENCE_COUNTS.items():
        if cname == name and cn == n and abs(tol - ctol) <= 1e-9 * ctol:
            return max(1, ref - 2), ref + 2
    return None


@dataclasses.dataclass
class BenchmarkRow:
    case_name: str
    n: int
    tolerance: float
    mode: int
    iterations: int
    seconds: float
    dual_value: float
    exact_cost: float
    converged: bool
    expected: Optional[Tuple[int, int]]
    status: str  # "ok", "FAIL", or "n/a" when no reference count exists


def run_benchmark_case(case: BenchmarkCase, n: int, tol: float,
                       mode: int = BACK_AND_FORTH) -> BenchmarkRow:
    """benchmark.hpp:84-124 on the GPU solver."""
    shape = (n, n) if case.dim == 2 else (n, n, n)
    mu = normalize(builtin_density(shape, case.mu_spec))
    nu = normalize(builtin_density(shape, case.nu_spec))
    cfg = SolverConfig(mode=mode, tolerance=-1.0, exact_cost=case.exact_cost, exact_tolerance=tol,
                       max_iterations=1000 if mode == BACK_AND_FORTH else 20000)
    rep = solve(mu, nu, cfg)
    converged = rep.termination == "cost_target_met"
    expected = expected_iterations(case.name, n, tol) if mode == BACK_AND_FORTH else None
    if not converged:
        status = "FAIL"
    elif expected is not None:
        status = "ok" if expected[0] <= rep.iterations <= expected[1] else "FAIL"
    else:
        status = "n/a"
    return BenchmarkRow(case.name, n, tol, mode, rep.iterations, rep.wall_seconds, rep.dual_value,
                        case.exact_cost, converged, expected, status)


def write_benchmark_csv(out: IO[str], rows: List[BenchmarkRow]) -> None:
    """benchmark.hpp:126-147 column layout."""
    out.write("case,n,tolerance,mode,iterations,seconds,dual_value,exact_cost,"
              "expected_lo,expected_hi,status\n")
    for r in rows:
        mode = "bfm" if r.mode == BACK_AND_FORTH else "gradient-ascent"
        lo, hi = (str(r.expected[0]), str(r.expected[1])) if r.expected else ("", "")
        out.write(f"{r.case_name},{r.n},{r.tolerance:g},{mode},{r.iterations},{r.seconds:g},"
                  f"{r.dual_value:.12g},{r.exact_cost:.12g},{lo},{hi},{r.status}\n")
