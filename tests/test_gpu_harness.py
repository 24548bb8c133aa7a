"""Paper cases (benchmark.hpp:27-124) on the GPU solver: the exact-cost
stopping rule reaches the known optimal costs within the reference's
published iteration counts (±2), and — in 2-D, where the reference solver
is quick on the CPU — with exactly the reference's iteration count, dual
value (1e-12) and fields (bitwise)."""
import io

import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import benchmark as B

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


CASES = {c.name: c for c in B.standard_benchmark_cases()}


@pytest.mark.parametrize("name,n,tol", [("two_discs", 128, 1e-4), ("two_discs", 128, 1e-8),
                                        ("two_discs", 256, 1e-4), ("four_squares", 256, 1e-4),
                                        ("eight_cubes", 128, 1e-3), ("two_balls", 128, 1e-4)])
def test_paper_case_status_ok(name, n, tol):
    row = B.run_benchmark_case(CASES[name], n, tol)
    assert row.converged and row.status == "ok", row
    assert abs(row.dual_value - row.exact_cost) <= tol
    out = io.StringIO()
    B.write_benchmark_csv(out, [row])
    assert out.getvalue().splitlines()[1].endswith(",ok")


@pytest.mark.parametrize("name,n,tol", [("two_discs", 128, 1e-8), ("four_squares", 256, 1e-4)])
def test_paper_case_matches_reference(name, n, tol, ref):
    c = CASES[name]
    shape = (n, n)
    mu = bfm.normalize(bfm.builtin_density(shape, c.mu_spec))
    nu = bfm.normalize(bfm.builtin_density(shape, c.nu_spec))
    cfg = bfm.SolverConfig(tolerance=-1.0, exact_cost=c.exact_cost, exact_tolerance=tol,
                           max_iterations=1000)
    got = bfm.Solver(mu, nu, cfg).run()
    want = ref.RefSolver(mu, nu, cfg).run()
    assert got.termination == want.termination == "cost_target_met"
    assert got.iterations == want.iterations
    assert abs(got.dual_value - want.dual_value) <= 1e-12 * max(1.0, abs(want.dual_value))
    assert O.n_bit_diff(got.phi, want.phi) == 0 and O.n_bit_diff(got.psi, want.psi) == 0
