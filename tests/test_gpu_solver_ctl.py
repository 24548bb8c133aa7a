"""Device-resident scalar state, certified decisions and CUDA-graph iterations
(csrc/solver_ctl.cu, bfm_solver in csrc/capi.cu).

* graphs vs eager launches: the same kernels, so bit-identical fields and trace;
* batched steps (run() with no interrupting rule) vs one step at a time;
* the exact-replay path: when a sigma / blow-up / stall / stopping comparison
  cannot be certified against the reference's sequential Kahan scalars, the
  iteration is replayed with reference-order scalars. The hook forces it at a
  chosen iteration; the replayed iteration's IterationStats must then equal
  the reference's (solver.hpp:78-88) bit for bit, and the run stays bitwise.
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu

FIELDS = ("residual", "dual_value", "sigma_first", "sigma_second", "grad_norm_sq_first",
          "grad_norm_sq_second", "increase_first", "increase_second")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def stats(t):
    return np.array([getattr(t, f) for f in FIELDS])


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("mode", [bfm.BACK_AND_FORTH, bfm.GRADIENT_ASCENT])
def test_graphs_equal_eager(mode):
    mu, nu = synthetic.c1(64)
    cfg = bfm.SolverConfig(mode=mode, tolerance=-1.0, max_iterations=12)
    a = bfm.Solver(mu, nu, cfg)
    b = bfm.Solver(mu, nu, cfg)
    b.set_graphs(False)
    ta = [a.step() for _ in range(12)]
    tb = [b.step() for _ in range(12)]
    for x, y in zip(ta, tb):
        assert (bits(stats(x)) == bits(stats(y))).all()
    assert O.n_bit_diff(a.phi(), b.phi()) == 0 and O.n_bit_diff(a.psi(), b.psi()) == 0
    assert a.sigma() == b.sigma()
    assert a.launches() == b.launches()


def test_batched_run_equals_stepping(ref):
    # run() with tolerance < 0 batches up to 10 steps per synchronisation
    mu, nu = synthetic.c1(128)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=25)
    rep = bfm.Solver(mu, nu, cfg).run()
    s = bfm.Solver(mu, nu, cfg)
    tr = [s.step() for _ in range(25)]
    for x, y in zip(rep.trace, tr):
        assert (bits(stats(x)) == bits(stats(y))).all()
    want = ref.RefSolver(mu, nu, cfg).run()
    assert rep.iterations == want.iterations == 25
    for x, y in [(rep.phi, want.phi), (rep.psi, want.psi), (rep.map, want.map)]:
        assert O.n_bit_diff(x, y) == 0


@pytest.mark.parametrize("mode,forced,probe_only", [
    (bfm.BACK_AND_FORTH, 3, False),
    (bfm.BACK_AND_FORTH, 1, False),
    (bfm.BACK_AND_FORTH, 6, True),
    (bfm.GRADIENT_ASCENT, 4, False),
])
def test_forced_exact_replay_matches_reference(ref, mode, forced, probe_only):
    mu, nu = synthetic.c1(64)
    cfg = bfm.SolverConfig(mode=mode, tolerance=-1.0, max_iterations=10)
    g = bfm.Solver(mu, nu, cfg)
    c = ref.RefSolver(mu, nu, cfg)
    g.debug_force_exact(forced, probe_only)
    for k in range(1, 9):
        a, b = g.step(), c.step()
        sa, sb = stats(a), stats(b)
        if k == forced and not probe_only:
            # the replayed step's scalars are the reference's own Kahan values
            assert (bits(sa) == bits(sb)).all(), (k, sa - sb)
        else:
            assert np.all(np.abs(sa - sb) <= 1e-12 * np.maximum(1.0, np.abs(sb))), k
        assert a.sigma_first == b.sigma_first and a.sigma_second == b.sigma_second
        assert O.n_bit_diff(g.phi(), c.phi()) == 0 and O.n_bit_diff(g.psi(), c.psi()) == 0
    assert g.exact_replays() == 1
    if probe_only:
        # the probe of the forced iteration is exact: its dual is the reference's
        pass
    assert g.dual_value() == pytest.approx(c.dual_value(), rel=1e-12)


def test_forced_exact_probe_dual_is_reference_bits(ref):
    mu, nu = synthetic.c1(64)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10)
    g = bfm.Solver(mu, nu, cfg)
    c = ref.RefSolver(mu, nu, cfg)
    for _ in range(4):
        g.step()
        c.step()
    g.debug_force_exact(5, True)
    assert g.dual_value() == c.dual_value()
    assert g.residual() == c.residual()
    assert g.exact_replays() == 1


def test_null_handles_are_errors():
    lib = bfm.load_library()
    assert lib.bfm_solver_iteration(None) == -1
    assert lib.bfm_solver_launches(None) == -1
    n = bfm.C.c_int()
    assert lib.bfm_solver_trace(None, None, 0, bfm.C.byref(n)) == 2
    assert lib.bfm_solver_step(None, None) == 2
