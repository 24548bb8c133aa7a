"""Full-length parity at BASELINE.json's configs against the unmodified
reference solver (north_star: "potentials, map and dual value within 1e-9
relative ... and the same iteration count").

The goldens (tests/golden/fullrun_<cfg>.npz) were written by
tests/golden/make_fullrun.py from oracle/_ref (the reference headers compiled
unmodified, solver.hpp:146-368) on the same generator inputs: per iteration the
IterationStats, sigma and SHA-256 of phi/psi bits; then the gauge-fixed report
of run() (finish, solver.hpp:330-349). Here the GPU solver is stepped the same
way and every iteration is compared; the first mismatching iteration is
reported together with the number of differing sampled nodes and their rel-inf
size, so a failure says where the trajectories forked.

Bar: zero differing bits in phi and psi at every iteration, the identical
sigma trace and iteration count, the same termination, a bitwise-equal
gauge-fixed report (phi, psi, every map component) and scalars within 1e-12
relative (the reference's Kahan sums vs our double-double reductions)."""
import hashlib
import os

import numpy as np
import pytest

import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SCALAR_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def close(a, b, rtol=SCALAR_RTOL):
    return abs(a - b) <= rtol * max(1.0, abs(b))


def load(name):
    path = os.path.join(HERE, "golden", f"fullrun_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_fullrun.py {name})")
    return np.load(path)


def sample_report(kind, it, got, want_sample, idx):
    g = got.reshape(-1)[idx]
    bad = int(np.count_nonzero(g.view(np.uint64) != want_sample.view(np.uint64)))
    rel = float(np.max(np.abs(g - want_sample)) / max(1e-300, np.max(np.abs(want_sample))))
    return f"{kind} differs at iteration {it}: {bad}/{idx.size} sampled nodes, rel-inf {rel:.3e}"


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_fullrun_matches_reference(name):
    g = load(name)
    config, n, seed = (int(v) for v in g["generator"])
    mu, nu = synthetic._shared(config, n, seed)
    assert sha(mu) == str(g["mu_sha"]) and sha(nu) == str(g["nu_sha"]), "generator inputs changed"
    steps = int(g["steps"])
    idx = g["sample_index"]
    fields = [str(f) for f in g["stat_fields"]]
    s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=steps))
    prev = 0.0
    for k in range(steps):
        st = s.step()
        phi, psi = s.phi(), s.psi()
        want = g["trace"][k]
        got = [getattr(st, f) for f in fields]
        assert got[0] == want[0]
        for f, a, b in zip(fields[1:], got[1:], want[1:]):
            assert close(a, b), f"{f} at iteration {k + 1}: {a!r} vs reference {b!r}"
        assert st.sigma_first == want[fields.index("sigma_first")], f"sigma fork at iteration {k + 1}"
        assert st.sigma_second == want[fields.index("sigma_second")], f"sigma fork at iteration {k + 1}"
        assert s.sigma() == g["sigma"][k]
        assert sha(phi) == str(g["phi_sha"][k]), sample_report("phi", k + 1, phi, g["phi_sample"][k], idx)
        assert sha(psi) == str(g["psi_sha"][k]), sample_report("psi", k + 1, psi, g["psi_sample"][k], idx)
        if name == "c2" and k + 1 < steps:
            # SURVEY Appendix B stop rule: not crossed before the reference's
            # stopping iteration ...
            assert abs(st.dual_value - prev) >= 1e-6
        prev = st.dual_value
    if name == "c2":  # ... and crossed at it
        assert abs(g["trace"][steps - 1][fields.index("dual_value")] - g["trace"][steps - 2][
            fields.index("dual_value")]) < 1e-6
    rep = s.run()
    it, dual, primal, resid = g["rep_scalars"]
    assert rep.iterations == int(it) == steps
    assert rep.termination == str(g["rep_termination"])
    assert close(rep.dual_value, dual) and close(rep.primal_cost, primal) and close(rep.residual, resid)
    assert sha(rep.phi) == str(g["rep_phi_sha"]), sample_report("report phi", steps, rep.phi,
                                                                g["rep_phi_sample"], idx)
    assert sha(rep.psi) == str(g["rep_psi_sha"]), sample_report("report psi", steps, rep.psi,
                                                                g["rep_psi_sample"], idx)
    for a in range(rep.map.shape[0]):
        assert sha(rep.map[a]) == str(g["rep_map_sha"][a]), sample_report(
            f"map[{a}]", steps, rep.map[a], g["rep_map_sample"][a], idx)
    assert len(rep.trace) == int(g["rep_trace_len"])
