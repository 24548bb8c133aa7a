"""The C++ multi-GPU solver (csrc/dist_solver.cu, bfm_dist_solver_*): the
reference's Solver loop (solver.hpp:146-368) over an axis-0 slab
decomposition with the library's own pack/unpack kernels and exchanges.

On the single test GPU, P ranks run as threads with the in-process
communicator (host-synchronised exchanges: no kernel waits on another rank);
the NCCL communicator runs at P = 1. Every result must equal the single-GPU
solver bit for bit (fields, sigma trace, report)."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import dist_cpp as DC
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def single(shape, mu, nu, cfg, steps):
    s = bfm.Solver(mu, nu, cfg)
    tr = [s.step() for _ in range(steps)]
    return s, tr


@pytest.mark.parametrize("shape,parts", [((32, 24), 1), ((32, 24), 2), ((33, 20), 3), ((16, 12, 10), 2),
                                         ((24, 16, 8), 4), ((64, 64), 4)])
def test_cpp_dist_steps_bitwise(shape, parts):
    mu, nu = synthetic.c1_like(shape)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=100)
    ref, tr = single(shape, mu, nu, cfg, 4)
    res = DC.run_local(shape, mu, nu, cfg, parts=parts, steps=4)
    phi = np.concatenate([r[1] for r in res])
    psi = np.concatenate([r[2] for r in res])
    assert O.n_bit_diff(phi, ref.phi()) == 0 and O.n_bit_diff(psi, ref.psi()) == 0
    for r in res:
        for a, b in zip(r[0], tr):
            assert a.sigma_first == b.sigma_first and a.sigma_second == b.sigma_second
            assert abs(a.dual_value - b.dual_value) <= 1e-12 * max(1.0, abs(b.dual_value))


@pytest.mark.parametrize("mode", [bfm.BACK_AND_FORTH, bfm.GRADIENT_ASCENT])
def test_cpp_dist_run_report_bitwise(mode):
    shape = (40, 36)
    mu, nu = synthetic.c1_like(shape)
    cfg = bfm.SolverConfig(mode=mode, tolerance=-1.0, max_iterations=6)
    want = bfm.Solver(mu, nu, cfg).run()
    res = DC.run_local(shape, mu, nu, cfg, parts=3, report=True)
    for _, _, _, rep in res:  # every rank holds the full report
        assert rep.iterations == want.iterations and rep.termination == want.termination
        for x, y in [(rep.phi, want.phi), (rep.psi, want.psi), (rep.map, want.map)]:
            assert O.n_bit_diff(x, y) == 0
        assert abs(rep.primal_cost - want.primal_cost) <= 1e-12 * abs(want.primal_cost)
        assert abs(rep.dual_value - want.dual_value) <= 1e-12 * abs(want.dual_value)


def test_cpp_dist_nccl_single_rank():
    """The NCCL communicator end to end at P = 1 (self send/recv)."""
    try:
        uid = DC.nccl_unique_id()
    except bfm.Error as e:
        pytest.skip(f"NCCL unavailable: {e}")
    shape = (32, 32)
    mu, nu = synthetic.c1_like(shape)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=3)
    comm = DC.nccl_comm(uid, 0, 1)
    s = DC.CppDistSolver(comm, shape, mu, nu, cfg)
    rep = s.run()
    want = bfm.Solver(mu, nu, cfg).run()
    assert O.n_bit_diff(rep.phi, want.phi) == 0 and O.n_bit_diff(rep.map, want.map) == 0
    s.close()
    comm.close()
