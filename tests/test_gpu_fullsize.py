"""Full-size checks at BASELINE.json's sizes (C3 4096^2, C4 384^3).

At these sizes the exact CPU oracles take seconds to minutes per operator, so
besides one direct comparison of a full C3 iteration with the reference, the
checks are size-independent properties the operators must satisfy exactly:
the c-transform's Galois identity phi^ccc = phi^c (transforms.hpp; KAT at
test_transforms.cpp:255-283 on small grids), the identity map's pushforward
(test_pushforward.cpp:54-81: rho == mu bit for bit), mass conservation of a
general pushforward, and a Poisson eigenmode (test_poisson.cpp:41-62)."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("shape", [(4096, 4096), (384, 384, 384)])
def test_galois_identity_fullsize(shape):
    phi = synthetic.c5_potential(shape)[0]
    c1 = bfm.ctransform(phi)
    c3 = bfm.ctransform(bfm.ctransform(c1))
    assert O.n_bit_diff(c3, c1) == 0


def test_identity_pushforward_fullsize_bitwise():
    shape = (4096, 4096)
    mu, _ = synthetic.c3()
    disp = bfm.map_from_conjugate(np.zeros(shape))
    assert not disp.any()
    assert O.n_bit_diff(bfm.pushforward_density(disp, mu), mu) == 0


def test_pushforward_mass_fullsize():
    shape = (4096, 4096)
    mu, _ = synthetic.c3()
    u = synthetic.c5_pushforward_potential(shape)
    rho = bfm.pushforward_density(bfm.map_from_conjugate(u), mu)
    m0 = np.sum(mu, dtype=np.float64)
    assert abs(np.sum(rho, dtype=np.float64) - m0) <= 1e-12 * m0
    assert (rho >= 0).all()


def test_poisson_eigenmode_fullsize():
    n = 4096
    x = (np.arange(n) + 0.5) / n
    k0, k1 = 3, 7
    r = np.outer(np.cos(np.pi * k0 * x), np.cos(np.pi * k1 * x))
    lam = (2 - 2 * np.cos(np.pi * k0 / n)) * n * n + (2 - 2 * np.cos(np.pi * k1 / n)) * n * n
    out = bfm.solve_neumann(r)
    assert np.max(np.abs(out - r / lam)) <= 1e-12 * np.max(np.abs(r / lam))


def test_c3_iteration_matches_reference_bitwise(ref):
    # one full BFM iteration (probe + step) at 4096^2 against the unmodified
    # reference solver (about 10 s of CPU)
    mu, nu = synthetic.c3()
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10)
    gpu = bfm.Solver(mu, nu, cfg)
    cpu = ref.RefSolver(mu, nu, cfg)
    a = gpu.step()
    b = cpu.step()
    assert O.n_bit_diff(gpu.phi(), cpu.phi()) == 0
    assert O.n_bit_diff(gpu.psi(), cpu.psi()) == 0
    assert abs(a.dual_value - b.dual_value) <= 1e-12 * max(1.0, abs(b.dual_value))
    assert a.sigma_second == b.sigma_second
