"""Multi-GPU slab decomposition (paper_1905_12154_b200/dist.py) on the GPU.

The gpurun box has one B200, so the P ranks run as threads of one process
(LocalComm) on that device: every rank-local kernel is the real sm_100a
bfm_slab_* path and every exchange is the real row/column/record routing;
only the transport differs from NCCL. The bar is the single-GPU result, bit
for bit (fields), and 1e-12 relative for the reduced scalars."""
import numpy as np
import pytest
import torch

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import dist as D
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def _rows(L, r, a):
    r0, nr = L.rows(r)
    return torch.from_numpy(np.ascontiguousarray(a[r0:r0 + nr]).reshape(-1).copy()).cuda()


def _assemble(L, parts):
    return np.concatenate([p.reshape(L.nrows[r], *L.shape[1:]) for r, p in enumerate(parts)], 0)


SHAPES = [(64, 48), (48, 64), (30, 20), (24, 18, 10), (16, 16, 16)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 2, 3])
def test_dist_ctransform_bitwise(shape, P):
    rng = np.random.default_rng(P * 100 + len(shape))
    L = D.SlabLayout(shape, P)
    for kind in range(2):
        phi = rng.uniform(-1, 1, shape) if kind == 0 else synthetic.c5_potential(shape)[0]

        def fn(r, comm, ops):
            x = D.SlabExchange(L, comm)
            cols = x.rows_to_cols(_rows(L, r, phi))
            chain, q = ops.ct_cols(cols)
            out = ops.ct_rows(x.cols_to_rows(chain), x.cols_to_rows(q))
            return out.cpu().numpy()

        got = _assemble(L, D.spmd_local(L, fn))
        assert O.n_bit_diff(got, bfm.ctransform(phi)) == 0, (shape, P, kind)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("P", [1, 2, 3])
def test_dist_poisson_bitwise(shape, P):
    rng = np.random.default_rng(7 + P)
    L = D.SlabLayout(shape, P)
    rhs = rng.standard_normal(shape)

    def fn(r, comm, ops):
        x = D.SlabExchange(L, comm)
        y = ops.poisson_rows_forward(_rows(L, r, rhs))
        z = x.cols_to_rows(ops.poisson_cols(x.rows_to_cols(y)))
        return ops.poisson_rows_inverse(z).cpu().numpy()

    got = _assemble(L, D.spmd_local(L, fn))
    assert O.n_bit_diff(got, bfm.solve_neumann(rhs)) == 0, (shape, P)


def _pf_cases(shape):
    rng = np.random.default_rng(len(shape) * 13 + shape[0])
    u1 = synthetic.c5_pushforward_potential(shape)
    mu = rng.uniform(0, 1, shape) * (rng.uniform(0, 1, shape) > 0.3)
    g = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in shape], indexing="ij")
    # concentrated: everything towards one interior point (heavy targets that
    # receive deposits from every rank)
    u2 = sum(0.5 * x * x - c * x for x, c in zip(g, (0.37, 0.61, 0.5)))
    return [(u1, mu), (u2, rng.lognormal(0, 2, shape))]


@pytest.mark.parametrize("shape", [(64, 48), (30, 20), (16, 12, 10), (40, 40)])
@pytest.mark.parametrize("P", [1, 2, 3])
def test_dist_pushforward_residual_bitwise(shape, P):
    L = D.SlabLayout(shape, P)
    for u, mu in _pf_cases(shape):
        target = np.random.default_rng(3).uniform(0, 2, shape)

        def fn(r, comm, ops):
            x = D.SlabExchange(L, comm)
            src = _rows(L, r, mu)
            key, w, cm, _ = ops.pf_map(x.halo(_rows(L, r, u)), src)
            recs = x.route_records(key, w, cm, src, ops)
            return ops.pf_gather(*recs, _rows(L, r, target)).cpu().numpy()

        got = _assemble(L, D.spmd_local(L, fn))
        want = target - bfm.pushforward_density(bfm.map_from_conjugate(u), mu)
        assert O.n_bit_diff(got, want) == 0, (shape, P)


@pytest.mark.parametrize("shape,P", [((64, 64), 2), ((64, 64), 3), ((48, 40), 4), ((16, 16, 12), 2)])
def test_dist_solver_matches_single_gpu(shape, P):
    if len(shape) == 2:
        mu, nu = synthetic.c1(shape[0]) if shape[0] == shape[1] else synthetic.c1_like(shape)
    else:
        mu, nu = synthetic.c1_like(shape)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=100)
    steps = 4
    single = bfm.Solver(mu, nu, cfg)
    for _ in range(steps):
        single.step()
    single.dual_value()  # the next probe, as run_local(steps=...) leaves it
    res = D.run_local(shape, mu, nu, cfg, parts=P, steps=steps)
    L = D.SlabLayout(shape, P)
    phi = _assemble(L, [s.phi.cpu().numpy() for s, _ in res])
    psi = _assemble(L, [s.psi.cpu().numpy() for s, _ in res])
    assert O.n_bit_diff(phi, single.phi()) == 0
    assert O.n_bit_diff(psi, single.psi()) == 0
    t1 = single.trace()
    t2 = res[0][0].trace
    assert len(t1) == len(t2) == steps
    for a, b in zip(t1, t2):
        for f in ("dual_value", "sigma_first", "sigma_second", "grad_norm_sq_first",
                  "grad_norm_sq_second", "residual"):
            x, y = getattr(a, f), getattr(b, f)
            assert abs(x - y) <= 1e-12 * max(1.0, abs(x)), (f, x, y)
    for s, _ in res[1:]:  # every rank holds the same scalars
        assert [t.dual_value for t in s.trace] == [t.dual_value for t in t2]


def test_dist_run_and_report_matches_single_gpu():
    shape = (48, 48)
    mu, nu = synthetic.c1_like(shape)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=6)
    want = bfm.Solver(mu, nu, cfg).run()
    res = D.run_local(shape, mu, nu, cfg, parts=3)
    rep = res[0][1]
    assert rep.termination == want.termination and rep.iterations == want.iterations
    assert O.n_bit_diff(rep.phi, want.phi) == 0
    assert O.n_bit_diff(rep.psi, want.psi) == 0
    assert O.n_bit_diff(rep.map, want.map) == 0
    assert abs(rep.primal_cost - want.primal_cost) <= 1e-12 * abs(want.primal_cost)
    assert abs(rep.dual_value - want.dual_value) <= 1e-12 * max(1.0, abs(want.dual_value))
