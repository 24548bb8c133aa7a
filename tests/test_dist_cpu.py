"""Multi-GPU slab decomposition, host logic on CPU: 2 ranks over
torch.distributed/gloo (one process each), the rank-local operators from
tests/dist_cpu_ops.py. Checks that the exchanges (row/column transposes,
halo rows, deposit-record routing, rank-ordered scalar merges) reproduce the
single-process oracle bit for bit (fields) on tiny grids; the GPU version of
the same checks (real sm_100a slab kernels) is tests/test_gpu_dist.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

CASES = {
    "ct2": (12, 10),
    "ct3": (6, 5, 4),
    "pois2": (12, 10),
    "pois3": (6, 8, 4),
    "pf2": (14, 12),
    "pf3": (8, 6, 5),
    "solve2": (10, 12),
}


def _inputs():
    rng = np.random.default_rng(42)
    data = {}
    for k in ("ct2", "ct3"):
        data[k] = rng.uniform(-1, 1, CASES[k])
    for k in ("pois2", "pois3"):
        data[k] = rng.standard_normal(CASES[k])
    for k in ("pf2", "pf3"):
        shp = CASES[k]
        g = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in shp], indexing="ij")
        # strong contraction towards an interior point: deposits cross ranks
        u = sum(0.5 * x * x - c * x for x, c in zip(g, (0.45, 0.6, 0.5)))
        u = u * 0.9 + 0.01 * synthetic.c5_pushforward_potential(shp)
        mu = rng.lognormal(0, 1, shp) * (rng.uniform(0, 1, shp) > 0.2)
        target = rng.uniform(0, 2, shp)
        data[k] = (u, mu, target)
    data["solve2"] = synthetic.c1_like(CASES["solve2"])
    return data


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from paper_1905_12154_b200 import SolverConfig
    from paper_1905_12154_b200 import dist as D
    from dist_cpu_ops import CpuSlabOps

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    comm = D.TorchComm()
    data = _inputs()
    res = {}

    def rows(L, a):
        r0, nr = L.rows(rank)
        return torch.from_numpy(np.ascontiguousarray(a[r0:r0 + nr]).reshape(-1).copy())

    for k in ("ct2", "ct3"):
        L = D.SlabLayout(CASES[k], world)
        x = D.SlabExchange(L, comm)
        ops = CpuSlabOps(L, rank)
        chain, q = ops.ct_cols(x.rows_to_cols(rows(L, data[k])))
        res[k] = ops.ct_rows(x.cols_to_rows(chain), x.cols_to_rows(q)).numpy()
    for k in ("pois2", "pois3"):
        L = D.SlabLayout(CASES[k], world)
        x = D.SlabExchange(L, comm)
        ops = CpuSlabOps(L, rank)
        y = ops.poisson_rows_forward(rows(L, data[k]))
        z = x.cols_to_rows(ops.poisson_cols(x.rows_to_cols(y)))
        res[k] = ops.poisson_rows_inverse(z).numpy()
    for k in ("pf2", "pf3"):
        u, mu, target = data[k]
        L = D.SlabLayout(CASES[k], world)
        x = D.SlabExchange(L, comm)
        ops = CpuSlabOps(L, rank)
        src = rows(L, mu)
        key, w, cm, _ = ops.pf_map(x.halo(rows(L, u)), src)
        recs = x.route_records(key, w, cm, src, None)
        res[k] = ops.pf_gather(*recs, rows(L, target)).numpy()
    L = D.SlabLayout(CASES["solve2"], world)
    mu, nu = data["solve2"]
    r0, nr = L.rows(rank)
    s = D.DistSolver(L, comm, CpuSlabOps(L, rank), mu[r0:r0 + nr], nu[r0:r0 + nr],
                     SolverConfig(tolerance=-1.0, max_iterations=10), mu_full=mu, nu_full=nu)
    for _ in range(2):
        s.step()
    res["solve2_phi"] = s.phi.numpy()
    res["solve2_psi"] = s.psi.numpy()
    res["solve2_dual"] = np.array([t.dual_value for t in s.trace])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    out = tmp_path_factory.mktemp("dist")
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(out)), nprocs=world,
                       start_method="spawn", join=True)
    parts = [dict(np.load(out / f"rank{r}.npz")) for r in range(world)]
    return parts


def _full(parts, key, shape):
    return np.concatenate([p[key] for p in parts]).reshape(shape)


def test_dist_ctransform_gloo(results):
    data = _inputs()
    for k in ("ct2", "ct3"):
        assert O.n_bit_diff(_full(results, k, CASES[k]), O.orc_ctransform(data[k])) == 0, k


def test_dist_poisson_gloo(results):
    data = _inputs()
    for k in ("pois2", "pois3"):
        assert O.n_bit_diff(_full(results, k, CASES[k]), O.orc_solve_neumann(data[k])) == 0, k


def test_dist_pushforward_gloo(results):
    data = _inputs()
    for k in ("pf2", "pf3"):
        u, mu, target = data[k]
        want = target - O.orc_pushforward_density(O.orc_map_from_conjugate(u), mu)
        assert O.n_bit_diff(_full(results, k, CASES[k]), want) == 0, k


def test_dist_solver_gloo(results):
    mu, nu = _inputs()["solve2"]
    phi, psi, duals = O.orc_run_steps(mu, nu, 2)
    shp = CASES["solve2"]
    assert O.n_bit_diff(_full(results, "solve2_phi", shp), phi) == 0
    assert O.n_bit_diff(_full(results, "solve2_psi", shp), psi) == 0
    for r in results:
        np.testing.assert_allclose(r["solve2_dual"], duals, rtol=1e-12, atol=1e-15)


def test_cpp_dist_layout_and_comm_handles():
    """The C++ multi-GPU driver's row partition matches the Python layout, and
    the in-process communicator group can be made without a device (the
    solver itself needs the GPU: tests/test_gpu_dist_cpp.py)."""
    from paper_1905_12154_b200 import dist as D
    from paper_1905_12154_b200 import dist_cpp as DC

    for n0, parts in [(32, 1), (33, 3), (4096, 8), (384, 8), (10, 4)]:
        L = D.SlabLayout((n0, 16), parts)
        assert DC.split_rows(n0, parts) == (L.row0, L.nrows)
    comms = DC.local_group(3)
    assert [c.rank for c in comms] == [0, 1, 2] and all(c.size == 3 for c in comms)
    for c in comms:
        c.close()
