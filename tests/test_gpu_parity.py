"""GPU parity: the sm_100a kernels (through the C ABI) against the reference.

Bar: every field-producing operator is BITWISE equal
to the reference built with the shared DCT (oracle/_ref): c-transform (exactly
rounded), map, pushforward, Poisson. Scalars from reductions (pair values,
gn) feed only decisions and are compared with rel tol 1e-12 (they are not
sequential Kahan sums on the GPU). Goldens in tests/golden/ come from the
unmodified reference (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


# ------------------------------------------------------------- c-transform
def test_ctransform_goldens_bitwise():
    g = load("ctransform.npz")
    for k in [k for k in g if k.startswith("ct_in_")]:
        name = k[len("ct_in_"):]
        out = bfm.ctransform(g[k])
        assert O.n_bit_diff(out, g["ct_out_" + name]) == 0, name


@pytest.mark.parametrize("shape", [(1024,), (256, 256), (512, 512), (384, 96), (96, 384), (48, 48, 48),
                                   (32, 64, 16), (24, 24, 24), (2, 2), (3, 5), (2, 3, 2)])
def test_ctransform_random_vs_restatement_or_reference(shape, ref):
    rng = np.random.default_rng(sum(shape))
    for kind in range(3):
        if kind == 0:
            phi = rng.uniform(-1, 1, shape)
        elif kind == 1:
            phi = synthetic.c5_potential(shape)[0]
        else:
            g = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in shape], indexing="ij")
            phi = sum(0.5 * x * x for x in g) + 1e-13 * rng.standard_normal(shape)
        out = bfm.ctransform(phi)
        want = ref.ref_ctransform(phi)
        assert O.n_bit_diff(out, want) == 0, (shape, kind)


@pytest.mark.parametrize("shape", [(2048, 2048), (4096, 512), (128, 128, 128)])
def test_ctransform_large_vs_reference(shape, ref):
    phi = synthetic.c5_potential(shape)[0]
    out = bfm.ctransform(phi)
    want = ref.ref_ctransform(phi)
    assert O.n_bit_diff(out, want) == 0


@pytest.mark.parametrize("shape", [(64,), (24, 24), (8, 8, 8), (33, 17)])
def test_galois_laws_exact(shape):
    # test_transforms.cpp:255-283: phi <= phi^cc pointwise, phi^ccc == phi^c bitwise
    rng = np.random.default_rng(149)
    for _ in range(20):
        phi = rng.uniform(0, 1, shape)
        c = bfm.ctransform(phi)
        cc = bfm.ctransform(c)
        assert np.all(phi <= cc)
        assert O.n_bit_diff(bfm.ctransform(cc), c) == 0


def test_ctransform_c5_4096_matches_reference(ref):
    phi = synthetic.c5_potential((4096, 4096))[0]
    out = bfm.ctransform(phi)
    want = ref.ref_ctransform(phi)
    assert O.n_bit_diff(out, want) == 0


# ------------------------------------------------------------- Poisson
def test_poisson_goldens_bitwise():
    g = load("poisson.npz")
    for k in [k for k in g if k.startswith("pois_in_")]:
        key = k[len("pois_in_"):]
        out = bfm.solve_neumann(g[k])
        assert O.n_bit_diff(out, g["pois_out_" + key]) == 0, key


@pytest.mark.parametrize("shape", [(4096, 64), (64, 4096), (1024, 1024), (384, 48), (48, 384, 8), (96, 96, 96),
                                   (30, 50), (130,)])
def test_poisson_vs_restatement(shape):
    r = np.random.default_rng(11).uniform(-1, 1, shape)
    assert O.n_bit_diff(bfm.solve_neumann(r), O.orc_solve_neumann(r)) == 0


# ------------------------------------------------------------- pushforward
def test_pushforward_goldens_bitwise():
    g = load("pushforward.npz")
    for k in [k for k in g if k.startswith("pf_u_")]:
        key = k[len("pf_u_"):]
        disp = bfm.map_from_conjugate(g[k])
        assert O.n_bit_diff(disp, g["pf_disp_" + key]) == 0, key
        rho = bfm.pushforward_density(disp, g["pf_mu_" + key])
        assert O.n_bit_diff(rho, g["pf_rho_" + key]) == 0, key
        half = bfm.displacement_interpolant(disp, g["pf_mu_" + key], 0.5)
        assert O.n_bit_diff(half, g["pf_half_" + key]) == 0, key
        d2 = bfm.map_from_conjugate(g["pf_u2_" + key])
        assert O.n_bit_diff(d2, g["pf_disp2_" + key]) == 0, key
        assert O.n_bit_diff(bfm.pushforward_density(d2, g["pf_mu_" + key]), g["pf_rho2_" + key]) == 0


@pytest.mark.parametrize("shape", [(512, 512), (64, 64, 64), (1000, 7)])
def test_pushforward_vs_restatement(shape):
    rng = np.random.default_rng(5)
    u = synthetic.c5_pushforward_potential(shape)
    mu = rng.uniform(0, 1, shape) * (rng.uniform(0, 1, shape) > 0.4)
    disp = bfm.map_from_conjugate(u)
    assert O.n_bit_diff(disp, O.orc_map_from_conjugate(u)) == 0
    assert O.n_bit_diff(bfm.pushforward_density(disp, mu), O.orc_pushforward_density(disp, mu)) == 0


def test_pushforward_concentrated_map():
    # many sources into few cells: exercises large sorted buckets
    n = 256
    x = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(x, x, indexing="ij")
    u = 0.5 * (X * X + Y * Y) - 0.5 * X - 0.5 * Y  # grad u = x - 0.5 -> everything to the centre
    mu = np.ones((n, n))
    disp = bfm.map_from_conjugate(u)
    rho = bfm.pushforward_density(disp, mu)
    assert O.n_bit_diff(rho, O.orc_pushforward_density(disp, mu)) == 0


@pytest.mark.parametrize("n", [40, 128, 300])
def test_pushforward_concentrated_random_mass(n):
    # medium (K <= 2048), heavy with shared-memory ranks, heavy with global ranks
    rng = np.random.default_rng(n)
    x = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(x, x, indexing="ij")
    u = 0.5 * (X * X + Y * Y) - 0.31 * X - 0.67 * Y
    mu = rng.lognormal(0.0, 2.0, (n, n)) * (rng.uniform(0, 1, (n, n)) > 0.1)
    disp = bfm.map_from_conjugate(u)
    rho = bfm.pushforward_density(disp, mu)
    assert O.n_bit_diff(rho, O.orc_pushforward_density(disp, mu)) == 0


def _seq_fold(w):
    r = 0.0
    for x in w.tolist():
        r = r + x
    return r


def _fold_cases():
    rng = np.random.default_rng(11)
    cases = []
    for K in [0, 1, 2, 31, 32, 33, 255, 256, 257, 4095, 4096, 4097, 20000]:
        cases.append(rng.lognormal(0.0, 3.0, K))
    cases.append(np.zeros(5000))
    w = rng.uniform(0, 1, 9000)
    w[:3000] = 0.0
    w[rng.uniform(0, 1, 9000) < 0.3] = 0.0
    cases.append(w)
    # ties: half-ulp and odd multiples of half-ulps around 1.0 (round half to even)
    ulp = 2.0 ** -52
    t = rng.integers(0, 4, 6000) * (ulp / 2)
    t[0] = 1.0
    cases.append(t)
    t2 = rng.integers(0, 8, 6000) * (ulp / 4) + (rng.uniform(0, 1, 6000) < 0.5) * ulp * 3.5
    t2[0] = 1.0 + 3 * ulp
    cases.append(t2)
    cases.append(2.0 ** np.arange(0, 700, 0.5))                   # a binade crossing per step
    cases.append(np.concatenate([[1.0], np.full(5000, 2.0 ** -53)]))  # ties that never round up
    cases.append(np.concatenate([[1.0 + ulp], np.full(5000, 2.0 ** -53)]))  # ties that round up
    cases.append(rng.uniform(0, 1, 3000) * 1e-310)                # subnormal weights
    cases.append(np.concatenate([rng.uniform(0, 1, 100), [np.inf], rng.uniform(0, 1, 100)]))
    cases.append(np.concatenate([rng.uniform(0, 1, 100), [np.nan], rng.uniform(0, 1, 100)]))
    cases.append(rng.uniform(-1, 1, 3000))                        # negative weights (not produced, still exact)
    cases.append(rng.uniform(0, 1, 5000) * 2.0 ** rng.integers(-60, 60, 5000))
    return cases


@pytest.mark.parametrize("mode", [0, 1])
def test_exact_fold_matches_sequential(mode):
    import ctypes as C
    lib = bfm.load_library()
    cases = _fold_cases()
    off = np.zeros(len(cases) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(c) for c in cases])
    w = np.ascontiguousarray(np.concatenate(cases).astype(np.float64)) if off[-1] else np.zeros(1)
    out = np.empty(len(cases))
    rc = lib.bfm_debug_fold(w.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p),
                            C.c_int(len(cases)), C.c_int(mode), out.ctypes.data_as(C.c_void_p))
    assert rc == 0, lib.bfm_last_error()
    for i, c in enumerate(cases):
        want = _seq_fold(c)
        got = float(out[i])
        same = (np.isnan(want) and np.isnan(got)) or np.float64(want).view(np.int64) == np.float64(got).view(np.int64)
        assert same, (i, len(c), want.hex() if not np.isnan(want) else "nan", got.hex() if not np.isnan(got) else "nan")


def test_pushforward_kats():
    # test_pushforward.cpp:104-116 fractional split; :137-150 boundary deposits
    mu = np.zeros(8)
    mu[2] = 8.0
    disp = np.zeros((1, 8))
    disp[0, 2] = 0.7 * (1.0 / 8)
    rho = bfm.pushforward_density(disp, mu)
    assert abs(rho[2] - 8 * 0.3) < 1e-13 and abs(rho[3] - 8 * 0.7) < 1e-13
    mu = np.zeros(8)
    mu[1] = mu[6] = 4.0
    disp = np.zeros((1, 8))
    disp[0, 1] = 0.0 - (1.5 / 8)
    disp[0, 6] = 1.0 - (6.5 / 8)
    rho = bfm.pushforward_density(disp, mu)
    assert rho[0] == 4.0 and rho[7] == 4.0


# ------------------------------------------------------------- solver
def _scal(rep):
    return np.array([rep.iterations, rep.dual_value, rep.primal_cost, rep.residual])


@pytest.mark.parametrize("case,cfg", [
    ("c1_64", bfm.SolverConfig(tolerance=-1.0, max_iterations=8)),
    ("discs", bfm.SolverConfig(tolerance=-1.0, max_iterations=40, exact_cost=0.25, exact_tolerance=1e-4)),
    ("balls", bfm.SolverConfig(tolerance=-1.0, max_iterations=4)),
])
def test_solver_goldens(case, cfg):
    g = load("solver.npz")
    rep = bfm.Solver(g[case + "_mu"], g[case + "_nu"], cfg).run()
    want = g[case + "_scalars"]
    assert rep.iterations == int(want[0])
    assert abs(rep.dual_value - want[1]) <= 1e-12 * max(1.0, abs(want[1]))
    assert abs(rep.primal_cost - want[2]) <= 1e-12 * max(1.0, abs(want[2]))
    assert O.n_bit_diff(rep.phi, g[case + "_phi"]) == 0
    assert O.n_bit_diff(rep.psi, g[case + "_psi"]) == 0
    assert O.n_bit_diff(rep.map, g[case + "_map"]) == 0


def test_solver_c1_full_vs_reference(ref):
    """C1: 256^2, 100 iterations, tolerance disabled (BASELINE configs[0])."""
    mu, nu = synthetic.c1()
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=100)
    a = bfm.Solver(mu, nu, cfg).run()
    b = ref.RefSolver(mu, nu, cfg).run()
    assert a.iterations == b.iterations == 100 or a.termination == b.termination
    assert a.termination == b.termination
    for x, y in [(a.phi, b.phi), (a.psi, b.psi), (a.map, b.map)]:
        assert O.n_bit_diff(x, y) == 0
    ta = np.array([t.dual_value for t in a.trace])
    tb = np.array([t.dual_value for t in b.trace])
    assert np.abs(ta - tb).max() <= 1e-12 * np.abs(tb).max()


def test_solver_deterministic():
    mu, nu = synthetic.c1(64)
    cfg = bfm.SolverConfig(tolerance=1e-5, max_iterations=30)
    a = bfm.Solver(mu, nu, cfg).run()
    b = bfm.Solver(mu, nu, cfg).run()
    assert a.iterations == b.iterations and a.dual_value == b.dual_value
    assert O.n_bit_diff(a.phi, b.phi) == 0


def test_identical_marginals_terminate_immediately():
    # test_solver.cpp:57-70
    x = (np.arange(32) + 0.5) / 32
    X, Y = np.meshgrid(x, x, indexing="ij")
    raw = ((X - 0.5) ** 2 + (Y - 0.5) ** 2 <= 0.04).astype(float)
    mu = raw / (raw.sum() / 1024)
    for mode in (bfm.BACK_AND_FORTH, bfm.GRADIENT_ASCENT):
        rep = bfm.solve(mu, mu, bfm.SolverConfig(mode=mode, tolerance=1e-4))
        assert rep.termination == "tolerance_met" and rep.iterations == 0
        assert rep.residual == 0.0 and rep.dual_value == 0.0


def test_gradient_ascent_mode_matches_reference(ref):
    g = load("solver.npz")
    cfg = bfm.SolverConfig(mode=bfm.GRADIENT_ASCENT, tolerance=-1.0, max_iterations=10)
    a = bfm.Solver(g["discs_mu"], g["discs_nu"], cfg).run()
    b = ref.RefSolver(g["discs_mu"], g["discs_nu"], cfg).run()
    assert O.n_bit_diff(a.phi, b.phi) == 0 and O.n_bit_diff(a.psi, b.psi) == 0


@pytest.mark.parametrize("driver", ["facade_drive", "workspace_drive"])
def test_cpp_facade_driver_runs_on_gpu(tmp_path, driver):
    """Drivers written against the reference's C++ API (solver, operators,
    TransformWorkspace) compile unchanged against include/bfm_b200/bfm.hpp and
    pass the reference's own checks on the GPU."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / driver
    libdir = os.path.join(root, "paper_1905_12154_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(root, "include"),
                        os.path.join(root, "tests", "cxx", driver + ".cpp"), "-L" + libdir,
                        "-l:libbfm_b200.so", "-Wl,-rpath," + libdir, "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr


@pytest.mark.parametrize("shape", [(512, 512), (40, 48, 56)])
def test_pushforward_tier_boundaries(shape):
    # blocks of consecutive sources sent to one interior point each: its 2^d
    # corner targets receive exactly K deposits, K straddling every gather
    # tier boundary (one thread / warp merge / CTA merge / warp fold / exact
    # parallel fold); the other sources stay put
    rng = np.random.default_rng(sum(shape))
    d = len(shape)
    N = int(np.prod(shape))
    sizes = [48, 49, 512, 513, 4096, 4097, 16384, 16385]
    if N < 2 * sum(sizes):
        sizes = [48, 49, 512, 513, 4096, 4097]
    coords = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in shape], indexing="ij")
    disp = [np.zeros(shape) for _ in range(d)]
    flat = [x.reshape(-1) for x in disp]
    src = [c.reshape(-1) for c in coords]
    start = 0
    for b, K in enumerate(sizes):
        tgt = rng.uniform(0.1, 0.9, d)
        for a in range(d):
            flat[a][start:start + K] = tgt[a] - src[a][start:start + K]
        start += K + 1000
    mu = rng.lognormal(0.0, 1.5, shape)
    got = bfm.pushforward_density(np.stack(disp), mu)
    want = O.orc_pushforward_density(np.stack(disp), mu)
    assert O.n_bit_diff(got, want) == 0


def test_solver_c2_until_dual_gap_vs_reference(ref):
    """C2 (BASELINE configs[1]): 1024^2, run until |dual_n - dual_(n-1)| < 1e-6
    (capped at 120 steps here). Both solvers step in
    lockstep: the same stopping iteration, bitwise-equal potentials there,
    duals within 1e-12 relative throughout."""
    mu, nu = synthetic.c2()
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6)
    a = bfm.Solver(mu, nu, cfg)
    b = ref.RefSolver(mu, nu, cfg)
    prev_a = prev_b = None
    stop_a = stop_b = None
    for it in range(1, 121):
        da = a.step().dual_value
        db = b.step().dual_value
        assert abs(da - db) <= 1e-12 * max(1.0, abs(db)), it
        if stop_a is None and prev_a is not None and abs(da - prev_a) < 1e-6:
            stop_a = it
        if stop_b is None and prev_b is not None and abs(db - prev_b) < 1e-6:
            stop_b = it
        prev_a, prev_b = da, db
        if stop_a is not None or stop_b is not None:
            break
    assert stop_a == stop_b and stop_a is not None
    print(f"C2: |dual gap| < 1e-6 at iteration {stop_a} (dual {prev_a!r})")
    assert O.n_bit_diff(a.phi(), b.phi()) == 0 and O.n_bit_diff(a.psi(), b.psi()) == 0
