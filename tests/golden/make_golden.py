"""Generates tests/golden/*.npz from the UNMODIFIED reference
(oracle/_ref/libbfmref.so = /root/reference/proj/include/bfm + FFTW shim).

Run in the build container (needs oracle/_ref built):
    python tests/golden/make_golden.py
The fixtures are small (< 2 MB total) and committed; tests compare the
restatement oracle and the B200 kernels against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402
from paper_1905_12154_b200 import SolverConfig, synthetic  # noqa: E402


def ct_inputs():
    rng = np.random.default_rng(20261020)
    cases = {}
    cases["1d_n40_rand"] = rng.uniform(-1, 1, 40)
    cases["2d_24x17_rand"] = rng.uniform(-1, 1, (24, 17))
    cases["3d_6x5x7_rand"] = rng.uniform(-1, 1, (6, 5, 7))
    cases["2d_64x64_c5"] = synthetic.c5_potential((64, 64))[0]
    cases["3d_12x12x12_c5"] = synthetic.c5_potential((12, 12, 12))[0]
    cases["2d_48x48_c5"] = synthetic.c5_potential((48, 48))[0]
    cases["3d_12x10x8_c5"] = synthetic.c5_potential((12, 10, 8))[0]
    cases["2d_64x64_zero"] = np.zeros((64, 64))
    g = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in (32, 32)], indexing="ij")
    cases["2d_32x32_quadratic"] = 0.5 * (g[0] ** 2 + g[1] ** 2)
    cases["2d_32x32_quadnoise"] = cases["2d_32x32_quadratic"] + 1e-12 * rng.standard_normal((32, 32))
    sp = np.zeros((16, 16))
    sp[5, 9] = 1.0
    cases["2d_16x16_spike"] = sp
    g = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in (96, 40)], indexing="ij")
    cases["2d_96x40_affine"] = 0.125 * g[0] + 0.1 * g[1]
    cases["2d_128x96_tiny"] = rng.uniform(0, 1, (128, 96)) * 1e-3
    return cases


def main():
    if O.ref_lib() is None:
        raise SystemExit("oracle/_ref not built")
    out = {}
    for name, phi in ct_inputs().items():
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out["ct_in_" + name] = phi
        out["ct_out_" + name] = O.ref_ctransform(phi)
    np.savez_compressed(os.path.join(HERE, "ctransform.npz"), **out)

    rng = np.random.default_rng(7)
    out = {}
    for shape in [(64,), (384,), (2, 2), (32, 16), (17, 29), (48, 48), (24, 48), (12, 10, 8),
                  (6, 9, 11), (16, 16, 16), (8, 12, 6)]:
        key = "x".join(map(str, shape))
        r = rng.uniform(-1, 1, shape)
        out["pois_in_" + key] = r
        out["pois_out_" + key] = O.ref_solve_neumann(r)
    np.savez_compressed(os.path.join(HERE, "poisson.npz"), **out)

    out = {}
    for shape in [(32, 32), (24, 20), (12, 12, 12), (40,)]:
        key = "x".join(map(str, shape))
        u = synthetic.c5_pushforward_potential(shape)
        mu = synthetic._normalize(1.0 + rng.uniform(0, 1, shape) * (rng.uniform(0, 1, shape) > 0.3))
        disp = O.ref_map_from_conjugate(u)
        out["pf_u_" + key] = u
        out["pf_mu_" + key] = mu
        out["pf_disp_" + key] = disp
        out["pf_rho_" + key] = O.ref_pushforward_density(disp, mu)
        out["pf_half_" + key] = O.ref_displacement_interpolant(disp, mu, 0.5)
        # a far-moving steep potential (cap + clamp) on the same grid
        g = np.meshgrid(*[(np.arange(n) + 0.5) / n for n in shape], indexing="ij")
        u2 = 0.7 * sum(gg * gg for gg in g) - 0.9 * g[0]
        out["pf_u2_" + key] = u2
        d2 = O.ref_map_from_conjugate(u2)
        out["pf_disp2_" + key] = d2
        out["pf_rho2_" + key] = O.ref_pushforward_density(d2, mu)
    np.savez_compressed(os.path.join(HERE, "pushforward.npz"), **out)

    out = {}
    # C1-like at 64^2: fixed 8 iterations
    mu, nu = synthetic.c1(64)
    cfg = SolverConfig(tolerance=-1.0, max_iterations=8)
    s = O.RefSolver(mu, nu, cfg)
    rep = s.run()
    out["c1_64_mu"], out["c1_64_nu"] = mu, nu
    out["c1_64_phi"], out["c1_64_psi"], out["c1_64_map"] = rep.phi, rep.psi, rep.map
    out["c1_64_trace"] = np.array([[getattr(t, f) for f in
                                    ("residual", "dual_value", "sigma_first", "sigma_second",
                                     "grad_norm_sq_first", "grad_norm_sq_second",
                                     "increase_first", "increase_second")] for t in rep.trace])
    out["c1_64_scalars"] = np.array([rep.iterations, rep.dual_value, rep.primal_cost, rep.residual])
    # two discs 64^2 with the exact-cost stop (test_solver.cpp:98-124)
    d1 = O.ref_builtin((64, 64), "disc:0.25,0.25,0.125")
    d2 = O.ref_builtin((64, 64), "disc:0.75,0.75,0.125")
    mu2, nu2 = synthetic._normalize(d1), synthetic._normalize(d2)
    cfg = SolverConfig(tolerance=-1.0, max_iterations=40, exact_cost=0.25, exact_tolerance=1e-4)
    rep = O.RefSolver(mu2, nu2, cfg).run()
    out["discs_mu"], out["discs_nu"] = mu2, nu2
    out["discs_phi"], out["discs_psi"], out["discs_map"] = rep.phi, rep.psi, rep.map
    out["discs_scalars"] = np.array([rep.iterations, rep.dual_value, rep.primal_cost, rep.residual])
    # 3D balls 16^3, 4 iterations
    b1 = O.ref_builtin((16, 16, 16), "ball:0.3,0.3,0.3,0.2")
    b2 = O.ref_builtin((16, 16, 16), "ball:0.65,0.6,0.7,0.25")
    mu3, nu3 = synthetic._normalize(b1), synthetic._normalize(b2)
    cfg = SolverConfig(tolerance=-1.0, max_iterations=4)
    rep = O.RefSolver(mu3, nu3, cfg).run()
    out["balls_mu"], out["balls_nu"] = mu3, nu3
    out["balls_phi"], out["balls_psi"], out["balls_map"] = rep.phi, rep.psi, rep.map
    out["balls_scalars"] = np.array([rep.iterations, rep.dual_value, rep.primal_cost, rep.residual])
    np.savez_compressed(os.path.join(HERE, "solver.npz"), **out)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
