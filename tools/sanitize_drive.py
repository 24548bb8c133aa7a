"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): c-transforms (dyadic and non-dyadic, 2-D and 3-D), pushforward,
Poisson, a few solver iterations with graphs, power costs, and the C++
multi-GPU driver with two in-process ranks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import dist_cpp as DC  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

for shape in [(64, 48), (64, 64), (12, 10, 8), (16, 16, 16)]:
    phi = synthetic.c5_potential(shape)[0]
    bfm.ctransform(phi)
    u = 0.05 * synthetic.c5_potential(shape)[1]
    mu = synthetic.c1_like(shape)[0]
    bfm.pushforward_density(bfm.map_from_conjugate(u), mu)
    bfm.solve_neumann(u - u.mean())
bfm.ctransform(synthetic.c5_potential((40, 40))[0], exponents=(1.5, 2.5))
mu, nu = synthetic.c1(64)
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=5))
rep = s.run()
s2 = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=3), exponents=(1.5, 3.0))
s2.run()
DC.run_local((32, 24), *synthetic.c1_like((32, 24)), bfm.SolverConfig(tolerance=-1.0, max_iterations=4),
             parts=2, steps=2)
print("sanitize drive ok", rep.iterations, rep.dual_value)
