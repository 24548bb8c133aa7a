"""Profiling driver (not a test): C3 4096^2, a couple of BFM iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mu, nu = synthetic.CONFIGS[cfg]()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=100))
for _ in range(iters):
    st = s.step()
    print(st.iteration, st.dual_value, flush=True)
