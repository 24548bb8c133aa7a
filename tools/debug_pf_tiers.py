"""Diagnostic (not a test): gather-tier target counts of each pushforward
half step (solver.hpp:245-260) over a few BFM iterations."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
mu, nu = synthetic.CONFIGS[cfg]()
lib = bfm.load_library()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=100))
for it in range(5):
    s.step()
    out = (C.c_int * 3)()
    lib.bfm_debug_pf_tiers(C.c_void_p(s._h.value), out)
    print(it, "warp tier", out[0], "CTA tier", out[1], "huge", out[2], flush=True)
