"""Per-pass line statistics of the dyadic c-transform inside a C3 iteration
(BFM_CT_STATS=1 builds the plan with the diagnostic counters): lines on the
convex fast path, the kept-convex path and the merge tree."""
import ctypes as C
import os
import sys

os.environ["BFM_CT_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
mu, nu = getattr(synthetic, name)()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
lib = bfm.load_library()
lib.bfm_debug_ct_stats.argtypes = [C.c_void_p, C.c_void_p]
buf = (C.c_ulonglong * 32)()
prev = [0] * 32
for it in range(6):
    s.step()
    lib.bfm_debug_ct_stats(s._h, buf)
    cur = list(buf)
    d = [c - p for c, p in zip(cur, prev)]
    prev = cur
    print(f"iter {it + 1}: points {d[0]} flagged {d[1]} kept-convex lines {d[28]} merged lines {d[29]}", flush=True)
