"""Phase clocks of the dyadic c-transform inside C3 iterations (BFM_CT_STATS=1):
every line's thread 0 adds its clock64 deltas per phase (slots 8..13), per
merge level (18..26) and the merge tail (27); slots 0..5 are the counters
(points, flagged queries, walked corners, exact chunk / merge tests, merge
tests), 28/29 the kept-convex / merged line counts."""
import ctypes as C
import os
import sys

os.environ["BFM_CT_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
mu, nu = getattr(synthetic, name)()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
lib = bfm.load_library()
lib.bfm_debug_ct_stats.argtypes = [C.c_void_p, C.c_void_p]
buf = (C.c_ulonglong * 32)()
prev = [0] * 32
names = ["f~/max", "local corners", "chunk hulls", "1b/merge", "tangents", "resolve"]
for it in range(iters):
    s.step()
    lib.bfm_debug_ct_stats(s._h, buf)
    cur = list(buf)
    d = [c - p for c, p in zip(cur, prev)]
    prev = cur
    tot = sum(d[8:14]) or 1
    print(f"iter {it + 1}: points {d[0]} flagged {d[1]} walked {d[2]} xchunk {d[3]} xmerge {d[4]} "
          f"mergetests {d[5]} kept-convex {d[28]} merged {d[29]}")
    print("   phases (share of thread-0 clocks): "
          + ", ".join(f"{n} {100.0 * d[8 + i] / tot:.1f}%" for i, n in enumerate(names)))
    mt = sum(d[18:28]) or 1
    print("   merge levels (share of merge clocks): "
          + " ".join(f"L{i}:{100.0 * d[18 + i] / mt:.1f}" for i in range(9)) + f" tail:{100.0 * d[27] / mt:.1f}"
          + f"  merge/total {100.0 * mt / tot:.1f}%", flush=True)
    print("   raw phase clocks 8..17: " + " ".join(f"{100.0 * x / (sum(d[8:18]) or 1):.1f}" for x in d[8:18])
          + "  counters 0..7: " + " ".join(str(x) for x in d[0:8]), flush=True)
