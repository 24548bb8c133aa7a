"""A/B of the c-transform kernels inside a C3/C2/C1 iteration (per-op CUDA
events) — run twice, with BFM_CT_HULL=1 (exact-hull kernel) and without
(divide-and-conquer kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mu, nu = getattr(synthetic, name)()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
for _ in range(3):
    s.step()
s.set_timing(True)
ms = s.time_steps(steps)
ops = s.op_times()
print(f"{name} hull={os.environ.get('BFM_CT_HULL', '0')} B={os.environ.get('BFM_DC_B', '-')} "
      f"lpc={os.environ.get('BFM_DC_LPC', '-')}: {ms / steps:.3f} ms/iter; ctransform "
      f"{ops['ctransform'][0] / ops['ctransform'][1]:.4f} ms/call; per iter "
      + " ".join(f"{k} {v[0] / steps:.3f}" for k, v in ops.items()) + f"; dual {s.dual_value()!r}", flush=True)
