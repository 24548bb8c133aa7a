"""C1/C2 latency path: ms per iteration with graphs / eager, timing on / off."""
import sys
import numpy as np
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c1"
mu, nu = getattr(synthetic, cfgname)()
cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6)
for graphs in (True, False):
    for timing in (False, True):
        s = bfm.Solver(mu, nu, cfg)
        s.set_graphs(graphs)
        for _ in range(5):
            s.step()
        s.time_steps(5)
        s.set_timing(timing)
        ms = s.time_steps(100)
        ops = s.op_times() if timing else {}
        print(f"{cfgname} graphs={graphs} timing={timing}: {ms/100:.4f} ms/iter", 
              {k: round(v[0] / 100, 4) for k, v in ops.items()}, flush=True)
