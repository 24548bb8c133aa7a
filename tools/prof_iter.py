"""Profiling driver: `warm` BFM iterations of a config, then one iteration
(probe + step) between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (tools/launches.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mu, nu = synthetic.CONFIGS[cfg]()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
s.set_graphs(False)  # kernel-by-kernel launches for the profiler
for _ in range(warm):
    s.step()
s.dual_value()
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
import torch  # noqa: E402

torch.cuda.profiler.start()
s.step()
s.dual_value()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one iteration after", warm)
