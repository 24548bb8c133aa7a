"""Profiling driver (not a test): where the end-to-end time of bench.py's e2e
leg goes (solver creation, K steps, field readback)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

mu, nu = synthetic.c3()
cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6)
s0 = bfm.Solver(mu, nu, cfg)
s0.step()
del s0
pin_mu = torch.from_numpy(mu).pin_memory().numpy()
pin_nu = torch.from_numpy(nu).pin_memory().numpy()
import ctypes as C  # noqa: E402
lib = bfm.load_library()
c = cfg._c()
for rep in range(2):
    t0 = time.perf_counter()
    rc = lib.bfm_validate_inputs(2, (C.c_int * 2)(4096, 4096), pin_mu.ctypes.data_as(C.c_void_p),
                                 pin_nu.ctypes.data_as(C.c_void_p), C.byref(c))
    print(f"host validation {1e3*(time.perf_counter()-t0):.1f} ms rc={rc}", flush=True)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = bfm.Solver(pin_mu, pin_nu, cfg)
    t1 = time.perf_counter()
    for _ in range(5):
        s.step()
    s.dual_value()
    t2 = time.perf_counter()
    a = s.phi()
    b = s.psi()
    t3 = time.perf_counter()
    del s
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  5 steps {1e3*(t2-t1):.1f} ms  readback {1e3*(t3-t2):.1f} ms  destroy {1e3*(t4-t3):.1f} ms", flush=True)
