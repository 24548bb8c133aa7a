"""Times the c-transform operator on C3 solver iterates: the generic potential
(phi right after an ascent step is not available from outside, so psi + a
smooth bump stands in) and the c-concave ones (phi and psi as the solver
leaves them). Run once per BFM_CT_QG setting."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

mu, nu = synthetic.c3()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    s.step()
phi, psi = s.phi(), s.psi()
del s
lib = bfm.load_library()
shape = phi.shape
ws = C.c_void_p()
assert lib.bfm_workspace_create(len(shape), (C.c_int * len(shape))(*shape), C.byref(ws)) == 0
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
x = (np.arange(shape[0]) + 0.5) / shape[0]
bump = 1e-3 * np.add.outer(np.sin(7 * x), np.cos(5 * x))
cases = {"phi (c-concave)": phi, "psi (c-concave)": psi, "psi + bump (generic)": psi + bump}
for name, a in cases.items():
    d_in = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_out = torch.empty_like(d_in)
    for _ in range(2):
        assert lib.bfm_ctransform_device(ws, C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()), st) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lib.bfm_ctransform_device(ws, C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()), st)
    e1.record()
    torch.cuda.synchronize()
    print(f"QG={os.environ.get('BFM_CT_QG', 'default')} {name}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
