"""Phase clocks (BFM_CT_STATS=1) of the dyadic c-transform on C3 solver
iterates, separately for the c-concave potential (phi = psi^c as the solver
leaves it) and the generic one (psi after its ascent step)."""
import ctypes as C
import os
import sys

os.environ["BFM_CT_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

mu, nu = synthetic.c3()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
for _ in range(6):
    s.step()
phi, psi = s.phi(), s.psi()
del s
lib = bfm.load_library()
shape = phi.shape
ws = C.c_void_p()
assert lib.bfm_workspace_create(len(shape), (C.c_int * len(shape))(*shape), C.byref(ws)) == 0
lib.bfm_debug_ws_ct_stats.argtypes = [C.c_void_p, C.c_void_p]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
buf = (C.c_ulonglong * 32)()
names = ["load+f~", "local corners", "chunk hulls", "1b/merge tail", "tangents", "resolve"]
for name, a in (("c-concave (phi)", phi), ("generic (psi)", psi)):
    d_in = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_out = torch.empty_like(d_in)
    lib.bfm_ctransform_device(ws, C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()), st)
    torch.cuda.synchronize()
    lib.bfm_debug_ws_ct_stats(ws, buf)
    b0 = list(buf)
    lib.bfm_ctransform_device(ws, C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()), st)
    torch.cuda.synchronize()
    lib.bfm_debug_ws_ct_stats(ws, buf)
    d = [x - y for x, y in zip(list(buf), b0)]
    lines = 2 * shape[0]
    ph = d[8:14]
    mt = sum(d[18:28])
    tot = sum(ph) + mt
    print(f"QG={os.environ.get('BFM_CT_QG', 'default')} {name}: clocks per line {tot / lines:.0f}; "
          + ", ".join(f"{n} {100.0 * x / tot:.1f}%" for n, x in zip(names, ph)) + f", merge levels {100.0 * mt / tot:.1f}%")
    print(f"    flagged {d[1]} walked {d[2]} exact local {d[3]} exact merge {d[4]} merge tests {d[5]} "
          f"kept-convex lines {d[28]} merged lines {d[29]}", flush=True)
