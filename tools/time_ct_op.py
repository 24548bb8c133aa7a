"""Times the c-transform operator (device pointers, CUDA events) on the C5
potential of one grid, on phi and on the c-concave phi^c: time_ct_op.py 4096x4096"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

shape = tuple(int(x) for x in (sys.argv[1].split("x") if len(sys.argv) > 1 else ["4096", "4096"]))
lib = bfm.load_library()
phi = torch.from_numpy(synthetic.c5_potential(shape)[0]).cuda()
psi = torch.empty_like(phi)
phi2 = torch.empty_like(phi)
ws = C.c_void_p()
assert lib.bfm_workspace_create(len(shape), (C.c_int * len(shape))(*shape), C.byref(ws)) == 0
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def run(a, b):
    assert lib.bfm_ctransform_device(ws, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), s) == 0


for _ in range(2):
    run(phi, psi)
    run(psi, phi2)
torch.cuda.synchronize()
res = []
for a, b in ((phi, psi), (psi, phi2)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run(a, b)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 5)
print(f"{'x'.join(map(str, shape))}: phi -> psi {res[0]:.3f} ms, psi -> phi'' {res[1]:.3f} ms "
      f"(QG={os.environ.get('BFM_CT_QG', 'default')}, T0={os.environ.get('BFM_CT_T0', 'default')})", flush=True)
