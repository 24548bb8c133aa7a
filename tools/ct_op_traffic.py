"""Profiling driver (not a test): the c-transform operator of bench.py's
roofline (C5 potential at 4096^2) — run under ncu for the DRAM bytes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

shape = (4096, 4096)
lib = bfm.load_library()
phi = torch.from_numpy(synthetic.c5_potential(shape)[0]).cuda()
out = torch.empty_like(phi)
ws = C.c_void_p()
assert lib.bfm_workspace_create(2, (C.c_int * 2)(*shape), C.byref(ws)) == 0
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    assert lib.bfm_ctransform_device(ws, C.c_void_p(phi.data_ptr()), C.c_void_p(out.data_ptr()), sp) == 0
torch.cuda.synchronize()
print("ok")
