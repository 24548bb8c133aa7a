"""Profiling driver: the c-transform operator on C5 phi at 4096^2 (the bench's roofline case)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

shape = tuple(int(x) for x in (sys.argv[1].split("x") if len(sys.argv) > 1 else ["4096", "4096"]))
lib = bfm.load_library()
phi = torch.from_numpy(synthetic.c5_potential(shape)[0]).cuda()
out = torch.empty_like(phi)
ws = C.c_void_p()
assert lib.bfm_workspace_create(len(shape), (C.c_int * len(shape))(*shape), C.byref(ws)) == 0
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    assert lib.bfm_ctransform_device(ws, C.c_void_p(phi.data_ptr()), C.c_void_p(out.data_ptr()), s) == 0
torch.cuda.synchronize()
print("ok", float(out.sum()))
