import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from fractions import Fraction as F
import paper_1905_12154_b200 as bfm
lib = bfm.load_library()
rng = np.random.default_rng(1)
for m in (2, 3, 5, 7):
    t = rng.uniform(-1, 1, (20000, m)) * np.ldexp(1.0, rng.integers(-30, 30, (20000, m)))
    t[::3, 1] = -t[::3, 0] * (1 + 1e-16 * rng.uniform(-1, 1, t[::3, 0].shape))
    out = np.empty(20000)
    assert lib.bfm_debug_round_down(t.ctypes.data_as(C.c_void_p), m, 20000, out.ctypes.data_as(C.c_void_p)) == 0
    bad = 0
    for i in range(2000):
        v = sum(F(x) for x in t[i])
        d = float(v)
        if F(d) > v: d = np.nextafter(d, -np.inf)
        if d == 0: d = 0.0
        if np.float64(d).view(np.int64) != out[i].view(np.int64):
            bad += 1
            if bad < 4: print(m, i, t[i].tolist(), out[i].hex(), float(d).hex())
    print("m", m, "bad", bad)
