import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_12154_b200 as bfm
rng = np.random.default_rng(0)
for shape in [(3,), (5,), (6,), (7,), (12,), (3, 5), (2, 3, 2), (5, 3), (6, 10)]:
    for kind in range(2):
        phi = rng.uniform(-1, 1, shape)
        if shape == (6, 10) and kind == 1:
            np.save("gpurun_out/crash_phi.npy", phi)
            print("calling", flush=True)
            bfm.ctransform(phi)
            print("ok")
