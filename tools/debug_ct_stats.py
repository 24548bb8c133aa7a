import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BFM_CT_STATS"] = "1"
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic
lib = bfm.load_library()
mu, nu = synthetic.c3()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=100))
for it in range(3):
    s.step()
    out = (C.c_ulonglong * 32)()
    lib.bfm_debug_ct_stats(C.c_void_p(s._h.value), out)
    names = ["queries", "nonlone", "sum(R-L)", "edges_checked", "edges_scanned", "scan_len", "near_corner_Mw", "near_corner_Mc"]
    print(it, {n: out[i] for i, n in enumerate(names)}, flush=True); ph=["load","convex","hull","merge","compact","suspect","tangent","certify","flagged","final"]; tot=sum(out[8+i] for i in range(10)); print("  phases %:", {ph[i]: round(100*out[8+i]/max(1,tot),1) for i in range(10)})
