"""Diagnostics (not a test): c-transform per-phase clocks and query statistics
in the C3 solver (BFM_CT_STATS=1) and on the C5 operator."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BFM_CT_STATS"] = "1"
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = bfm.load_library()
names = ["queries", "flagged", "walk", "exact_chunk", "exact_merge", "merge_tests", "-", "-"]
ph = ["load", "convex", "hull", "merge", "compact", "suspect", "tangent", "certify", "flagged", "final"]
if os.environ.get("BFM_DY", "1") == "1":  # dyadic exact-hull kernel phase slots
    ph = ["load+max", "convex", "hull", "merge", "tangent", "resolve", "-", "-", "-", "-"]
if cfg == "c5":  # the C5 operator on a 4096^2 potential
    import torch
    phi = torch.from_numpy(synthetic.c5_potential((4096, 4096))[0]).cuda()
    out = torch.empty_like(phi)
    ws = C.c_void_p()
    assert lib.bfm_workspace_create(2, (C.c_int * 2)(4096, 4096), C.byref(ws)) == 0
    assert lib.bfm_ctransform_device(ws, C.c_void_p(phi.data_ptr()), C.c_void_p(out.data_ptr()), None) == 0
    torch.cuda.synchronize()
    raw = (C.c_ulonglong * 32)()
    lib.bfm_debug_ws_ct_stats(ws, raw)
    tot = sum(raw[8 + i] for i in range(10))
    print("c5", {n: raw[i] for i, n in enumerate(names)}, {ph[i]: round(100 * raw[8 + i] / max(1, tot), 1) for i in range(10)})
    sys.exit(0)
mu, nu = synthetic.CONFIGS[cfg]()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=100))
# dyadic exact-hull kernel: 0 queries, 1 flagged, 2 exact orientation tests, 3 walked corners;
# non-dyadic kernel: see ctransform.cu (phases in slots 8..17)
ph = ["load", "convex", "hull", "merge", "compact", "suspect", "tangent", "certify", "flagged", "final"]
if os.environ.get("BFM_DY", "1") == "1":  # dyadic exact-hull kernel phase slots
    ph = ["load+max", "convex", "hull", "merge", "tangent", "resolve", "-", "-", "-", "-"]
prev = [0] * 32
for it in range(iters):
    s.step()
    out = (C.c_ulonglong * 32)()
    lib.bfm_debug_ct_stats(C.c_void_p(s._h.value), out)
    cur = list(out)
    dlt = [cur[i] - prev[i] for i in range(32)]
    prev = cur
    print(it, {n: dlt[i] for i, n in enumerate(names)}, flush=True)
    tot = sum(dlt[8 + i] for i in range(10))
    print("  phases %:", {ph[i]: round(100 * dlt[8 + i] / max(1, tot), 1) for i in range(10)},
          " total Mclk (line-thread-0 sum):", round(tot / 1e6, 1), flush=True)
    print("  merge levels Mclk:", [round(dlt[18 + i] / 1e6, 1) for i in range(10)], flush=True)
