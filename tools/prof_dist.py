"""Profiling driver (not a test): per-operator time of the slab driver at P=1
over NCCL (single process) on C3, vs the fused single-GPU solver."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import dist as D  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29577")
tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
mu, nu = synthetic.c3()
L = D.SlabLayout(mu.shape, 1)
comm = D.TorchComm()
ops = D.CudaSlabOps(L, 0, torch.device("cuda", 0))
s = D.DistSolver(L, comm, ops, mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=100),
                 device=torch.device("cuda", 0))
for _ in range(2):
    s.step()


def t(name, f, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    print(f"{name:28s} {1e3 * (time.perf_counter() - t0) / reps:8.3f} ms", flush=True)


x = s.x
t("rows_to_cols", lambda: x.rows_to_cols(s.phi))
cols = x.rows_to_cols(s.phi)
t("ct_cols", lambda: ops.ct_cols(cols))
chain, q = ops.ct_cols(cols)
t("cols_to_rows(chain)", lambda: x.cols_to_rows(chain))
t("cols_to_rows(q)", lambda: x.cols_to_rows(q))
cr, qr = x.cols_to_rows(chain), x.cols_to_rows(q)
t("ct_rows", lambda: ops.ct_rows(cr, qr))
t("ctransform total", lambda: s.ctransform(s.phi))
import ctypes as C  # noqa: E402
lib = bfm.load_library()
ws = C.c_void_p()
assert lib.bfm_workspace_create(2, (C.c_int * 2)(4096, 4096), C.byref(ws)) == 0
outp = torch.empty_like(s.phi)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
t("single-GPU ctransform", lambda: lib.bfm_ctransform_device(ws, C.c_void_p(s.phi.data_ptr()), C.c_void_p(outp.data_ptr()), sp))
dist_out = s.ctransform(s.phi)
lib.bfm_ctransform_device(ws, C.c_void_p(s.phi.data_ptr()), C.c_void_p(outp.data_ptr()), sp)
torch.cuda.synchronize()
print("bitwise equal:", bool(torch.equal(dist_out.view(torch.int64), outp.view(torch.int64))))
t("halo", lambda: x.halo(s.psi))
uh = x.halo(s.psi)
t("pf_map", lambda: ops.pf_map(uh, s.mu))
key, w, cm, _ = ops.pf_map(uh, s.mu)
t("route_records", lambda: x.route_records(key, w, cm, s.mu, ops))
recs = x.route_records(key, w, cm, s.mu, ops)
t("pf_gather", lambda: ops.pf_gather(*recs, s.nu))

t("pushforward total", lambda: s.pushforward_residual(s.psi, s.mu, s.nu))
r = s.pushforward_residual(s.psi, s.mu, s.nu)
t("solve_neumann", lambda: s.solve_neumann(r))
t("pair_value", lambda: s.pair_value())
t("step", lambda: s.step(), reps=3)
tdist.destroy_process_group()
