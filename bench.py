#!/usr/bin/env python
"""BFM benchmark: grid-point-iterations/s (float64) at BASELINE.json's two
headline sizes — C3 (4096^2, configs[2]) is the line's `value`, C4 (384^3,
configs[3]) is reported in the same line under "c4" (skip with --no-c4);
--config c4 makes C4 the headline.

A "step" is one steady-state back-and-forth iteration (the reference's
run() loop body: probe + step(), solver.hpp:211-226, i.e. 4 c-transforms, 2
ascent directions, 4 pair values, 2 axpys). Inputs are the seeded synthetic
densities of the BASELINE shapes from the library's shared generator
(bfm_synthetic_densities).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4|c5]
  (K defaults to the config's own iteration count: C3 50, C4 30, C1 100)
  python bench.py --impl reference ...   (the reference's own CPU solver,
        oracle/_ref = unmodified headers + FFTW shim, on the host cores)

--gpus N > 1 without torchrun re-executes itself under torch.distributed.run
(one process per GPU). Prints ONE JSON line (rank 0)."""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "BFM grid-point-iterations/sec (float64) at 4096² and 384³; c-transform HBM GB/s"
UNIT = "grid-point-iterations/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


ITERATIONS = {"c1": 100, "c2": 50, "c3": 50, "c4": 30}


def workload(cfg):
    """(mu, nu, config dict). The config dict is identical for both arms."""
    from paper_1905_12154_b200 import synthetic

    names = {
        "c3": ("C3: 2D 4096x4096 quadratic BFM, masked Gaussian mixtures (BASELINE configs[2])", [4096, 4096]),
        "c4": ("C4: 3D 384^3 quadratic BFM, Gaussian mixture -> ball (BASELINE configs[3])", [384, 384, 384]),
        "c1": ("C1: 2D 256x256 quadratic BFM, 3 Gaussians -> disc (BASELINE configs[0])", [256, 256]),
        "c2": ("C2: 2D 1024x1024 quadratic BFM, rectangles -> annulus-masked Gaussians (BASELINE configs[1])",
               [1024, 1024]),
    }
    if cfg not in names:
        raise SystemExit(f"unknown config {cfg}")
    mu, nu = getattr(synthetic, cfg)()
    desc = {"workload": names[cfg][0], "grid": names[cfg][1],
            "inputs": "bfm_synthetic_densities (std::mt19937_64, SURVEY 8(d)), seed %s" % cfg[1],
            "step": "one BFM iteration: probe + step() (4 c-transforms, 2 ascent directions, 4 pair values, 2 axpys)",
            "l2": "inputs larger than L2 (about 10 resident float64 fields of the grid)" if cfg in ("c3", "c4")
            else "fields fit in L2 (small config)"}
    return mu, nu, desc


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.samples = []
        self.index = index
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def quiet_stdout(fn):
    """Runs fn with file descriptor 1 pointed at stderr (native libraries that
    print banners at initialisation would otherwise break the one-JSON-line
    stdout contract)."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        return fn()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def reference_arm(args):
    """--impl reference: the reference's own CPU BFM (oracle/_ref) on the host."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    from paper_1905_12154_b200 import SolverConfig

    if O.ref_lib() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbfmref.so not built"}))
        return
    if args.config == "c5":
        # the reference's c-transform operator (transforms.hpp:396-432) on all
        # host threads, bounded sample: the 1024^2 C5 potential
        from paper_1905_12154_b200 import synthetic

        shape = (1024, 1024)
        phi = synthetic.c5_potential(shape)[0]
        O.ref_ctransform(phi)
        t0 = time.perf_counter()
        done = 0
        while done < max(1, args.steps) and time.perf_counter() - t0 < 120.0:
            O.ref_ctransform(phi)
            done += 1
        dt = (time.perf_counter() - t0) / done
        v = 16.0 * 2 * phi.size / dt / 1e9
        cores = os.cpu_count()
        print(json.dumps({
            "impl": "reference", "metric": "C5 isolated operator sweep: c-transform HBM GB/s (float64)",
            "value": v, "unit": "GB/s", "n_gpus": world, "steps": done, "warmup": 1,
            "ms_per_step": 1e3 * dt, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded C5 potential)",
            "config": {"workload": "C5: c-transform operator, 1024^2 sample (BASELINE configs[4])"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": f"{done} reference c-transforms of the 1024^2 C5 potential"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    mu, nu, desc = workload(args.config)
    N = mu.size
    s = O.RefSolver(mu, nu, SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
    s.dual_value()  # first probe (setup)
    budget = 240.0
    warm = 0
    t_start = time.perf_counter()
    for _ in range(args.warmup):
        s.step()
        s.dual_value()
        warm += 1
        if time.perf_counter() - t_start > budget / 3:
            break
    done = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.step()
        s.dual_value()  # trailing probe = next iteration's run() loop head
        done += 1
        if time.perf_counter() - t0 > budget:
            break
    dt = time.perf_counter() - t0
    v = N * done / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": done, "warmup": warm, "ms_per_step": 1e3 * dt / max(1, done),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE shapes)",
        "config": desc,
        "impl_detail": "reference bfm::Solver (oracle/_ref: unmodified headers + FFTW-subset shim) on all host threads",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
                         "sample": f"{done} full BFM iterations (probe+step) of {desc['workload']} on "
                                   f"{cores} host threads ({cpu_model()}); Poisson via the FFTW-subset shim"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.config == "c3" and not args.no_c4:
        # the C4 half of the metric: one bounded reference iteration (about a
        # minute on 16 host threads)
        mu4, nu4, desc4 = workload("c4")
        s4 = O.RefSolver(mu4, nu4, SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
        s4.dual_value()
        t4 = time.perf_counter()
        s4.step()
        s4.dual_value()
        dt4 = time.perf_counter() - t4
        v4 = mu4.size / dt4
        line["c4"] = {"workload": desc4["workload"], "grid": desc4["grid"], "steps": 1, "value": v4,
                      "unit": UNIT, "ms_per_step": 1e3 * dt4,
                      "cpu_baseline": {"value": v4, "unit": UNIT, "cores": cores, "kind": "reference",
                                       "cpu_model": cpu_model(),
                                       "sample": f"1 full BFM iteration (probe+step) of {desc4['workload']}"},
                      "e2e": {"value": v4, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_baseline(mu, nu, desc):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        import oracle_lib as O
        from paper_1905_12154_b200 import SolverConfig

        if O.ref_lib() is None:
            return None
        s = O.RefSolver(mu, nu, SolverConfig(tolerance=-1.0, max_iterations=10 ** 6))
        s.dual_value()
        t0 = time.perf_counter()
        s.step()
        s.dual_value()
        dt = time.perf_counter() - t0
        cores = os.cpu_count()
        return {"value": mu.size / dt, "unit": UNIT, "cores": cores, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"1 full BFM iteration (probe+step) of {desc['workload']} with the reference "
                          f"bfm::Solver (oracle/_ref, FFTW-subset shim) on {cores} host threads "
                          f"({cpu_model()}), {dt:.1f} s"}
    except Exception as e:  # the baseline is reported, never fatal
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"failed: {e}"}


def traffic_table():
    """ncu DRAM bytes (read + write) per call of each operator inside the BFM
    iteration, keyed "<op>@<grid>" (profiles/dram_bytes.json, written from
    the committed ncu captures by tools/dram_table.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "dram_bytes.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def op_rooflines(ops, shape, steps, hbm, hbm_kind):
    """Per-operator rooflines from the live per-operator CUDA events of the
    timed region (on the solver stream). Algorithmic bytes,
    per call: c-transform 16 d B/node (d axis-pass launches), pushforward +
    residual 32 B/node, Neumann solve 16 (2d - 1) B/node; the reductions op
    (4 pair values x 32 B/node, 2 gn x 16 B/node, 2 axpys x 24 B/node, plus
    the one-thread decision kernels) is reported per iteration (208 B/node)."""
    d = len(shape)
    N = int(np.prod(shape))
    key = "x".join(map(str, shape))
    tt = traffic_table()
    per_node = {"ctransform": 16.0 * d, "pushforward": 32.0, "poisson": 16.0 * (2 * d - 1)}
    out = {}
    for op, bpn in per_node.items():
        ms_total, calls = ops[op]
        ms = ms_total / max(calls, 1)
        b = bpn * N
        ach = b / (ms * 1e-3) / 1e9
        out[op] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                   "traffic": tt.get(f"{op}@{key}"), "ms_per_call": ms, "calls": calls,
                   "algorithmic_bytes_per_call": b, "algorithmic_bytes_per_node": bpn, "peak_kind": hbm_kind}
    ms_total, calls = ops["reduce"]
    ms = ms_total / max(steps, 1)
    b = 208.0 * N
    ach = b / (ms * 1e-3) / 1e9
    out["reductions"] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "traffic": tt.get(f"reductions@{key}"), "ms_per_iteration": ms,
                         "algorithmic_bytes_per_iteration": b, "algorithmic_bytes_per_node": 208.0,
                         "peak_kind": hbm_kind}
    out["ctransform"]["kernel"] = (f"c-transform: {d} axis-pass launches per call (ct_dy_kernel on dyadic "
                                   f"grids, ct_pass_kernel otherwise)")
    return out


def ctransform_roofline(lib, shape, torch, hbm, hbm_kind, reps=10):
    """Times the c-transform operator (d kernel launches, one per axis pass)
    on resident data with CUDA events on its launch stream; L2 flushed
    between launches. Algorithmic bytes: 16*d per node."""
    import ctypes as C

    from paper_1905_12154_b200 import synthetic

    d = len(shape)
    N = int(np.prod(shape))
    phi = torch.from_numpy(synthetic.c5_potential(tuple(shape))[0]).cuda()
    out = torch.empty_like(phi)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ws = C.c_void_p()
    ext = (C.c_int * d)(*shape)
    assert lib.bfm_workspace_create(d, ext, C.byref(ws)) == 0
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    for _ in range(3):
        assert lib.bfm_ctransform_device(ws, C.c_void_p(phi.data_ptr()), C.c_void_p(out.data_ptr()), sp) == 0
    launches = lib.bfm_workspace_last_launches(ws)
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.bfm_ctransform_device(ws, C.c_void_p(phi.data_ptr()), C.c_void_p(out.data_ptr()), sp)
        e1.record(stream)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    lib.bfm_workspace_destroy(ws)
    ms = tot / reps
    bytes_alg = 16.0 * d * N
    achieved = bytes_alg / (ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ctransform_dram_bytes.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("x".join(map(str, shape)))
        except Exception:
            traffic = None
    return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic,
            "kernel": f"c-transform operator ({launches} axis-pass launches) on {'x'.join(map(str, shape))}",
            "ms_per_launch_group": ms, "algorithmic_bytes": bytes_alg, "peak_kind": hbm_kind}


def c5_sweep(args):
    """BASELINE configs[4]: each operator timed separately
    on resident float64 data — ctransform(phi), solve_neumann(P - mean), and
    the fused map + pushforward + residual of the uniform mu through u — on
    2D 512^2..8192^2 and 3D 128^3..512^3, L2 flushed before every launch
    group, CUDA events on the launch stream. Algorithmic bytes per node:
    c-transform 16 d, Poisson 16 (2d - 1), pushforward + residual 32.
    Prints ONE JSON line; `sweep` lists every (operator, grid)."""
    import ctypes as C

    import torch

    import paper_1905_12154_b200 as bfm
    from paper_1905_12154_b200 import synthetic

    lib = bfm.load_library()
    hbm, hbm_kind = peaks()
    grids = [(n, n) for n in (512, 1024, 2048, 4096, 8192)] + [(n, n, n) for n in (128, 256, 384, 512)]
    if args.sweep_max:
        grids = [g for g in grids if int(np.prod(g)) <= args.sweep_max]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    reps = max(1, args.steps)
    rows = []
    launches = 0
    for shape in grids:
        d = len(shape)
        N = int(np.prod(shape))
        phi_np, P_np = synthetic.c5_potential(shape)
        u_np = synthetic.c5_pushforward_potential(shape)
        phi = torch.from_numpy(phi_np).cuda()
        rhs = torch.from_numpy(P_np - P_np.mean()).cuda()
        u = torch.from_numpy(u_np).cuda()
        mu = torch.ones(shape, dtype=torch.float64, device="cuda")
        tgt = torch.zeros_like(mu)
        out = torch.empty_like(phi)
        del phi_np, P_np, u_np
        ws = C.c_void_p()
        assert lib.bfm_workspace_create(d, (C.c_int * d)(*shape), C.byref(ws)) == 0
        ops = {
            "ctransform": (lambda: lib.bfm_ctransform_device(ws, C.c_void_p(phi.data_ptr()),
                                                             C.c_void_p(out.data_ptr()), sp), 16.0 * d),
            "solve_neumann": (lambda: lib.bfm_solve_neumann_device(ws, C.c_void_p(rhs.data_ptr()),
                                                                   C.c_void_p(out.data_ptr()), sp),
                              16.0 * (2 * d - 1)),
            "pushforward_residual": (lambda: lib.bfm_pushforward_residual_device(
                ws, C.c_void_p(u.data_ptr()), C.c_void_p(mu.data_ptr()), C.c_void_p(tgt.data_ptr()),
                C.c_void_p(out.data_ptr()), sp), 32.0),
        }
        for name, (fn, bpn) in ops.items():
            for _ in range(max(1, args.warmup)):
                assert fn() == 0
            nl = lib.bfm_workspace_last_launches(ws)
            tot = 0.0
            for _ in range(reps):
                flush.fill_(1.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                assert fn() == 0
                e1.record(stream)
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
                launches += nl
            ms = tot / reps
            gbs = bpn * N / (ms * 1e-3) / 1e9
            rows.append({"op": name, "grid": list(shape), "ms": ms, "launches_per_call": nl,
                         "algorithmic_bytes_per_node": bpn, "achieved_gbs": gbs, "frac": gbs / hbm})
            print(f"# {name:22s} {'x'.join(map(str, shape)):>14s} {ms:9.3f} ms {gbs:8.1f} GB/s "
                  f"{100 * gbs / hbm:5.2f}%", file=sys.stderr, flush=True)
        lib.bfm_workspace_destroy(ws)
        del phi, rhs, u, mu, tgt, out
        torch.cuda.empty_cache()
    ct = [r for r in rows if r["op"] == "ctransform"]
    head = max(ct, key=lambda r: int(np.prod(r["grid"]))) if ct else rows[0]
    line = {"metric": "C5 isolated operator sweep: c-transform HBM GB/s (float64)",
            "value": head["achieved_gbs"], "unit": "GB/s", "n_gpus": 1, "steps": reps,
            "warmup": args.warmup, "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded C5 potentials, SURVEY §8(d))",
            "config": {"workload": "C5: isolated operator sweep (BASELINE configs[4])",
                       "l2": "flushed (256 MiB write) before every launch group"},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": head["achieved_gbs"], "peak": hbm, "unit": "GB/s",
                         "frac": head["achieved_gbs"] / hbm, "traffic": None, "peak_kind": hbm_kind,
                         "kernel": f"c-transform operator on {'x'.join(map(str, head['grid']))}"},
            "sweep": rows}
    print(json.dumps(line), flush=True)


def ours_dist(args):
    """N > 1: the C++ multi-GPU solver (csrc/dist_solver.cu, bfm_dist_solver_*):
    one problem split into axis-0 slabs over N GPUs (strong scaling), NCCL
    send/recv exchanges issued by the library on its own stream, the NCCL
    unique id broadcast over torch.distributed (plumbing only)."""
    rank, world, local = dist_env()
    import torch
    import torch.distributed as tdist

    import paper_1905_12154_b200 as bfm
    from paper_1905_12154_b200 import dist_cpp as DC

    torch.cuda.set_device(local)
    bfm.set_device(local)
    dev = torch.device("cuda", local)

    def setup():
        tdist.init_process_group("nccl", device_id=dev)
        obj = [DC.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        return DC.nccl_comm(obj[0], rank, world)

    comm = quiet_stdout(setup)  # NCCL's init banner must not precede the JSON line
    mu, nu, desc = workload(args.config)
    N = mu.size
    starts, sizes = DC.split_rows(mu.shape[0], world)
    r0, nr = starts[rank], sizes[rank]
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6)
    s = DC.CppDistSolver(comm, mu.shape, mu[r0:r0 + nr], nu[r0:r0 + nr], cfg)
    for _ in range(args.warmup):
        s.step()
    clocks = ClockSampler(local)
    tdist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ms = s.time_steps(args.steps)  # CUDA events on the solver stream
    ck = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    tdist.barrier()
    ms_max = float(t.item())
    value = N * args.steps / (ms_max * 1e-3)
    s.close()

    # end to end: pinned host slabs in, K iterations, phi/psi slabs back
    pin_mu = torch.from_numpy(np.ascontiguousarray(mu[r0:r0 + nr])).pin_memory().numpy()
    pin_nu = torch.from_numpy(np.ascontiguousarray(nu[r0:r0 + nr])).pin_memory().numpy()
    tdist.barrier()
    t0 = time.perf_counter()
    s2 = DC.CppDistSolver(comm, mu.shape, pin_mu, pin_nu, cfg)
    for _ in range(args.steps):
        s2.step()
    phi_h = s2.field_rows(0)
    psi_h = s2.field_rows(1)
    e2e_local = time.perf_counter() - t0
    s2.close()
    te = torch.tensor([e2e_local], dtype=torch.float64, device=dev)
    tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
    e2e_s = float(te.item())
    del phi_h, psi_h
    e2e = {"value": N * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(2 * 8 * N / args.steps),
           "d2h_bytes_per_step": int(2 * 8 * N / args.steps),
           "note": "bfm_dist_solver from pinned host slabs + K steps + phi/psi slab readback, wall clock, "
                   "max over ranks"}
    if rank == 0:
        hbm, hbm_kind = peaks()
        d = len(desc["grid"])
        # NVLink bytes per rank and iteration (4 c-transforms x (8 + 12) B/node, 2
        # Neumann solves x 16 B/node, of which (P-1)/P leave the rank) against
        # 900 GB/s per direction
        nvl_bytes = (4 * 20 + 2 * 16) * (N / world) * (world - 1) / world
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE shapes; no public dataset)",
            "config": desc,
            "impl_detail": f"C++ multi-GPU solver, axis-0 slabs x{world}, NCCL send/recv exchanges",
            "gpu_launches": None,
            "clocks": ck,
            "roofline": {"bound": "nvlink", "achieved": nvl_bytes / (ms_max / args.steps * 1e-3) / 1e9,
                         "peak": 900.0, "unit": "GB/s",
                         "frac": nvl_bytes / (ms_max / args.steps * 1e-3) / 1e9 / 900.0, "traffic": None,
                         "kernel": "all-to-all exchange volume per iteration per rank over the whole step time",
                         "hbm_peak": hbm, "peak_kind": hbm_kind},
            "cpu_baseline": None,
            "e2e": e2e,
        }
        print(json.dumps(line))
    comm.close()
    tdist.destroy_process_group()


def ours_dist_python(args):
    """N > 1: the axis-0 slab decomposition (paper_1905_12154_b200/dist.py):
    one problem split over N GPUs (strong scaling), NCCL all-to-alls for the
    transposes and deposit records, rank-ordered scalar merges."""
    rank, world, local = dist_env()
    import torch
    import torch.distributed as tdist

    import paper_1905_12154_b200 as bfm
    from paper_1905_12154_b200 import dist as D

    torch.cuda.set_device(local)
    bfm.set_device(local)
    dev = torch.device("cuda", local)
    quiet_stdout(lambda: (tdist.init_process_group("nccl", device_id=dev), tdist.barrier()))
    comm = D.TorchComm()
    mu, nu, desc = workload(args.config)
    N = mu.size
    L = D.SlabLayout(mu.shape, world)
    r0, nr = L.rows(rank)
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6)
    ops = D.CudaSlabOps(L, rank, dev)
    s = D.DistSolver(L, comm, ops, mu[r0:r0 + nr], nu[r0:r0 + nr], cfg, mu_full=mu, nu_full=nu,
                     device=dev)
    for _ in range(args.warmup):
        s.step()
    s.ensure_probe()
    l0 = ops.launches
    clocks = ClockSampler(local)
    tdist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        s.step()
    s.ensure_probe()  # the next iteration's probe belongs to this step's work
    e1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    launches = ops.launches - l0
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    tdist.barrier()
    ms_max = float(t.item())
    value = N * args.steps / (ms_max * 1e-3)

    # rank-local kernels and all-to-alls, timed with CUDA events on a few
    # further steps (outside the timed region: the events add host syncs)
    timer = D.EventTimer()
    ops.timer = comm.timer = timer
    k_prof = max(1, min(3, args.steps))
    for _ in range(k_prof):
        s.step()
    s.ensure_probe()
    prof = timer.resolve()
    ops.timer = comm.timer = None
    del s

    # end to end: pinned host slabs in, K iterations, phi/psi slabs back
    pin_mu = torch.from_numpy(np.ascontiguousarray(mu[r0:r0 + nr])).pin_memory()
    pin_nu = torch.from_numpy(np.ascontiguousarray(nu[r0:r0 + nr])).pin_memory()
    tdist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = D.DistSolver(L, comm, ops, pin_mu.numpy(), pin_nu.numpy(), cfg, device=dev)
    for _ in range(args.steps):
        s2.step()
    phi_h = s2.phi.cpu()
    psi_h = s2.psi.cpu()
    e2e_local = time.perf_counter() - t0
    te = torch.tensor([e2e_local], dtype=torch.float64, device=dev)
    tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
    e2e_s = float(te.item())
    del s2, phi_h, psi_h
    e2e = {"value": N * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(2 * 8 * N / args.steps),
           "d2h_bytes_per_step": int(2 * 8 * N / args.steps),
           "note": "DistSolver from pinned host slabs + K step() + phi/psi slab readback, wall clock, max over ranks"}
    if rank == 0:
        hbm, hbm_kind = peaks()
        d = len(desc["grid"])
        n_local = nr * (N // L.shape[0])
        ct_ms, ct_calls, _ = prof.get("ctransform", (0.0, 1, 0))
        calls = max(1, ct_calls // d)  # d rank-local launches groups per c-transform call
        ct_call_ms = ct_ms / calls
        ct_bytes = 16.0 * d * n_local
        a2a_ms, a2a_calls, a2a_bytes = prof.get("alltoall", (0.0, 1, 0))
        nvl = a2a_bytes / max(a2a_ms * 1e-3, 1e-12) / 1e9
        roof = {"bound": "hbm", "achieved": ct_bytes / (ct_call_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": ct_bytes / (ct_call_ms * 1e-3) / 1e9 / hbm, "traffic": None,
                "kernel": f"rank-0 local c-transform kernels ({d} axis passes over its column and row slabs)",
                "ms_per_call": ct_call_ms, "algorithmic_bytes_per_call": ct_bytes, "peak_kind": hbm_kind,
                "alltoall": {"bound": "nvlink", "achieved": nvl, "peak": 900.0, "unit": "GB/s",
                             "frac": nvl / 900.0, "bytes": a2a_bytes, "ms": a2a_ms, "calls": a2a_calls,
                             "note": f"rank 0: bytes sent to other ranks over {k_prof} profiled steps, "
                                     "NCCL all_to_all_single time (CUDA events)"},
                "profiled_steps": k_prof,
                "op_ms_per_step": {c: v[0] / k_prof for c, v in prof.items()}}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE shapes; no public dataset)",
            "config": desc,
            "impl_detail": f"axis-0 slabs x{world} (NCCL all-to-all transposes and deposit routing)",
            "gpu_launches": int(launches),
            "clocks": ck,
            "roofline": roof,
            "cpu_baseline": None,
            "e2e": e2e,
        }
        print(json.dumps(line))
    ops.close()
    tdist.destroy_process_group()


def measure(cfg, steps, warmup, local=0):
    """Our arm on one GPU for one config: device-timed steps (value), live
    per-operator rooflines, and the end-to-end run through the public API."""
    import torch

    import paper_1905_12154_b200 as bfm

    mu, nu, desc = workload(cfg)
    N = mu.size
    conf = bfm.SolverConfig(tolerance=-1.0, max_iterations=10 ** 6)
    s = bfm.Solver(mu, nu, conf)
    for _ in range(warmup):
        s.step()
    s.time_steps(1)  # the graphs of the timed loop are captured outside the timed region
    l0 = s.launches()
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    clocks.start()
    ms = s.time_steps(steps)  # graphs, side-stream overlap, no per-operator events
    ck = clocks.stop()
    launches = s.launches() - l0
    # profiled pass right after: the same iterations' kernels with per-operator
    # CUDA events on their stream, the side-stream work serialised so each
    # event pair times one operator (the live rooflines)
    k_prof = max(1, min(steps, 10))
    s.set_timing(True)
    s.time_steps(1)  # capture of the profiled graphs
    s.set_timing(False)
    s.set_timing(True)
    ms_prof = s.time_steps(k_prof)
    ops = s.op_times()
    s.set_timing(False)
    del s

    # end to end through the public API with host buffers: solver creation
    # from pinned host arrays (H2D of mu, nu), K steps, phi/psi read back (D2H)
    pin_mu = torch.from_numpy(mu).pin_memory().numpy()
    pin_nu = torch.from_numpy(nu).pin_memory().numpy()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = bfm.Solver(pin_mu, pin_nu, conf)
    for _ in range(steps):
        s2.step()
    phi_h = s2.phi()
    psi_h = s2.psi()
    e2e_s = time.perf_counter() - t0
    del s2, phi_h, psi_h
    e2e = {"value": N * steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(2 * 8 * N / steps),
           "d2h_bytes_per_step": int(2 * 8 * N / steps),
           "note": "bfm.Solver(mu, nu) from pinned host arrays + K step() + phi()/psi() readback, wall clock"}
    hbm, hbm_kind = peaks()
    roofs = op_rooflines(ops, desc["grid"], k_prof, hbm, hbm_kind)
    for r in roofs.values():
        r["measured_over"] = f"{k_prof} profiled steps right after the timed region ({ms_prof / k_prof:.3f} ms/step)"
    return {"mu": mu, "nu": nu, "desc": desc, "N": N, "ms": ms, "value": N * steps / (ms * 1e-3),
            "ops": ops, "k_prof": k_prof, "ms_prof": ms_prof, "rooflines": roofs, "clocks": ck,
            "launches": launches, "e2e": e2e}


def ours(args):
    rank, world, local = dist_env()
    if (world > 1 and not args.replicas) or args.slabs:
        return ours_dist_python(args) if args.py_dist else ours_dist(args)
    import torch

    import paper_1905_12154_b200 as bfm

    torch.cuda.set_device(local)
    bfm.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        quiet_stdout(lambda: (dist.init_process_group("nccl", device_id=torch.device("cuda", local)),
                              dist.barrier()))
    m = measure(args.config, args.steps, args.warmup, local)
    t = torch.tensor([m["ms"]], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_max = float(t.item())
    value = m["N"] * args.steps * world / (ms_max * 1e-3)
    sub = None
    if args.config == "c3" and not args.no_c4:
        c4_steps = ITERATIONS["c4"] if args.c4_steps is None else args.c4_steps
        m4 = measure("c4", c4_steps, args.warmup, local)
        sub = {"workload": m4["desc"]["workload"], "grid": m4["desc"]["grid"], "steps": c4_steps,
               "value": m4["value"] * world, "unit": UNIT, "ms_per_step": m4["ms"] / c4_steps,
               "roofline": m4["rooflines"]["ctransform"], "rooflines": m4["rooflines"],
               "op_breakdown_ms_per_step": {k: v[0] / m4["k_prof"] for k, v in m4["ops"].items()},
               "gpu_launches": int(m4["launches"]), "clocks": m4["clocks"], "e2e": m4["e2e"]}
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    hbm, hbm_kind = peaks()
    lib = bfm.load_library()
    roof = dict(m["rooflines"]["ctransform"])
    roof["c5_operator"] = ctransform_roofline(lib, m["desc"]["grid"], torch, hbm, hbm_kind)
    cpu = cpu_baseline(m["mu"], m["nu"], m["desc"]) if world == 1 and not args.no_cpu_baseline else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE shapes; no public dataset)",
        "config": m["desc"],
        "impl_detail": ("independent single-GPU replicas" if world > 1 else "single B200") +
                       "; iterations as CUDA graphs, certified device-side scalar decisions",
        "gpu_launches": int(m["launches"]),
        "clocks": m["clocks"],
        "roofline": roof,
        "rooflines": m["rooflines"],
        "op_breakdown_ms_per_step": {k: v[0] / m["k_prof"] for k, v in m["ops"].items()},
        "cpu_baseline": cpu,
        "e2e": m["e2e"],
    }
    if sub is not None:
        line["c4"] = sub
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def respawn_under_torchrun(args):
    """--gpus N > 1 outside torchrun: one process per GPU via torch.distributed.run."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the config's own iteration count, BASELINE configs: "
                         "C1 100, C3 50, C4 30; C2 50; the C5 sweep 3; the reference arm 5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--sweep-max", type=int, default=0,
                    help="c5: skip grids with more nodes than this (0: all)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="c3: skip the C4 (384^3) sub-object")
    ap.add_argument("--c4-steps", type=int, default=None, help="c3: timed steps of the C4 sub-object (default 30)")
    ap.add_argument("--slabs", action="store_true",
                    help="use the slab-decomposition driver even at N = 1 (checks the NCCL path)")
    ap.add_argument("--py-dist", action="store_true",
                    help="N > 1: the Python slab driver (dist.py) instead of the C++ one")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent single-GPU replicas instead of the slab decomposition")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0 and args.impl == "ours":
        respawn_under_torchrun(args)
    if world and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.steps is None:
        args.steps = 5 if args.impl == "reference" else {"c1": 100, "c2": 50, "c3": 50, "c4": 30, "c5": 3}[args.config]
    if args.impl == "reference":
        reference_arm(args)
    elif args.config == "c5":
        if dist_env()[0] == 0:
            c5_sweep(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
