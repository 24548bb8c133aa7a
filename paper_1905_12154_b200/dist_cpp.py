"""Python handle on the C++ multi-GPU solver (csrc/dist_solver.cu, the
bfm_dist_solver_* C ABI): bfm::Solver (solver.hpp:146-368) on an axis-0 slab
decomposition, one process per GPU, exchanges as NCCL send/recv issued by the
library. The host loop is C++; this module only creates communicators and
moves host arrays.

    uid = nccl_unique_id()            # on rank 0, then broadcast it
    comm = nccl_comm(uid, rank, world)
    s = CppDistSolver(comm, shape, mu_rows, nu_rows, config)
    s.step(); rep = s.run()

local_group(P) gives P communicators whose ranks run as threads of this
process on one device (host-synchronised exchanges) — how a single GPU
checks P > 1.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import List, Optional, Sequence

import numpy as np

from . import (_ERRORS, TERMINATION_NAMES, Error, IterationStats, SolveReport, SolverConfig, _extents,
               load_library)


def _lib():
    lib = load_library()
    if getattr(lib, "_dist_declared", False):
        return lib
    P, I, D = C.c_void_p, C.c_int, C.c_double
    sig = {
        "bfm_nccl_unique_id": (I, [P]),
        "bfm_comm_create_nccl": (I, [P, I, I, P]),
        "bfm_comm_create_local_group": (I, [I, P]),
        "bfm_comm_destroy": (None, [P]),
        "bfm_dist_solver_create": (I, [P, I, P, P, P, P, P]),
        "bfm_dist_solver_destroy": (None, [P]),
        "bfm_dist_solver_rows": (I, [P, P, P]),
        "bfm_dist_solver_step": (I, [P, P]),
        "bfm_dist_solver_probe": (I, [P, P, P]),
        "bfm_dist_solver_run": (I, [P, P]),
        "bfm_dist_solver_field": (I, [P, I, P]),
        "bfm_dist_solver_report_field": (I, [P, I, P]),
        "bfm_dist_solver_trace": (I, [P, P, I, P]),
        "bfm_dist_solver_iteration": (I, [P]),
        "bfm_dist_solver_time_steps": (I, [P, I, P]),
        "bfm_dist_solver_sigma": (D, [P]),
        "bfm_dist_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    lib._dist_declared = True
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, Error)(_lib().bfm_dist_last_error().decode())


def split_rows(n0: int, parts: int):
    """The library's row partition (lower ranks take the remainder rows)."""
    base, rem = divmod(n0, parts)
    sizes = [base + (1 if r < rem else 0) for r in range(parts)]
    starts = [sum(sizes[:r]) for r in range(parts)]
    return starts, sizes


class Comm:
    def __init__(self, handle: C.c_void_p, rank: int, size: int):
        self.h, self.rank, self.size = handle, rank, size

    def close(self):
        if self.h:
            _lib().bfm_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(_lib().bfm_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm(uid: bytes, rank: int, size: int) -> Comm:
    h = C.c_void_p()
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    _check(_lib().bfm_comm_create_nccl(buf, int(rank), int(size), C.byref(h)))
    return Comm(h, rank, size)


def local_group(parts: int) -> List[Comm]:
    hs = (C.c_void_p * parts)()
    _check(_lib().bfm_comm_create_local_group(int(parts), hs))
    return [Comm(C.c_void_p(hs[r]), r, parts) for r in range(parts)]


class CppDistSolver:
    """One rank of the C++ multi-GPU solver (bfm_dist_solver_*)."""

    def __init__(self, comm: Comm, shape: Sequence[int], mu_rows, nu_rows,
                 config: Optional[SolverConfig] = None):
        lib = _lib()
        self.shape = tuple(int(n) for n in shape)
        self.comm = comm
        mu_rows = np.ascontiguousarray(mu_rows, dtype=np.float64)
        nu_rows = np.ascontiguousarray(nu_rows, dtype=np.float64)
        c = (config or SolverConfig())._c()
        h = C.c_void_p()
        _check(lib.bfm_dist_solver_create(comm.h, len(self.shape), _extents(self.shape),
                                          mu_rows.ctypes.data_as(C.c_void_p),
                                          nu_rows.ctypes.data_as(C.c_void_p), C.byref(c), C.byref(h)))
        self.h = h
        r0, nr = C.c_int(), C.c_int()
        _check(lib.bfm_dist_solver_rows(h, C.byref(r0), C.byref(nr)))
        self.row0, self.nrows = r0.value, nr.value

    def close(self):
        if self.h:
            _lib().bfm_dist_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stats(s) -> IterationStats:
        return IterationStats(iteration=s.iteration, residual=s.residual, dual_value=s.dual_value,
                              sigma_first=s.sigma_first, sigma_second=s.sigma_second,
                              grad_norm_sq_first=s.grad_norm_sq_first,
                              grad_norm_sq_second=s.grad_norm_sq_second,
                              increase_first=s.increase_first, increase_second=s.increase_second)

    def step(self) -> IterationStats:
        from . import _Stats

        st = _Stats()
        _check(_lib().bfm_dist_solver_step(self.h, C.byref(st)))
        return self._stats(st)

    def dual_value(self) -> float:
        v = C.c_double()
        _check(_lib().bfm_dist_solver_probe(self.h, C.byref(v), None))
        return v.value

    def residual(self) -> float:
        v = C.c_double()
        _check(_lib().bfm_dist_solver_probe(self.h, None, C.byref(v)))
        return v.value

    def time_steps(self, k: int) -> float:
        """k steps (+ the trailing probes) between CUDA events on the solver stream: ms."""
        ms = C.c_double()
        _check(_lib().bfm_dist_solver_time_steps(self.h, int(k), C.byref(ms)))
        return ms.value

    def sigma(self) -> float:
        return float(_lib().bfm_dist_solver_sigma(self.h))

    def field_rows(self, which: int = 0) -> np.ndarray:
        M = int(np.prod(self.shape[1:]))
        out = np.empty((self.nrows,) + self.shape[1:], dtype=np.float64)
        _check(_lib().bfm_dist_solver_field(self.h, int(which), out.ctypes.data_as(C.c_void_p)))
        assert out.size == self.nrows * M
        return out

    def trace(self) -> List[IterationStats]:
        from . import _Stats

        n = C.c_int()
        _check(_lib().bfm_dist_solver_trace(self.h, None, 0, C.byref(n)))
        arr = (_Stats * max(1, n.value))()
        _check(_lib().bfm_dist_solver_trace(self.h, arr, n.value, C.byref(n)))
        return [self._stats(arr[i]) for i in range(n.value)]

    def run(self) -> SolveReport:
        from . import _Report

        rep = _Report()
        _check(_lib().bfm_dist_solver_run(self.h, C.byref(rep)))
        d = len(self.shape)

        def full(which):
            out = np.empty(self.shape, dtype=np.float64)
            _check(_lib().bfm_dist_solver_report_field(self.h, int(which), out.ctypes.data_as(C.c_void_p)))
            return out

        return SolveReport(termination=TERMINATION_NAMES[rep.termination], iterations=rep.iterations,
                           dual_value=rep.dual_value, primal_cost=rep.primal_cost, residual=rep.residual,
                           wall_seconds=rep.wall_seconds, trace=self.trace(), phi=full(0), psi=full(1),
                           map=np.stack([full(2 + a) for a in range(d)]))


def run_local(shape, mu, nu, config: Optional[SolverConfig] = None, parts: int = 2, steps: int = 0,
              report: bool = False, device: int = 0):
    """P ranks of the C++ solver as threads of this process on one device.
    Returns per rank (trace, phi rows, psi rows, report or None)."""
    from . import set_device

    comms = local_group(parts)
    starts, sizes = split_rows(shape[0], parts)
    results: list = [None] * parts
    errors: list = [None] * parts

    def body(r):
        try:
            set_device(device)
            s = CppDistSolver(comms[r], shape, mu[starts[r]:starts[r] + sizes[r]],
                              nu[starts[r]:starts[r] + sizes[r]], config)
            for _ in range(steps):
                s.step()
            rep = s.run() if report else None
            results[r] = (s.trace(), s.field_rows(0), s.field_rows(1), rep)
            s.close()
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errors[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(parts)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    for e in errors:
        if e is not None:
            raise e
    return results
