"""Multi-GPU BFM: one process per GPU, axis-0 slab decomposition.

The reference (solver.hpp:146-368) is single-node CPU code; this is the
B200-side scale-out of the same iteration:

* Rank r owns rows [row0_r, row0_r + nrows_r) of the grid (axis 0 split into
  P contiguous blocks) for every field, and, for axis-0 work, the flattened
  columns [col0_r, col0_r + ncols_r) of the n1*n2 non-axis-0 index.
* c-transform (transforms.hpp:396-432): phi rows -> columns (one all-to-all,
  8 B/node); pass 0 along axis 0 on the column slab writes the argmin j0* and
  Q = phi(j0*, column); (j0*, Q) columns -> rows (12 B/node); passes 1..d-1 are
  row-local. The exact minimum does not depend on how the candidates are
  grouped, so the result equals the single-GPU transform bit for bit.
* Neumann Poisson (poisson.hpp:87-106): DCT-II along axes d-1..1 on rows,
  rows -> columns, the fused axis-0 [DCT-II, divide, DCT-III] on columns,
  columns -> rows, DCT-III along 1..d-1. Every line sees the same arithmetic.
* Pushforward (pushforward.hpp:70-91,141-172): u with one halo row from each
  neighbour; every source becomes a deposit record (global lo-corner cell,
  weights, clamp mask, mass) sent to the owners of the target rows it reaches
  (one all-to-all-v). Received records are concatenated in sender-rank order,
  which is the global source order, so each target folds its deposits in the
  reference's sequential order.
* Scalars (pair value, gn, primal): per-rank unscaled double-double partial
  sums, all-gathered and merged in rank order (deterministic).

The rank-local kernels are the C ABI bfm_slab_* entry points (hand-written
sm_100a kernels, CudaSlabOps). Collectives go through a Comm: TorchComm
(torch.distributed, NCCL between GPUs, one process per GPU) or LocalComm
(ranks as threads of one process, used to check the decomposition on one
device; ranks only exchange host-synchronised buffers, no kernel ever waits
on another rank). Ops and Comm are plain objects so the exchange logic can be
exercised on CPU (gloo) by the tests with a test-side implementation of the
rank-local operators.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
import time
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import (BACK_AND_FORTH, TERMINATION_NAMES, IterationStats, NumericalBlowup, SolveReport,
               SolverConfig, _check, _extents, load_library)


# ---------------------------------------------------------------- layout
def _split(n: int, parts: int) -> Tuple[List[int], List[int]]:
    base, rem = divmod(n, parts)
    sizes = [base + (1 if r < rem else 0) for r in range(parts)]
    starts = [0]
    for s in sizes[:-1]:
        starts.append(starts[-1] + s)
    return starts, sizes


class SlabLayout:
    """Axis-0 row blocks and flattened column blocks of a d-dimensional grid."""

    def __init__(self, shape: Sequence[int], parts: int):
        self.shape = tuple(int(n) for n in shape)
        self.d = len(self.shape)
        if self.d < 2:
            raise ValueError("slab decomposition needs d >= 2")
        self.P = int(parts)
        self.n0 = self.shape[0]
        self.M = int(np.prod(self.shape[1:]))
        if self.n0 < self.P or self.M < self.P:
            raise ValueError(f"grid {self.shape} too small for {self.P} ranks")
        self.row0, self.nrows = _split(self.n0, self.P)
        self.col0, self.ncols = _split(self.M, self.P)
        self.N = self.n0 * self.M
        self.vol = 1.0
        for n in self.shape:
            self.vol *= 1.0 / n  # grid.hpp:71 (product of fl(1/n) in axis order)

    def rows(self, r: int) -> Tuple[int, int]:
        return self.row0[r], self.nrows[r]

    def cols(self, r: int) -> Tuple[int, int]:
        return self.col0[r], self.ncols[r]

    def row_owner(self, rows: torch.Tensor) -> torch.Tensor:
        starts = torch.tensor(self.row0[1:], dtype=rows.dtype, device=rows.device)
        return torch.bucketize(rows, starts, right=True)


# ---------------------------------------------------------------- communicators
class EventTimer:
    """Per-category device time (CUDA events on the current stream) and byte
    counts; bench.py's rank-local kernel and all-to-all rooflines at N > 1."""

    def __init__(self):
        self.pending = []
        self.ms = {}
        self.calls = {}
        self.bytes = {}

    def span(self, cat: str, nbytes: int = 0):
        timer = self

        class _Span:
            def __enter__(self):
                self.a = torch.cuda.Event(enable_timing=True)
                self.b = torch.cuda.Event(enable_timing=True)
                self.a.record()

            def __exit__(self, *exc):
                self.b.record()
                timer.pending.append((cat, self.a, self.b))
                timer.bytes[cat] = timer.bytes.get(cat, 0) + nbytes
                return False

        return _Span()

    def resolve(self):
        torch.cuda.synchronize()
        for cat, a, b in self.pending:
            self.ms[cat] = self.ms.get(cat, 0.0) + a.elapsed_time(b)
            self.calls[cat] = self.calls.get(cat, 0) + 1
        self.pending = []
        return {c: (self.ms[c], self.calls[c], self.bytes.get(c, 0)) for c in self.ms}


class _NoSpan:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


def _span(timer, cat, nbytes=0):
    return timer.span(cat, nbytes) if timer is not None else _NoSpan()


class TorchComm:
    """torch.distributed process group (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.timer = None  # EventTimer: all-to-all time and bytes leaving this rank

    def alltoallv(self, sends: List[torch.Tensor],
                  recv_counts: Optional[List[int]] = None) -> List[torch.Tensor]:
        """sends[q] goes to rank q; returns what every rank sent here. The
        receive sizes are exchanged first unless the caller knows them."""
        dist = self.dist
        ref = sends[0]
        sc = [int(x.numel()) for x in sends]
        if recv_counts is None:
            counts = torch.tensor(sc, dtype=torch.int64, device=ref.device)
            rcounts = torch.empty_like(counts)
            dist.all_to_all_single(rcounts, counts, group=self.group)
            recv_counts = [int(c) for c in rcounts.tolist()]
        out = torch.empty(sum(recv_counts), dtype=ref.dtype, device=ref.device)
        sent = (sum(sc) - sc[self.rank]) * ref.element_size()
        with _span(self.timer, "alltoall", sent):
            dist.all_to_all_single(out, torch.cat([x.reshape(-1) for x in sends]), recv_counts, sc,
                                   group=self.group)
        return list(torch.split(out, recv_counts))

    def alltoall_flat(self, send: torch.Tensor, send_counts: List[int],
                      recv_counts: List[int]) -> torch.Tensor:
        """send is already packed by destination (send_counts elements per
        rank, in rank order); returns the packed receive buffer."""
        out = torch.empty(sum(recv_counts), dtype=send.dtype, device=send.device)
        sent = (sum(send_counts) - send_counts[self.rank]) * send.element_size()
        with _span(self.timer, "alltoall", sent):
            self.dist.all_to_all_single(out, send, recv_counts, send_counts, group=self.group)
        return out

    def allgather(self, values: Sequence[float]) -> np.ndarray:
        dist = self.dist
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        mine = torch.tensor(list(values), dtype=torch.float64, device=dev)
        outs = [torch.empty_like(mine) for _ in range(self.size)]
        dist.all_gather(outs, mine, group=self.group)
        return np.stack([o.cpu().numpy() for o in outs])


class LocalComm:
    """P ranks as threads of one process (checks the decomposition on one
    device). Buffers are exchanged only after the sender's work is complete."""

    class _Shared:
        def __init__(self, size: int):
            self.size = size
            self.barrier = threading.Barrier(size)
            self.box: list = [None] * size

    def __init__(self, shared: "LocalComm._Shared", rank: int):
        self.sh = shared
        self.rank = rank
        self.size = shared.size

    @staticmethod
    def group(size: int) -> List["LocalComm"]:
        sh = LocalComm._Shared(size)
        return [LocalComm(sh, r) for r in range(size)]

    def _exchange(self, item):
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        self.sh.barrier.wait()
        self.sh.box[self.rank] = item
        self.sh.barrier.wait()
        got = list(self.sh.box)
        self.sh.barrier.wait()
        return got

    def alltoallv(self, sends: List[torch.Tensor],
                  recv_counts: Optional[List[int]] = None) -> List[torch.Tensor]:
        boxes = self._exchange([s.reshape(-1).clone() for s in sends])
        return [boxes[r][self.rank] for r in range(self.size)]

    def alltoall_flat(self, send: torch.Tensor, send_counts: List[int],
                      recv_counts: List[int]) -> torch.Tensor:
        got = self.alltoallv(list(torch.split(send.reshape(-1), send_counts)), recv_counts)
        return torch.cat(got)

    def allgather(self, values: Sequence[float]) -> np.ndarray:
        boxes = self._exchange(np.asarray(list(values), dtype=np.float64))
        return np.stack(boxes)


# ---------------------------------------------------------------- rank-local ops
class CudaSlabOps:
    """Rank-local halves of the operators: the bfm_slab_* C ABI (sm_100a)."""

    def __init__(self, layout: SlabLayout, rank: int, device: torch.device):
        self.L = layout
        self.rank = rank
        self.device = device
        self.lib = load_library()
        lib = self.lib
        P = C.c_void_p
        lib.bfm_slab_create.argtypes = [C.c_int, P, C.c_int, C.c_int, C.c_long, C.c_int, P]
        lib.bfm_slab_destroy.argtypes = [P]
        for fn in ("bfm_slab_ct_cols", "bfm_slab_ct_rows", "bfm_slab_poisson_rows_forward",
                   "bfm_slab_poisson_cols", "bfm_slab_poisson_rows_inverse", "bfm_slab_pf_map",
                   "bfm_slab_pf_gather", "bfm_slab_dot", "bfm_slab_primal"):
            getattr(lib, fn).restype = C.c_int
        lib.bfm_slab_ct_cols.argtypes = [P] * 5
        lib.bfm_slab_ct_rows.argtypes = [P] * 5
        lib.bfm_slab_poisson_rows_forward.argtypes = [P] * 4
        lib.bfm_slab_poisson_cols.argtypes = [P] * 4
        lib.bfm_slab_poisson_rows_inverse.argtypes = [P] * 3
        lib.bfm_slab_pf_map.argtypes = [P] * 8
        lib.bfm_slab_pf_num_cells.argtypes = [P]
        lib.bfm_slab_pf_num_cells.restype = C.c_long
        lib.bfm_slab_pf_gather.argtypes = [P, C.c_long] + [P] * 7
        lib.bfm_slab_dot.argtypes = [P] * 7
        lib.bfm_slab_primal.argtypes = [P] * 5
        lib.bfm_slab_axpy.argtypes = [P, P, C.c_double, P, P]
        lib.bfm_slab_axpy.restype = C.c_int
        lib.bfm_slab_last_launches.argtypes = [P]
        lib.bfm_slab_set_partition.argtypes = [P, C.c_int, P]
        lib.bfm_slab_set_partition.restype = C.c_int
        lib.bfm_slab_pf_route.argtypes = [P] * 8
        lib.bfm_slab_pf_route.restype = C.c_int
        lib.bfm_slab_pf_unpack.argtypes = [P, C.c_long] + [P] * 6
        lib.bfm_slab_pf_unpack.restype = C.c_int
        r0, nr = layout.rows(rank)
        c0, nc = layout.cols(rank)
        h = C.c_void_p()
        _check(lib, lib.bfm_slab_create(layout.d, _extents(layout.shape), r0, nr, c0, nc, C.byref(h)))
        self.h = h
        self.launches = 0
        self.timer = None  # EventTimer: rank-local operator kernels
        starts = (C.c_int * (layout.P + 1))(*(layout.row0 + [layout.n0]))
        _check(lib, lib.bfm_slab_set_partition(h, layout.P, starts))

    def close(self):
        if self.h:
            self.lib.bfm_slab_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # helpers
    def _s(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t: Optional[torch.Tensor]):
        return C.c_void_p(t.data_ptr() if t is not None else 0)

    def _run(self, rc):
        _check(self.lib, rc)
        self.launches += int(self.lib.bfm_slab_last_launches(self.h))

    def empty(self, n: int, dtype=torch.float64) -> torch.Tensor:
        return torch.empty(n, dtype=dtype, device=self.device)

    # operators
    def ct_cols(self, phi_cols: torch.Tensor):
        n = phi_cols.numel()
        chain = self.empty(n, torch.int32)
        q = self.empty(n)
        with _span(self.timer, "ctransform"):
            self._run(self.lib.bfm_slab_ct_cols(self.h, self._p(phi_cols), self._p(chain), self._p(q),
                                                self._s()))
        return chain, q

    def ct_rows(self, chain: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
        out = self.empty(q.numel())
        with _span(self.timer, "ctransform"):
            self._run(self.lib.bfm_slab_ct_rows(self.h, self._p(chain), self._p(q), self._p(out), self._s()))
        return out

    def poisson_rows_forward(self, x: torch.Tensor) -> torch.Tensor:
        out = self.empty(x.numel())
        with _span(self.timer, "poisson"):
            self._run(self.lib.bfm_slab_poisson_rows_forward(self.h, self._p(x), self._p(out), self._s()))
        return out

    def poisson_cols(self, x: torch.Tensor) -> torch.Tensor:
        out = self.empty(x.numel())
        with _span(self.timer, "poisson"):
            self._run(self.lib.bfm_slab_poisson_cols(self.h, self._p(x), self._p(out), self._s()))
        return out

    def poisson_rows_inverse(self, x: torch.Tensor) -> torch.Tensor:
        with _span(self.timer, "poisson"):
            self._run(self.lib.bfm_slab_poisson_rows_inverse(self.h, self._p(x), self._s()))
        return x

    def pf_map(self, u_halo: torch.Tensor, source: torch.Tensor, want_disp: bool = False):
        n = source.numel()
        d = self.L.d
        key = self.empty(n, torch.int32)
        w = self.empty(d * n)
        cmask = self.empty(n, torch.uint8)
        disp = self.empty(d * n) if want_disp else None
        self._run(self.lib.bfm_slab_pf_map(self.h, self._p(u_halo), self._p(source), self._p(key),
                                           self._p(w), self._p(cmask), self._p(disp), self._s()))
        return key, w, cmask, disp

    def pf_num_cells(self) -> int:
        return int(self.lib.bfm_slab_pf_num_cells(self.h))

    def pf_route(self, key, w, cmask, mass):
        """Packed records per destination rank (see SlabExchange.route_records)."""
        d = self.L.d
        packed = self.empty(2 * mass.numel() * (3 + d))
        counts = (C.c_long * self.L.P)()
        self._run(self.lib.bfm_slab_pf_route(self.h, self._p(key), self._p(w), self._p(cmask),
                                             self._p(mass), self._p(packed), counts, self._s()))
        return packed, [int(c) for c in counts]

    def pf_unpack(self, packed, nrec: int):
        d = self.L.d
        keys = self.empty(nrec, torch.int32)
        mass = self.empty(nrec)
        w = self.empty(d * nrec)
        cmask = self.empty(nrec, torch.uint8)
        self._run(self.lib.bfm_slab_pf_unpack(self.h, int(nrec), self._p(packed), self._p(keys),
                                              self._p(mass), self._p(w), self._p(cmask), self._s()))
        return keys, mass, w, cmask

    def pf_gather(self, keys, mass, w, cmask, target) -> torch.Tensor:
        nloc = self.L.nrows[self.rank] * self.L.M
        out = self.empty(nloc)
        self._run(self.lib.bfm_slab_pf_gather(self.h, int(keys.numel()), self._p(keys), self._p(mass),
                                              self._p(w), self._p(cmask), self._p(target),
                                              self._p(out), self._s()))
        return out

    def dot(self, a1, b1, a2=None, b2=None) -> Tuple[float, float, float, float]:
        out = (C.c_double * 4)()
        self._run(self.lib.bfm_slab_dot(self.h, self._p(a1), self._p(b1), self._p(a2), self._p(b2),
                                        out, self._s()))
        return tuple(out)

    def primal(self, disp, mu) -> Tuple[float, float]:
        out = (C.c_double * 2)()
        self._run(self.lib.bfm_slab_primal(self.h, self._p(disp), self._p(mu), out, self._s()))
        return tuple(out)

    def axpy(self, u: torch.Tensor, sigma: float, d: torch.Tensor) -> None:
        self._run(self.lib.bfm_slab_axpy(self.h, self._p(u), float(sigma), self._p(d), self._s()))


# ---------------------------------------------------------------- exchanges
def _two_sum(a: float, b: float) -> Tuple[float, float]:
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def merge_dd(parts: np.ndarray) -> Tuple[float, float]:
    """Rank-ordered double-double merge of (hi, lo) partials (reduce.cu dd_merge)."""
    s, c = 0.0, 0.0
    for hi, lo in parts:
        s, e = _two_sum(s, float(hi))
        c = (c + float(lo)) + e
    return s, c


class SlabExchange:
    """The collectives of the decomposition (identical for every Ops)."""

    def __init__(self, layout: SlabLayout, comm):
        self.L = layout
        self.comm = comm
        self.rank = comm.rank

    def rows_to_cols(self, x_rows: torch.Tensor) -> torch.Tensor:
        """Row slab (nrows_r x M) -> column slab (n0 x ncols_r). Packing by
        destination is one strided copy when the column blocks are equal;
        the received blocks (source-rank order = row order) ARE the column
        slab, so nothing is copied after the exchange."""
        L, r = self.L, self.rank
        nr = L.nrows[r]
        nc = L.ncols[r]
        x = x_rows.reshape(nr, L.M)
        if len(set(L.ncols)) == 1:
            send = x.reshape(nr, L.P, nc).transpose(0, 1).contiguous().reshape(-1)
        else:
            send = torch.cat([x[:, L.col0[q]:L.col0[q] + L.ncols[q]].reshape(-1) for q in range(L.P)])
        return self.comm.alltoall_flat(send, [nr * L.ncols[q] for q in range(L.P)],
                                       [L.nrows[q] * nc for q in range(L.P)])

    def cols_to_rows(self, x_cols: torch.Tensor) -> torch.Tensor:
        """Column slab (n0 x ncols_r) -> row slab (nrows_r x M). The row
        blocks of the column slab are already packed by destination; one
        strided copy interleaves the received column blocks."""
        L, r = self.L, self.rank
        nc = L.ncols[r]
        nr = L.nrows[r]
        out = self.comm.alltoall_flat(x_cols.reshape(-1), [L.nrows[q] * nc for q in range(L.P)],
                                      [nr * L.ncols[q] for q in range(L.P)])
        if len(set(L.ncols)) == 1:
            return out.reshape(L.P, nr, nc).transpose(0, 1).contiguous().reshape(-1)
        parts = torch.split(out, [nr * L.ncols[q] for q in range(L.P)])
        return torch.cat([parts[q].reshape(nr, L.ncols[q]) for q in range(L.P)], 1).reshape(-1)

    def halo(self, u_rows: torch.Tensor) -> torch.Tensor:
        """u with the neighbours' boundary rows above and below (zeros at the
        grid boundary, where the one-sided gradient never reads them)."""
        L, r = self.L, self.rank
        nr = L.nrows[r]
        u = u_rows.reshape(nr, L.M)
        empty = u[:0].reshape(-1)
        sends = [empty] * L.P
        if r > 0:
            sends[r - 1] = u[0].contiguous()
        if r < L.P - 1:
            sends[r + 1] = u[nr - 1].contiguous()
        recv = self.comm.alltoallv(sends, [L.M if abs(q - r) == 1 else 0 for q in range(L.P)])
        top = recv[r - 1] if r > 0 else torch.zeros(L.M, dtype=u.dtype, device=u.device)
        bot = recv[r + 1] if r < L.P - 1 else torch.zeros(L.M, dtype=u.dtype, device=u.device)
        return torch.cat([top.reshape(1, -1), u, bot.reshape(1, -1)], 0).reshape(-1)

    def route_records(self, key, w, cmask, mass, ops=None):
        """Sends each deposit record to the owners of the target rows it
        reaches; returns this rank's records in global source order with keys
        relative to its cells (global cell - (row0 - 1) * M). Records travel
        packed as (3 + d) float64 words: key bits, mass, d weights, mask.
        With CudaSlabOps the packing and unpacking are the bfm_slab_pf_route /
        _unpack kernels; otherwise (CPU test operators) torch ops."""
        L, r = self.L, self.rank
        if ops is not None and hasattr(ops, "pf_route"):
            rec = 3 + L.d
            packed, counts = ops.pf_route(key, w, cmask, mass)
            sends = list(torch.split(packed[:sum(counts) * rec], [c * rec for c in counts]))
            got = torch.cat(self.comm.alltoallv(sends))
            return ops.pf_unpack(got, got.numel() // rec)
        d = L.d
        nloc = mass.numel()
        dev = mass.device
        key64 = key.to(torch.int64) & 0xFFFFFFFF
        valid = key64 != L.N
        i0 = torch.where(valid, torch.div(key64, L.M, rounding_mode="floor"), torch.zeros_like(key64))
        own_lo = L.row_owner(i0)
        up_ok = valid & ((cmask.to(torch.int64) & 1) == 0) & (i0 + 1 < L.n0)
        own_hi = L.row_owner(torch.clamp(i0 + 1, max=L.n0 - 1))
        second = up_ok & (own_hi != own_lo)  # then own_hi == own_lo + 1 (no empty ranks)
        # copy slots 2s (owner of row i0) and 2s+1 (owner of row i0+1 when it
        # differs), destination P = none; a stable sort by destination keeps
        # every destination's records in source order
        slot_dst = torch.stack([torch.where(valid, own_lo, torch.full_like(own_lo, L.P)),
                                torch.where(second, own_hi, torch.full_like(own_hi, L.P))], 1)
        slot_dst = slot_dst.reshape(-1).to(torch.int16)
        sorted_dst, order = torch.sort(slot_dst, stable=True)
        bounds = torch.searchsorted(sorted_dst, torch.arange(L.P + 1, device=dev, dtype=torch.int16))
        counts = bounds[1:] - bounds[:-1]
        total = int(bounds[L.P].item())
        sid = torch.div(order[:total], 2, rounding_mode="floor")
        dst = sorted_dst[:total].to(torch.int64)
        row0s = torch.tensor(L.row0, dtype=torch.int64, device=dev)
        rel = key64[sid] - (row0s[dst] - 1) * L.M
        wv = w.reshape(d, nloc)
        rec = torch.empty((sid.numel(), 3 + d), dtype=torch.float64, device=dev)
        rec[:, 0] = rel.view(torch.float64) if rel.numel() else rec[:, 0]
        rec[:, 1] = mass[sid]
        rec[:, 2:2 + d] = wv[:, sid].t()
        rec[:, 2 + d] = cmask[sid].to(torch.float64)
        sends = list(torch.split(rec.reshape(-1), [int(c) * (3 + d) for c in counts.tolist()]))
        got = torch.cat(self.comm.alltoallv(sends)).reshape(-1, 3 + d)
        keys = got[:, 0].contiguous().view(torch.int64).to(torch.int32)
        masses = got[:, 1].contiguous()
        wcat = got[:, 2:2 + d].t().contiguous().reshape(-1)
        cmasks = got[:, 2 + d].to(torch.uint8)
        return keys, masses, wcat, cmasks

    def allgather(self, values) -> np.ndarray:
        return self.comm.allgather(values)


# ---------------------------------------------------------------- solver
class DistSolver:
    """bfm::Solver (solver.hpp:146-368) on P ranks; one instance per rank.

    mu_rows / nu_rows: this rank's rows of the densities (host arrays);
    validation and sigma_0 use the full arrays when given (every rank runs
    the same host checks, as the single-GPU solver does)."""

    def __init__(self, layout: SlabLayout, comm, ops, mu_rows, nu_rows,
                 config: Optional[SolverConfig] = None, mu_full=None, nu_full=None,
                 device: Optional[torch.device] = None):
        self.L = layout
        self.comm = comm
        self.ops = ops
        self.rank = comm.rank
        self.x = SlabExchange(layout, comm)
        self.cfg = config or SolverConfig()
        self.start = time.perf_counter()
        dev = device if device is not None else torch.device("cpu")
        self.device = dev
        if mu_full is not None and nu_full is not None:
            lib = load_library()
            mf = np.ascontiguousarray(mu_full, dtype=np.float64)
            nf = np.ascontiguousarray(nu_full, dtype=np.float64)
            c = self.cfg._c()
            _check(lib, lib.bfm_validate_inputs(layout.d, _extents(layout.shape),
                                                mf.ctypes.data_as(C.c_void_p),
                                                nf.ctypes.data_as(C.c_void_p), C.byref(c)))
        mu_rows = np.ascontiguousarray(mu_rows, dtype=np.float64).reshape(-1)
        nu_rows = np.ascontiguousarray(nu_rows, dtype=np.float64).reshape(-1)
        self.mu = torch.from_numpy(mu_rows.copy()).to(dev)
        self.nu = torch.from_numpy(nu_rows.copy()).to(dev)
        n = self.mu.numel()
        self.phi = torch.zeros(n, dtype=torch.float64, device=dev)
        self.psi = torch.zeros(n, dtype=torch.float64, device=dev)
        sups = self.x.allgather([float(mu_rows.max(initial=0.0)), float(nu_rows.max(initial=0.0))])
        sup = float(sups.max())
        self.sigma = self.cfg.sigma_init if self.cfg.sigma_init > 0.0 else 8.0 / sup
        self.last_pair = 0.0
        self.prev_dual = float("nan")
        self.probe_dual = 0.0
        self.probe_gn = 0.0
        self.dir = None
        self.fresh = False
        self.iteration = 0
        self.stall = 0
        self.trace: List[IterationStats] = []

    # operators over the decomposition
    def ctransform(self, u_rows: torch.Tensor) -> torch.Tensor:
        cols = self.x.rows_to_cols(u_rows)
        chain, q = self.ops.ct_cols(cols)
        chain_r = self.x.cols_to_rows(chain)
        q_r = self.x.cols_to_rows(q)
        return self.ops.ct_rows(chain_r, q_r)

    def solve_neumann(self, r_rows: torch.Tensor) -> torch.Tensor:
        y = self.ops.poisson_rows_forward(r_rows)
        yc = self.x.rows_to_cols(y)
        zc = self.ops.poisson_cols(yc)
        z = self.x.cols_to_rows(zc)
        return self.ops.poisson_rows_inverse(z)

    def pushforward_residual(self, u_rows, source, target) -> torch.Tensor:
        uh = self.x.halo(u_rows)
        key, w, cmask, _ = self.ops.pf_map(uh, source)
        keys, masses, ws, cms = self.x.route_records(key, w, cmask, source, self.ops)
        return self.ops.pf_gather(keys, masses, ws, cms, target)

    def _dot(self, a1, b1, a2=None, b2=None) -> float:
        parts = self.x.allgather(self.ops.dot(a1, b1, a2, b2))
        s1, c1 = merge_dd(parts[:, 0:2])
        v = (s1 + c1) * self.L.vol
        if a2 is not None:
            s2, c2 = merge_dd(parts[:, 2:4])
            v = v + (s2 + c2) * self.L.vol
        return v

    def pair_value(self) -> float:  # solver.hpp:240
        return self._dot(self.phi, self.nu, self.psi, self.mu)

    def ascent_direction(self, u, source, target):  # solver.hpp:245-260
        r = self.pushforward_residual(u, source, target)
        d = self.solve_neumann(r)
        gn = self._dot(r, d)
        return d, gn

    def ensure_probe(self) -> None:  # solver.hpp:264-280
        if self.fresh:
            return
        if self.cfg.mode == BACK_AND_FORTH:
            self.psi = self.ctransform(self.phi)
            v = self.pair_value()
            if v < self.last_pair - 1e-10:
                raise NumericalBlowup("solve: conjugation decreased the dual pair value")
            self.last_pair = v
            self.probe_dual = v
        else:
            self.probe_dual = self.last_pair
        self.dir, self.probe_gn = self.ascent_direction(self.psi, self.mu, self.nu)
        self.fresh = True

    def _update_sigma(self, sigma, increase, gn):  # solver.hpp:68-76
        c = self.cfg
        pred = sigma * gn
        if increase < c.beta_1 * pred:
            sigma *= c.alpha_2
        elif increase > c.beta_2 * pred:
            sigma *= c.alpha_1
        return max(sigma, c.sigma_min)

    def step(self) -> IterationStats:  # solver.hpp:189-207, 286-328
        self.ensure_probe()
        st = IterationStats(iteration=self.iteration + 1,
                            residual=math.sqrt(max(self.probe_gn, 0.0)))
        if self.cfg.mode == BACK_AND_FORTH:
            v2 = self.probe_dual
            st.sigma_first = self.sigma
            st.grad_norm_sq_first = self.probe_gn
            self.ops.axpy(self.phi, self.sigma, self.dir)
            self.psi = self.ctransform(self.phi)
            v3 = self.pair_value()
            st.increase_first = v3 - v2
            self.sigma = self._update_sigma(self.sigma, st.increase_first, self.probe_gn)
            self.phi = self.ctransform(self.psi)
            v4 = self.pair_value()
            if v4 < v3 - 1e-10:
                raise NumericalBlowup("solve: conjugation decreased the dual pair value")
            dir2, gn2 = self.ascent_direction(self.phi, self.nu, self.mu)
            st.sigma_second = self.sigma
            st.grad_norm_sq_second = gn2
            self.ops.axpy(self.psi, self.sigma, dir2)
            self.phi = self.ctransform(self.psi)
            v5 = self.pair_value()
            st.increase_second = v5 - v4
            self.sigma = self._update_sigma(self.sigma, st.increase_second, gn2)
            st.dual_value = v5
            self.last_pair = v5
        else:
            v1 = self.probe_dual
            st.sigma_first = self.sigma
            st.grad_norm_sq_first = self.probe_gn
            self.ops.axpy(self.phi, self.sigma, self.dir)
            self.psi = self.ctransform(self.phi)
            v2 = self.pair_value()
            st.increase_first = v2 - v1
            self.sigma = self._update_sigma(self.sigma, st.increase_first, self.probe_gn)
            self.phi = self.ctransform(self.psi)
            v3 = self.pair_value()
            if v3 < v2 - 1e-10:
                raise NumericalBlowup("solve: conjugation decreased the dual pair value")
            st.dual_value = v3
            self.last_pair = v3
        self.fresh = False
        self.iteration += 1
        if abs(st.dual_value - self.prev_dual) < 1e-12:
            self.stall += 1
        else:
            self.stall = 0
        self.prev_dual = st.dual_value
        self.trace.append(st)
        return st

    def run(self) -> Tuple[str, float]:  # solver.hpp:211-226 (stopping rules only)
        c = self.cfg
        while True:
            self.ensure_probe()
            residual = math.sqrt(max(self.probe_gn, 0.0))
            if c.tolerance >= 0.0 and residual <= c.tolerance:
                return TERMINATION_NAMES[0], residual
            if c.exact_cost is not None and c.exact_tolerance > 0.0 and \
                    abs(self.probe_dual - c.exact_cost) <= c.exact_tolerance:
                return TERMINATION_NAMES[3], residual
            if self.iteration >= c.max_iterations:
                return TERMINATION_NAMES[1], residual
            if self.stall >= 10:
                return TERMINATION_NAMES[2], residual
            self.step()

    def gather_rows(self, x_rows: torch.Tensor) -> Optional[np.ndarray]:
        """Full field on every rank (host array), rows in rank order."""
        L = self.L
        parts = self.comm.alltoallv([x_rows.reshape(-1)] * L.P)
        return torch.cat(parts).cpu().numpy().reshape(L.shape)

    def report(self, termination: str, residual: float) -> SolveReport:
        """solver.hpp:330-349: gauge fix with the reference's sequential Kahan
        integral (host), displacement map of psi, primal cost."""
        L = self.L
        phi = self.gather_rows(self.phi)
        psi = self.gather_rows(self.psi)
        s, c = 0.0, 0.0  # grid.hpp:124-133,179-183
        for v in phi.reshape(-1).tolist():
            y = v - c
            t = s + y
            c = (t - s) - y
            s = t
        shift = s * L.vol
        phi = phi - shift
        psi = psi + shift
        r0, nr = L.rows(self.rank)
        psi_rows = torch.from_numpy(np.ascontiguousarray(psi[r0:r0 + nr]).reshape(-1)).to(self.device)
        uh = self.x.halo(psi_rows)
        _, _, _, disp = self.ops.pf_map(uh, self.mu, want_disp=True)
        parts = self.x.allgather(self.ops.primal(disp, self.mu))
        ps, pc = merge_dd(parts[:, 0:2])
        primal = (ps + pc) * L.vol
        disp_full = [self.gather_rows(disp.reshape(L.d, -1)[a].contiguous()) for a in range(L.d)]
        return SolveReport(termination=termination, iterations=self.iteration,
                           dual_value=self.probe_dual, primal_cost=primal, residual=residual,
                           wall_seconds=time.perf_counter() - self.start, trace=list(self.trace),
                           phi=phi, psi=psi, map=np.stack(disp_full))


def spmd_local(layout: SlabLayout, fn, device: str = "cuda", ops_factory=None) -> list:
    """Runs fn(rank, comm, ops) for every rank of `layout` as threads of this
    process (LocalComm) and returns the per-rank results. ops_factory(layout,
    rank, device) defaults to CudaSlabOps."""
    parts = layout.P
    comms = LocalComm.group(parts)
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    make_ops = ops_factory or (lambda L, r, d: CudaSlabOps(L, r, d))
    results: list = [None] * parts
    errors: list = [None] * parts

    def body(r):
        try:
            if dev.type == "cuda":
                torch.cuda.set_device(dev)
                torch.cuda.set_stream(torch.cuda.Stream(dev))
            ops = make_ops(layout, r, dev)
            results[r] = fn(r, comms[r], ops)
            if dev.type == "cuda":
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errors[r] = e
            comms[r].sh.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(parts)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errors:
        if e is not None:
            raise e
    return results


def run_local(shape, mu, nu, config: Optional[SolverConfig] = None, parts: int = 2,
              steps: Optional[int] = None, device: str = "cuda") -> list:
    """The solver with `parts` ranks as threads of this process on one device
    (a check of the decomposition, not a performance path). Returns per-rank
    (DistSolver, SolveReport or None): after `steps` steps (plus the next
    probe), or after run() and the report."""
    L = SlabLayout(shape, parts)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    nu = np.ascontiguousarray(nu, dtype=np.float64)

    def fn(r, comm, ops):
        r0, nr = L.rows(r)
        s = DistSolver(L, comm, ops, mu[r0:r0 + nr], nu[r0:r0 + nr], config,
                       mu_full=mu, nu_full=nu, device=torch.device(device))
        if steps is None:
            term, res = s.run()
            return s, s.report(term, res)
        for _ in range(steps):
            s.step()
        s.ensure_probe()
        return s, None

    return spmd_local(L, fn, device)
