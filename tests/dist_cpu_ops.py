"""TEST INFRASTRUCTURE: a CPU stand-in for the rank-local operators of the
multi-GPU slab decomposition (paper_1905_12154_b200/dist.py, CudaSlabOps), so
the exchange logic (row/column transposes, halos, deposit-record routing,
rank-ordered scalar merges) runs under torch.distributed/gloo on CPU.

Each method restates the contract of the matching bfm_slab_* entry point
(include/bfm_b200.h) from the reference's semantics:
* c-transform passes: exact minimisation with Python Fractions
  (transforms.hpp:396-432; the last pass rounds the exact minimum toward -inf,
  -0 -> +0, exact.hpp:167-179). Tiny grids only.
* Poisson: the oracle's per-line DCT (oracle/bfm_oracle.cpp orc_dct_axis,
  orc_poisson_cols: the shared dct_line.h routine, poisson.hpp:87-106).
* map / locate / splat: pushforward.hpp:51-63,70-91,141-172 (sequential
  deposits in global source order, restricted to the rank's target rows).
* dot / primal: math.fsum partials (the driver only needs an accurate
  (hi, lo) pair per rank).
"""
from __future__ import annotations

import ctypes as C
import math
from fractions import Fraction

import numpy as np
import torch

import oracle_lib as O


def _coord(h: float, i: int) -> float:
    return (float(i) + 0.5) * h


def _g_exact(h: float, k: int, j: int) -> Fraction:
    """hs(x) + hs(y) - x*y exactly (transforms.hpp:253,374-375)."""
    x = _coord(h, k)
    y = _coord(h, j)
    return Fraction(0.5 * x * x) + Fraction(0.5 * y * y) - Fraction(x) * Fraction(y)


def _round_down(v: Fraction) -> float:
    f = float(v)
    if Fraction(f) > v:
        f = float(np.nextafter(f, -np.inf))
    return 0.0 if f == 0.0 else f


class CpuSlabOps:
    def __init__(self, layout, rank: int, device=None):
        self.L = layout
        self.rank = rank
        self.shape = layout.shape
        self.d = layout.d
        self.h = [1.0 / n for n in self.shape]
        self.row0, self.nrows = layout.rows(rank)
        self.col0, self.ncols = layout.cols(rank)
        self.launches = 0

    # ---- c-transform
    def ct_cols(self, phi_cols: torch.Tensor):
        L = self.L
        nc = self.ncols
        phi = phi_cols.numpy().reshape(L.n0, nc)
        chain = np.zeros((L.n0, nc), dtype=np.int32)
        q = np.zeros((L.n0, nc))
        h0 = self.h[0]
        for c in range(nc):
            for k in range(L.n0):
                best, bj = None, -1
                for j in range(L.n0):
                    v = _g_exact(h0, k, j) - Fraction(float(phi[j, c]))
                    if best is None or v < best:
                        best, bj = v, j
                chain[k, c] = bj
                q[k, c] = phi[bj, c]
        return torch.from_numpy(chain.reshape(-1)), torch.from_numpy(q.reshape(-1))

    def ct_rows(self, chain: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
        L = self.L
        nr = self.nrows
        rest = self.shape[1:]
        ch = chain.numpy().reshape((nr,) + rest)
        qq = q.numpy().reshape((nr,) + rest)
        out = np.zeros((nr,) + rest)
        h = self.h
        for i in range(nr):
            X0 = self.row0 + i
            if self.d == 2:
                for k1 in range(rest[0]):
                    best = None
                    for j1 in range(rest[0]):
                        v = _g_exact(h[0], X0, int(ch[i, j1])) + _g_exact(h[1], k1, j1) - Fraction(float(qq[i, j1]))
                        if best is None or v < best:
                            best = v
                    out[i, k1] = _round_down(best)
            else:
                n1, n2 = rest
                # pass 1 (axis 1) for every (k1, y2), then pass 2 (axis 2)
                v1 = [[None] * n2 for _ in range(n1)]
                for k1 in range(n1):
                    for y2 in range(n2):
                        best = None
                        for j1 in range(n1):
                            v = _g_exact(h[0], X0, int(ch[i, j1, y2])) + _g_exact(h[1], k1, j1) - \
                                Fraction(float(qq[i, j1, y2]))
                            if best is None or v < best:
                                best = v
                        v1[k1][y2] = best
                for k1 in range(n1):
                    for k2 in range(n2):
                        best = min(v1[k1][j2] + _g_exact(h[2], k2, j2) for j2 in range(n2))
                        out[i, k1, k2] = _round_down(best)
        return torch.from_numpy(out.reshape(-1))

    # ---- Poisson
    def _orc(self):
        lib = O.orc_lib()
        lib.orc_dct_axis.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        lib.orc_poisson_cols.argtypes = [C.c_int, C.c_void_p, C.c_long, C.c_int, C.c_void_p, C.c_void_p]
        return lib

    def _ext(self, shape):
        return (C.c_int * len(shape))(*shape)

    def poisson_rows_forward(self, x: torch.Tensor) -> torch.Tensor:
        a = np.ascontiguousarray(x.numpy().copy())
        shp = (self.nrows,) + self.shape[1:]
        lib = self._orc()
        for ax in range(self.d - 1, 0, -1):
            assert lib.orc_dct_axis(self.d, self._ext(shp), ax, 0, a.ctypes.data_as(C.c_void_p)) == 0
        return torch.from_numpy(a)

    def poisson_cols(self, x: torch.Tensor) -> torch.Tensor:
        a = np.ascontiguousarray(x.numpy())
        out = np.empty_like(a)
        lib = self._orc()
        assert lib.orc_poisson_cols(self.d, self._ext(self.shape), self.col0, self.ncols,
                                    a.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)) == 0
        return torch.from_numpy(out)

    def poisson_rows_inverse(self, x: torch.Tensor) -> torch.Tensor:
        a = np.ascontiguousarray(x.numpy().copy())
        shp = (self.nrows,) + self.shape[1:]
        lib = self._orc()
        for ax in range(1, self.d):
            assert lib.orc_dct_axis(self.d, self._ext(shp), ax, 1, a.ctypes.data_as(C.c_void_p)) == 0
        return torch.from_numpy(a)

    # ---- pushforward
    def _locate(self, n, h, x):  # pushforward.hpp:51-63
        c0 = _coord(h, 0)
        cl = _coord(h, n - 1)
        if x <= c0:
            return 0, True, 0.0
        if x >= cl:
            return n - 1, True, 0.0
        i = int(x * float(n) - 0.5)
        i = max(0, min(i, n - 2))
        while i + 1 < n - 1 and _coord(h, i + 1) <= x:
            i += 1
        while i > 0 and _coord(h, i) > x:
            i -= 1
        clo = _coord(h, i)
        chi = _coord(h, i + 1)
        return i, False, (x - clo) / (chi - clo)

    def pf_map(self, u_halo: torch.Tensor, source: torch.Tensor, want_disp: bool = False):
        L = self.L
        d = self.d
        M = L.M
        nr = self.nrows
        u = u_halo.numpy()
        src = source.numpy()
        nloc = nr * M
        key = np.zeros(nloc, dtype=np.int64)
        w = np.zeros((d, nloc))
        cmask = np.zeros(nloc, dtype=np.uint8)
        disp = np.zeros((d, nloc))
        gstride = [int(np.prod(self.shape[a + 1:])) for a in range(d)]
        diam = math.sqrt(d)
        for s in range(nloc):
            idx = list(np.unravel_index(s, (nr,) + self.shape[1:]))
            idx[0] += self.row0
            su = s + M
            dsp = [0.0] * d
            for a in range(d):
                n = self.shape[a]
                x = _coord(self.h[a], idx[a])
                st = gstride[a]
                inv_h = float(n)
                j = idx[a]
                if j == 0:
                    gr = (u[su + st] - u[su]) * inv_h
                elif j == n - 1:
                    gr = (u[su] - u[su - st]) * inv_h
                else:
                    gr = (u[su + st] - u[su - st]) * (0.5 * inv_h)
                mag = abs(gr)
                if not (mag < diam):
                    mag = diam
                v = -mag if gr < 0.0 else mag
                t = min(max(x - v, 0.0), 1.0)
                dsp[a] = t - x
                disp[a, s] = dsp[a]
            m = src[s]
            if m == 0.0:
                key[s] = L.N
                continue
            k = 0
            mask = 0
            for a in range(d):
                x = _coord(self.h[a], idx[a])
                lo, cl, whi = self._locate(self.shape[a], self.h[a], x + 1.0 * dsp[a])
                k += lo * gstride[a]
                if cl:
                    mask |= 1 << a
                w[a, s] = whi
            key[s] = k
            cmask[s] = mask
        return (torch.from_numpy(key.astype(np.int32)), torch.from_numpy(w.reshape(-1)),
                torch.from_numpy(cmask), torch.from_numpy(disp.reshape(-1)) if want_disp else None)

    def pf_num_cells(self) -> int:
        return (self.nrows + 1) * self.L.M

    def pf_gather(self, keys, mass, w, cmask, target) -> torch.Tensor:
        L = self.L
        d = self.d
        M = L.M
        nr = self.nrows
        nrec = keys.numel()
        kk = keys.numpy().astype(np.int64)
        ms = mass.numpy()
        ww = w.numpy().reshape(d, nrec)
        cm = cmask.numpy()
        rest = self.shape[1:]
        rho = np.zeros(nr * M)
        for r in range(nrec):  # global source order
            cr, rem = divmod(int(kk[r]), M)
            cell = [self.row0 - 1 + cr] + list(np.unravel_index(rem, rest))
            for b in range(1 << d):
                if b & int(cm[r]):
                    continue
                tgt = [cell[a] + ((b >> a) & 1) for a in range(d)]
                li = tgt[0] - self.row0
                if li < 0 or li >= nr:
                    continue
                wt = ms[r]
                for a in range(d):
                    wt *= ww[a, r] if (b >> a) & 1 else 1.0 - ww[a, r]
                if wt != 0.0:
                    t = int(np.ravel_multi_index([li] + tgt[1:], (nr,) + rest))
                    rho[t] += wt
        out = rho if target is None else target.numpy() - rho
        return torch.from_numpy(out)

    # ---- scalars / elementwise
    def dot(self, a1, b1, a2=None, b2=None):
        s1 = math.fsum((a1.numpy() * b1.numpy()).tolist())
        s2 = math.fsum((a2.numpy() * b2.numpy()).tolist()) if a2 is not None else 0.0
        return (s1, 0.0, s2, 0.0)

    def primal(self, disp, mu):
        d = self.d
        dv = disp.numpy().reshape(d, -1)
        m = mu.numpy()
        c = np.zeros_like(m)
        for a in range(d):
            c = c + 0.5 * dv[a] * dv[a]
        terms = (c * m)[m != 0.0]
        return (math.fsum(terms.tolist()), 0.0)

    def axpy(self, u, sigma, dvec):
        u.copy_(u + sigma * dvec)
