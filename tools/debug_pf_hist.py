"""Diagnostic (not a test): distribution of deposits per target node of the
pushforward at C3 (numpy restatement of the map, approximate)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402


def kdist(u, src):
    n = u.shape[0]
    h = 1.0 / n
    x = (np.arange(n) + 0.5) * h
    keys = []
    lo = []
    for a in range(2):
        g = np.gradient(u, h, axis=a, edge_order=1)
        mag = np.minimum(np.abs(g), np.sqrt(2.0))
        v = np.sign(g) * mag
        xa = x[:, None] if a == 0 else x[None, :]
        t = np.clip(xa - v, 0, 1)
        i = np.clip(np.floor(t * n - 0.5).astype(np.int64), 0, n - 2)
        lo.append(i)
    cell = lo[0] * n + lo[1]
    cell = cell[src > 0]
    cnt = np.bincount(cell.ravel(), minlength=n * n).reshape(n, n)
    K = cnt.copy()
    K[1:, :] += cnt[:-1, :]
    K[:, 1:] += cnt[:, :-1]
    K[1:, 1:] += cnt[:-1, :-1]
    K = K.ravel()
    for lo_, hi_ in [(0, 48), (49, 4096), (4097, 10**12)]:
        sel = (K >= lo_) & (K <= hi_)
        print(f"  K in [{lo_},{hi_}]: targets {sel.sum()}, deposits {K[sel].sum()}")
    top = np.sort(K)[-10:]
    print("  top K:", top.tolist(), "sum K:", K.sum())


mu, nu = synthetic.c3()
s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=100))
for it in range(3):
    psi = s.psi() if hasattr(s, "psi") else None
    phi = s.phi()
    print("iter", it)
    if psi is not None:
        kdist(psi, mu)
    kdist(phi, nu)
    s.step()
