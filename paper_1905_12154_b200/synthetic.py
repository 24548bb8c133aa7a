"""Seeded synthetic inputs for the BASELINE.json configs C1-C5.

No public dataset is involved: the reference's benchmark instances are
closed-form shapes (benchmark.hpp:27-43), and BASELINE.json's configs are
seeded random densities. Draws use numpy's default_rng(seed) (PCG64), object
by object, fields in the listed order. Gaussians are unit-peak
exp(-|x-c|^2 / (2 s^2)) summed with equal weights, then normalised to unit
mass (grid.hpp:151-164). Indicators use the reference's closed cell-centre
membership (io.hpp:407-420). Both the GPU and the CPU reference arm receive
the identical float64 arrays.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

from . import axis_coords


def _normalize(raw: np.ndarray) -> np.ndarray:
    vol = 1.0
    for n in raw.shape:
        vol *= 1.0 / n
    mass = float(np.sum(raw, dtype=np.float64)) * vol
    if mass <= 0.0:
        raise ValueError("density has zero total mass")
    return np.ascontiguousarray(raw / mass)


def _gauss(shape, centers, sigmas) -> np.ndarray:
    d = len(shape)
    coords = [axis_coords(n) for n in shape]
    out = np.zeros(shape, dtype=np.float64)
    for c, s in zip(centers, sigmas):
        f = None
        for a in range(d):
            g = np.exp(-((coords[a] - c[a]) ** 2) / (2.0 * s * s))
            f = g if f is None else np.multiply.outer(f, g)
        out += f
    return out


def _ball(shape, center, radius) -> np.ndarray:
    """builtin_density disc/ball (io.hpp:407-414): d2 <= r*r, d2 summed in axis order."""
    d = len(shape)
    coords = [axis_coords(n) for n in shape]
    d2 = np.zeros(shape, dtype=np.float64)
    for a in range(d):
        dl = coords[a] - center[a]
        sh = [1] * d
        sh[a] = shape[a]
        d2 = d2 + (dl * dl).reshape(sh)
    return (d2 <= radius * radius).astype(np.float64)


def c1(n: int = 256, seed: int = 1) -> Tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    cs, ss = [], []
    for _ in range(3):
        cs.append(rng.uniform(0.2, 0.8, size=2))
        ss.append(rng.uniform(0.05, 0.15))
    mu = _normalize(_gauss((n, n), cs, ss))
    nu = _normalize(_ball((n, n), (0.5, 0.5), 0.3))
    return mu, nu


def c1_like(shape, seed: int = 1) -> Tuple[np.ndarray, np.ndarray]:
    """C1's recipe on any 2-D/3-D grid: 3 Gaussians vs a centred disc/ball
    (test-sized instances, e.g. the multi-GPU decomposition checks)."""
    d = len(shape)
    rng = np.random.default_rng(seed)
    cs, ss = [], []
    for _ in range(3):
        cs.append(rng.uniform(0.2, 0.8, size=d))
        ss.append(rng.uniform(0.05, 0.15))
    mu = _normalize(_gauss(tuple(shape), cs, ss))
    nu = _normalize(_ball(tuple(shape), (0.5,) * d, 0.3))
    return mu, nu


def c2(n: int = 1024, seed: int = 2) -> Tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    x = axis_coords(n)
    raw = np.zeros((n, n))
    for _ in range(5):
        w = rng.uniform(0.1, 0.4)
        h = rng.uniform(0.1, 0.4)
        x0 = rng.uniform(0.0, 1.0 - w)
        y0 = rng.uniform(0.0, 1.0 - h)
        m0 = (x >= x0) & (x <= x0 + w)
        m1 = (x >= y0) & (x <= y0 + h)
        raw[np.ix_(m0, m1)] = 1.0
    mu = _normalize(raw)
    cs, ss = [], []
    for _ in range(8):
        cs.append(rng.uniform(0.1, 0.9, size=2))
        ss.append(rng.uniform(0.02, 0.1))
    ca = rng.uniform(0.45, 0.55, size=2)
    g = _gauss((n, n), cs, ss)
    r = np.sqrt(_dist2((n, n), ca))
    g[(r < 0.15) | (r > 0.45)] = 0.0
    nu = _normalize(g)
    return mu, nu


def _dist2(shape, c) -> np.ndarray:
    coords = [axis_coords(n) for n in shape]
    d2 = np.zeros(shape)
    for a in range(len(shape)):
        sh = [1] * len(shape)
        sh[a] = shape[a]
        d2 = d2 + ((coords[a] - c[a]) ** 2).reshape(sh)
    return d2


def _masked_gauss(rng, n: int, k: int, block: int):
    cs, ss = [], []
    for _ in range(k):
        cs.append(rng.uniform(0.0, 1.0, size=2))
        ss.append(rng.uniform(0.01, 0.1))
    g = _gauss((n, n), cs, ss)
    nb = max(1, n // block)
    keep = rng.uniform(0.0, 1.0, size=(nb, nb)) >= 0.5
    if not keep.any():
        keep[0, 0] = True
    mask = np.kron(keep, np.ones((n // nb, n // nb), dtype=bool))
    g = np.where(mask, g, 0.0)
    if not (g > 0).any():
        g[mask] = 1.0
    return _normalize(g)


def c3(n: int = 4096, seed: int = 3) -> Tuple[np.ndarray, np.ndarray]:
    """16 Gaussians x Bernoulli(0.5) mask of 64x64-cell blocks, independently for mu, nu."""
    rng = np.random.default_rng(seed)
    block = max(1, n // 64)
    mu = _masked_gauss(rng, n, 16, block)
    nu = _masked_gauss(rng, n, 16, block)
    return mu, nu


def c4(n: int = 384, seed: int = 4) -> Tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    cs, ss = [], []
    for _ in range(6):
        cs.append(rng.uniform(0.0, 1.0, size=3))
        ss.append(rng.uniform(0.03, 0.12))
    mu = _normalize(_gauss((n, n, n), cs, ss))
    nu = _normalize(_ball((n, n, n), (0.5, 0.5, 0.5), 0.3))
    return mu, nu


def c5_potential(shape, seed: int = 5) -> Tuple[np.ndarray, np.ndarray]:
    """phi = |x|^2/2 + 0.05 P(x), P = sum_{m<32} cos(pi k_m . x + theta_m),
    k_m in {0..16}^d. Returns (phi, P)."""
    rng = np.random.default_rng(seed)
    d = len(shape)
    coords = [axis_coords(n) for n in shape]
    P = np.zeros(shape)
    for _ in range(32):
        k = rng.integers(0, 17, size=d)
        th = rng.uniform(0.0, 2.0 * math.pi)
        arg = np.zeros(shape)
        for a in range(d):
            sh = [1] * d
            sh[a] = shape[a]
            arg = arg + (math.pi * k[a] * coords[a]).reshape(sh)
        P += np.cos(arg + th)
    half = np.zeros(shape)
    for a in range(d):
        sh = [1] * d
        sh[a] = shape[a]
        half = half + (0.5 * coords[a] * coords[a]).reshape(sh)
    return np.ascontiguousarray(half + 0.05 * P), np.ascontiguousarray(P)


def c5_pushforward_potential(shape, seed: int = 5) -> np.ndarray:
    """u = -0.05 P * (0.05 / max|grad_h(0.05 P)|): maximum displacement 0.05
    (SURVEY Appendix B)."""
    _, P = c5_potential(shape, seed)
    g2 = np.zeros(shape)
    for a, n in enumerate(shape):
        g2 = g2 + (np.gradient(0.05 * P, 1.0 / n, axis=a)) ** 2
    scale = 0.05 / max(1e-300, float(np.sqrt(g2.max())))
    return np.ascontiguousarray(-0.05 * P * scale)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4}
