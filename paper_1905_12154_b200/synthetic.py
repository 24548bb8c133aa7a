"""Seeded synthetic inputs for the BASELINE.json configs C1-C5.

No public dataset is involved: the reference's benchmark instances are
closed-form shapes (benchmark.hpp:27-43), and BASELINE.json's configs are
seeded random densities.

C1-C4 come from the library's shared generator (bfm_synthetic_densities,
csrc/synthetic.cpp): std::mt19937_64(seed), uniforms (rng()>>11)*2^-53, object
by object with fields in the listed order, unit-peak Gaussians
exp(-|x-c|^2 / (2 s^2)) summed with equal weights, closed cell-centre
indicators (io.hpp:407-420), Kahan normalisation (grid.hpp:151-164) — so a C++
driver regenerates the identical arrays. Test-sized helpers
(c1_like) and the C5 operator-sweep potentials use numpy's default_rng
(PCG64). Both the GPU and the CPU reference arm receive the identical float64
arrays.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

from . import axis_coords


def _shared(config: int, n: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    from . import synthetic_densities

    return synthetic_densities(config, n, seed)


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
    """C1: 3 Gaussians (centre ~U[0.2,0.8]^2, s ~U[0.05,0.15]) vs disc:0.5,0.5,0.3."""
    return _shared(1, n, seed)


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
    """C2: union of 5 rectangles vs 8 Gaussians masked to an annulus."""
    return _shared(2, n, seed)


def _dist2(shape, c) -> np.ndarray:
    coords = [axis_coords(n) for n in shape]
    d2 = np.zeros(shape)
    for a in range(len(shape)):
        sh = [1] * len(shape)
        sh[a] = shape[a]
        d2 = d2 + ((coords[a] - c[a]) ** 2).reshape(sh)
    return d2


def c3(n: int = 4096, seed: int = 3) -> Tuple[np.ndarray, np.ndarray]:
    """C3: 16 Gaussians x Bernoulli(0.5) mask of 64x64 blocks, independently for mu, nu."""
    return _shared(3, n, seed)


def c4(n: int = 384, seed: int = 4) -> Tuple[np.ndarray, np.ndarray]:
    """C4: 6 3-D Gaussians vs ball:0.5,0.5,0.5,0.3."""
    return _shared(4, n, seed)


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
