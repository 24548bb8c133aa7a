"""BFMG field files (reference io.hpp:242-348): little-endian "BFMG", u32 dim,
u32 extents, f64 spacings (1/n), f64 values row-major (last axis fastest)."""
from __future__ import annotations

import struct
from typing import Tuple

import numpy as np

from . import InvalidArgument, IoError


def write_bfmg(path: str, values: np.ndarray) -> None:
    a = np.ascontiguousarray(values, dtype="<f8")
    if not 1 <= a.ndim <= 3:
        raise InvalidArgument("bfmg: grids are 1-, 2- or 3-dimensional")
    with open(path, "wb") as f:
        f.write(b"BFMG")
        f.write(struct.pack("<I", a.ndim))
        f.write(struct.pack(f"<{a.ndim}I", *a.shape))
        f.write(struct.pack(f"<{a.ndim}d", *[1.0 / n for n in a.shape]))
        f.write(a.tobytes())


def read_bfmg(path: str) -> np.ndarray:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"bfmg: cannot open '{path}'") from e
    if len(data) < 8 or data[:4] != b"BFMG":
        raise IoError("bfmg: bad magic")
    (dim,) = struct.unpack_from("<I", data, 4)
    if not 1 <= dim <= 3:
        raise IoError("bfmg: unsupported dimension")
    off = 8
    if len(data) < off + 4 * dim:
        raise IoError("bfmg: truncated header")
    ext: Tuple[int, ...] = struct.unpack_from(f"<{dim}I", data, off)
    off += 4 * dim
    total = 1
    for e in ext:
        if e == 0 or e > (1 << 20):
            raise IoError("bfmg: implausible extent")
        total *= e
        if total > (1 << 31):
            raise IoError("bfmg: implausible size")
    if len(data) < off + 8 * dim:
        raise IoError("bfmg: truncated payload")
    sp = struct.unpack_from(f"<{dim}d", data, off)
    off += 8 * dim
    for a, n in enumerate(ext):
        h = 1.0 / n
        if abs(sp[a] - h) > 1e-9 * h:
            raise IoError("bfmg: spacing does not match a unit-domain grid")
    if len(data) < off + 8 * total:
        raise IoError("bfmg: truncated payload")
    return np.frombuffer(data, dtype="<f8", count=total, offset=off).reshape(ext).astype(np.float64)
