"""Test-only access to the CPU oracles (never imported by the product).

* ``ref``: oracle/_ref/libbfmref.so — the UNMODIFIED reference headers
  (/root/reference/proj/include/bfm) compiled with the FFTW-subset shim
  (oracle/fftw3.h) by oracle/Makefile. Travels to the GPU box as a built
  file; absent only if the reference was never present where it was built.
* ``orc``: oracle/liboracle.so — our independent CPU restatement
  (oracle/bfm_oracle.cpp).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

import paper_1905_12154_b200 as bfm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libbfmref.so")
ORC_PATH = os.path.join(ROOT, "oracle", "liboracle.so")

_ref = None
_orc = None


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            return None
        _ref = C.CDLL(REF_PATH)
        bfm._declare(_ref, "ref_")
        _ref.ref_ctransform.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _ref.ref_ctransform.restype = C.c_int
        _ref.ref_builtin_density.argtypes = [C.c_int, C.c_void_p, C.c_char_p, C.c_void_p]
        _ref.ref_normalize.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _ref.ref_hm1dot_norm_sq.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _ref.ref_config_default.argtypes = [C.c_void_p]
    return _ref


def orc_lib():
    global _orc
    if _orc is None:
        _orc = C.CDLL(ORC_PATH)
        for name in ("orc_ctransform", "orc_solve_neumann"):
            getattr(_orc, name).argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _orc.orc_map_from_conjugate.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        _orc.orc_pushforward_density.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _orc.orc_displacement_interpolant.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                      C.c_double, C.c_void_p]
        _orc.orc_integrate.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _orc.orc_run_steps.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        _orc.orc_update_sigma.restype = C.c_double
        _orc.orc_update_sigma.argtypes = [C.c_double, C.c_double, C.c_double, C.c_void_p]
        _orc.orc_last_error.restype = C.c_char_p
    return _orc


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _ext(shape):
    return (C.c_int * len(shape))(*shape)


def _chk(lib, rc, prefix):
    if rc != 0:
        raise bfm._ERRORS.get(rc, bfm.Error)(getattr(lib, prefix + "last_error")().decode())


class RefSolver(bfm.Solver):
    _prefix = "ref_"

    def __init__(self, mu, nu, config=None, exponents=None):
        super().__init__(mu, nu, config, _lib=ref_lib(), exponents=exponents)

    def launches(self):
        return 0


# ---- reference (unmodified headers) -------------------------------------
def ref_ctransform(phi, threads=0):
    lib = ref_lib()
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    out = np.empty_like(phi)
    _chk(lib, lib.ref_ctransform(phi.ndim, _ext(phi.shape), _p(phi), _p(out), threads), "ref_")
    return out


def ref_solve_neumann(rhs):
    lib = ref_lib()
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    out = np.empty_like(rhs)
    _chk(lib, lib.ref_solve_neumann(rhs.ndim, _ext(rhs.shape), _p(rhs), _p(out)), "ref_")
    return out


def ref_map_from_conjugate(u):
    lib = ref_lib()
    u = np.ascontiguousarray(u, dtype=np.float64)
    disp = np.empty((u.ndim,) + u.shape)
    _chk(lib, lib.ref_map_from_conjugate(u.ndim, _ext(u.shape), _p(u), 0, _p(disp)), "ref_")
    return disp


def ref_pushforward_density(disp, mu):
    lib = ref_lib()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    disp = np.ascontiguousarray(disp, dtype=np.float64)
    rho = np.empty_like(mu)
    _chk(lib, lib.ref_pushforward_density(mu.ndim, _ext(mu.shape), _p(disp), _p(mu), _p(rho)), "ref_")
    return rho


def ref_displacement_interpolant(disp, mu, t):
    lib = ref_lib()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    disp = np.ascontiguousarray(disp, dtype=np.float64)
    rho = np.empty_like(mu)
    _chk(lib, lib.ref_displacement_interpolant(mu.ndim, _ext(mu.shape), _p(disp), _p(mu), t, _p(rho)),
         "ref_")
    return rho


def ref_integrate(f, w=None):
    lib = ref_lib()
    f = np.ascontiguousarray(f, dtype=np.float64)
    v = C.c_double()
    wp = None if w is None else _p(np.ascontiguousarray(w, dtype=np.float64))
    _chk(lib, lib.ref_integrate(f.ndim, _ext(f.shape), _p(f), wp, C.byref(v)), "ref_")
    return v.value


def ref_primal_cost_cost(disp, mu, exponents):
    lib = ref_lib()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    disp = np.ascontiguousarray(disp, dtype=np.float64)
    ex = (C.c_double * 3)(*([float(e) for e in exponents] + [2.0] * (3 - len(exponents))))
    lib.ref_primal_cost_cost.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    v = C.c_double()
    _chk(lib, lib.ref_primal_cost_cost(mu.ndim, _ext(mu.shape), ex, _p(disp), _p(mu), C.byref(v)), "ref_")
    return v.value


def ref_primal_cost(disp, mu):
    lib = ref_lib()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    disp = np.ascontiguousarray(disp, dtype=np.float64)
    v = C.c_double()
    _chk(lib, lib.ref_primal_cost(mu.ndim, _ext(mu.shape), _p(disp), _p(mu), C.byref(v)), "ref_")
    return v.value


def ref_builtin(shape, spec):
    lib = ref_lib()
    out = np.empty(shape)
    _chk(lib, lib.ref_builtin_density(len(shape), _ext(shape), spec.encode(), _p(out)), "ref_")
    return out


def ref_update_sigma(sigma, inc, gn, config=None):
    return bfm.update_sigma(sigma, inc, gn, config, _lib_override=ref_lib(), _prefix="ref_")


# ---- our restatement ------------------------------------------------------
def orc_ctransform(phi):
    lib = orc_lib()
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    out = np.empty_like(phi)
    _chk(lib, lib.orc_ctransform(phi.ndim, _ext(phi.shape), _p(phi), _p(out)), "orc_")
    return out


def orc_solve_neumann(rhs):
    lib = orc_lib()
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    out = np.empty_like(rhs)
    _chk(lib, lib.orc_solve_neumann(rhs.ndim, _ext(rhs.shape), _p(rhs), _p(out)), "orc_")
    return out


def orc_map_from_conjugate(u):
    lib = orc_lib()
    u = np.ascontiguousarray(u, dtype=np.float64)
    disp = np.empty((u.ndim,) + u.shape)
    _chk(lib, lib.orc_map_from_conjugate(u.ndim, _ext(u.shape), _p(u), 0, _p(disp)), "orc_")
    return disp


def orc_pushforward_density(disp, mu):
    lib = orc_lib()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    disp = np.ascontiguousarray(disp, dtype=np.float64)
    rho = np.empty_like(mu)
    _chk(lib, lib.orc_pushforward_density(mu.ndim, _ext(mu.shape), _p(disp), _p(mu), _p(rho)), "orc_")
    return rho


def orc_integrate(f, w=None):
    lib = orc_lib()
    f = np.ascontiguousarray(f, dtype=np.float64)
    v = C.c_double()
    wp = None if w is None else _p(np.ascontiguousarray(w, dtype=np.float64))
    _chk(lib, lib.orc_integrate(f.ndim, _ext(f.shape), _p(f), wp, C.byref(v)), "orc_")
    return v.value


def orc_run_steps(mu, nu, iters):
    lib = orc_lib()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    nu = np.ascontiguousarray(nu, dtype=np.float64)
    phi = np.empty_like(mu)
    psi = np.empty_like(mu)
    duals = np.empty(iters)
    _chk(lib, lib.orc_run_steps(mu.ndim, _ext(mu.shape), _p(mu), _p(nu), iters, _p(phi), _p(psi),
                                _p(duals)), "orc_")
    return phi, psi, duals


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def n_bit_diff(a, b):
    return int(np.count_nonzero(bits(a) != bits(b)))


def ref_normalize(raw):
    lib = ref_lib()
    raw = np.ascontiguousarray(raw, dtype=np.float64)
    out = np.empty_like(raw)
    _chk(lib, lib.ref_normalize(raw.ndim, _ext(raw.shape), _p(raw), _p(out)), "ref_")
    return out


def ref_ctransform_cost(phi, exponents, threads=0):
    lib = ref_lib()
    lib.ref_ctransform_cost.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    out = np.empty_like(phi)
    ex = (C.c_double * 3)(*([float(e) for e in exponents] + [2.0] * (3 - len(exponents))))
    _chk(lib, lib.ref_ctransform_cost(phi.ndim, _ext(phi.shape), ex, _p(phi), _p(out), threads), "ref_")
    return out


def ref_map_from_conjugate_cost(u, exponents, side=0):
    lib = ref_lib()
    lib.ref_map_from_conjugate_cost.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                                C.c_void_p]
    u = np.ascontiguousarray(u, dtype=np.float64)
    disp = np.empty((u.ndim,) + u.shape)
    ex = (C.c_double * 3)(*([float(e) for e in exponents] + [2.0] * (3 - len(exponents))))
    _chk(lib, lib.ref_map_from_conjugate_cost(u.ndim, _ext(u.shape), ex, _p(u), side, _p(disp)), "ref_")
    return disp
