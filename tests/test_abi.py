"""CPU-only checks of the C-ABI boundary: the library loads, exports every
entry point include/bfm_b200.h declares, validates inputs exactly like the
reference (solver.hpp:105-142, grid.hpp:60-76) and fails loudly without a
device (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1905_12154_b200 as bfm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bfm_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(bfm_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = bfm.load_library()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bfm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_update_sigma_kats_host_only():
    # test_solver.cpp:43-55 through the C ABI (pure host function)
    assert abs(bfm.update_sigma(1.0, 0.1, 1.0) - 0.8) <= 1e-15
    assert abs(bfm.update_sigma(1.0, 0.9, 1.0) - 1.25) <= 1e-15
    assert bfm.update_sigma(1.0, 0.5, 1.0) == 1.0
    assert bfm.update_sigma(0.012, 0.0, 1.0) == 0.01
    assert bfm.update_sigma(0.7, 0.0, 0.0) == 0.7


def _disc(n, cx, cy, r):
    x = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(x, x, indexing="ij")
    raw = ((X - cx) ** 2 + (Y - cy) ** 2 <= r * r).astype(float)
    return raw / (raw.sum() / (n * n))


def test_input_validation_matches_reference_error_types():
    # test_solver.cpp:255-290
    ok = _disc(16, 0.5, 0.5, 0.25)
    with pytest.raises(bfm.InfeasibleInput):
        bfm.Solver(2 * ok, ok)
    neg = ok.copy()
    neg[0, 3] = -0.5
    with pytest.raises(bfm.NegativeInput):
        bfm.Solver(neg, ok)
    nan = ok.copy()
    nan[0, 7] = np.nan
    with pytest.raises(bfm.InfeasibleInput):
        bfm.Solver(nan, ok)
    with pytest.raises(bfm.GridMismatch):
        bfm.Solver(ok, _disc(8, 0.5, 0.5, 0.25))
    with pytest.raises(bfm.InvalidArgument):
        bfm.Solver(ok, ok, bfm.SolverConfig(max_iterations=-2))
    with pytest.raises(bfm.InvalidArgument):
        bfm.Solver(ok, ok, bfm.SolverConfig(beta_1=0.8))
    with pytest.raises(bfm.InvalidArgument):
        bfm.ctransform(np.zeros((1, 4)))


@pytest.mark.skipif(bfm.device_available(), reason="a CUDA device is present")
def test_no_cpu_fallback_without_device():
    with pytest.raises(bfm.DeviceError):
        bfm.ctransform(np.zeros((8, 8)))
    with pytest.raises(bfm.DeviceError):
        bfm.Solver(_disc(16, 0.5, 0.5, 0.25), _disc(16, 0.5, 0.5, 0.25))


def test_facade_header_compiles():
    src = os.path.join(ROOT, "tests", "cxx", "facade_drive.cpp")
    if not os.path.exists(src):
        pytest.skip("no C++ facade driver")
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I" + os.path.join(ROOT, "include"), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_displacement_shape_is_checked():
    """A wrongly shaped displacement is a GridMismatch (require_same_grid in
    pushforward.hpp), not an out-of-bounds read of the C ABI."""
    mu = np.ones((8, 8))
    for bad in (np.zeros((8, 8)), np.zeros((2, 8, 4)), np.zeros((3, 8, 8))):
        with pytest.raises(bfm.GridMismatch):
            bfm.pushforward_density(bad, mu)
        with pytest.raises(bfm.GridMismatch):
            bfm.displacement_interpolant(bad, mu, 0.5)
        with pytest.raises(bfm.GridMismatch):
            bfm.primal_cost(bad, mu)


def test_solver_null_handles_fail_cleanly():
    lib = bfm.load_library()
    import ctypes as C

    assert lib.bfm_solver_iteration(None) == -1
    n = C.c_int()
    assert lib.bfm_solver_trace(None, None, 0, C.byref(n)) == 2
    assert lib.bfm_solver_step(None, None) == 2
    assert lib.bfm_solver_run(None, None) == 2
    v = C.c_double()
    assert lib.bfm_solver_dual_value(None, C.byref(v)) == 2


def test_synthetic_generator_is_deterministic_and_normalised():
    """The shared mt19937_64 generator (bfm_synthetic_densities): same bits
    twice, unit Kahan mass (grid.hpp:151-164), C3's 64x64 block masks."""
    a = bfm.synthetic_densities(3, 256, 3)
    b = bfm.synthetic_densities(3, 256, 3)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    for x in a:
        assert abs(np.sum(x) / x.size - 1.0) < 1e-12  # (integrate() needs the GPU)
        blocks = x.reshape(64, 4, 64, 4).max(axis=(1, 3))
        assert 0.2 < (blocks == 0).mean() < 0.8  # Bernoulli(0.5) blocks
    with pytest.raises(bfm.InvalidArgument):
        bfm.synthetic_densities(7, 64, 1)


@pytest.mark.parametrize("driver", ["facade_drive", "workspace_drive"])
def test_cpp_drivers_compile_against_the_facade(driver, tmp_path):
    """The reference-API drivers compile and link against the facade and the
    C ABI library here (they run on the GPU in test_gpu_parity.py)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1905_12154_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(root, "include"),
                        os.path.join(root, "tests", "cxx", driver + ".cpp"), "-L" + libdir,
                        "-l:libbfm_b200.so", "-Wl,-rpath," + libdir, "-o", str(tmp_path / driver)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
