"""Adversarial c-transform parity for the exact-hull kernel (dyadic grids,
csrc/ctransform.cu ct_dy_kernel) and the non-dyadic kernel, bitwise against
the unmodified reference (transforms.hpp:396-432, exact.hpp:167-179).

Each input targets one exact path of the kernel:
  * c-concave inputs (psi^c): exactly collinear runs -> local-corner drops
    and exact ties between hull corners (the common case inside a BFM step);
  * affine and constant lines: every interior point exactly collinear;
  * plateaus of a few distinct values: many exact ties between candidates;
  * magnitudes from 1e-300 (gradual underflow) to 1e+150, and lines mixing
    them: the 127-bit integer orientation path fails (exponent spread) and the
    error-free cascades / expansion fallback must decide;
  * signed zeros and ulp-level noise on a quadratic (near-degenerate hulls).
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def _grid(shape):
    return np.meshgrid(*[(np.arange(n) + 0.5) / n for n in shape], indexing="ij")


def _cases(shape, rng):
    g = _grid(shape)
    quad = sum(0.5 * x * x for x in g)
    out = {
        "affine": 0.3 * g[0] - 0.7 * g[-1] + 0.125,
        "constant": np.full(shape, 0.25),
        "zeros_signed": np.where(rng.uniform(size=shape) < 0.5, 0.0, -0.0),
        "plateaus": np.round(rng.uniform(-1, 1, shape) * 3) / 3,
        "quadratic_ulp_noise": quad * (1.0 + 2.0 ** -52 * rng.integers(-2, 3, shape)),
        "tiny": 1e-300 * rng.uniform(-1, 1, shape),
        "huge": 1e150 * rng.uniform(-1, 1, shape),
        "mixed_exponents": rng.uniform(-1, 1, shape) * 10.0 ** rng.integers(-30, 30, shape),
        "c5": synthetic.c5_potential(shape)[0],
    }
    # c-concave inputs: psi^c of the above (what every other c-transform of a
    # BFM iteration sees); their lines carry exactly collinear runs
    out["cconcave_c5"] = bfm.ctransform(out["c5"])
    out["cconcave_random"] = bfm.ctransform(rng.uniform(-1, 1, shape))
    out["cconcave_plateaus"] = bfm.ctransform(out["plateaus"])
    return out


@pytest.mark.parametrize("shape", [(256,), (2, 2), (4, 8), (64, 64), (256, 128), (1024, 256), (32, 32, 32),
                                   (16, 64, 8)])
def test_ctransform_adversarial_dyadic(shape, ref):
    rng = np.random.default_rng(7 * sum(shape) + len(shape))
    for name, phi in _cases(shape, rng).items():
        got = bfm.ctransform(phi)
        want = ref.ref_ctransform(phi)
        assert O.n_bit_diff(got, want) == 0, (shape, name)


@pytest.mark.parametrize("shape", [(96, 40), (48, 24, 12), (384, 6)])
def test_ctransform_adversarial_non_dyadic(shape, ref):
    rng = np.random.default_rng(11 * sum(shape))
    for name, phi in _cases(shape, rng).items():
        got = bfm.ctransform(phi)
        want = ref.ref_ctransform(phi)
        assert O.n_bit_diff(got, want) == 0, (shape, name)


def test_ctransform_bfm_iterates_full_size(ref):
    """Both inputs of a C3 iteration (phi and its c-concave image) at 4096^2
    after two BFM steps of the solver, bitwise vs the reference."""
    mu, nu = synthetic.c3()
    s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10))
    s.step()
    s.step()
    for phi in (s.phi(), s.psi()):
        got = bfm.ctransform(phi)
        want = ref.ref_ctransform(phi)
        assert O.n_bit_diff(got, want) == 0


def test_ctransform_c4_iterates_full_size(ref):
    """Both inputs of a C4 iteration at 384^3 (non-dyadic: the fixed-point
    exact evaluations) after two BFM steps, bitwise vs the reference."""
    mu, nu = synthetic.c4()
    s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10))
    s.step()
    s.step()
    for phi in (s.phi(), s.psi()):
        got = bfm.ctransform(phi)
        want = ref.ref_ctransform(phi)
        assert O.n_bit_diff(got, want) == 0
