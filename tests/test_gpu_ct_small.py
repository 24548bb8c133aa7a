"""Small and oddly shaped dyadic grids through the exact-hull c-transform: every thread /
chunk layout the plan can pick for short lines (one to eight points per
thread, lines shorter than a warp, one-point axes' neighbours) against the
CPU restatement, on a generic potential and on its c-transform (exactly
collinear runs). Reference: transforms.hpp:396-432."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu

SHAPES = [(2, 2), (4, 4), (8, 8), (16, 16), (32, 32), (64, 64), (128, 128), (256, 256), (8, 256), (256, 8),
          (2, 256), (128, 2), (256,), (64,), (4, 4, 4), (8, 8, 8), (16, 16, 4),
          # long lines: the small-state form (lines of 4096 points and more) in 1-D, thin 2-D and 3-D
          # grids; lines too long for the staged form (16384 points) on the last axis and, through the
          # transposed pass 0, on axis 0 of a 2-D grid
          (4096,), (8192,), (8, 4096), (4096, 8), (2, 8192), (4, 4, 4096), (16384,), (4, 16384), (16384, 4)]


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("shape", SHAPES)
def test_small_dyadic_grids_bitwise(shape):
    rng = np.random.default_rng(sum(shape))
    phi = synthetic.c5_potential(shape)[0] + 0.01 * rng.standard_normal(shape)
    psi = bfm.ctransform(phi)
    want = O.orc_ctransform(phi)
    assert O.n_bit_diff(psi, want) == 0
    assert O.n_bit_diff(bfm.ctransform(psi), O.orc_ctransform(want)) == 0


@pytest.mark.parametrize("shape", [(32768,), (16384, 4, 4), (4, 16384, 4)])
def test_lines_beyond_shared_memory_are_rejected(shape):
    # 32768-point lines, and 16384-point lines on a strided axis of a 3-D grid, do not fit
    with pytest.raises(bfm.InvalidArgument):
        bfm.ctransform(np.zeros(shape))
