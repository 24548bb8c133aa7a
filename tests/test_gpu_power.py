"""Power costs c = sum_a |y_a - x_a|^p_a / p_a (cost.hpp:24-48; SURVEY §8(f)
#4) on the GPU against the unmodified reference's generic path."""
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


@pytest.mark.parametrize("shape,exps", [((96,), (1.5,)), ((64, 48), (1.5, 2.5)), ((48, 64), (3.0, 3.0)),
                                        ((40, 40), (2.0, 1.25)), ((12, 10, 8), (1.2, 2.0, 4.0)),
                                        ((16, 16, 16), (1.5, 1.5, 1.5))])
def test_power_ctransform_bitwise_vs_reference(shape, exps, ref):
    rng = np.random.default_rng(len(shape) * 7 + shape[0])
    for kind in range(3):
        if kind == 0:
            phi = rng.uniform(-1, 1, shape)
        elif kind == 1:
            phi = synthetic.c5_potential(shape)[0]
        else:  # plateaus: exact ties between many candidates
            phi = np.round(rng.uniform(-1, 1, shape) * 4) / 4
        got = bfm.ctransform(phi, exps)
        want = ref.ref_ctransform_cost(phi, exps)
        assert O.n_bit_diff(got, want) == 0, (shape, exps, kind)


def test_power_all_quadratic_is_the_shortcut():
    phi = synthetic.c5_potential((32, 24))[0]
    assert O.n_bit_diff(bfm.ctransform(phi, (2.0, 2.0)), bfm.ctransform(phi)) == 0


def test_power_rejects_bad_exponents():
    with pytest.raises(bfm.InvalidArgument):
        bfm.ctransform(np.zeros((8, 8)), (1.0, 2.0))
