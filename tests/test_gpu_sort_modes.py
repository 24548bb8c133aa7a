"""The pushforward's two sorting paths (one-sweep radix sort with decoupled
look-back, and the multi-kernel passes) must give bit-identical densities:
both are stable sorts of the same (cell, source) pairs, so every target folds
its deposits in the reference's order (pushforward.hpp:141-178). The path is
chosen per process (BFM_PF_SORT), so each mode runs in its own subprocess and
reports a SHA-256 of the output; the default mode is checked against the CPU
restatement as well."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic
shape = tuple(int(x) for x in sys.argv[2].split("x"))
rng = np.random.default_rng(11)
u = synthetic.c5_pushforward_potential(shape)
mu = rng.uniform(0, 1, shape) * (rng.uniform(0, 1, shape) > 0.5)
disp = bfm.map_from_conjugate(u)
rho = bfm.pushforward_density(disp, mu)
# a concentrated map as well: long buckets, every gather tier
x = [(np.arange(n) + 0.5) / n for n in shape]
X = np.meshgrid(*x, indexing="ij")
u2 = sum(0.5 * Xi * Xi - 0.5 * Xi for Xi in X) * 0.97
rho2 = bfm.pushforward_density(bfm.map_from_conjugate(u2), mu)
# no mass at all (every key is the sentinel), and a single massive source
rho3 = bfm.pushforward_density(disp, np.zeros(shape))
one = np.zeros(shape)
one.flat[one.size // 3] = 2.5
rho4 = bfm.pushforward_density(disp, one)
assert not rho3.any() and abs(rho4.sum() - 2.5) < 1e-12
print(hashlib.sha256(rho.tobytes()).hexdigest(), hashlib.sha256(rho2.tobytes()).hexdigest(),
      hashlib.sha256(rho4.tobytes()).hexdigest())
"""


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def run_mode(mode, shape):
    env = dict(os.environ)
    env.pop("BFM_PF_SORT", None)
    if mode:
        env["BFM_PF_SORT"] = mode
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, "x".join(map(str, shape))], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.split()


@pytest.mark.parametrize("shape", [(1536, 1024), (160, 160, 96), (100000,), (37, 23)])
def test_sort_paths_agree_bitwise(shape):
    a = run_mode("onesweep", shape)
    b = run_mode("legacy", shape)
    assert a == b


def test_default_path_matches_restatement():
    shape = (700, 900)
    rng = np.random.default_rng(3)
    u = synthetic.c5_pushforward_potential(shape)
    mu = rng.uniform(0, 1, shape) * (rng.uniform(0, 1, shape) > 0.3)
    disp = bfm.map_from_conjugate(u)
    assert O.n_bit_diff(bfm.pushforward_density(disp, mu), O.orc_pushforward_density(disp, mu)) == 0
