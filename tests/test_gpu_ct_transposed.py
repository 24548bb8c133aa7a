"""The dyadic c-transform's two forms of pass 0 — strided columns, and rows of
the transposed potential between two tiled transposes — must give identical
bits (the exact minimum does not depend on how the lines are laid out;
transforms.hpp:396-432). BFM_CT_T0 selects the form when a plan is built, so
each form runs in its own subprocess and reports SHA-256 digests; the
transposed form is also checked against the CPU restatement."""
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
SHAPES = [(64, 256), (512, 128), (256, 256), (2048, 1024), (32, 4096)]

SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic
out = []
for spec in sys.argv[2:]:
    shape = tuple(int(x) for x in spec.split("x"))
    phi = synthetic.c5_potential(shape)[0]
    psi = bfm.ctransform(phi)        # a generic potential
    phi2 = bfm.ctransform(psi)       # a c-concave one (collinear runs, exact ties)
    out.append(hashlib.sha256(psi.tobytes()).hexdigest() + hashlib.sha256(phi2.tobytes()).hexdigest())
print(" ".join(out))
"""


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not bfm.device_available():
        pytest.skip("no CUDA device")


def run_mode(t0):
    env = dict(os.environ)
    env["BFM_CT_T0"] = t0
    specs = ["x".join(map(str, s)) for s in SHAPES]
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT] + specs, env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.split()


def test_transposed_pass0_matches_strided_bitwise():
    a = run_mode("1")
    b = run_mode("0")
    assert len(a) == len(SHAPES) and a == b


def test_transposed_pass0_matches_restatement():
    shape = (128, 512)
    phi = synthetic.c5_potential(shape)[0]
    want = O.orc_ctransform(phi)
    env = dict(os.environ)
    env["BFM_CT_T0"] = "1"
    code = (SCRIPT.split("out = []")[0]
            + "shape = (128, 512)\nphi = synthetic.c5_potential(shape)[0]\n"
              "print(hashlib.sha256(bfm.ctransform(phi).tobytes()).hexdigest())\n")
    out = subprocess.run([sys.executable, "-c", code, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split()[-1] == hashlib.sha256(np.ascontiguousarray(want).tobytes()).hexdigest()
