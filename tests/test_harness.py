"""Paper-case harness and BFMG I/O, host side: fixture
densities bitwise against the reference's builtin_density / normalize, error
behaviour, BFMG round trip and rejection of malformed files, CSV layout."""
import io
import struct

import numpy as np
import pytest

import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import benchmark as B
from paper_1905_12154_b200.bfmg import read_bfmg, write_bfmg


@pytest.mark.parametrize("case", B.standard_benchmark_cases(), ids=lambda c: c.name)
def test_case_densities_bitwise_vs_reference(case, ref):
    shape = (40, 36) if case.dim == 2 else (14, 12, 10)
    for spec in (case.mu_spec, case.nu_spec):
        raw = bfm.builtin_density(shape, spec)
        assert O.n_bit_diff(raw, ref.ref_builtin(shape, spec)) == 0
        assert O.n_bit_diff(bfm.normalize(raw), ref.ref_normalize(raw)) == 0


def test_builtin_and_normalize_errors():
    with pytest.raises(bfm.InvalidArgument):
        bfm.builtin_density((8, 8), "")
    with pytest.raises(bfm.InvalidArgument):
        bfm.builtin_density((8, 8), "blob:0.5,0.5,0.1")
    with pytest.raises(bfm.InvalidArgument):
        bfm.builtin_density((8, 8), "disc:0.5,0.5")
    with pytest.raises(bfm.InvalidArgument):
        bfm.builtin_density((8, 8), "ball:0.5,0.5,0.5,0.1")  # 3-D shape on a 2-D grid
    with pytest.raises(bfm.InvalidArgument):
        bfm.builtin_density((8, 8), "disc:0.5,0.5,-1")
    # '+' before a digit is an exponent, not a union
    a = bfm.builtin_density((8, 8), "disc:0.5,0.5,3e-1")
    b = bfm.builtin_density((8, 8), "disc:0.5,0.5,0.03e+1")
    assert (a == b).all() and a.sum() > 0
    with pytest.raises(bfm.NegativeInput):
        bfm.normalize(-np.ones((4, 4)))
    with pytest.raises(bfm.AllZeroInput):
        bfm.normalize(np.zeros((4, 4)))


def test_expected_iteration_table():
    assert B.expected_iterations("two_discs", 256, 1e-4) == (1, 5)
    assert B.expected_iterations("four_squares", 512, 1e-6) == (11, 15)
    assert B.expected_iterations("two_discs", 64, 1e-4) is None


def test_csv_layout():
    row = B.BenchmarkRow("two_discs", 128, 1e-4, bfm.BACK_AND_FORTH, 3, 0.5, 0.2500001, 0.25, True,
                         (1, 5), "ok")
    out = io.StringIO()
    B.write_benchmark_csv(out, [row])
    lines = out.getvalue().splitlines()
    assert lines[0] == ("case,n,tolerance,mode,iterations,seconds,dual_value,exact_cost,"
                        "expected_lo,expected_hi,status")
    assert lines[1] == "two_discs,128,0.0001,bfm,3,0.5,0.2500001,0.25,1,5,ok"


def test_bfmg_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    for shape in [(7,), (5, 6), (3, 4, 5)]:
        a = rng.standard_normal(shape)
        p = str(tmp_path / f"f{len(shape)}.bfmg")
        write_bfmg(p, a)
        b = read_bfmg(p)
        assert b.shape == a.shape and O.n_bit_diff(a, b) == 0
        raw = open(p, "rb").read()
        assert raw[:4] == b"BFMG" and struct.unpack_from("<I", raw, 4)[0] == len(shape)


def test_bfmg_rejects_malformed(tmp_path):
    p = str(tmp_path / "x.bfmg")
    write_bfmg(p, np.ones((4, 4)))
    raw = bytearray(open(p, "rb").read())
    for bad, what in [(b"XFMG" + raw[4:], "magic"), (raw[:20], "truncated"),
                      (raw[:4] + struct.pack("<I", 5) + raw[8:], "dimension")]:
        open(p, "wb").write(bytes(bad))
        with pytest.raises(bfm.IoError):
            read_bfmg(p)
    spoil = bytearray(raw)
    struct.pack_into("<d", spoil, 16, 0.3)  # spacing of axis 0 is not 1/4
    open(p, "wb").write(bytes(spoil))
    with pytest.raises(bfm.IoError):
        read_bfmg(p)
    with pytest.raises(bfm.IoError):
        read_bfmg(str(tmp_path / "missing.bfmg"))
