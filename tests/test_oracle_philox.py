"""Pins for the oracle's random stream (reading R10): Philox4x32-10 against
library routines, bit-exact.  No GPU."""
import json
import os
import subprocess
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _h(s):
    return int(s, 16)


def test_random123_known_answers():
    kat = json.load(open(os.path.join(HERE, "golden", "philox_kat.json")))
    for v in kat["vectors"]:
        out = O.philox_raw([_h(c) for c in v["ctr"]], [_h(k) for k in v["key"]])
        assert out == [_h(o) for o in v["out"]]


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("pin") / "curand_pin")
    subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", "-o", exe,
                           os.path.join(HERE, "pins", "curand_philox_pin.cpp")])
    return exe


def test_against_curand_raw_block(curand_host):
    g = np.random.default_rng(123)
    rows = g.integers(0, 2**32, size=(300, 6), dtype=np.uint64)
    rows[0] = 0
    rows[1] = 2**32 - 1
    inp = "\n".join(" ".join("%x" % int(v) for v in r) for r in rows) + "\n"
    res = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for r, line in zip(rows, res):
        want = [int(w, 16) for w in line.split()]
        got = O.philox_raw([int(v) for v in r[:4]], [int(v) for v in r[4:]])
        assert got == want


def test_counter_layout_against_curand(curand_host):
    """Block (seed, trajectory i, step k) = Philox(ctr=(k_lo,k_hi,i_lo,i_hi), key=(seed_lo,seed_hi)):
    the cuRAND layout with subsequence = i and offset = 4k (SURVEY §8(c) pin table)."""
    triples = [(1, 0, 0), (1, 1, 0), (1, 0, 1), (2**64 - 1, 2**40 + 7, 2**33 + 5), (12345, 999_999, 17_000),
               (0, 2**64 - 1, 2**64 - 1)]
    inp = ""
    for s, i, k in triples:
        inp += "%x %x %x %x %x %x\n" % (k & 0xFFFFFFFF, k >> 32, i & 0xFFFFFFFF, i >> 32, s & 0xFFFFFFFF, s >> 32)
    res = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for (s, i, k), line in zip(triples, res):
        assert O.philox(s, i, k) == [int(w, 16) for w in line.split()]


def test_worked_example_seed1():
    """SURVEY §8(c) known answer (seed 1, i = 0, k = 0), itself re-derived above from cuRAND."""
    assert O.philox(1, 0, 0) == [0xE3E80670, 0xE50A0EBC, 0x95F222C0, 0xB615AA27]


def test_u53_mapping_exact():
    """u1 = (((r0<<32|r1)>>11)+1) 2^-53 in (0,1], u2 = ((r2<<32|r3)>>11) 2^-53 in [0,1): exact rationals."""
    for s, i, k in [(1, 0, 0), (7, 3, 11), (2**63 + 1, 2**35, 77)]:
        r = O.philox(s, i, k)
        w1 = (r[0] << 32) | r[1]
        w2 = (r[2] << 32) | r[3]
        u1, u2 = O.uniforms(s, i, k)
        assert Fraction(u1) == Fraction((w1 >> 11) + 1, 2**53)
        assert Fraction(u2) == Fraction(w2 >> 11, 2**53)
    # edge words: all-zero -> (2^-53, 0); all-ones -> (1, 1 - 2^-53)
    assert Fraction((0 >> 11) + 1, 2**53) == Fraction(float(2.0**-53))
    assert float(Fraction(((2**64 - 1) >> 11) + 1, 2**53)) == 1.0
    assert float(Fraction((2**64 - 1) >> 11, 2**53)) == 1.0 - 2.0**-53


def test_uniforms_distribution():
    from scipy import stats
    u = np.array([O.uniforms(9, i, k) for i in range(200) for k in range(100)])
    assert (u[:, 0] > 0).all() and (u[:, 0] <= 1).all() and (u[:, 1] >= 0).all() and (u[:, 1] < 1).all()
    assert stats.kstest(u[:, 0], "uniform").pvalue > 1e-3
    assert stats.kstest(u[:, 1], "uniform").pvalue > 1e-3
    # u1 and u2 of the same block are independent (correlation ~ 0)
    assert abs(np.corrcoef(u[:, 0], u[:, 1])[0, 1]) < 0.03
