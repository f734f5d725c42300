"""Pins for the oracle's counter-based RNG (reading R1).

The paper is silent on its generator ("Each experiment uses different initial
random seed"), so the pins are the generator's published
definition (known-answer vectors) and distribution properties.
"""
import math
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_known_answers(ctr, key, expect):
    assert O.philox4x32_10(ctr, key) == expect


def test_draw_packs_counter_and_key():
    # draw(seed, tag, i, j): key = (seed lo, seed hi), ctr = (i lo, i hi, j, tag)
    seed, tag, i, j = 0x0123456789ABCDEF, 7, 0xFEDCBA9876543210, 3
    x = O.philox4x32_10(
        [i & 0xFFFFFFFF, i >> 32, j, tag], [seed & 0xFFFFFFFF, seed >> 32]
    )
    a, b = O.draw(seed, tag, i, j)
    assert a == x[0] | (x[1] << 32)
    assert b == x[2] | (x[3] << 32)


def test_u01_and_uint_edges():
    assert O.u01(0) == 0.0
    assert O.u01((1 << 64) - 1) == 1.0 - 2.0**-53
    assert O.u01o(0) == 2.0**-53
    assert O.u01o((1 << 64) - 1) == 1.0
    assert O.uint(0, 1007) == 0
    assert O.uint((1 << 64) - 1, 1007) == 1006
    assert O.uint(1 << 63, 1 << 20) == 1 << 19
    # exact floor(a*m/2^64) against Python big integers
    rng = np.random.default_rng(0)
    for _ in range(200):
        a = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        m = int(rng.integers(1, 2**40))
        assert O.uint(a, m) == (a * m) >> 64


def test_u01_moments_and_uniformity():
    n = 40000
    u = np.array([O.u01(O.draw(11, O.TAG_GATE, i, 0)[0]) for i in range(n)])
    assert abs(u.mean() - 0.5) < 4 * math.sqrt(1 / 12 / n)
    assert abs(u.var() - 1 / 12) < 0.004
    hist, _ = np.histogram(u, bins=20, range=(0, 1))
    chi2 = ((hist - n / 20) ** 2 / (n / 20)).sum()
    assert chi2 < 43.8  # chi-square 19 dof, p = 0.001


def test_normal_moments():
    n = 40000
    z = np.array([O.normal(5, O.TAG_OPNOISE, i, 1) for i in range(n)])
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 0.03
    assert abs((z**4).mean() - 3.0) < 0.15  # Gaussian kurtosis


def test_streams_are_distinct():
    a = {O.draw(1, t, 0, 0) for t in range(1, 10)}
    assert len(a) == 9
    assert O.draw(1, 1, 0, 0) != O.draw(2, 1, 0, 0)
    assert O.draw(1, 1, 0, 0) != O.draw(1, 1, 0, 1)
    assert O.draw(1, 1, 0, 0) != O.draw(1, 1, 1 << 32, 0)
