"""Host logic of the library's Shor post-processing (row f3; no GPU needed).

qsim_shor_candidates / qsim_shor_try / qsim_shor_prob_succ are plain host
code in libqsim; they are checked here against the same brute-force and
Table 5 pins as the oracle (tests/test_oracle_shor.py) and against the
oracle element by element.
"""
import math

import numpy as np
import pytest

import oracle as O
from _closed_forms import order
from test_oracle_shor import brute_candidates, table5

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")


def test_prob_succ_table5():
    for n, p, q, th, *_ in table5():
        inv = 1.0 / Q.qsim_shor_prob_succ(n, (p - 1) * (q - 1))
        assert th <= inv < th + 0.01
        assert Q.qsim_shor_prob_succ(n, (p - 1) * (q - 1)) == pytest.approx(
            O.shor_prob_succ(n, (p - 1) * (q - 1)), rel=1e-15)
    assert math.isnan(Q.qsim_shor_prob_succ(2, 1))


@pytest.mark.parametrize("N,m", [(15, 8), (35, 11), (143, 16), (21311, 30)])
def test_candidates(N, m):
    rng = np.random.default_rng(7 + N)
    M = 1 << m
    ys = [int(v) for v in rng.integers(1, M, 300)] + [1, M - 1, M // 2]
    for y in ys:
        got = Q.qsim_shor_candidates(y, m, N)
        assert got == O.shor_candidates(y, m, N)
        if N < 200:
            assert got == brute_candidates(y, m, N)
    assert Q.qsim_shor_candidates(0, m, N) == []
    with pytest.raises(Q.QsimError):
        Q.qsim_shor_candidates(1, 0, N)


def test_candidates_full_size_peaks():
    """At the paper's size (N = 21311, 2l = 30) the peak nearest k 2^30 / r
    recovers r / gcd(k, r) for every k (the continued-fraction guarantee)."""
    N, m = 21311, 30
    M = 1 << m
    x = 2
    r = order(x, N)
    for k in [1, 2, 3, 5, 7, r - 1, r // 2 + 1]:
        y = round(k * M / r)
        d = r // math.gcd(k, r)
        assert Q.qsim_shor_candidates(y, m, N)[-1] == d


@pytest.mark.parametrize("N", [15, 21, 35, 143, 221])
def test_try(N):
    for x in range(2, N):
        if math.gcd(x, N) != 1:
            continue
        r = order(x, N)
        for rr in range(1, 2 * r + 3):
            for g in (False, True):
                assert Q.qsim_shor_try(N, x, rr, g) == O.shor_try(N, x, rr, g)
