"""Pins for the oracle's Shor semantic mode and post-processing (row f3).

Each check is fixed by something other than the oracle itself: Table 5 of
the paper, brute force over small integers, Legendre's theorem on continued
fractions, number theory of the order, and the closed-form QFT of a periodic
register.  PAPER.md:827-859 (algorithm), 896-903 (semantic mode), 907-920
(Prob_succ), 944-998 (Table 5 and the improvements).
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from _closed_forms import fejer_branch, order

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "shor_table5.txt")


def table5():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        n, p, q, th, orig, imp = line.split()
        rows.append((int(n), int(p), int(q), float(th), float(orig), float(imp)))
    return rows


def is_prime(v):
    return v > 1 and all(v % d for d in range(2, int(math.isqrt(v)) + 1))


def test_table5_rows_are_rsa_type():
    """n = p q with p, q prime, 14-15 bits."""
    for n, p, q, *_ in table5():
        assert n == p * q and is_prime(p) and is_prime(q)
        assert 14 <= n.bit_length() <= 15


def test_prob_succ_reproduces_table5_theoretical():
    """1/Prob_succ(n) with phi = (p-1)(q-1) and natural logs equals the
    Theoretical column, which the paper prints truncated to two decimals."""
    for n, p, q, th, *_ in table5():
        inv = 1.0 / O.shor_prob_succ(n, (p - 1) * (q - 1))
        assert th <= inv < th + 0.01, (n, inv, th)


def test_prob_succ_limits():
    # phi(n) = n - 1 (n prime): the step-2 term vanishes
    n = 10007
    pp = O.shor_prob_succ(n, n - 1)
    assert pp == pytest.approx(0.5 * 4 / math.pi**2 * math.exp(-0.5772156649015329) / math.log(math.log(n)),
                               rel=1e-14)
    # the bound is a probability and grows with the share of non-coprime x
    assert 0 < O.shor_prob_succ(21311, 21000) < O.shor_prob_succ(21311, 15000) < 1


def brute_candidates(y, m, N):
    """All r in [1, N) with a k >= 1, gcd(k, r) = 1, |y/2^m - k/r| <= 2^-(m+1)."""
    M = 1 << m
    out = []
    for r in range(1, N):
        for k in {(y * r) // M, (y * r) // M + 1}:
            if k >= 1 and math.gcd(k, r) == 1 and 2 * abs(y * r - k * M) <= r:
                out.append(r)
    return sorted(set(out))


def test_candidates_example():
    # 85/256 ~ 1/3; 128/256 = 1/2; 64/256 = 1/4 (N = 15, m = 8)
    assert O.shor_candidates(85, 8, 15) == [3]
    assert O.shor_candidates(128, 8, 15) == [2]
    assert O.shor_candidates(64, 8, 15) == [4]
    assert O.shor_candidates(0, 8, 15) == []


@pytest.mark.parametrize("N,m", [(15, 8), (21, 10), (35, 11), (143, 16)])
def test_candidates_equal_brute_force(N, m):
    """With N^2 <= 2^m every fraction within 1/2^(m+1) of y/2^m has
    |y/2^m - k/r| < 1/(2 r^2), so by Legendre's theorem it is a convergent:
    the convergent list equals the brute-force set (which has <= 1 element)."""
    rng = np.random.default_rng(N)
    M = 1 << m
    ys = list(range(1, min(M, 600))) + [int(v) for v in rng.integers(1, M, 400)]
    for y in ys:
        got = O.shor_candidates(y, m, N)
        assert got == brute_candidates(y, m, N), (y, got)
        assert len(got) <= 1


@pytest.mark.parametrize("N", [15, 21, 33, 35, 143, 221])
def test_try_with_true_order(N):
    """Steps 4-5 on the exact order r = ord_N(x): a factor exactly when r is
    even and x^(r/2) != -1 (mod N), and then it divides N."""
    for x in range(2, N):
        if math.gcd(x, N) != 1:
            continue
        r = order(x, N)
        f = O.shor_try(N, x, r)
        good = r % 2 == 0 and pow(x, r // 2, N) != N - 1
        if good:
            assert 1 < f < N and N % f == 0, (x, r, f)
        else:
            assert f == 0
        # the GCD check only adds tests: never a wrong factor
        for rr in range(1, 2 * r + 3):
            g = O.shor_try(N, x, rr, gcd_check=True)
            assert g == 0 or (1 < g < N and N % g == 0)
            if O.shor_try(N, x, rr) != 0:
                assert g != 0


def test_semantic_state_support_and_norm():
    """Uniform over {a : x^a = v mod N}: the arithmetic progression
    a0, a0 + r, ... with r = ord_N(x)."""
    for (m, x, N, v) in [(8, 7, 15, 4), (10, 2, 21, 8), (16, 5, 143, 125), (12, 3, 35, 27)]:
        psi = O.shor_semantic_state(m, x, N, v)
        r = order(x, N)
        a0 = next(a for a in range(r) if pow(x, a, N) == v)
        support = np.arange(a0, 1 << m, r)
        assert np.flatnonzero(psi).tolist() == support.tolist()
        assert np.allclose(psi[support], 1 / math.sqrt(len(support)), rtol=0, atol=1e-15)
        assert abs(np.vdot(psi, psi) - 1) < 1e-13


def test_semantic_qft_closed_form():
    """QFT of the periodic register: r | 2^m gives exact peaks 1/r at
    multiples of 2^m/r; otherwise the Fejer closed form of one branch."""
    m, x, N, v = 8, 7, 15, 4          # r = 4
    psi = O.shor_semantic_state(m, x, N, v)
    O.qft(psi, 0, m)
    P = np.abs(psi) ** 2
    peaks = np.zeros(1 << m)
    peaks[:: (1 << m) // 4] = 0.25
    assert np.allclose(P, peaks, atol=1e-14)
    for (m, x, N, v) in [(10, 2, 21, 8), (16, 5, 143, 125)]:
        psi = O.shor_semantic_state(m, x, N, v)
        O.qft(psi, 0, m)
        r = order(x, N)
        a0 = next(a for a in range(r) if pow(x, a, N) == v)
        c = len(range(a0, 1 << m, r))
        ref = fejer_branch(1 << m, r, c, np.arange(1 << m))
        assert np.allclose(np.abs(psi) ** 2, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("N,m", [(15, 8), (21, 10), (143, 16)])
def test_run_finds_factors(N, m):
    for run in range(12):
        for improved in (False, True):
            t, f = O.shor_run(N, m, 11, run, improved)
            assert t >= 1 and 1 < f < N and N % f == 0


def test_run_iterations_statistics():
    """Over many runs at N = 143: every run succeeds, the improved
    post-processing needs no more iterations on average than the original
    (same draws: it only adds checks), and the original mean stays below
    the paper's 1/Prob_succ bound (PAPER.md:907-920 is a lower bound on
    the per-iteration success probability)."""
    N, m, runs = 143, 16, 60
    orig = [O.shor_run(N, m, 3, r, False)[0] for r in range(runs)]
    imp = [O.shor_run(N, m, 3, r, True)[0] for r in range(runs)]
    assert all(t >= 1 for t in orig + imp)
    assert all(b <= a for a, b in zip(orig, imp))
    assert np.mean(orig) < 1 / O.shor_prob_succ(N, 120)


@pytest.mark.parametrize("improved", [False, True])
def test_run_tallies_are_consistent(improved):
    """Table 6 bookkeeping: every run ends with exactly
    one success; an iteration runs a check only after the earlier ones
    failed; the iteration count is the number of quantum iterations plus
    the step-2 ending."""
    N, m, runs = 437, 18, 40
    st = np.zeros(len(O.SHOR_STATS), np.int64)
    total = 0
    for r in range(runs):
        t, f = O.shor_run(N, m, 5, r, improved, 200, st)
        assert t >= 1 and N % f == 0
        total += t
    S = dict(zip(O.SHOR_STATS, st.tolist()))
    assert S["quantum"] + S["step2"] == total
    assert S["step2"] + S["basic_s"] + S["gcd_s"] + S["sf_s"] + S["lcm_s"] == runs
    if improved:
        assert S["quantum"] == S["basic_s"] + S["basic_f"] + S["neighbor_f"]
        assert S["gcd_s"] + S["gcd_f"] <= S["basic_f"]
        assert S["sf_s"] + S["sf_f"] <= S["basic_f"] - S["gcd_s"]
        assert S["lcm_s"] + S["lcm_f"] <= S["basic_f"] - S["gcd_s"] - S["sf_s"]
    else:
        assert S["neighbor_s"] == S["neighbor_f"] == S["gcd_s"] == S["sf_s"] == S["lcm_s"] == 0
        assert S["basic_s"] + S["basic_f"] <= S["quantum"]
