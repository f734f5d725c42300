"""Pins for the oracle's error model (§3, §4.3).

The paper prints two closed forms for the |0><0| term after k applications of
H_n under each error model; trajectory averages of the oracle's primitives
must reproduce them within sampling error:
  * depolarizing channel:   ((1 + (1 - 4p/3)^k) / 2)^n
  * operational error:   ((1 + e^{-9 k sigma^2 / 4}) / 2)^n
with H(x, y) = U_R(pi/4 + x) U_P1(pi + y), fresh x, y ~ N(0, sigma^2) per
application.  A dropped Pauli, a wrong Pauli, a channel
applied to the wrong qubit set, or noise reused across applications moves
the mean by many standard errors.
"""
import math

import numpy as np

import oracle as O


def _mean_se(x):
    x = np.asarray(x)
    return x.mean(), x.std(ddof=1) / math.sqrt(len(x))


def test_depolarizing_ht_decay_law():
    n, p, k, trials = 3, 0.06, 4, 3000
    allq = (1 << n) - 1
    vals = []
    for t in range(trials):
        psi = np.zeros(1 << n, complex); psi[0] = 1
        for i in range(k):
            O.hadamard_range(psi, 0, n)
            O.inject_paulis(psi, seed=99, epoch=t * k + i, qmask=allq, p=p)
        vals.append(abs(psi[0]) ** 2)
    m, se = _mean_se(vals)
    law = ((1 + (1 - 4 * p / 3) ** k) / 2) ** n
    assert abs(m - law) < 4 * se, (m, law, se)


def test_depolarizing_law_paper_example_value():
    # survey value for n = 20, p = 1e-2, k = 2
    assert ((1 + (1 - 4 * 1e-2 / 3) ** 2) / 2) ** 20 == \
        __import__("pytest").approx(0.765934, abs=1e-6)


def test_operational_ht_decay_law():
    n, sigma, k, trials = 2, 0.15, 6, 3000
    nz = O.Noise(seed=7, sigma=sigma)
    vals = []
    for _ in range(trials):
        psi = np.zeros(1 << n, complex); psi[0] = 1
        for _i in range(k):
            for q in range(n):
                O.apply_angles(psi, nz, O.RP, [math.pi / 4, math.pi], 0, 0, q)
        vals.append(abs(psi[0]) ** 2)
    assert nz.g == trials * k * n
    m, se = _mean_se(vals)
    law = ((1 + math.exp(-9 * k * sigma**2 / 4)) / 2) ** n
    assert abs(m - law) < 4 * se, (m, law, se)


def test_operational_law_value_corrects_spec_example():
    # ((1 + e^{-9*100*1e-4/4}) / 2)^20 = 0.79953 (the exponent is -0.0225)
    v = ((1 + math.exp(-9 * 100 * 1e-4 / 4)) / 2) ** 20
    assert abs(v - 0.799527) < 1e-6


def test_depolarizing_p_zero_and_p_one():
    psi = np.zeros(2, complex); psi[0] = 1
    assert O.inject_paulis(psi, seed=1, epoch=0, qmask=1, p=0.0) == []
    assert psi[0] == 1
    # p = 1: every draw is an event; sigma_x|0> = |1>, sigma_y|0> = i|1>, sigma_z|0> = |0>
    seen = set()
    for e in range(60):
        psi = np.zeros(2, complex); psi[0] = 1
        ev = O.inject_paulis(psi, seed=1, epoch=e, qmask=1, p=1.0)
        assert len(ev) == 1
        k = ev[0][2]; seen.add(k)
        expect = {1: [0, 1], 2: [0, 1j], 3: [1, 0]}[k]
        assert np.array_equal(psi, np.array(expect, complex))
    assert seen == {1, 2, 3}


def test_depolarizing_event_rate_binomial():
    p, n, epochs = 0.01, 10, 4000
    psi = np.zeros(1 << n, complex); psi[0] = 1
    cnt = 0
    for e in range(epochs):
        cnt += len(O.inject_paulis(psi, seed=3, epoch=e, qmask=(1 << n) - 1, p=p))
    N = n * epochs
    assert abs(cnt - N * p) < 4 * math.sqrt(N * p * (1 - p))
