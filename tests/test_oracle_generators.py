"""Pins for the oracle's config generators that round 1 pinned only through
limits and moments: each is replayed here from the
config text and the DESIGN.md reading, with dense matrices and formulas
written out in numpy / Python, sharing nothing with oracle.c but the raw
Philox draws (themselves pinned to the published known-answer vectors in
test_oracle_rng.py).

* orc_cfg4 (BASELINE.json configs[4], reading R18): brickwork layout, Haar
  index l*n + q, CNOT direction (control = lower index), noisy NOT angles,
  Pauli rule -- dense 2^n x 2^n kron products at n = 5..7;
* orc_gaussian_state (configs[2], reading R19): Box-Muller branches (re = cos,
  im = sin), u01o for the radius and u01 for the angle, normalisation;
* orc_shor_base (configs[3], reading R11): the rejection rule.
"""
import math

import numpy as np
import pytest

import oracle as O

SEED4 = 5


# ------------------------------------------------------------------ written-out primitives
def u01(a):          # (a >> 11) 2^-53  (R1)
    return (a >> 11) * 2.0**-53


def u01o(a):         # ((a >> 11) + 1) 2^-53  (R1)
    return ((a >> 11) + 1) * 2.0**-53


def uint(a, m):      # floor(a m / 2^64)  (R1)
    return (a * m) >> 64


def normal(seed, tag, i, j):   # Box-Muller, cos branch (R1)
    a, b = O.draw(seed, tag, i, j)
    return math.sqrt(-2.0 * math.log(u01o(a))) * math.cos(2.0 * math.pi * u01(b))


def UR(t):
    return np.array([[math.cos(t), -math.sin(t)], [math.sin(t), math.cos(t)]], complex)


def UP1(p):
    return np.array([[1, 0], [0, np.exp(1j * p)]], complex)


def UP2(p):
    return np.array([[np.exp(1j * p), 0], [0, 1]], complex)


PAULI = {1: np.array([[0, 1], [1, 0]], complex), 2: np.array([[0, -1j], [1j, 0]], complex),
         3: np.array([[1, 0], [0, -1]], complex)}


def one_qubit(n, q, U):
    """I_{2^q} (x) U (x) I_{2^(n-1-q)} (qubit 0 = MSB, reading R3)."""
    return np.kron(np.eye(1 << q), np.kron(U, np.eye(1 << (n - 1 - q))))


def controlled(n, c, t, U):
    """Dense controlled-U: rows where bit c is 1 get U on t."""
    N = 1 << n
    M = np.zeros((N, N), complex)
    for j in range(N):
        if not (j >> (n - 1 - c)) & 1:
            M[j, j] = 1
            continue
        b = (j >> (n - 1 - t)) & 1
        j0 = j & ~(1 << (n - 1 - t))
        j1 = j0 | (1 << (n - 1 - t))
        M[j, j0] += U[b, 0]
        M[j, j1] += U[b, 1]
    return M


def cfg4_replay(n, layers, seed, sigma, p):
    """BASELINE.json configs[4] as the text states it: per layer a Haar gate on
    every qubit, a CNOT brickwork on (2k, 2k+1) for even layers and
    (2k+1, 2k+2) for odd ones, then a per-qubit Pauli draw; angle noise
    sigma on every angle, counter g in gate order (R14/R15/R18)."""
    psi = np.zeros(1 << n, complex)
    psi[0] = 1
    g = 0
    ev = []
    for l in range(layers):
        for q in range(n):
            i = l * n + q
            a0, b0 = O.draw(seed, O.TAG_HAAR, i, 0)
            a1, b1 = O.draw(seed, O.TAG_HAAR, i, 1)
            theta = math.acos(math.sqrt(u01(a0)))
            alpha, beta, gamma = 2 * math.pi * u01(b0), 2 * math.pi * u01(a1), 2 * math.pi * u01(b1)
            z = [sigma * normal(seed, O.TAG_OPNOISE, g, s) for s in range(4)]
            U = UP2(alpha + z[0]) @ UP1(beta + z[1]) @ UR(theta + z[2]) @ UP1(gamma + z[3])
            psi = one_qubit(n, q, U) @ psi
            g += 1
        first = 0 if l % 2 == 0 else 1
        for c in range(first, n - 1, 2):
            z = [sigma * normal(seed, O.TAG_OPNOISE, g, s) for s in range(2)]
            X = UR(math.pi / 2 + z[0]) @ UP1(math.pi + z[1])
            psi = controlled(n, c, c + 1, X) @ psi
            g += 1
        for q in range(n):
            u = u01(O.draw(seed, O.TAG_PAULI, l, q)[0])
            if u < p:
                k = 1 if u < p / 3 else 2 if u < 2 * p / 3 else 3
                psi = one_qubit(n, q, PAULI[k]) @ psi
                ev.append((l, q, k))
    return psi, ev


@pytest.mark.parametrize("n,layers,sigma,p", [(5, 4, 1e-3, 0.1), (6, 5, 1e-2, 0.2), (7, 3, 1e-3, 0.0),
                                              (6, 2, 0.0, 0.3)])
def test_cfg4_generator_dense_replay(n, layers, sigma, p):
    psi, ev = O.cfg4(n=n, layers=layers, seed=SEED4, sigma=sigma, p=p)
    ref, rev = cfg4_replay(n, layers, SEED4, sigma, p)
    assert ev == rev
    assert np.max(np.abs(psi - ref)) < 1e-13
    if p >= 0.1:
        assert len(ev) > 0   # the replay exercises the Pauli branch


def test_cfg4_brickwork_layout_matters():
    """A replay with the odd layers' pairs shifted (or the CNOT reversed) is far
    from the oracle: the comparison above can see those mistakes."""
    n, layers = 5, 2
    psi, _ = O.cfg4(n=n, layers=layers, seed=SEED4, sigma=0.0, p=0.0)
    ref, _ = cfg4_replay(n, layers, SEED4, 0.0, 0.0)
    assert np.max(np.abs(psi - ref)) < 1e-13
    # reversed CNOT on the first layer's first pair
    bad = np.zeros(1 << n, complex); bad[0] = 1
    for q in range(n):
        a0, b0 = O.draw(SEED4, O.TAG_HAAR, q, 0)
        a1, b1 = O.draw(SEED4, O.TAG_HAAR, q, 1)
        U = UP2(2 * math.pi * u01(b0)) @ UP1(2 * math.pi * u01(a1)) @ UR(math.acos(math.sqrt(u01(a0)))) \
            @ UP1(2 * math.pi * u01(b1))
        bad = one_qubit(n, q, U) @ bad
    X = UR(math.pi / 2) @ UP1(math.pi)
    bad_rev = controlled(n, 1, 0, X) @ bad
    good = controlled(n, 0, 1, X) @ bad
    assert np.max(np.abs(bad_rev - good)) > 1e-3


# ------------------------------------------------------------------ configs[2] Gaussian
@pytest.mark.parametrize("n,seed", [(3, 3), (6, 3), (5, 17)])
def test_gaussian_state_hand_box_muller(n, seed):
    """alpha_idx = Box-Muller(u1 = u01o(a), u2 = u01(b)) of draw(seed, GAUSS, idx, 0),
    re = cos branch, im = sin branch, then / sqrt(sum |alpha|^2) (R19)."""
    raw = []
    for idx in range(1 << n):
        a, b = O.draw(seed, O.TAG_GAUSS, idx, 0)
        r = math.sqrt(-2.0 * math.log(u01o(a)))
        t = 2.0 * math.pi * u01(b)
        raw.append(complex(r * math.cos(t), r * math.sin(t)))
    raw = np.array(raw)
    ref = raw / math.sqrt(math.fsum(abs(x) ** 2 for x in raw))
    got = O.gaussian_state(n, seed)
    assert np.max(np.abs(got - ref)) < 1e-15
    # the swapped branches / u01 radius would differ visibly
    alt = np.conj(ref) * 1j   # re <-> im
    assert np.max(np.abs(got - alt)) > 1e-3


def test_gaussian_state_first_amplitudes_golden():
    """The raw (unnormalised) first amplitude of configs[2]'s seed, from the
    Philox known answer for counter (0, 0, 0, GAUSS), key (3, 0)."""
    x = O.philox4x32_10([0, 0, 0, O.TAG_GAUSS], [3, 0])
    a, b = x[0] | (x[1] << 32), x[2] | (x[3] << 32)
    assert (a, b) == O.draw(3, O.TAG_GAUSS, 0, 0)
    r = math.sqrt(-2.0 * math.log(((a >> 11) + 1) * 2.0**-53))
    t = 2.0 * math.pi * ((b >> 11) * 2.0**-53)
    psi = O.gaussian_state(4, 3)
    raw0 = complex(r * math.cos(t), r * math.sin(t))
    # psi_0 / raw_0 is the common positive real normalisation factor
    ratio = psi[0] / raw0
    assert abs(ratio.imag) < 1e-15 and ratio.real > 0


# ------------------------------------------------------------------ configs[3] base
def shor_base_rule(seed, N):
    """R11: t = 0, 1, ...: a_t = 2 + uint(draw(seed, BASE, t, 0).a, N - 3), the
    first a_t with gcd(a_t, N) = 1."""
    t = 0
    while True:
        a = 2 + uint(O.draw(seed, O.TAG_BASE, t, 0)[0], N - 3)
        if math.gcd(a, N) == 1:
            return a
        t += 1


@pytest.mark.parametrize("seed,N", [(4, 1007), (4, 15), (1, 21), (9, 35), (4, 143), (7, 1023), (4, 4095)])
def test_shor_base_rule(seed, N):
    a = O.shor_base(seed, N)
    assert a == shor_base_rule(seed, N)
    assert 2 <= a <= N - 2 and math.gcd(a, N) == 1


def test_shor_base_configs3_value():
    assert O.shor_base(4, 1007) == 558 == shor_base_rule(4, 1007)
