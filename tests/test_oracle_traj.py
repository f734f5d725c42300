"""Pins for the oracle's noise-experiment trajectories (SURVEY.md §8(f) row
f2; R33-R36).

What fixes each value:
  * HT experiment: sigma = p = 0 and k even returns |0..0>
    exactly, k odd gives the uniform state; trajectory averages of
    |<0|psi>|^2 follow the paper's two closed forms ((1 + (1-4p/3)^k)/2)^n
     and ((1 + e^{-9k sigma^2/4})/2)^n;
  * Grover experiment: without errors the ancilla stays
    |-> and P(register = k) after t iterations is sin^2((2t+1) theta),
    sin theta = 2^{-n/2}, with the full register state in
    closed form;
  * QFT with decoherence: p = 0 is the QFT circuit with
    the same gate noise, bit for bit; for m = 2 from |00> with sigma = 0 the
    only injection point sits after R_1 where the state is |+>|0>, so the
    fidelity of a trajectory is |<+|P0|+>| |<0|P1|0>| and its mean is
    (1 - 2p/3)^2.
"""
import math

import numpy as np

import oracle as O


def _mean_se(x):
    x = np.asarray(x, float)
    return x.mean(), x.std(ddof=1) / math.sqrt(len(x))


# ------------------------------------------------------------------ HT
def test_ht_noiseless_even_and_odd():
    n = 5
    psi = O.traj_ht(n, 6, seed=3, sigma=0.0, p=0.0)
    assert abs(abs(psi[0]) ** 2 - 1) < 1e-12
    psi = O.traj_ht(n, 3, seed=3, sigma=0.0, p=0.0)
    assert np.max(np.abs(np.abs(psi) ** 2 - 1 / 32)) < 1e-12


def test_ht_depolarizing_average_is_the_papers_closed_form():
    n, k, p, T = 3, 6, 0.04, 3000
    vals = [abs(O.traj_ht(n, k, seed=1000 + t, sigma=0.0, p=p)[0]) ** 2 for t in range(T)]
    m, se = _mean_se(vals)
    law = ((1 + (1 - 4 * p / 3) ** k) / 2) ** n
    assert abs(m - law) < 4 * se, (m, law, se)


def test_ht_operational_average_is_the_papers_closed_form():
    n, k, sigma, T = 2, 8, 0.12, 3000
    vals = [abs(O.traj_ht(n, k, seed=5000 + t, sigma=sigma, p=0.0)[0]) ** 2 for t in range(T)]
    m, se = _mean_se(vals)
    law = ((1 + math.exp(-9 * k * sigma ** 2 / 4)) / 2) ** n
    assert abs(m - law) < 4 * se, (m, law, se)


def test_ht_trajectories_differ_only_through_the_seed():
    a = O.traj_ht(4, 4, seed=77, sigma=1e-2, p=0.1)
    b = O.traj_ht(4, 4, seed=77, sigma=1e-2, p=0.1)
    c = O.traj_ht(4, 4, seed=78, sigma=1e-2, p=0.1)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


# ------------------------------------------------------------------ Grover
def test_grover_noiseless_closed_form_with_ancilla():
    n, k, iters = 6, 41, 7
    psi, trace = O.traj_grover(n, k, iters, seed=1, sigma=0.0, p=0.0)
    th = math.asin(2 ** (-n / 2))
    for t in range(iters):
        assert abs(trace[t] - math.sin((2 * t + 3) * th) ** 2) < 1e-12
    # register amplitudes: sin((2T+1)th) on k, cos((2T+1)th)/sqrt(N-1) elsewhere,
    # times the ancilla |-> = (|0> - |1>)/sqrt2, up to one global sign
    N = 1 << n
    a = (2 * iters + 1) * th
    reg = np.full(N, math.cos(a) / math.sqrt(N - 1))
    reg[k] = math.sin(a)
    ref = np.kron(reg, np.array([1, -1]) / math.sqrt(2))
    s = np.sign(np.real(np.vdot(ref, psi)))
    assert np.max(np.abs(psi - s * ref)) < 1e-12


def test_grover_errors_keep_the_norm_and_change_the_trace():
    psi, trace = O.traj_grover(5, 7, 5, seed=9, sigma=0.05, p=0.05)
    assert abs(np.linalg.norm(psi) - 1) < 1e-12
    _, clean = O.traj_grover(5, 7, 5, seed=9, sigma=0.0, p=0.0)
    assert np.max(np.abs(trace - clean)) > 1e-6


# ------------------------------------------------------------------ QFT with decoherence
def test_qft_decoherent_without_depolarizing_is_the_qft_circuit():
    m = 6
    rng = np.random.default_rng(1)
    v = rng.normal(size=1 << m) + 1j * rng.normal(size=1 << m)
    v /= np.linalg.norm(v)
    a, b = v.copy(), v.copy()
    na, nb = O.Noise(seed=4, sigma=1e-3), O.Noise(seed=4, sigma=1e-3)
    O.qft_decoherent(a, 0, m, noise=na, p=0.0)
    O.qft(b, 0, m, noise=nb)
    assert np.array_equal(a, b) and na.g == nb.g


def test_qft_decoherent_two_qubit_fidelity_closed_form():
    p, T = 0.3, 4000
    ideal = np.zeros(4, complex)
    ideal[0] = 1
    O.qft(ideal, 0, 2)
    vals = []
    for t in range(T):
        psi = np.zeros(4, complex)
        psi[0] = 1
        O.qft_decoherent(psi, 0, 2, noise=O.Noise(seed=20000 + t, sigma=0.0), p=p)
        vals.append(abs(O.inner(ideal, psi)))
    m, se = _mean_se(vals)
    assert abs(m - (1 - 2 * p / 3) ** 2) < 4 * se, (m, se)
