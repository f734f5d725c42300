"""Pins for the oracle's circuits, reductions and config generators.

What fixes each value:
  * Hadamard transform closed form H_n|x> and H_n^2 = I;
  * QFT definition beta_x = 2^{-n/2} sum_y w^{xy} alpha_y
    on basis states and against numpy's FFT (a library routine);
  * Grover's closed form for -H V_f0 H V_fk: after t
    iterations alpha_k = sin((2t+1) theta), the rest cos((2t+1) theta)/sqrt(N-1);
  * order finding: classical modpow per basis state and the
    exact (Fejer-kernel) distribution of the exponent register;
  * norm preservation; measurement examples;
  * configs[0] replayed with brute-force dense matrices.
"""
import math

import numpy as np
import pytest

import oracle as O
from _closed_forms import fejer_distribution, order


def rand_state(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


# ------------------------------------------------------------------ H_n
@pytest.mark.parametrize("n", [1, 3, 6])
def test_hadamard_closed_form_every_basis_state(n):
    N = 1 << n
    for x in range(N):
        psi = np.zeros(N, complex); psi[x] = 1
        O.hadamard_range(psi, 0, n)
        ref = np.array([(-1) ** bin(x & y).count("1") for y in range(N)]) / math.sqrt(N)
        assert np.max(np.abs(psi - ref)) < 1e-15


def test_hadamard_twice_is_identity_and_zero_maps_uniform():
    rng = np.random.default_rng(1)
    psi = rand_state(10, rng); orig = psi.copy()
    O.hadamard_range(psi, 0, 10); O.hadamard_range(psi, 0, 10)
    assert np.max(np.abs(psi - orig)) < 1e-14
    z = np.zeros(1 << 12, complex); z[0] = 1
    O.hadamard_range(z, 0, 12)
    assert np.max(np.abs(z - 2.0**-6)) < 1e-16


def test_hadamard_spec_example():
    psi = np.zeros(4, complex); psi[1] = 1          # |01>
    O.hadamard_range(psi, 0, 2)
    assert np.allclose(psi, [0.5, -0.5, 0.5, -0.5], atol=1e-16)


# ------------------------------------------------------------------ QFT
@pytest.mark.parametrize("inverse", [False, True])
def test_qft_basis_state_closed_form(inverse):
    n = 5; N = 1 << n
    s = -1 if inverse else 1
    for y in range(N):
        psi = np.zeros(N, complex); psi[y] = 1
        O.qft(psi, 0, n, inverse)
        ref = np.exp(s * 2j * np.pi * ((np.arange(N) * y) % N) / N) / math.sqrt(N)
        assert np.max(np.abs(psi - ref)) < 1e-14


@pytest.mark.parametrize("n", [1, 2, 4, 7, 12])
def test_qft_matches_numpy_fft(n):
    rng = np.random.default_rng(n)
    N = 1 << n
    a = rand_state(n, rng)
    f = a.copy(); O.qft(f, 0, n, False)
    assert np.max(np.abs(f - np.fft.ifft(a) * math.sqrt(N))) < 1e-13
    b = a.copy(); O.qft(b, 0, n, True)
    assert np.max(np.abs(b - np.fft.fft(a) / math.sqrt(N))) < 1e-13


def test_qft_subrange_matches_fft_along_axis():
    rng = np.random.default_rng(5)
    n, lo, m = 9, 2, 4
    a = rand_state(n, rng)
    f = a.copy(); O.qft(f, lo, m, True)
    t = a.reshape(1 << lo, 1 << m, 1 << (n - lo - m))
    ref = (np.fft.fft(t, axis=1) / math.sqrt(1 << m)).reshape(-1)
    assert np.max(np.abs(f - ref)) < 1e-14


def test_qft_spec_example_n3():
    psi = np.zeros(8, complex); psi[0] = psi[4] = 1 / math.sqrt(2)
    O.qft(psi, 0, 3)
    ref = np.array([0.5 if x % 2 == 0 else 0 for x in range(8)])
    assert np.max(np.abs(psi - ref)) < 1e-15


def test_dft_samples_is_the_definition():
    rng = np.random.default_rng(3)
    n = 12
    a = rand_state(n, rng)
    xs = [0, 1, 77, 2048, 4095]
    for inv in (False, True):
        ref = (np.fft.fft(a) / 64) if inv else (np.fft.ifft(a) * 64)
        got = O.dft_samples(a, xs, inv)
        assert np.max(np.abs(got - ref[xs])) < 1e-14


def test_qft_gate_counter_counts_h_and_rd():
    # configs[2]: 28 H + 378 R_d (28*27/2) -> g = 406 after the circuit
    psi = np.zeros(1 << 6, complex); psi[0] = 1
    nz = O.Noise()
    O.qft(psi, 0, 6, False, nz)
    assert nz.g == 6 + 15


def test_gaussian_state_is_normalised_and_gaussian():
    psi = O.gaussian_state(14, 3)
    assert abs(O.norm(psi) - 1) < 1e-15
    z = psi * math.sqrt(1 << 14)          # ~ complex normal, E|z|^2 = 1 after normalisation
    assert abs(np.mean(z.real)) < 0.05 and abs(np.var(z.real) - 0.5) < 0.03


# ------------------------------------------------------------------ Grover
def test_grover_n2_single_iteration_is_exact():
    psi, tr = O.cfg1(n=2, seed=2, iters=1)
    k = O.grover_mark(2, 2)
    assert abs(psi[k] - 1) < 1e-15 and tr[0] == pytest.approx(1, abs=1e-15)


@pytest.mark.parametrize("n,iters", [(10, 80), (12, 60)])
def test_grover_full_vector_closed_form(n, iters):
    N = 1 << n
    psi, trace = O.cfg1(n=n, seed=2, iters=iters)
    k = O.grover_mark(2, n)
    th = math.asin(2 ** (-n / 2))
    t = np.arange(1, iters + 1)
    assert np.max(np.abs(trace - np.sin((2 * t + 1) * th) ** 2)) < 1e-12
    ref = np.full(N, math.cos((2 * iters + 1) * th) / math.sqrt(N - 1))
    ref[k] = math.sin((2 * iters + 1) * th)
    assert np.max(np.abs(psi - ref)) < 1e-12


def test_grover_n20_mark_and_optimum():
    k = O.grover_mark(2, 20)
    assert 0 <= k < 1 << 20
    K = math.floor(math.pi / 4 * math.sqrt(1 << 20))
    assert K == 804
    th = math.asin(2**-10)
    assert math.sin((2 * K + 1) * th) ** 2 == pytest.approx(0.999999756965, abs=1e-12)


# ------------------------------------------------------------------ order finding
def test_modmul_is_classical_modpow_on_basis_states():
    ne, nw, N, a = 5, 4, 15, 7
    n = ne + nw
    for e in range(1 << ne):
        for w in [1, 2, 7, 14, 15]:       # 15 >= N: identity (reading R10)
            psi = np.zeros(1 << n, complex); psi[(e << nw) | w] = 1
            for j in range(ne):
                c = O.powmod(a, 1 << j, N)
                O.modmul(psi, ne, nw, 1 << (ne - 1 - j), 1 << (ne - 1 - j), c, N)
            w2 = (w * pow(a, e, N)) % N if w < N else w
            assert psi[(e << nw) | w2] == 1


def test_modmul_is_a_bijection():
    rng = np.random.default_rng(0)
    n = 10
    psi = rand_state(n, rng)
    before = np.sort_complex(psi.copy())
    O.modmul(psi, 4, 6, 0b1010, 0b1000, 35, 61)
    assert np.array_equal(np.sort_complex(psi), before)


@pytest.mark.parametrize("N,a,ne,nw", [(15, 7, 8, 4), (15, 11, 8, 4), (21, 2, 9, 5),
                                       (35, 3, 10, 6), (1007, 558, 12, 10)])
def test_order_finding_matches_fejer_closed_form(N, a, ne, nw):
    P = O.cfg3(ne=ne, nw=nw, N=N, a=a, seed=4, sigma=0.0)
    ref = fejer_distribution(1 << ne, order(a, N))
    assert np.max(np.abs(P - ref)) < 1e-13
    assert abs(P.sum() - 1) < 1e-13


def test_spec_order_finding_examples():
    # N = 15: x = 11 -> y in {0, 128}; x = 7 -> {0, 64, 128, 192} (2l = 8)
    P = O.cfg3(ne=8, nw=4, N=15, a=11, seed=4, sigma=0.0)
    assert set(np.nonzero(P > 1e-12)[0]) == {0, 128}
    P = O.cfg3(ne=8, nw=4, N=15, a=7, seed=4, sigma=0.0)
    assert set(np.nonzero(P > 1e-12)[0]) == {0, 64, 128, 192}


def test_shor_base_for_config3():
    a = O.shor_base(4, 1007)
    assert 2 <= a <= 1005 and math.gcd(a, 1007) == 1


def test_noisy_order_finding_stays_close():
    # soft check: TV distance grows like sigma, small for 1e-3
    ne, nw, N = 10, 6, 35
    a = 3
    P0 = O.cfg3(ne=ne, nw=nw, N=N, a=a, seed=4, sigma=0.0)
    P1 = O.cfg3(ne=ne, nw=nw, N=N, a=a, seed=4, sigma=1e-3)
    P2 = O.cfg3(ne=ne, nw=nw, N=N, a=a, seed=4, sigma=1e-2)
    tv1, tv2 = 0.5 * np.abs(P1 - P0).sum(), 0.5 * np.abs(P2 - P0).sum()
    assert 0 < tv1 < 0.02 and tv1 < tv2 < 0.2
    assert abs(P1.sum() - 1) < 1e-13


# ------------------------------------------------------------------ reductions
def test_norm_and_probs_against_definitions():
    rng = np.random.default_rng(11)
    n = 12
    psi = rand_state(n, rng) * 1.3
    assert O.norm(psi) == pytest.approx(math.fsum(np.abs(psi) ** 2), rel=1e-15)
    for lo, m in [(0, 3), (4, 5), (9, 3), (0, 12)]:
        ref = (np.abs(psi) ** 2).reshape(1 << lo, 1 << m, -1).sum(axis=(0, 2))
        assert np.max(np.abs(O.probs(psi, lo, m) - ref)) < 1e-15


def test_pairwise_norm_is_accurate_at_scale():
    psi = O.gaussian_state(22, 9)
    assert abs(O.norm(psi) - 1) < 2e-15


def test_measurement_examples():
    u = np.full(4, 0.5, complex)                 # uniform n = 2, cumulative .25 .5 .75 1
    assert O.measure(u, 0.70) == 2
    assert O.measure(u, 0.0) == 0
    assert O.measure(u, 0.25) == 1               # sum_{j<i} <= r < sum_{j<=i}
    b = np.zeros(8, complex); b[5] = 1
    for r in (0.0, 0.3, 0.999999):
        assert O.measure(b, r) == 5
    z = np.zeros(8, complex); z[3] = 1 - 1e-17; z[6] = 0
    assert O.measure(z, 0.9999999999999999) == 3  # r >= total -> last nonzero


def test_measurement_frequencies_chi_square():
    rng = np.random.default_rng(2)
    psi = rand_state(3, rng)
    p = np.abs(psi) ** 2
    S = 20000
    counts = np.zeros(8)
    for s in range(S):
        a, _ = O.draw(123, O.TAG_MEASURE, s, 0)
        counts[O.measure(psi, O.u01(a))] += 1
    chi2 = ((counts - S * p) ** 2 / (S * p)).sum()
    assert chi2 < 24.3   # 7 dof, p = 0.001


# ------------------------------------------------------------------ configs[0]
def test_cfg0_replayed_with_dense_matrices():
    n, seed, ng = 10, 1, 200
    psi, kinds, qs = O.cfg0(n, seed, ng)
    ref = np.zeros(1 << n, complex); ref[0] = 1
    for g in range(ng):
        a, b = O.draw(seed, O.TAG_GATE, g, 0)
        if O.u01(a) < 0.7:
            q = O.uint(b, n)
            assert kinds[g] == 0 and qs[g][0] == q
            U = O.mat_angles(O.HAAR, O.haar_angles(seed, g))
            ref = np.kron(np.eye(1 << q), np.kron(U, np.eye(1 << (n - 1 - q)))) @ ref
        else:
            a2, b2 = O.draw(seed, O.TAG_PAIR, g, 0)
            c = O.uint(a2, n); t = O.uint(b2, n - 1); t += t >= c
            assert kinds[g] == 1 and tuple(qs[g]) == (t, c)
            idx = np.arange(1 << n)
            src = np.where((idx >> (n - 1 - c)) & 1, idx ^ (1 << (n - 1 - t)), idx)
            ref = ref[src]
    assert np.max(np.abs(psi - ref)) < 1e-13
    assert abs(O.norm(psi) - 1) < 1e-13
    assert 100 < (kinds == 0).sum() < 180


# ------------------------------------------------------------------ configs[4]
def test_cfg4_small_norm_and_noise_free_limit():
    psi, ev = O.cfg4(n=8, layers=4, seed=5, sigma=0.0, p=0.0)
    assert ev == [] and abs(O.norm(psi) - 1) < 1e-13
    psi2, ev2 = O.cfg4(n=8, layers=4, seed=5, sigma=1e-3, p=0.0)
    d = np.linalg.norm(psi2 - psi)
    assert 1e-5 < d < 0.1


def test_cfg4_forced_decoherence_events():
    # forcing variant: n = 12, 20 layers, p = 0.05 -> ~12 events
    psi, ev = O.cfg4(n=12, layers=20, seed=5, sigma=1e-3, p=0.05)
    assert 3 <= len(ev) <= 30
    assert all(0 <= l < 20 and 0 <= q < 12 and 1 <= k <= 3 for l, q, k in ev)
    assert abs(O.norm(psi) - 1) < 1e-13
    # event decisions are exactly the u01 < p rule of the channel
    for l in range(20):
        for q in range(12):
            u = O.u01(O.draw(5, O.TAG_PAULI, l, q)[0])
            hit = [e for e in ev if e[0] == l and e[1] == q]
            if u < 0.05:
                assert hit and hit[0][2] == (1 if u < 0.05 / 3 else 2 if u < 0.1 / 3 else 3)
            else:
                assert not hit
