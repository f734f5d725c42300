"""Pins for the oracle's SURVEY.md §8(f) rows f1/f4: the approximate QFT,
sub-register (partial) measurement and the inner product / fidelity.

What fixes each value (readings R30-R32):
  * AQFT on a basis state |x>: the QFT circuit leaves output qubit m-1-j in
    (|0> + e^{i phi_j}|1>)/sqrt2 with phi_j = sum_d x_{j+d} pi / 2^d over the
    R_d it applies (d <= b), so the amplitudes are a closed-form product; the
    full band (b >= m-1) is the DFT definition; the
    fidelity to the exact QFT is prod_j |cos(delta_j / 2)| with delta_j the
    dropped phase, non-decreasing in b;
  * partial measurement: m = n is the full measurement;
    on |+>^k (x) |phi> the marginal is uniform, so y = floor(r 2^k) and the
    post-state is |y>|phi> exactly; a second measurement repeats y;
  * inner product: <e_i|e_j> = delta_ij, <psi|psi> = the (fsum-pinned) norm,
    <psi| e^{i t} psi> = e^{i t}, conjugate symmetry, closed-form overlaps of
    DFT basis vectors.
"""
import cmath
import math

import numpy as np
import pytest

import oracle as O


def rand_state(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def bit(x, q, m):
    """Value of qubit q (qubit 0 = MSB) of the m-bit value x."""
    return (x >> (m - 1 - q)) & 1


def aqft_basis_closed_form(m, x, b, inverse=False):
    sg = -1.0 if inverse else 1.0
    phi = []
    for j in range(m):
        s = 0.0
        for d in range(0, m - j):
            if d <= b:
                s += bit(x, j + d, m) * math.pi / 2 ** d
        phi.append(sg * s)
    out = np.empty(1 << m, complex)
    for y in range(1 << m):
        a = 1.0
        for j in range(m):
            if bit(y, m - 1 - j, m):        # after the swaps, qubit j sits at m-1-j
                a *= cmath.exp(1j * phi[j])
        out[y] = a / math.sqrt(1 << m)
    return out


# ------------------------------------------------------------------ AQFT
@pytest.mark.parametrize("m", [1, 3, 5])
@pytest.mark.parametrize("inverse", [False, True])
def test_aqft_basis_states_closed_form_every_band(m, inverse):
    for x in range(1 << m):
        for b in range(0, m + 1):
            psi = np.zeros(1 << m, complex)
            psi[x] = 1
            O.aqft(psi, 0, m, b, inverse)
            ref = aqft_basis_closed_form(m, x, b, inverse)
            assert np.max(np.abs(psi - ref)) < 1e-14, (x, b)


def test_aqft_full_band_is_the_dft_definition():
    m = 6
    w = cmath.exp(2j * math.pi / (1 << m))
    for x in (0, 1, 37, 63):
        psi = np.zeros(1 << m, complex)
        psi[x] = 1
        O.aqft(psi, 0, m, m - 1)
        ref = np.array([w ** (x * y) for y in range(1 << m)]) / math.sqrt(1 << m)
        assert np.max(np.abs(psi - ref)) < 1e-14


def test_aqft_band_zero_is_hadamard_then_bit_reversal():
    m = 4
    rng = np.random.default_rng(3)
    psi = rand_state(m, rng)
    a = psi.copy()
    O.aqft(a, 0, m, 0)
    ref = np.empty_like(psi)
    for y in range(1 << m):
        yr = int(format(y, f"0{m}b")[::-1], 2)
        ref[y] = sum(psi[x] * (-1) ** bin(x & yr).count("1") for x in range(1 << m)) / 4.0
    assert np.max(np.abs(a - ref)) < 1e-14


def test_aqft_fidelity_closed_form_and_monotone_in_band():
    m = 7
    for x in (1, 45, 127, 86):
        fids = []
        exact = np.zeros(1 << m, complex)
        exact[x] = 1
        O.qft(exact, 0, m)
        for b in range(m):
            psi = np.zeros(1 << m, complex)
            psi[x] = 1
            O.aqft(psi, 0, m, b)
            f = abs(O.inner(exact, psi))
            dropped = [sum(bit(x, j + d, m) * math.pi / 2 ** d for d in range(b + 1, m - j)) for j in range(m)]
            assert f == pytest.approx(math.prod(abs(math.cos(dl / 2)) for dl in dropped), abs=1e-13)
            fids.append(f)
        assert all(fids[i] <= fids[i + 1] + 1e-15 for i in range(len(fids) - 1))
        assert fids[-1] == pytest.approx(1.0, abs=1e-14)


def test_aqft_counts_only_applied_gates():
    m, b = 6, 2
    nz = O.Noise(seed=4, sigma=1e-3)
    psi = np.zeros(1 << m, complex)
    psi[0] = 1
    O.aqft(psi, 0, m, b, noise=nz)
    applied = m + sum(1 for j in range(m) for k in range(j + 1, m) if k - j <= b)
    assert nz.g == applied


def test_aqft_on_a_sub_register_acts_per_slice():
    """AQFT on qubits [lo, lo+m) of n qubits = the m-qubit AQFT on every slice
    of the other qubits (tensor structure)."""
    n, lo, m, b = 7, 2, 4, 1
    rng = np.random.default_rng(9)
    psi = rand_state(n, rng)
    a = psi.copy()
    O.aqft(a, lo, m, b)
    t = psi.reshape(1 << lo, 1 << m, 1 << (n - lo - m)).copy()
    for i in range(t.shape[0]):
        for k in range(t.shape[2]):
            v = np.ascontiguousarray(t[i, :, k])
            O.aqft(v, 0, m, b)
            t[i, :, k] = v
    assert np.max(np.abs(a - t.reshape(-1))) < 1e-14


# ------------------------------------------------------------------ partial measurement
def test_measure_range_full_register_is_measure():
    n = 6
    rng = np.random.default_rng(5)
    psi = rand_state(n, rng)
    for s in range(200):
        r = O.u01(O.draw(9, O.TAG_MEASURE, s, 0)[0])
        a = psi.copy()
        assert O.measure_range(a, 0, n, r, collapse=False) == O.measure(psi, r)


@pytest.mark.parametrize("k,lo", [(3, 0), (2, 4)])
def test_measure_range_uniform_marginal_closed_form(k, lo):
    """Qubits [lo, lo+k) in |+>^k, the rest in a fixed state: P(y) = 2^-k, so
    y = floor(r 2^k) and the post-state is |y> on the register, the rest untouched."""
    n = 7
    rng = np.random.default_rng(11)
    rest = rand_state(n - k, rng)
    plus = np.ones(1 << k) / math.sqrt(1 << k)
    hi = rest.reshape(1 << lo, -1)
    psi = np.zeros((1 << lo, 1 << k, 1 << (n - lo - k)), complex)
    for a in range(1 << lo):
        for y in range(1 << k):
            psi[a, y, :] = hi[a, :] * plus[y]
    psi = psi.reshape(-1)
    for r in (0.0, 0.124, 0.49, 0.61, 0.999):   # away from the 2^-k ties (R22)
        p = psi.copy()
        y = O.measure_range(p, lo, k, r)
        assert y == math.floor(r * (1 << k))
        ref = np.zeros((1 << lo, 1 << k, 1 << (n - lo - k)), complex)
        ref[:, y, :] = hi
        assert np.max(np.abs(p - ref.reshape(-1))) < 1e-14
        # a collapsed register measures the same value again, whatever r
        for r2 in (0.0, 0.3, 0.99):
            assert O.measure_range(p.copy(), lo, k, r2) == y


def test_measure_range_frequencies_follow_marginal():
    n, lo, m = 8, 3, 3
    rng = np.random.default_rng(2)
    psi = rand_state(n, rng)
    P = O.probs(psi, lo, m)
    counts = np.zeros(1 << m)
    trials = 4000
    for s in range(trials):
        r = O.u01(O.draw(21, O.TAG_MEASURE, s, 0)[0])
        counts[O.measure_range(psi.copy(), lo, m, r, collapse=False)] += 1
    chi2 = float(np.sum((counts - trials * P) ** 2 / (trials * P)))
    assert chi2 < 30.0           # 7 dof: p ~ 1e-4


# ------------------------------------------------------------------ inner product
def test_inner_basis_and_norm_and_phase():
    n = 5
    for i in (0, 3, 31):
        for j in (0, 3, 31):
            a = np.zeros(1 << n, complex); a[i] = 1
            b = np.zeros(1 << n, complex); b[j] = 1
            assert O.inner(a, b) == (1 if i == j else 0)
    rng = np.random.default_rng(4)
    psi = rand_state(n, rng) * 0.7
    assert O.inner(psi, psi).real == pytest.approx(O.norm(psi), abs=1e-15)
    t = 0.913
    assert O.inner(psi, psi * cmath.exp(1j * t)) == pytest.approx(cmath.exp(1j * t) * O.norm(psi), abs=1e-15)
    phi = rand_state(n, rng)
    assert O.inner(psi, phi) == pytest.approx(O.inner(phi, psi).conjugate(), abs=1e-15)
    assert abs(O.inner(rand_state(n, rng), rand_state(n, rng))) <= 1.0


def test_inner_of_fourier_vectors_closed_form():
    """<f_x|g> with f_x the DFT vector of frequency x and g = f_z shifted in
    phase by e^{i t y}: a geometric sum (written out here, not from numpy)."""
    m = 6
    N = 1 << m
    x, z, t = 5, 9, 0.37
    f = np.array([cmath.exp(2j * math.pi * x * y / N) for y in range(N)]) / math.sqrt(N)
    g = np.array([cmath.exp(2j * math.pi * z * y / N + 1j * t * y) for y in range(N)]) / math.sqrt(N)
    q = cmath.exp(1j * (2 * math.pi * (z - x) / N + t))
    ref = (1 - q ** N) / (1 - q) / N
    assert O.inner(f, g) == pytest.approx(ref, abs=1e-14)
