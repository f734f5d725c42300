"""Edge and degenerate cases through the C-ABI against the oracle: one-qubit
and tiny registers (unfused kernels), empty ranges, single-wire transforms,
band 0 of the approximate QFT, p = 0 / p = 1 error injection, sigma = 0
angle gates, registers just above the fused-path threshold (9 local qubits),
odd register sizes whose tiles leave ragged passive parts, and reads of
single amplitudes at the ends of the state."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")

TOL = 1e-10


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


@pytest.fixture
def mk():
    made = []

    def make(n, state=None):
        h = Q.qsim_create(n)
        made.append(h)
        if state is not None:
            Q.qsim_set_state(h, 0, state)
        return h

    yield make
    for h in made:
        Q.qsim_destroy(h)


def get(h, n):
    return Q.qsim_get_state(h, 0, 1 << n)


def test_one_qubit_register(mk):
    h = mk(1)
    U = np.array([[0.6, 0.8j], [0.8j, 0.6]])
    Q.qsim_apply_1q(h, 0, U)
    assert np.max(np.abs(get(h, 1) - U[:, 0])) < 1e-15
    Q.qsim_qft(h, 0, 1)
    ref = U[:, 0].copy()
    O.qft(ref, 0, 1)
    assert np.max(np.abs(get(h, 1) - ref)) < 1e-15
    assert Q.qsim_measure(h, 0.0) == O.measure(ref, 0.0)


@pytest.mark.parametrize("n", [9, 10, 11, 13, 15])
def test_transforms_with_empty_and_single_wire_ranges(mk, n):
    psi = rand_state(n, n)
    h = mk(n, psi)
    ref = psi.copy()
    for lo, m in [(0, 0), (n - 1, 1), (0, 1), (n // 2, 0)]:
        Q.qsim_qft(h, lo, m, False)
        Q.qsim_fft(h, lo, m, True)
        Q.qsim_hadamard(h, lo, m)
        O.qft(ref, lo, m, False)
        O.qft(ref, lo, m, True)
        O.hadamard_range(ref, lo, m)
    assert np.max(np.abs(get(h, n) - ref)) < TOL


@pytest.mark.parametrize("n", [9, 11, 14])
def test_aqft_band_zero_and_ragged_sizes(mk, n):
    psi = rand_state(n, 3 * n)
    h = mk(n, psi)
    Q.qsim_aqft(h, 1, n - 1, 0, False)
    ref = psi.copy()
    O.aqft(ref, 1, n - 1, 0)
    assert np.max(np.abs(get(h, n) - ref)) < TOL


def test_error_injection_p_zero_and_one(mk):
    n = 10
    psi = rand_state(n, 8)
    h = mk(n, psi)
    assert Q.qsim_inject_errors(h, 5, 0.0, (1 << n) - 1, 0) == []
    assert np.array_equal(get(h, n), psi)
    ev = Q.qsim_inject_errors(h, 5, 1.0, (1 << n) - 1, 1)
    ref = psi.copy()
    rev = O.inject_paulis(ref, 5, 1, (1 << n) - 1, 1.0)
    assert ev == rev and len(ev) == n
    assert np.array_equal(get(h, n), ref)


def test_sigma_zero_angle_gates_equal_nominal_matrices(mk):
    n = 12
    psi = rand_state(n, 4)
    h = mk(n, psi)
    Q.qsim_set_gate_noise(h, 9, 0.0)
    ref = psi.copy()
    nz = O.Noise(seed=9, sigma=0.0)
    for q in range(n):
        a = O.haar_angles(3, q)
        Q.qsim_apply_angles(h, Q.QSIM_GATE_HAAR, a, 0, 0, q)
        O.apply_angles(ref, nz, O.HAAR, a, 0, 0, q)
    assert np.max(np.abs(get(h, n) - ref)) < TOL


def test_single_amplitude_reads_at_the_ends(mk):
    n = 16
    psi = rand_state(n, 6)
    h = mk(n, psi)
    Q.qsim_qft(h, 0, n)
    O.qft(psi, 0, n)
    for idx in (0, 1, (1 << n) - 2, (1 << n) - 1):
        got = Q.qsim_get_state(h, idx, 1)[0]
        assert abs(got - psi[idx]) < TOL
        assert Q.qsim_prob_index(h, idx) == pytest.approx(abs(psi[idx]) ** 2, abs=1e-15)


def test_flush_of_an_empty_queue_and_repeated_sync(mk):
    n = 14
    psi = rand_state(n, 1)
    h = mk(n, psi)
    for _ in range(3):
        Q.qsim_sync(h)
    assert np.array_equal(get(h, n), psi)
    assert abs(Q.qsim_norm(h) - 1) < 1e-13


def test_gate_list_equals_single_calls(mk):
    """qsim_apply_gates = the same gates through qsim_apply_1q / _ctrl /
    _angles one by one (gate noise and counter included); an invalid entry
    stops the list with its error and leaves the applied prefix."""
    n = 12
    psi = rand_state(n, 21)
    h1, h2 = mk(n, psi), mk(n, psi)
    for h in (h1, h2):
        Q.qsim_set_gate_noise(h, 5, 1e-2)
    rng = np.random.default_rng(3)
    gl = []
    for i in range(60):
        q = int(rng.integers(n))
        if i % 3 == 0:
            U = np.linalg.qr(rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2)))[0]
            gl.append(("matrix", q, U, 0, 0))
            Q.qsim_apply_1q(h2, q, U)
        elif i % 3 == 1:
            c = (q + 1 + int(rng.integers(n - 1))) % n
            U = np.array([[0, 1], [1, 0]], complex)
            gl.append(("matrix", q, U, 1 << c, 1 << c))
            Q.qsim_apply_ctrl(h2, 1 << c, 1 << c, q, U)
        else:
            a = [float(x) for x in rng.uniform(0, 6, 4)]
            gl.append(("angles", q, Q.QSIM_GATE_HAAR, a, 0, 0))
            Q.qsim_apply_angles(h2, Q.QSIM_GATE_HAAR, a, 0, 0, q)
    Q.qsim_apply_gates(h1, gl)
    assert np.max(np.abs(get(h1, n) - get(h2, n))) < 1e-13
    assert Q.qsim_get_gate_counter(h1) == Q.qsim_get_gate_counter(h2)
    with pytest.raises(Q.QsimError):
        Q.qsim_apply_gates(h1, [("matrix", 0, np.eye(2), 0, 0), ("matrix", n + 3, np.eye(2), 0, 0)])
