"""Pins for the oracle's evolution kernels and gate matrices (§2.2, §3).

Each kernel is checked against a brute-force 2^n x 2^n matrix built here with
numpy from the paper's definitions -- X = I_{2^i} (x) U (x) I_{2^{n-1-i}}
(caption "Total unitary matrix", reading R3) and the CTX row
rule -- never from the oracle's own code.  General
(non-unitary, non-symmetric) complex matrices are used so that a transposed
operand or a swapped u12/u21 cannot pass.
"""
import itertools

import numpy as np
import pytest

import oracle as O


def rand_state(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def rand_mat(rng):
    return rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))


def dense_X(n, q, U):
    return np.kron(np.eye(1 << q), np.kron(U, np.eye(1 << (n - 1 - q))))


def dense_CTX(n, ctrl, vals, q, U):
    """Row rule of PAPER.md:366-371 generalised to several controls."""
    X = dense_X(n, q, U)
    Id = np.eye(1 << n)
    M = np.empty_like(X)
    for j in range(1 << n):
        ok = all(((j >> (n - 1 - c)) & 1) == ((vals >> c) & 1) for c in ctrl)
        M[j] = X[j] if ok else Id[j]
    return M


@pytest.mark.parametrize("n", [1, 2, 3, 5, 6])
def test_apply_1q_equals_dense_X(n):
    rng = np.random.default_rng(100 + n)
    for q in range(n):
        U = rand_mat(rng)
        psi = rand_state(n, rng)
        ref = dense_X(n, q, U) @ psi
        O.apply_1q(psi, q, U)
        assert np.max(np.abs(psi - ref)) < 1e-13


def test_apply_1q_in_place_uses_old_values():
    # storing t1 first would give (x u11 + y u12) u21 + y u22
    U = np.array([[1, 2], [3, 4]], dtype=complex)
    psi = np.array([1.0, 10.0], dtype=complex)
    O.apply_1q(psi, 0, U)
    assert psi[0] == 21 and psi[1] == 43


@pytest.mark.parametrize("n", [2, 3, 4, 6])
def test_apply_ctrl_equals_row_rule(n):
    rng = np.random.default_rng(200 + n)
    for q in range(n):
        others = [c for c in range(n) if c != q]
        for k in range(1, min(3, len(others)) + 1):
            for ctrl in itertools.combinations(others, k):
                vals_bits = rng.integers(0, 2, size=k)
                mask = sum(1 << c for c in ctrl)
                vals = sum(int(b) << c for b, c in zip(vals_bits, ctrl))
                U = rand_mat(rng)
                psi = rand_state(n, rng)
                ref = dense_CTX(n, ctrl, vals, q, U) @ psi
                O.apply_ctrl(psi, mask, vals, q, U)
                assert np.max(np.abs(psi - ref)) < 1e-13


def test_spec_examples_cnot_and_not():
    X = [[0, 1], [1, 0]]
    psi = np.zeros(4, complex); psi[0] = 1
    O.apply_1q(psi, 0, X)                 # NOT on qubit 0 of |00> -> |10> (index 2)
    assert psi[2] == 1
    psi = np.zeros(4, complex); psi[2] = 1
    O.apply_ctrl(psi, 1, 1, 1, X)          # CNOT(q0 -> q1) on |10> -> |11>
    assert psi[3] == 1
    psi = np.zeros(4, complex); psi[0] = 1
    O.apply_ctrl(psi, 1, 1, 1, X)          # control not satisfied
    assert psi[0] == 1


@pytest.mark.parametrize("n", [2, 3, 5])
def test_swap_is_bit_exchange(n):
    rng = np.random.default_rng(300 + n)
    for q1, q2 in itertools.combinations(range(n), 2):
        psi = rand_state(n, rng)
        ref = np.empty_like(psi)
        for j in range(1 << n):
            b1 = (j >> (n - 1 - q1)) & 1
            b2 = (j >> (n - 1 - q2)) & 1
            k = j & ~((1 << (n - 1 - q1)) | (1 << (n - 1 - q2)))
            k |= (b2 << (n - 1 - q1)) | (b1 << (n - 1 - q2))
            ref[k] = psi[j]
        O.swap(psi, q1, q2)
        assert np.array_equal(psi, ref)


def test_swap_equals_three_cnots():
    rng = np.random.default_rng(7)
    n = 4
    X = [[0, 1], [1, 0]]
    psi = rand_state(n, rng)
    ref = psi.copy()
    O.apply_ctrl(ref, 1 << 1, 1 << 1, 3, X)
    O.apply_ctrl(ref, 1 << 3, 1 << 3, 1, X)
    O.apply_ctrl(ref, 1 << 1, 1 << 1, 3, X)
    O.swap(psi, 1, 3)
    assert np.max(np.abs(psi - ref)) < 1e-15


def test_unitary_then_adjoint_restores():
    rng = np.random.default_rng(8)
    n = 8
    psi = rand_state(n, rng)
    orig = psi.copy()
    for q in range(n):
        a = O.haar_angles(9, q)
        U = O.mat_angles(O.HAAR, a)
        O.apply_1q(psi, q, U)
        O.apply_ctrl(psi, 1 << ((q + 1) % n), 1 << ((q + 1) % n), q, U)
        O.apply_ctrl(psi, 1 << ((q + 1) % n), 1 << ((q + 1) % n), q, U.conj().T)
        O.apply_1q(psi, q, U.conj().T)
    assert np.max(np.abs(psi - orig)) < 1e-13


# ------------------------------------------------------------ matrices (§3.2)
def test_rotation_and_phase_definitions():
    t, p = 0.3, 1.1
    assert np.allclose(O.mat_ur(t), [[np.cos(t), -np.sin(t)], [np.sin(t), np.cos(t)]], atol=0)
    assert np.allclose(O.mat_up1(p), [[1, 0], [0, np.exp(1j * p)]], atol=1e-16)
    assert np.allclose(O.mat_up2(p), [[np.exp(1j * p), 0], [0, 1]], atol=1e-16)


def test_H_and_NOT_decompositions():
    # H = U_R(pi/4) U_P1(pi), NOT = U_R(pi/2) U_P1(pi)
    H = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    assert np.max(np.abs(O.mat_angles(O.RP, [np.pi / 4, np.pi]) - H)) < 1e-15
    assert np.max(np.abs(O.mat_angles(O.RP, [np.pi / 2, np.pi]) - [[0, 1], [1, 0]])) < 1e-15
    # R_d = U_P1(pi / 2^d)
    for d in range(1, 6):
        assert np.max(np.abs(O.mat_angles(O.P1, [np.pi / 2**d]) -
                             np.diag([1, np.exp(1j * np.pi / 2**d)]))) < 1e-16


def test_haar_form_is_product_and_haar_distributed():
    a = O.haar_angles(1, 0)
    U = O.mat_angles(O.HAAR, a)
    ref = (np.diag([np.exp(1j * a[0]), 1]) @ np.diag([1, np.exp(1j * a[1])]) @
           np.array([[np.cos(a[2]), -np.sin(a[2])], [np.sin(a[2]), np.cos(a[2])]]) @
           np.diag([1, np.exp(1j * a[3])]))
    assert np.max(np.abs(U - ref)) < 1e-15
    # Haar moments on U(2): E|tr U|^2 = 1, E|tr U|^4 = 2 (reading R12)
    tr = np.array([np.trace(O.mat_angles(O.HAAR, O.haar_angles(77, i))) for i in range(20000)])
    m2, m4 = np.mean(np.abs(tr) ** 2), np.mean(np.abs(tr) ** 4)
    assert abs(m2 - 1.0) < 0.04 and abs(m4 - 2.0) < 0.12
    # unitarity
    for i in range(50):
        V = O.mat_angles(O.HAAR, O.haar_angles(3, i))
        assert np.max(np.abs(V @ V.conj().T - np.eye(2))) < 1e-15


def test_angle_noise_is_fresh_gaussian_per_slot():
    # each error angle is Gaussian(sigma), drawn per gate g, slot s
    seed, sig, g = 4, 1e-3, 17
    ang = [np.pi / 4, np.pi]
    z = [O.normal(seed, O.TAG_OPNOISE, g, s) for s in range(2)]
    U = O.mat_angles(O.RP, ang, seed=seed, sigma=sig, g=g)
    V = O.mat_angles(O.RP, [ang[0] + sig * z[0], ang[1] + sig * z[1]])
    assert np.array_equal(U, V)
    assert np.array_equal(O.mat_angles(O.RP, ang, seed=seed, sigma=0.0, g=g),
                          O.mat_angles(O.RP, ang))


def test_pauli_matrices():
    assert np.array_equal(O.pauli(1), [[0, 1], [1, 0]])
    assert np.array_equal(O.pauli(2), [[0, -1j], [1j, 0]])
    assert np.array_equal(O.pauli(3), [[1, 0], [0, -1]])
