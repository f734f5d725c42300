"""Cross-feature sequences through the C-ABI against the oracle: random
interleavings of queued gates (dense, controlled, angle-form with gate
noise), swaps (relabels), phase flips, exact and noisy fused transforms
(QFT / inverse, approximate QFT, FFT, constant and angle-form Hadamard
ranges), Pauli injection and the modular multiplication permutation, on a
single GPU and on in-process rank groups.  Each API call leaves the
logical -> physical layout in some state the next call must honour; the
gate counter ties every noisy gate to one Philox draw, so the whole
sequence is element-wise comparable (1e-10)."""
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


def rand_u(rng):
    a = O.haar_angles(11, int(rng.integers(1 << 30)))
    return O.mat_angles(O.HAAR, a)


@pytest.fixture
def mk():
    made = []

    def make(n, world, psi):
        h = Q.qsim_create(n) if world == 1 else Q.qsim_create_group(n, world)
        made.append(h)
        Q.qsim_set_state(h, 0, psi)
        return h

    yield make
    for h in made:
        Q.qsim_destroy(h)


@pytest.mark.parametrize("world,seed,n,nsteps", [(w, s, 15, 40) for w in (1, 2, 4) for s in range(1, 9)] +
                         [(w, s, 22, 25) for w in (1, 2) for s in (11, 12)])
def test_mixed_api_sequence_matches_oracle(mk, world, seed, n, nsteps):
    sigma = 1e-2
    rng = np.random.default_rng(seed)
    psi = rand_state(n, 100 + seed)
    h = mk(n, world, psi)
    Q.qsim_set_gate_noise(h, 30 + seed, sigma)
    Q.qsim_set_gate_counter(h, 0)
    nz = O.Noise(seed=30 + seed, sigma=sigma)
    ref = psi.copy()
    log = []
    for _ in range(nsteps):
        op = int(rng.integers(13))
        q = int(rng.integers(n))
        lo = int(rng.integers(n - 1))
        m = int(rng.integers(1, n - lo + 1))
        inv = bool(rng.integers(2))
        log.append((op, q, lo, m, inv))
        if op == 0:
            U = rand_u(rng)
            Q.qsim_apply_1q(h, q, U)
            O.apply_1q(ref, q, U)
        elif op == 1:
            c = int(rng.integers(n))
            if c == q:
                continue
            v = int(rng.integers(2))
            U = rand_u(rng)
            Q.qsim_apply_ctrl(h, 1 << c, v << c, q, U)
            O.apply_ctrl(ref, 1 << c, v << c, q, U)
        elif op == 2:
            a = O.haar_angles(5, int(rng.integers(1 << 20)))
            Q.qsim_apply_angles(h, Q.QSIM_GATE_HAAR, a, 0, 0, q)
            O.apply_angles(ref, nz, O.HAAR, a, 0, 0, q)
        elif op == 3:
            q2 = int(rng.integers(n))
            if q2 == q:
                continue
            Q.qsim_swap(h, q, q2)
            O.swap(ref, q, q2)
        elif op == 4:
            Q.qsim_qft(h, lo, m, inv)
            O.qft(ref, lo, m, inv, noise=nz)
        elif op == 5:
            Q.qsim_fft(h, lo, m, inv)
            O.qft(ref, lo, m, inv)
        elif op == 6:
            b = int(rng.integers(0, m))
            Q.qsim_aqft(h, lo, m, b, inv)
            O.aqft(ref, lo, m, b, inv, noise=nz)
        elif op == 7:
            Q.qsim_hadamard(h, lo, m)
            O.hadamard_range(ref, lo, m)
        elif op == 8:
            Q.qsim_hadamard_angles(h, lo, m)
            for qq in range(lo, lo + m):
                O.apply_angles(ref, nz, O.RP, [math.pi / 4, math.pi], 0, 0, qq)
        elif op == 9:
            idx = int(rng.integers(1 << n))
            Q.qsim_phase_flip(h, idx)
            O.phase_flip(ref, idx)
        elif op == 10:
            ev = Q.qsim_inject_errors(h, 7 + seed, 0.2, (1 << n) - 1, len(log))
            rev = O.inject_paulis(ref, 7 + seed, len(log), (1 << n) - 1, 0.2)
            assert ev == rev
        elif op == 11:
            # MODMUL by 4 mod 31 on a 5-qubit work register, one control
            wlo = int(rng.integers(1, n - 5 + 1))
            c = int(rng.integers(0, wlo))
            Q.qsim_apply_perm(h, Q.QSIM_PERM_MODMUL, wlo, 5, ctrl_mask=1 << c, ctrl_vals=1 << c, mult=4, modulus=31)
            O.modmul(ref, wlo, 5, 1 << c, 1 << c, 4, 31)
        else:
            # a sampled amplitude read in the middle (forces a flush)
            idx = int(rng.integers(1 << n))
            got = Q.qsim_get_state(h, idx, 1)[0]
            assert abs(got - ref[idx]) < TOL, log
    got = Q.qsim_get_state(h, 0, 1 << n)
    assert np.max(np.abs(got - ref)) < TOL, log
    assert Q.qsim_get_gate_counter(h) == nz.g
    assert abs(Q.qsim_norm(h) - 1) < 1e-12
