"""GPU parity for Shor's semantic mode.

libqsim's order-finding register (k_shor_semantic), its fused QFT and the
whole factoring run (device state + host post-processing) against the
oracle: amplitudes within 1e-10 (north_star), measured y, iteration counts
and factors bit-exact.  At the paper's size (N = 21311, 2l = 30 qubits,
PAPER.md:922-966) the register is checked on sampled indices against the
predicate x^a = v (mod N) and the QFT output against the Fejer closed form.
"""
import math

import numpy as np
import pytest

import oracle as O
from _closed_forms import fejer_branch, order

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")

TOL = 1e-10


@pytest.fixture
def reg():
    made = []

    def make(n):
        h = Q.qsim_create(n)
        made.append(h)
        return h

    yield make
    for h in made:
        Q.qsim_destroy(h)


# ragged shards (2^8 < one warp run of 2048), several tiles, and odd N
CASES = [(8, 7, 15, 4), (10, 2, 21, 8), (12, 3, 35, 27), (16, 5, 143, 125), (18, 2, 437, 16), (20, 6, 899, 36)]


@pytest.mark.parametrize("m,x,N,v", CASES)
def test_semantic_state_parity(reg, m, x, N, v):
    h = reg(m)
    Q.qsim_shor_semantic_state(h, x, N, v)
    got = Q.qsim_get_state(h, 0, 1 << m)
    ref = O.shor_semantic_state(m, x, N, v)
    assert float(np.max(np.abs(got - ref))) <= TOL
    assert np.array_equal(np.flatnonzero(got), np.flatnonzero(ref))


@pytest.mark.parametrize("m,x,N,v", CASES[1:])
def test_semantic_qft_parity(reg, m, x, N, v):
    h = reg(m)
    Q.qsim_shor_semantic_state(h, x, N, v)
    Q.qsim_qft(h, 0, m, False)
    got = Q.qsim_get_state(h, 0, 1 << m)
    ref = O.shor_semantic_state(m, x, N, v)
    O.qft(ref, 0, m)
    assert float(np.max(np.abs(got - ref))) <= TOL


def test_semantic_state_errors(reg):
    h = reg(10)
    with pytest.raises(Q.QsimError):
        Q.qsim_shor_semantic_state(h, 2, 2, 1)          # N < 3
    with pytest.raises(Q.QsimError):
        Q.qsim_shor_semantic_state(h, 22, 21, 1)        # x >= N
    with pytest.raises(Q.QsimError):
        Q.qsim_shor_semantic_state(h, 2, 21, 3)         # 3 is not a power of 2 mod 21
    h2 = reg(10)
    with pytest.raises(Q.QsimError):
        Q.qsim_shor_run(h2, 143, 1, 0)                  # 2^10 < 143^2


@pytest.mark.parametrize("N,m", [(15, 8), (21, 10), (143, 16), (437, 18)])
@pytest.mark.parametrize("improved", [False, True])
def test_run_parity(reg, N, m, improved):
    """Same draws, same register, same measurement: iterations and factors
    agree with the oracle run for run."""
    h = reg(m)
    sg = np.zeros(len(Q.SHOR_STATS), np.int64)
    so = np.zeros(len(O.SHOR_STATS), np.int64)
    for run in range(8):
        got = Q.qsim_shor_run(h, N, 11, run, improved, 200, sg)
        ref = O.shor_run(N, m, 11, run, improved, 200, so)
        assert got == ref, (run, got, ref)
        t, f = got
        assert t >= 1 and 1 < f < N and N % f == 0
    assert Q.SHOR_STATS == O.SHOR_STATS
    assert np.array_equal(sg, so)


def test_full_size_register_sampled(reg):
    """N = 21311 = 211 * 101 (Table 5), 2l = 30 qubits: sampled amplitudes
    against the predicate, the norm, then the QFT output on sampled y
    against the closed form of the periodic register."""
    N, m, x = 21311, 30, 2
    M = 1 << m
    r = order(x, N)
    v = pow(x, 12345, N)
    h = reg(m)
    Q.qsim_shor_semantic_state(h, x, N, v)
    a0 = 12345 % r
    c = len(range(a0, M, r))
    rng = np.random.default_rng(1)
    idx = np.concatenate([rng.integers(0, M, 2000), a0 + r * rng.integers(0, c, 2000), [0, M - 1, a0]])
    for i in idx:
        i = int(i)
        amp = Q.qsim_get_state(h, i, 1)[0]
        want = 1 / math.sqrt(c) if pow(x, i, N) == v else 0.0
        assert abs(amp - want) <= TOL, i
    assert abs(Q.qsim_norm(h) - 1) <= 1e-12
    Q.qsim_qft(h, 0, m, False)
    ys = np.concatenate([rng.integers(0, M, 500), [round(k * M / r) + d for k in range(0, r, max(1, r // 200))
                                                   for d in (-1, 0, 1)]]) % M
    P = np.array([Q.qsim_prob_index(h, int(y)) for y in ys])
    ref = fejer_branch(M, r, c, ys)
    assert np.max(np.abs(P - ref)) <= 1e-12
    assert abs(Q.qsim_norm(h) - 1) <= 1e-12


def test_full_size_runs_factor(reg):
    """Factoring runs at the paper's size succeed with valid factors."""
    N, m = 21311, 30
    h = reg(m)
    for run in range(3):
        for improved in (False, True):
            t, f = Q.qsim_shor_run(h, N, 2002, run, improved, 200)
            assert t >= 1 and f in (101, 211)
