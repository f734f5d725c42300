"""The largest single-GPU register: 2^33 amplitudes fill 128 GiB of the
B200's ~180 GB, leaving no room for an out-of-place copy.  The fused QFT then
runs its passes in place with the closing swaps as a relabel, and layout
restores use in-place position swaps.  Checked against closed forms on
sampled amplitudes (the state is too large for a host-side oracle copy):
QFT of a basis state, H_n of a basis state
(PAPER.md:420-436), marginals and the norm."""
import cmath
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")

N = 33


def free_bytes():
    import torch
    f, _ = torch.cuda.mem_get_info()
    return f


@pytest.fixture(scope="module")
def big():
    if free_bytes() < (1 << (N + 4)) + (4 << 30):
        pytest.skip("not enough device memory for a 2^33 state")
    h = Q.qsim_create(N)
    yield h
    Q.qsim_destroy(h)


def test_qft_of_basis_state_in_place(big):
    x = 0x1_2345_6789 & ((1 << N) - 1)
    Q.qsim_set_basis(big, x)
    Q.qsim_qft(big, 0, N, False)
    rng = np.random.default_rng(33)
    ys = [0, 1, (1 << N) - 1] + [int(v) for v in rng.integers(0, 1 << N, size=13)]
    for y in ys:
        got = Q.qsim_get_state(big, y, 1)[0]
        want = cmath.exp(2j * math.pi * ((x * y) % (1 << N)) / (1 << N)) / math.sqrt(1 << N)
        assert abs(got - want) < 1e-12, (y, got, want)
    assert abs(Q.qsim_norm(big) - 1) < 1e-12


def test_inverse_qft_returns_the_basis_state(big):
    x = 987654321
    Q.qsim_set_basis(big, x)
    Q.qsim_qft(big, 0, N, False)
    Q.qsim_qft(big, 0, N, True)
    assert abs(Q.qsim_get_state(big, x, 1)[0] - 1) < 1e-10
    assert abs(Q.qsim_prob_index(big, x) - 1) < 1e-10


def test_hadamard_and_marginals(big):
    x = 5
    Q.qsim_set_basis(big, x)
    Q.qsim_hadamard(big, 0, N)
    amp = 1 / math.sqrt(1 << N)
    for y in (0, 7, (1 << N) - 1):
        sign = -1 if bin(x & y).count("1") % 2 else 1
        assert abs(Q.qsim_get_state(big, y, 1)[0] - sign * amp) < 1e-15
    P = Q.qsim_probs(big, 3, 10)
    assert np.max(np.abs(P - 1 / 1024)) < 1e-12
