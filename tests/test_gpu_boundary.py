"""The §8(b) boundary calls added in round 2, each against the oracle or the
plain definition:

* qsim_create(n, ngpus > 1): the sharded handle over devices 0..ngpus-1 (on a
  one-GPU box every rank shares device 0);
* qsim_diffusion(lo, m): D = -H_m V_f0 H_m = 2|s><s| - I
  on the whole register (mean form) and on sub-registers (literal form);
* qsim_grover on sharded handles vs the oracle's literal iteration (configs[1]);
* strict unitarity (QSIM_ENONUNITARY);
* the noisy / approximate QFT with the block-move layout switched off (the
  dry-run relabel bug of round 1: the closing swaps were applied twice).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def diffusion_definition(psi, lo, m):
    """2|s><s| - I on qubits [lo, lo+m) written out: for every value of the
    other qubits, alpha_y <- 2 mean_y(alpha) - alpha_y (qubit 0 = MSB)."""
    n = int(np.log2(psi.size))
    t = psi.reshape(1 << lo, 1 << m, 1 << (n - lo - m))
    mean = t.mean(axis=1, keepdims=True)
    return (2 * mean - t).reshape(-1)


def diffusion_oracle(psi, lo, m):
    """The paper's literal -H_m V_f0 H_m with oracle primitives."""
    out = psi.copy()
    O.hadamard_range(out, lo, m)
    cm = sum(1 << q for q in range(lo, lo + m - 1))
    O.apply_ctrl(out, cm, 0, lo + m - 1, np.diag([-1.0, 1.0]).astype(complex)) if cm else \
        O.apply_1q(out, lo, np.diag([-1.0, 1.0]).astype(complex))
    O.hadamard_range(out, lo, m)
    return -out


def test_diffusion_oracle_pin():
    """The literal oracle form equals the mean-form definition (n = 7, every range)."""
    n = 7
    psi = rand_state(n, 1)
    for lo in range(n):
        for m in range(1, n - lo + 1):
            assert np.max(np.abs(diffusion_oracle(psi, lo, m) - diffusion_definition(psi, lo, m))) < 1e-13


@pytest.mark.parametrize("ngpus", [1, 2, 4])
@pytest.mark.parametrize("n", [6, 13])
def test_diffusion_every_range(n, ngpus):
    psi = rand_state(n, n + ngpus)
    rng = np.random.default_rng(n)
    ranges = [(0, n), (0, 1), (n - 1, 1), (0, n - 1), (1, n - 1)]
    ranges += [(int(lo), int(rng.integers(1, n - lo + 1))) for lo in rng.integers(0, n, 4)]
    for lo, m in ranges:
        h = Q.qsim_create(n, ngpus)
        try:
            Q.qsim_set_state(h, 0, psi)
            Q.qsim_diffusion(h, lo, m)
            got = Q.qsim_get_state(h, 0, 1 << n)
        finally:
            Q.qsim_destroy(h)
        ref = diffusion_oracle(psi, lo, m)
        assert np.max(np.abs(got - ref)) < TOL, (lo, m)


def test_diffusion_errors():
    h = Q.qsim_create(8)
    try:
        for lo, m in [(-1, 2), (0, 0), (0, 9), (7, 2)]:
            with pytest.raises(Q.QsimError) as e:
                Q.qsim_diffusion(h, lo, m)
            assert e.value.code == Q.QSIM_ERANGE
    finally:
        Q.qsim_destroy(h)


@pytest.mark.parametrize("ngpus", [2, 4, 8])
def test_grover_sharded_matches_oracle(ngpus):
    """configs[1] at n = 12 on a sharded handle: trace and final state vs the
    oracle's literal -H V_f0 H V_fk iterations."""
    n = 12
    iters = 50
    k = O.grover_mark(2, n)
    psi, rtrace = O.cfg1(n=n, seed=2, iters=iters)
    h = Q.qsim_create(n, ngpus)
    try:
        Q.qsim_hadamard(h, 0, n)
        trace = Q.qsim_grover(h, k, iters)
        got = Q.qsim_get_state(h, 0, 1 << n)
    finally:
        Q.qsim_destroy(h)
    assert np.max(np.abs(trace - rtrace)) < TOL
    assert np.max(np.abs(got - psi)) < TOL


@pytest.mark.parametrize("ngpus", [2, 4])
def test_create_ngpus_qft_and_probs(ngpus):
    n = 16
    psi = rand_state(n, 7)
    h = Q.qsim_create(n, ngpus)
    try:
        Q.qsim_set_state(h, 0, psi)
        Q.qsim_qft(h, 0, n, False)
        got = Q.qsim_get_state(h, 0, 1 << n)
        p = Q.qsim_probs(h, 0, 3)
    finally:
        Q.qsim_destroy(h)
    ref = psi.copy()
    O.qft(ref, 0, n, False)
    assert np.max(np.abs(got - ref)) < TOL
    assert np.max(np.abs(p - O.probs(ref, 0, 3))) < 1e-12


def test_create_ngpus_errors():
    for ng in [0, 3, 6, 128]:
        with pytest.raises(Q.QsimError) as e:
            Q.qsim_create(10, ng)
        assert e.value.code == Q.QSIM_EINVAL
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_create(2, 4)   # 2^n < 2 * ngpus
    assert e.value.code == Q.QSIM_ERANGE


def test_strict_unitarity():
    n = 8
    psi = rand_state(n, 3)
    h = Q.qsim_create(n)
    try:
        Q.qsim_set_state(h, 0, psi)
        Q.qsim_set_strict(h, True)
        bad = np.array([[1.0, 0.0], [0.0, 1.0 + 1e-9]], complex)
        for call in (lambda: Q.qsim_apply_1q(h, 3, bad), lambda: Q.qsim_apply_ctrl(h, 1, 1, 3, bad)):
            with pytest.raises(Q.QsimError) as e:
                call()
            assert e.value.code == Q.QSIM_ENONUNITARY
        # no effect on the state
        assert np.max(np.abs(Q.qsim_get_state(h, 0, 1 << n) - psi)) == 0.0
        # a unitary within rounding is accepted
        H = np.array([[1, 1], [1, -1]], complex) / np.sqrt(2)
        Q.qsim_apply_1q(h, 3, H)
        Q.qsim_set_strict(h, False)
        Q.qsim_apply_1q(h, 3, bad)   # off: applied as given
        ref = psi.copy()
        O.apply_1q(ref, 3, H)
        O.apply_1q(ref, 3, bad)
        assert np.max(np.abs(Q.qsim_get_state(h, 0, 1 << n) - ref)) < TOL
    finally:
        Q.qsim_destroy(h)


_NO_MOVES_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle as O
from paper_quant_ph_0201042_b200 import qsim as Q
n = 16
rng = np.random.default_rng(5)
psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n); psi /= np.linalg.norm(psi)
worst = 0.0
for (lo, m, b, sigma, inv) in [(0, 16, 4, 0.0, 0), (2, 12, 3, 0.0, 1), (0, 16, 15, 1e-3, 0), (3, 10, 9, 1e-3, 1), (0, 16, 5, 1e-3, 0)]:
    h = Q.qsim_create(n)
    Q.qsim_set_state(h, 0, psi)
    Q.qsim_set_gate_noise(h, 11, sigma)
    if b >= m - 1:
        Q.qsim_qft(h, lo, m, bool(inv))
    else:
        Q.qsim_aqft(h, lo, m, b, bool(inv))
    got = Q.qsim_get_state(h, 0, 1 << n)
    Q.qsim_destroy(h)
    ref = psi.copy()
    O.aqft(ref, lo, m, b, bool(inv), noise=O.Noise(11, sigma, 0))
    worst = max(worst, float(np.max(np.abs(got - ref))))
print("WORST", worst)
assert worst < 1e-10, worst
"""


def test_generalised_qft_without_block_moves():
    """with QSIM_NO_BLOCK_MOVES the dry runs of the
    generalised QFT used to apply the closing-swap relabel too."""
    env = dict(os.environ, QSIM_NO_BLOCK_MOVES="1")
    r = subprocess.run([sys.executable, "-c", _NO_MOVES_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("n,lo,m,inv", [(18, 0, 18, False), (17, 2, 12, True)])
def test_qft_host_stream(n, lo, m, inv):
    """Pipelined end-to-end QFTs of host states (qsim_qft_host_stream) equal
    the oracle's circuit on each state; the handle keeps the last result and
    keeps working afterwards."""
    count = 5
    rng = np.random.default_rng(n)
    states = rng.normal(size=(count, 1 << n)) + 1j * rng.normal(size=(count, 1 << n))
    states /= np.linalg.norm(states, axis=1, keepdims=True)
    inp = np.ascontiguousarray(states)
    out = np.zeros_like(inp)
    h = Q.qsim_create(n)
    try:
        Q.qsim_qft_host_stream(h, lo, m, inv, inp, out, count, 1 << n, 1 << n)
        last = Q.qsim_get_state(h, 0, 1 << n)
        # the handle still works: one more transform on the resident state
        Q.qsim_qft(h, lo, m, not inv)
        back = Q.qsim_get_state(h, 0, 1 << n)
        # stride 0: the same input every time, one output buffer
        one = np.zeros(1 << n, np.complex128)
        Q.qsim_qft_host_stream(h, lo, m, inv, inp[0].copy(), one, 3, 0, 0)
    finally:
        Q.qsim_destroy(h)
    for i in range(count):
        ref = states[i].copy()
        O.qft(ref, lo, m, inv)
        assert np.max(np.abs(out[i] - ref)) < TOL, i
    assert np.max(np.abs(last - out[-1])) == 0.0
    assert np.max(np.abs(back - states[-1])) < TOL
    ref0 = states[0].copy()
    O.qft(ref0, lo, m, inv)
    assert np.max(np.abs(one - ref0)) < TOL


def test_qft_host_stream_errors():
    h = Q.qsim_create(10)
    try:
        x = np.zeros(1 << 10, np.complex128)
        with pytest.raises(Q.QsimError) as e:
            Q.qsim_qft_host_stream(h, 3, 9, False, x, x, 1, 0, 0)
        assert e.value.code == Q.QSIM_ERANGE
        Q.qsim_set_gate_noise(h, 1, 1e-3)
        with pytest.raises(Q.QsimError) as e:
            Q.qsim_qft_host_stream(h, 0, 10, False, x, x, 1, 0, 0)
        assert e.value.code == Q.QSIM_EINVAL
    finally:
        Q.qsim_destroy(h)
    g = Q.qsim_create(12, 2)
    try:
        x = np.zeros(1 << 12, np.complex128)
        with pytest.raises(Q.QsimError) as e:
            Q.qsim_qft_host_stream(g, 0, 12, False, x, x, 1, 0, 0)
        assert e.value.code == Q.QSIM_EINVAL
    finally:
        Q.qsim_destroy(g)
