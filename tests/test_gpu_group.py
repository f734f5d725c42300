"""Sharded state over several ranks, run on one GPU as an in-process rank
group (qsim_create_group): the exchange plan, the rank-bit logic of every
kernel (controls / diagonal targets / QFT twiddles / permutation exponents on
rank bits), the canonical-layout restore and the fixed-order cross-rank sums
are the ones a multi-process NCCL world runs; only the transport differs
(device-to-device copies instead of ncclSend/ncclRecv).  Parity: the oracle.
"""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

TOL = 1e-10


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


@pytest.fixture
def grp():
    made = []

    def make(n, world, state=None):
        h = Q.qsim_create_group(n, world)
        made.append(h)
        if state is not None:
            Q.qsim_set_state(h, 0, state)
        return h

    yield make
    for h in made:
        Q.qsim_destroy(h)


def get(h, n):
    return Q.qsim_get_state(h, 0, 1 << n)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fuse", [True, False])
def test_group_random_gates(grp, world, fuse):
    n = 13
    rng = np.random.default_rng(world + 10 * fuse)
    psi = rand_state(n, world)
    h = grp(n, world, psi)
    Q.qsim_set_fusion(h, fuse)
    ref = psi.copy()
    for _ in range(120):
        q = int(rng.integers(n))
        kind = rng.integers(3)
        U = (rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))) / 2 if kind == 0 else \
            np.diag(np.exp(1j * rng.uniform(0, 6.3, 2))) if kind == 1 else np.array([[0, 1], [1, 0]], complex)
        others = [c for c in range(n) if c != q]
        k = int(rng.integers(0, 3))
        ctrl = rng.choice(others, size=k, replace=False) if k else []
        mask = sum(1 << int(c) for c in ctrl)
        vals = sum(int(rng.integers(2)) << int(c) for c in ctrl)
        if mask:
            Q.qsim_apply_ctrl(h, mask, vals, q, U)
            O.apply_ctrl(ref, mask, vals, q, U)
        else:
            Q.qsim_apply_1q(h, q, U)
            O.apply_1q(ref, q, U)
        if rng.random() < 0.05:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            Q.qsim_swap(h, a, b)
            O.swap(ref, a, b)
    assert np.max(np.abs(get(h, n) - ref)) < TOL
    assert abs(Q.qsim_norm(h) - O.norm(ref)) < 1e-12


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("n,lo,m,inv", [(14, 0, 14, False), (14, 0, 14, True), (15, 2, 10, False),
                                        (16, 0, 12, True), (13, 1, 12, False)])
def test_group_qft(grp, world, n, lo, m, inv):
    psi = rand_state(n, n + world)
    h = grp(n, world, psi)
    Q.qsim_qft(h, lo, m, inv)
    ref = psi.copy()
    O.qft(ref, lo, m, inv)
    assert np.max(np.abs(get(h, n) - ref)) < TOL


@pytest.mark.parametrize("world", [2, 8])
def test_group_hadamard_probs_measure(grp, world):
    n = 14
    psi = rand_state(n, 3)
    h = grp(n, world, psi)
    Q.qsim_hadamard(h, 0, n)
    ref = psi.copy()
    O.hadamard_range(ref, 0, n)
    for lo, m in [(0, 3), (0, 14), (2, 6), (8, 6)]:
        assert np.max(np.abs(Q.qsim_probs(h, lo, m) - O.probs(ref, lo, m))) < 1e-13
    cum = np.cumsum(np.abs(ref) ** 2)
    for s in range(20):
        r = O.u01(O.draw(4, O.TAG_MEASURE, s, 0)[0])
        i = O.measure(ref, r)
        margin = min(abs(r - cum[i]), abs(r - (cum[i - 1] if i else 0.0)))
        if margin > 1e-12:
            assert Q.qsim_measure(h, r) == i
    assert Q.qsim_prob_index(h, 12345) == pytest.approx(abs(ref[12345]) ** 2, abs=1e-16)


@pytest.mark.parametrize("world", [2, 4])
def test_group_gaussian_qft_cfg2(grp, world):
    n = 16
    h = grp(n, world)
    W.run_cfg2(h, n=n, seed=3)
    ref = O.cfg2(n=n, seed=3)
    assert np.max(np.abs(get(h, n) - ref)) < TOL
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("sigma", [0.0, 1e-3])
def test_group_order_finding(grp, world, sigma):
    ne, nw, N, a = 10, 6, 35, 3     # exponent bits sit on rank bits
    h = grp(ne + nw, world)
    P = W.run_cfg3(h, ne=ne, nw=nw, N=N, seed=4, sigma=sigma, a=a)
    pr = O.cfg3(ne=ne, nw=nw, N=N, seed=4, sigma=sigma, a=a)
    assert np.max(np.abs(P - pr)) < 1e-12


@pytest.mark.parametrize("world", [2, 4, 8])
def test_group_noisy_brickwork(grp, world):
    n = 12
    h = grp(n, world)
    ev = W.run_cfg4(h, n=n, layers=10, seed=5, sigma=1e-3, p=0.05)
    ref, rev = O.cfg4(n=n, layers=10, seed=5, sigma=1e-3, p=0.05)
    assert [tuple(e) for e in ev] == [tuple(e) for e in rev]
    assert np.max(np.abs(get(h, n) - ref)) < TOL


def test_group_matches_single_gpu_bitwise_for_permutations(grp):
    n = 14
    psi = rand_state(n, 9)
    h = grp(n, 4, psi)
    Q.qsim_apply_perm(h, Q.QSIM_PERM_MODEXP, 6, 8, elo=0, em=6, base=7, modulus=221)
    ref = psi.copy()
    for j in range(6):
        c = pow(7, 1 << j, 221)
        cm = 1 << (5 - j)
        O.modmul(ref, 6, 8, cm, cm, c, 221)
    assert np.array_equal(get(h, n), ref)


_CHUNK_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle as O
from paper_quant_ph_0201042_b200 import qsim as Q
worst = 0.0
for world in (2, 4, 8):
    n = 16
    rng = np.random.default_rng(world)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n); psi /= np.linalg.norm(psi)
    h = Q.qsim_create_group(n, world)
    Q.qsim_set_state(h, 0, psi)
    ref = psi.copy()
    Q.qsim_qft(h, 0, n, False); O.qft(ref, 0, n, False)
    for _ in range(40):
        q = int(rng.integers(n))
        U = (rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))) / 2
        Q.qsim_apply_1q(h, q, U); O.apply_1q(ref, q, U)
    Q.qsim_hadamard(h, 0, 5); O.hadamard_range(ref, 0, 5)
    worst = max(worst, float(np.max(np.abs(Q.qsim_get_state(h, 0, 1 << n) - ref))))
    Q.qsim_destroy(h)
print("WORST", worst)
assert worst < 1e-10, worst
"""


def test_group_exchanges_in_many_chunks():
    """Shard exchanges pipelined in 4 KiB chunks (QSIM_XCHG_CHUNK_KB): the
    chunked transport (two streams, per-chunk events) gives the oracle's state."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CHUNK_SCRIPT, root], env=dict(os.environ, QSIM_XCHG_CHUNK_KB="4"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
