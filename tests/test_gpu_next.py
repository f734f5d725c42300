"""GPU parity for SURVEY.md §8(f) rows f1 and f4 through the C-ABI:
qsim_fft (the paper's "FFT instead of the QFT circuit"),
qsim_aqft (approximate QFT), qsim_measure_range (partial
measurement with collapse) and qsim_inner (fidelity,
PAPER.md:1127-1128), against the pinned oracle (tests/test_oracle_next.py).
Single handles and in-process rank groups (sub-registers on rank bits)."""
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

    def make(n, state=None, world=1):
        h = Q.qsim_create(n) if world == 1 else Q.qsim_create_group(n, world)
        made.append(h)
        if state is not None:
            Q.qsim_set_state(h, 0, state)
        return h

    yield make
    for h in made:
        Q.qsim_destroy(h)


def get(h, n):
    return Q.qsim_get_state(h, 0, 1 << n)


def maxdiff(a, b):
    return float(np.max(np.abs(a - b)))


# ------------------------------------------------------------------ f1: FFT
@pytest.mark.parametrize("n,lo,m", [(12, 0, 12), (14, 3, 9), (17, 0, 17), (20, 5, 11), (13, 2, 3), (6, 1, 4)])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft_equals_dft(mk, n, lo, m, inverse):
    psi = rand_state(n, 100 + n + lo)
    h = mk(n, psi)
    Q.qsim_set_gate_noise(h, 7, 1e-3)        # the FFT is a black box: noise must not apply
    g0 = Q.qsim_get_gate_counter(h)
    Q.qsim_fft(h, lo, m, inverse)
    assert Q.qsim_get_gate_counter(h) == g0
    ref = psi.copy()
    O.qft(ref, lo, m, inverse)               # noiseless circuit = the DFT (pinned)
    assert maxdiff(get(h, n), ref) < TOL


def test_fft_full_register_sampled_against_definition(mk):
    n = 24
    h = mk(n)
    Q.qsim_init_gaussian(h, 3)
    psi = get(h, n)
    Q.qsim_fft(h, 0, n, False)
    xs = np.array([0, 1, 2, 12345, (1 << n) - 1, 777777, 1 << 23], np.uint64)
    ref = O.dft_samples(psi, xs)
    out = get(h, n)
    assert maxdiff(out[xs.astype(np.int64)], ref) < TOL
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


@pytest.mark.parametrize("world", [2, 4])
def test_fft_sharded(mk, world):
    n = 14
    psi = rand_state(n, 9 + world)
    h = mk(n, psi, world)
    Q.qsim_fft(h, 0, n, True)
    ref = psi.copy()
    O.qft(ref, 0, n, True)
    assert maxdiff(get(h, n), ref) < TOL


# ------------------------------------------------------------------ f4: approximate QFT
@pytest.mark.parametrize("n,lo,m,b", [(14, 0, 14, 3), (14, 2, 10, 1), (16, 0, 16, 6), (10, 1, 8, 0), (13, 0, 13, 12)])
@pytest.mark.parametrize("sigma", [0.0, 1e-3])
def test_aqft_matches_oracle(mk, n, lo, m, b, sigma):
    psi = rand_state(n, 7 * n + b)
    h = mk(n, psi)
    Q.qsim_set_gate_noise(h, 4, sigma)
    Q.qsim_set_gate_counter(h, 0)
    Q.qsim_aqft(h, lo, m, b, False)
    ref = psi.copy()
    nz = O.Noise(seed=4, sigma=sigma)
    O.aqft(ref, lo, m, b, False, noise=nz)
    assert maxdiff(get(h, n), ref) < TOL
    assert Q.qsim_get_gate_counter(h) == nz.g


def test_aqft_fidelity_against_exact_qft_via_inner(mk):
    """|<QFT psi | AQFT_b psi>| from the GPU equals the oracle's for every band,
    and reaches 1 at the full band."""
    n = 12
    psi = np.zeros(1 << n, complex)
    psi[1234] = 1
    he = mk(n, psi)
    Q.qsim_qft(he, 0, n, False)
    ex = psi.copy()
    O.qft(ex, 0, n)
    for b in range(0, n):
        ha = mk(n, psi)
        Q.qsim_aqft(ha, 0, n, b, False)
        ref = psi.copy()
        O.aqft(ref, 0, n, b)
        f = abs(Q.qsim_inner(he, ha))
        assert f == pytest.approx(abs(O.inner(ex, ref)), abs=1e-12)
    assert f == pytest.approx(1.0, abs=1e-12)


# ------------------------------------------------------------------ noisy QFT as fused passes
@pytest.mark.parametrize("n,lo,m,inverse", [(18, 0, 18, False), (18, 3, 12, True), (20, 0, 20, False),
                                            (12, 0, 9, False), (15, 2, 13, True), (11, 0, 8, False),
                                            (22, 1, 21, True)])
def test_noisy_qft_fused_matches_oracle(mk, n, lo, m, inverse):
    """Operational error on every H and R_d of the QFT: the
    generalised fused passes (k_qft_gen) against the oracle's gate-by-gate
    circuit with the same Philox draws, and the gate counter advanced by the
    number of gates."""
    psi = rand_state(n, 5 * n + m)
    h = mk(n, psi)
    Q.qsim_set_gate_noise(h, 11, 2e-2)
    Q.qsim_set_gate_counter(h, 100)
    Q.qsim_qft(h, lo, m, inverse)
    ref = psi.copy()
    nz = O.Noise(seed=11, sigma=2e-2, g=100)
    O.qft(ref, lo, m, inverse, noise=nz)
    assert maxdiff(get(h, n), ref) < TOL
    assert Q.qsim_get_gate_counter(h) == nz.g


@pytest.mark.parametrize("n,lo,m,sigma", [(20, 0, 20, 1e-2), (18, 3, 12, 5e-2), (12, 2, 3, 1e-2), (16, 0, 16, 0.0),
                                          (11, 0, 8, 1e-3)])
def test_hadamard_angles_equals_angle_gate_loop(mk, n, lo, m, sigma):
    """qsim_hadamard_angles = m angle-form H gates U_R(pi/4) U_P1(pi)
     in qubit order with the same Philox draws: the fused
    passes (k_qft_gen, no R_d, reversal undone by relabelling) against the
    oracle's gate loop, and the counter advanced by m."""
    psi = rand_state(n, 3 * n + m)
    h = mk(n, psi)
    Q.qsim_set_gate_noise(h, 21, sigma)
    Q.qsim_set_gate_counter(h, 7)
    Q.qsim_hadamard_angles(h, lo, m)
    ref = psi.copy()
    nz = O.Noise(seed=21, sigma=sigma, g=7)
    for q in range(lo, lo + m):
        O.apply_angles(ref, nz, O.RP, [math.pi / 4, math.pi], 0, 0, q)
    assert maxdiff(get(h, n), ref) < TOL
    assert Q.qsim_get_gate_counter(h) == nz.g == 7 + m
    # the layout stays consistent for what follows
    Q.qsim_qft(h, 0, n, False)
    O.qft(ref, 0, n, False, noise=nz)
    assert maxdiff(get(h, n), ref) < TOL


def test_noisy_qft_fused_equals_unfused_after_gates(mk):
    """A non-canonical layout (gates queued, swaps relabelled) before the noisy
    QFT: fused passes and the one-sweep-per-gate path give the same state."""
    n = 19
    psi = rand_state(n, 77)
    out = []
    for fuse in (True, False):
        h = mk(n, psi)
        Q.qsim_set_fusion(h, fuse)
        Q.qsim_set_gate_noise(h, 3, 1e-2)
        Q.qsim_swap(h, 0, 7)
        Q.qsim_hadamard(h, 2, 5)
        Q.qsim_qft(h, 1, 17, False)
        Q.qsim_qft(h, 0, 19, True)
        out.append(get(h, n))
    assert maxdiff(out[0], out[1]) < TOL


# ------------------------------------------------------------------ f4: partial measurement
@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("lo,m", [(0, 3), (4, 5), (9, 5), (0, 14), (2, 1)])
def test_measure_range_matches_oracle(mk, world, lo, m):
    n = 14
    psi = rand_state(n, 31 + lo + 3 * m)
    P = O.probs(psi, lo, m)
    cum = np.cumsum(P)
    for s in range(6):
        r = O.u01(O.draw(12, O.TAG_MEASURE, s, lo * 32 + m)[0])
        ref = psi.copy()
        y = O.measure_range(ref, lo, m, r, collapse=True)
        margin = min(abs(r - cum[y]), abs(r - (cum[y - 1] if y else 0.0)))
        if margin < 1e-12:
            continue                       # tie: parity unpinned (R22)
        h = mk(n, psi, world)
        assert Q.qsim_measure_range(h, lo, m, r, True) == y
        assert maxdiff(get(h, n), ref) < TOL
        assert abs(Q.qsim_norm(h) - 1) < 1e-12
        assert Q.qsim_measure_range(h, lo, m, 0.999, False) == y   # collapsed: same value again


def test_measure_range_after_circuit_layout(mk):
    """Measurement after a fused QFT (non-canonical layout until read-out)."""
    n = 16
    psi = rand_state(n, 5)
    h = mk(n, psi)
    Q.qsim_qft(h, 0, n, False)
    Q.qsim_apply_1q(h, 3, np.array([[0.6, 0.8j], [0.8j, 0.6]]))
    ref = psi.copy()
    O.qft(ref, 0, n)
    O.apply_1q(ref, 3, np.array([[0.6, 0.8j], [0.8j, 0.6]]))
    r = 0.4372
    y_ref = O.measure_range(ref, 2, 6, r)
    assert Q.qsim_measure_range(h, 2, 6, r) == y_ref
    assert maxdiff(get(h, n), ref) < TOL


# ------------------------------------------------------------------ f4: inner product
@pytest.mark.parametrize("world", [1, 2, 8])
def test_inner_matches_oracle(mk, world):
    n = 15
    a = rand_state(n, 1)
    b = rand_state(n, 2) * 0.8
    ha, hb = mk(n, a, world), mk(n, b, world)
    Q.qsim_apply_1q(hb, 4, np.array([[0, 1], [1, 0]]))     # leave b in a relabelled layout
    O.apply_1q(b, 4, np.array([[0, 1], [1, 0]]))
    got = Q.qsim_inner(ha, hb)
    ref = O.inner(a, b)
    assert abs(got - ref) < 1e-13
    assert abs(Q.qsim_inner(ha, ha) - O.norm(a)) < 1e-13


def test_inner_rejects_mismatched_registers(mk):
    ha, hb = mk(10), mk(11)
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_inner(ha, hb)
    assert e.value.code == Q.QSIM_EINVAL
