"""GPU parity: libqsim (sm_100a, through its C-ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): max |amplitude difference| <= 1e-10,
|norm - 1| <= 1e-12, bit-exact for permutations, error locations and measured
indices.  Inputs are seeded and synthetic; sizes span several
tiles of the fused kernels (tiles of 2^9..2^13 amplitudes) plus ragged cases.
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


def rand_mat(rng):
    return rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))


@pytest.fixture
def reg():
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


def maxdiff(a, b):
    return float(np.max(np.abs(a - b)))


# ------------------------------------------------------------------ single gates
@pytest.mark.parametrize("n", [1, 2, 5, 12, 17])
def test_apply_1q_every_qubit(reg, n):
    rng = np.random.default_rng(n)
    psi = rand_state(n, n)
    h = reg(n, psi)
    ref = psi.copy()
    for q in range(n):
        U = rand_mat(rng)
        U /= np.linalg.norm(U)          # keep magnitudes O(1); non-unitary on purpose
        Q.qsim_apply_1q(h, q, U)
        O.apply_1q(ref, q, U)
    assert maxdiff(get(h, n), ref) < TOL
    assert Q.qsim_launch_count(h) > 0


@pytest.mark.parametrize("n", [3, 8, 14])
def test_controlled_gates(reg, n):
    rng = np.random.default_rng(100 + n)
    psi = rand_state(n, 100 + n)
    h = reg(n, psi)
    ref = psi.copy()
    for _ in range(3 * n):
        q = int(rng.integers(n))
        others = [c for c in range(n) if c != q]
        k = int(rng.integers(1, min(3, len(others)) + 1))
        ctrl = rng.choice(others, size=k, replace=False)
        mask = sum(1 << int(c) for c in ctrl)
        vals = sum(int(rng.integers(2)) << int(c) for c in ctrl)
        if rng.random() < 0.3:
            U = np.diag(np.exp(1j * rng.uniform(0, 6.3, 2)))     # diagonal path
        else:
            U = rand_mat(rng) / 2
        Q.qsim_apply_ctrl(h, mask, vals, q, U)
        O.apply_ctrl(ref, mask, vals, q, U)
    assert maxdiff(get(h, n), ref) < TOL


def test_angle_gates_and_noise_counter(reg):
    n = 11
    psi = rand_state(n, 5)
    h = reg(n, psi)
    ref = psi.copy()
    Q.qsim_set_gate_noise(h, 77, 1e-2)
    nz = O.Noise(seed=77, sigma=1e-2)
    rng = np.random.default_rng(3)
    for i in range(40):
        kind = int(rng.integers(3))
        ang = list(rng.uniform(0, 6.28, 4))[: [2, 1, 4][kind]]
        q = int(rng.integers(n))
        c = (q + 1 + int(rng.integers(n - 1))) % n
        cm = (1 << c) if i % 3 == 0 else 0
        Q.qsim_apply_angles(h, kind, ang, cm, cm, q)
        O.apply_angles(ref, nz, kind, ang, cm, cm, q)
    assert Q.qsim_get_gate_counter(h) == nz.g == 40
    assert maxdiff(get(h, n), ref) < TOL


def test_swaps_are_exact_relabels(reg):
    n = 13
    psi = rand_state(n, 9)
    h = reg(n, psi)
    ref = psi.copy()
    for q1, q2 in [(0, 12), (3, 4), (12, 5), (1, 1), (7, 0)]:
        Q.qsim_swap(h, q1, q2)
        O.swap(ref, q1, q2)
    assert np.array_equal(get(h, n), ref)     # permutation: bit-exact


def test_phase_flip_after_relabel(reg):
    n = 10
    psi = rand_state(n, 4)
    h = reg(n, psi)
    ref = psi.copy()
    Q.qsim_swap(h, 0, 9)
    O.swap(ref, 0, 9)
    for idx in [0, 1, 513, 1023]:
        Q.qsim_phase_flip(h, idx)
        O.phase_flip(ref, idx)
    assert np.array_equal(get(h, n), ref)


# ------------------------------------------------------------------ H_n and QFT (fused)
@pytest.mark.parametrize("n,lo,m", [(12, 0, 12), (16, 3, 9), (20, 0, 20), (14, 5, 9), (8, 0, 8)])
def test_hadamard_range(reg, n, lo, m):
    psi = rand_state(n, n + lo)
    h = reg(n, psi)
    Q.qsim_hadamard(h, lo, m)
    ref = psi.copy()
    O.hadamard_range(ref, lo, m)
    assert maxdiff(get(h, n), ref) < TOL


@pytest.mark.parametrize("inverse", [False, True])
@pytest.mark.parametrize("n,lo,m", [(9, 0, 9), (12, 0, 12), (16, 0, 16), (21, 0, 21), (13, 0, 10),
                                    (13, 3, 10), (18, 2, 11), (17, 7, 10), (20, 0, 14), (6, 0, 6),
                                    # block partitions: 8,8,1+.. splits -- (8, r-8) and even splits of r
                                    (17, 0, 17), (19, 0, 19), (22, 0, 22), (23, 0, 23), (24, 1, 22),
                                    (24, 0, 24), (22, 3, 18)])
def test_qft_matches_oracle_circuit(reg, n, lo, m, inverse):
    psi = rand_state(n, 7 * n + lo)
    h = reg(n, psi)
    Q.qsim_qft(h, lo, m, inverse)
    ref = psi.copy()
    O.qft(ref, lo, m, inverse)
    assert maxdiff(get(h, n), ref) < TOL
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


def test_qft_then_inverse_is_identity(reg):
    n = 22
    psi = rand_state(n, 1)
    h = reg(n, psi)
    Q.qsim_qft(h, 0, n, False)
    Q.qsim_qft(h, 0, n, True)
    assert maxdiff(get(h, n), psi) < 1e-12


def test_qft_basis_state_closed_form(reg):
    n = 14
    N = 1 << n
    for y in [0, 1, 12345, N - 1]:
        h = reg(n)
        Q.qsim_set_basis(h, y)
        Q.qsim_qft(h, 0, n, False)
        ref = np.exp(2j * np.pi * ((np.arange(N) * y) % N) / N) / math.sqrt(N)   # exact reduction
        assert maxdiff(get(h, n), ref) < 1e-13


# ------------------------------------------------------------------ configs
def test_cfg0_random_circuit_full_parity(reg):
    h = reg(10)
    gates = W.run_cfg0(h, n=10, seed=1, ngates=200)
    ref, kinds, qs = O.cfg0(10, 1, 200)
    assert [0 if g[0] == "haar" else 1 for g in gates] == list(kinds)
    assert [(g[1], g[2]) for g in gates] == [tuple(x) for x in qs]
    assert maxdiff(get(h, 10), ref) < TOL
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


def test_cfg1_grover_small_full_parity(reg):
    n, iters = 12, 50
    h = reg(n)
    k, trace = W.run_cfg1(h, n=n, seed=2, iters=iters)
    ref, rtrace = O.cfg1(n=n, seed=2, iters=iters)
    assert k == O.grover_mark(2, n)
    assert np.max(np.abs(trace - rtrace)) < TOL
    assert maxdiff(get(h, n), ref) < TOL


def test_cfg1_grover_full_size_closed_form(reg):
    n = 20
    h = reg(n)
    k, trace = W.run_cfg1(h, n=n, seed=2)
    assert len(trace) == 804 and k == O.grover_mark(2, n)
    th = math.asin(2.0**-10)
    t = np.arange(1, 805)
    assert np.max(np.abs(trace - np.sin((2 * t + 1) * th) ** 2)) < TOL
    assert trace[-1] == pytest.approx(0.999999756965, abs=1e-10)
    psi = get(h, n)
    others = math.cos((2 * 804 + 1) * th) / math.sqrt((1 << n) - 1)
    assert abs(psi[k] - math.sin((2 * 804 + 1) * th)) < TOL
    mask = np.ones(1 << n, bool); mask[k] = False
    assert np.max(np.abs(psi[mask] - others)) < TOL


def test_cfg2_gaussian_init_parity(reg):
    n = 20
    h = reg(n)
    Q.qsim_init_gaussian(h, 3)
    ref = O.gaussian_state(n, 3)
    assert maxdiff(get(h, n), ref) < 1e-14
    assert abs(Q.qsim_norm(h) - 1) < 1e-14


def test_cfg2_mid_size_full_parity(reg):
    n = 20
    h = reg(n)
    W.run_cfg2(h, n=n, seed=3)
    ref = O.cfg2(n=n, seed=3)
    assert maxdiff(get(h, n), ref) < TOL


def test_cfg2_full_size_sampled(reg):
    """n = 28 (4 GiB), the launch configuration bench.py times: sampled
    outputs against the oracle's DFT definition."""
    n = 28
    h = reg(n)
    W.run_cfg2(h, n=n, seed=3)
    assert abs(Q.qsim_norm(h) - 1) < 1e-12
    alpha = O.gaussian_state(n, 3)
    rng = np.random.default_rng(28)
    xs = [0, 1, (1 << n) - 1, 1 << 27] + [int(x) for x in rng.integers(0, 1 << n, size=4)]
    ref = O.dft_samples(alpha, xs, inverse=False)
    got = np.array([Q.qsim_get_state(h, x, 1)[0] for x in xs])
    assert maxdiff(got, ref) < TOL


@pytest.mark.parametrize("N,a,ne,nw", [(15, 7, 8, 4), (35, 3, 10, 6), (1007, 558, 12, 10)])
@pytest.mark.parametrize("sigma", [0.0, 1e-3])
def test_cfg3_order_finding_small(reg, N, a, ne, nw, sigma):
    h = reg(ne + nw)
    P = W.run_cfg3(h, ne=ne, nw=nw, N=N, seed=4, sigma=sigma, a=a)
    pr, psi = O.cfg3(ne=ne, nw=nw, N=N, seed=4, sigma=sigma, a=a, want_state=True)
    assert np.max(np.abs(P - pr)) < 1e-12
    assert maxdiff(get(h, ne + nw), psi) < TOL


def test_cfg3_modexp_fused_equals_modmul_chain(reg):
    ne, nw, N, a = 9, 6, 35, 3
    psi = rand_state(ne + nw, 3)
    h1 = reg(ne + nw, psi)
    Q.qsim_apply_perm(h1, Q.QSIM_PERM_MODEXP, ne, nw, elo=0, em=ne, base=a, modulus=N)
    h2 = reg(ne + nw, psi)
    ref = psi.copy()
    for j in range(ne):
        c = pow(a, 1 << j, N)
        cm = 1 << (ne - 1 - j)
        Q.qsim_apply_perm(h2, Q.QSIM_PERM_MODMUL, ne, nw, ctrl_mask=cm, ctrl_vals=cm, mult=c, modulus=N)
        O.modmul(ref, ne, nw, cm, cm, c, N)
    s1, s2 = get(h1, ne + nw), get(h2, ne + nw)
    assert np.array_equal(s1, ref) and np.array_equal(s2, ref)   # bit-exact


@pytest.mark.parametrize("ne,nw,N,a", [(6, 5, 31, 3), (8, 11, 2047, 5), (12, 11, 1999, 7), (10, 10, 1007, 558),
                                        (4, 12, 4093, 3), (3, 6, 35, 1)])
def test_modexp_run_sizes_bit_exact(reg, ne, nw, N, a):
    """MODEXP on runs of 2^5 .. 2^12 amplitudes (the bulk-copy ring up to 2^11,
    the one-CTA-per-run kernel above), base 1 (every run inactive): bit-exact
    against the oracle's chain of controlled MODMULs."""
    psi = rand_state(ne + nw, ne * 31 + nw)
    h = reg(ne + nw, psi)
    Q.qsim_apply_perm(h, Q.QSIM_PERM_MODEXP, ne, nw, elo=0, em=ne, base=a, modulus=N)
    ref = psi.copy()
    for j in range(ne):
        cm = 1 << (ne - 1 - j)
        O.modmul(ref, ne, nw, cm, cm, pow(a, 1 << j, N), N)
    assert np.array_equal(get(h, ne + nw), ref)


@pytest.mark.parametrize("c", [1, 4, 1006])
def test_modmul_controlled_runs_bit_exact(reg, c):
    """MODMUL with a control qubit outside the work register (half the runs
    inactive) and c = 1 (identity): bit-exact against the oracle."""
    ne, nw, N = 7, 10, 1007
    psi = rand_state(ne + nw, c)
    h = reg(ne + nw, psi)
    Q.qsim_apply_perm(h, Q.QSIM_PERM_MODMUL, ne, nw, ctrl_mask=1 << 2, ctrl_vals=1 << 2, mult=c, modulus=N)
    ref = psi.copy()
    O.modmul(ref, ne, nw, 1 << 2, 1 << 2, c, N)
    assert np.array_equal(get(h, ne + nw), ref)


def test_cfg3_full_size_fejer(reg):
    """n = 30 (16 GiB), sigma = 0: P(e) against the exact closed form."""
    from _closed_forms import fejer_distribution, order
    h = reg(30)
    a = W.shor_base(4, 1007)
    assert a == O.shor_base(4, 1007)
    P = W.run_cfg3(h, ne=20, nw=10, N=1007, seed=4, sigma=0.0)
    ref = fejer_distribution(1 << 20, order(a, 1007))
    assert np.max(np.abs(P - ref)) < 1e-12
    assert abs(P.sum() - 1) < 1e-12


@pytest.mark.parametrize("n,p", [(12, 0.05), (14, 1e-4), (9, 0.2)])
def test_cfg4_noisy_brickwork_parity(reg, n, p):
    h = reg(n)
    ev = W.run_cfg4(h, n=n, layers=20, seed=5, sigma=1e-3, p=p)
    ref, rev = O.cfg4(n=n, layers=20, seed=5, sigma=1e-3, p=p)
    assert [tuple(e) for e in ev] == [tuple(e) for e in rev]     # bit-exact event list
    assert maxdiff(get(h, n), ref) < TOL
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


# ------------------------------------------------------------------ permutations / readout
def test_table_permutation_bit_exact(reg):
    n, lo, m = 12, 3, 5
    psi = rand_state(n, 8)
    h = reg(n, psi)
    rng = np.random.default_rng(0)
    table = rng.permutation(1 << m)
    Q.qsim_apply_perm(h, Q.QSIM_PERM_TABLE, lo, m, table=table, ctrl_mask=1, ctrl_vals=1)
    ref = np.empty_like(psi)
    shift = n - lo - m
    for j in range(1 << n):
        v = (j >> shift) & ((1 << m) - 1)
        ctrl = (j >> (n - 1)) & 1
        nv = table[v] if ctrl else v
        ref[(j & ~(((1 << m) - 1) << shift)) | (int(nv) << shift)] = psi[j]
    assert np.array_equal(get(h, n), ref)


@pytest.mark.parametrize("n,lo,m", [(24, 4, 16), (24, 0, 16), (24, 8, 16), (22, 2, 14), (26, 6, 18)])
def test_marginals_many_bins_match_oracle(reg, n, lo, m):
    """Marginals over many small bins (the warp-per-bin kernel), with the
    remaining positions above, below and on both sides of the range."""
    psi = rand_state(n, 100 + lo + m)
    h = reg(n, psi)
    got = Q.qsim_probs(h, lo, m)
    ref = O.probs(psi, lo, m)
    assert np.max(np.abs(got - ref)) < 1e-15
    assert abs(got.sum() - 1) < 1e-12


def test_norm_probs_measure(reg):
    n = 16
    psi = rand_state(n, 21) * 0.9
    h = reg(n, psi)
    assert Q.qsim_norm(h) == pytest.approx(O.norm(psi), abs=1e-14)
    for lo, m in [(0, 4), (5, 7), (10, 6), (0, 16)]:
        assert np.max(np.abs(Q.qsim_probs(h, lo, m) - O.probs(psi, lo, m))) < 1e-14
    psi /= np.linalg.norm(psi)
    Q.qsim_set_state(h, 0, psi)
    cum = np.cumsum(np.abs(psi) ** 2)
    for s in range(50):
        r = O.u01(O.draw(9, O.TAG_MEASURE, s, 0)[0])
        i = O.measure(psi, r)
        margin = min(abs(r - cum[i]), abs(r - (cum[i - 1] if i else 0.0)))
        if margin > 1e-12:
            assert Q.qsim_measure(h, r) == i
    assert Q.qsim_prob_index(h, 777) == pytest.approx(abs(psi[777]) ** 2, abs=1e-16)


def test_inject_errors_bit_exact_events(reg):
    n = 10
    psi = rand_state(n, 2)
    h = reg(n, psi)
    ref = psi.copy()
    for epoch in range(30):
        ev = Q.qsim_inject_errors(h, 11, 0.1, (1 << n) - 1, epoch)
        rev = O.inject_paulis(ref, 11, epoch, (1 << n) - 1, 0.1)
        assert ev == rev
    assert np.array_equal(get(h, n), ref)     # Paulis are exact


# ------------------------------------------------------------------ errors / edge cases
def test_validation_errors_have_no_effect(reg):
    n = 6
    psi = rand_state(n, 1)
    h = reg(n, psi)
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_apply_1q(h, n, np.eye(2))
    assert e.value.code == Q.QSIM_ERANGE
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_apply_ctrl(h, 1 << 2, 1 << 2, 2, np.eye(2))
    assert e.value.code == Q.QSIM_EINVAL
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_apply_perm(h, Q.QSIM_PERM_TABLE, 0, 3, table=[0, 1, 2, 3, 4, 5, 6, 6])
    assert e.value.code == Q.QSIM_ENOTBIJ
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_apply_perm(h, Q.QSIM_PERM_MODMUL, 2, 4, mult=5, modulus=15)
    assert e.value.code == Q.QSIM_ENOTBIJ
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_inject_errors(h, 1, 1.5, 1, 0)
    assert e.value.code == Q.QSIM_EINVAL
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_qft(h, 3, 4)
    assert e.value.code == Q.QSIM_ERANGE
    assert np.array_equal(get(h, n), psi)
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_create(0)
    assert e.value.code == Q.QSIM_ERANGE


def test_memory_bytes():
    assert Q.qsim_memory_bytes(20) == 16777216
    assert Q.qsim_memory_bytes(30) == 17179869184
    assert Q.qsim_memory_bytes(1) == 32


# ------------------------------------------------------------------ gate fusion
@pytest.mark.parametrize("n,ngates", [(9, 120), (13, 300), (17, 400), (20, 150)])
def test_fused_gate_passes_match_oracle(reg, n, ngates):
    """Random mix of dense, controlled (1-3 controls, both values), diagonal
    and controlled-diagonal gates: the fused tile passes (gate queue) and the
    unfused kernels both equal the oracle."""
    rng = np.random.default_rng(1000 + n)
    psi = rand_state(n, 50 + n)
    hf = reg(n, psi)
    hu = reg(n, psi)
    Q.qsim_set_fusion(hu, False)
    ref = psi.copy()
    for _ in range(ngates):
        q = int(rng.integers(n))
        kind = rng.integers(4)
        if kind == 0:
            U = rand_mat(rng) / 1.5
        elif kind == 1:
            U = np.diag(np.exp(1j * rng.uniform(0, 6.3, 2)))
        elif kind == 2:
            a = O.haar_angles(7, int(rng.integers(1 << 20)))
            U = O.mat_angles(O.HAAR, a)
        else:
            U = np.array([[0, 1], [1, 0]], complex)
        others = [c for c in range(n) if c != q]
        k = int(rng.integers(0, 4))
        ctrl = rng.choice(others, size=k, replace=False) if k else []
        mask = sum(1 << int(c) for c in ctrl)
        vals = sum(int(rng.integers(2)) << int(c) for c in ctrl)
        for h in (hf, hu):
            Q.qsim_apply_ctrl(h, mask, vals, q, U) if mask else Q.qsim_apply_1q(h, q, U)
        O.apply_ctrl(ref, mask, vals, q, U) if mask else O.apply_1q(ref, q, U)
    assert maxdiff(get(hf, n), ref) < TOL
    assert maxdiff(get(hu, n), ref) < TOL


@pytest.mark.parametrize("n,nq,ngates", [(14, 5, 400), (18, 7, 500), (22, 14, 600)])
def test_fused_merge_runs_match_oracle(reg, n, nq, ngates):
    """Runs the planner's merging hard: gates on a few qubits, each
    uncontrolled, singly controlled (either value) or a controlled phase, so
    consecutive gates on one target collapse into single / choice (DENSE2) /
    controlled (CDENSE) register updates and commute past each other."""
    rng = np.random.default_rng(77 + n)
    psi = rand_state(n, 90 + n)
    h = reg(n, psi)
    ref = psi.copy()
    qs = [int(x) for x in rng.choice(n, size=nq, replace=False)]
    for _ in range(ngates):
        q = qs[int(rng.integers(nq))]
        kind = int(rng.integers(5))
        if kind == 4:
            U = np.diag([1, np.exp(1j * rng.uniform(0, 6.3))])
        else:
            U = O.mat_angles(O.HAAR, O.haar_angles(9, int(rng.integers(1 << 20))))
        c = qs[int(rng.integers(nq))]
        if c != q and rng.integers(3):
            v = int(rng.integers(2))
            Q.qsim_apply_ctrl(h, 1 << c, v << c, q, U)
            O.apply_ctrl(ref, 1 << c, v << c, q, U)
        else:
            Q.qsim_apply_1q(h, q, U)
            O.apply_1q(ref, q, U)
    assert maxdiff(get(h, n), ref) < TOL
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


def test_fusion_is_a_single_pass_for_small_registers(reg):
    """configs[0]: all 200 gates of the n = 10 circuit fuse into one launch."""
    h = reg(10)
    Q.qsim_sync(h)
    l0 = Q.qsim_launch_count(h)
    W.run_cfg0(h, n=10, seed=1, ngates=200)
    Q.qsim_sync(h)
    assert Q.qsim_launch_count(h) - l0 <= 3
    ref, _, _ = O.cfg0(10, 1, 200)
    assert maxdiff(get(h, 10), ref) < TOL


# ------------------------------------------------------------------ full-size configs
def test_cfg1_full_size_oracle_parity(reg):
    """configs[1] exactly as specified (n = 20, 804 iterations) against the
    oracle's literal -H_n V_f0 H_n V_fk circuit, element by
    element, trace and final state."""
    n = 20
    h = reg(n)
    k, trace = W.run_cfg1(h, n=n, seed=2)
    ref, rtrace = O.cfg1(n=n, seed=2, iters=804)
    assert np.max(np.abs(trace - rtrace)) < TOL
    assert maxdiff(get(h, n), ref) < TOL


def _cfg4_inverse(h, n, layers, seed, sigma, events):
    """Apply the exact inverse of configs[4] (same noise realisation) through
    the C-ABI, with matrices built by the oracle's own angle code."""
    import math as _m
    g0s, g = [], 0
    for l in range(layers):
        g0s.append(g)
        g += n + len(range(l & 1, n - 1, 2))
    byl = {}
    for (l, q, k) in events:
        byl.setdefault(l, []).append((q, k))
    for l in reversed(range(layers)):
        for (q, k) in reversed(byl.get(l, [])):
            Q.qsim_apply_1q(h, q, O.pauli(k))              # Paulis are involutions
        g0 = g0s[l]
        cnots = list(range(l & 1, n - 1, 2))
        for i, c in reversed(list(enumerate(cnots))):
            U = O.mat_angles(O.RP, [_m.pi / 2, _m.pi], seed=seed, sigma=sigma, g=g0 + n + i)
            Q.qsim_apply_ctrl(h, 1 << c, 1 << c, c + 1, U.conj().T)
        for q in reversed(range(n)):
            U = O.mat_angles(O.HAAR, O.haar_angles(seed, l * n + q), seed=seed, sigma=sigma, g=g0 + q)
            Q.qsim_apply_1q(h, q, U.conj().T)


@pytest.mark.parametrize("n", [20, 32])
def test_cfg4_mirror_returns_to_zero(reg, n):
    """configs[4] (n = 32 is the full single-GPU size, 64 GiB): the circuit
    followed by its exact inverse built from the oracle's matrices returns to
    |0..0> -- pins every noisy gate applied by the GPU at a size the oracle
    cannot simulate; the norm stays 1 to 1e-12 throughout."""
    layers, seed, sigma, p = 20, 5, 1e-3, 1e-4 if n == 32 else 0.02
    h = reg(n)
    ev = W.run_cfg4(h, n=n, layers=layers, seed=seed, sigma=sigma, p=p)
    assert abs(Q.qsim_norm(h) - 1) < 1e-12
    _cfg4_inverse(h, n, layers, seed, sigma, ev)
    assert Q.qsim_prob_index(h, 0) > 1 - 1e-10
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


def test_cfg1_carried_sum_equals_reduced_sum():
    """k_grover_regs carries the amplitude sum through the iterations (D keeps
    <s|.>) instead of re-reducing it every iteration; the
    re-reducing variant (QSIM_GROVER_REDUCE) gives the same trace and state."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]);"
        "from paper_quant_ph_0201042_b200 import qsim as Q; from paper_quant_ph_0201042_b200 import workloads as W;"
        "h = Q.qsim_create(20); k, tr = W.run_cfg1(h, n=20, seed=2);"
        "np.save(sys.argv[2], np.concatenate([tr.astype(complex), Q.qsim_get_state(h, 0, 1 << 20)]))")
    res = []
    for env in ({}, {"QSIM_GROVER_REDUCE": "1"}):
        path = f"/tmp/grover_{len(env)}.npy"
        r = subprocess.run([sys.executable, "-c", script, root, path], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        res.append(np.load(path))
    assert np.max(np.abs(res[0] - res[1])) < 1e-13
