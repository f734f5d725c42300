"""GPU parity for row f2 (batched noisy trajectories, R33-R36)
through the C-ABI: every trajectory t of a batched handle equals the oracle's
single-register trajectory run with seed + t (element-wise, 1e-10), Pauli
events bit-exactly, and the batch averages (qsim_probs over the register,
qsim_batch_overlap) equal the means of the oracle's trajectories.  Single
handles and in-process rank groups (the trajectory index on rank bits)."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

TOL = 1e-10


@pytest.fixture
def mk():
    made = []

    def make(n, world=1):
        h = Q.qsim_create(n) if world == 1 else Q.qsim_create_group(n, world)
        made.append(h)
        return h

    yield make
    for h in made:
        Q.qsim_destroy(h)


def slices(h, n_total, b):
    psi = Q.qsim_get_state(h, 0, 1 << n_total)
    return psi.reshape(1 << b, -1) * math.sqrt(1 << b)


def oracle_events_ht(n, b, k, seed, p, ntraj):
    ev = []
    for t in range(ntraj):
        dummy = np.zeros(1 << n, complex)
        dummy[0] = 1
        for i in range(k):
            for (e, q, w) in O.inject_paulis(dummy, seed + t, i, (1 << n) - 1, p):
                ev.append((e, q + b, w, t))
    # library order: per epoch, qubit-major then trajectory
    return sorted(ev, key=lambda x: (x[0], x[1], x[3]))


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("sigma,p,k", [(2e-2, 0.03, 6), (0.0, 0.05, 9), (2e-2, 0.0, 12)])
def test_ht_batch_trajectories_match_oracle(mk, world, sigma, p, k):
    """Runs of per-trajectory gates on a qubit (noisy H's, Pauli tables,
    constant H's between them) are merged into device-side product tables by
    the planner: every trajectory still equals the oracle's."""
    n, b, seed = 10, 5, 100
    h = mk(n + b, world)
    p0, ev = W.run_ht_batch(h, n, b, k, seed, sigma, p)
    S = slices(h, n + b, b)
    refs = [O.traj_ht(n, k, seed + t, sigma, p) for t in range(1 << b)]
    for t in range(1 << b):
        assert np.max(np.abs(S[t] - refs[t])) < TOL, t
    assert ev == oracle_events_ht(n, b, k, seed, p, 1 << b)
    assert abs(p0 - np.mean([abs(r[0]) ** 2 for r in refs])) < 1e-12
    assert abs(Q.qsim_norm(h) - 1) < 1e-12


def test_ht_batch_noiseless_returns_zero_state(mk):
    n, b = 12, 4
    h = mk(n + b)
    p0, ev = W.run_ht_batch(h, n, b, 4, 1, 0.0, 0.0)
    assert ev == [] and abs(p0 - 1) < 1e-12


def test_grover_batch_trajectories_match_oracle(mk):
    n, b, mark, iters, seed, sigma, p = 8, 4, 177, 5, 300, 3e-2, 0.02
    h = mk(n + 1 + b)
    trace = W.run_grover_batch(h, n, b, mark, iters, seed, sigma, p)
    S = slices(h, n + 1 + b, b)
    traces = []
    for t in range(1 << b):
        ref, tr = O.traj_grover(n, mark, iters, seed + t, sigma, p)
        assert np.max(np.abs(S[t] - ref)) < TOL, t
        traces.append(tr)
    assert np.max(np.abs(np.array(trace) - np.mean(traces, axis=0))) < 1e-12


@pytest.mark.parametrize("world", [1, 2])
def test_qft_fidelity_batch_matches_oracle(mk, world):
    m, b, x, N, v, seed, sigma, p = 10, 3, 7, 33, 1, 55, 1e-2, 0.01
    h = mk(m + b, world)
    fid = W.run_qft_fidelity_batch(h, m, b, x, N, v, seed, sigma, p)
    psi0 = O.shor_semantic_state(m, x, N, v)
    ideal = psi0.copy()
    O.qft(ideal, 0, m)
    S = slices(h, m + b, b)
    for t in range(1 << b):
        ref = psi0.copy()
        O.qft_decoherent(ref, 0, m, noise=O.Noise(seed=seed + t, sigma=sigma), p=p)
        assert np.max(np.abs(S[t] - ref)) < TOL, t
        assert abs(fid[t] - abs(O.inner(ideal, ref))) < 1e-12


def test_batch_rejects_gates_on_the_trajectory_index(mk):
    h = mk(14)
    Q.qsim_set_batch(h, 3)
    Q.qsim_set_gate_noise(h, 1, 1e-3)
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, [0.1, 0.2], 0, 0, 1)
    assert e.value.code == Q.QSIM_EINVAL
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_apply_1q(h, 2, np.eye(2))
    assert e.value.code == Q.QSIM_EINVAL
    with pytest.raises(Q.QsimError) as e:
        Q.qsim_inject_errors(h, 1, 0.1, 1, 0)
    assert e.value.code == Q.QSIM_EINVAL
