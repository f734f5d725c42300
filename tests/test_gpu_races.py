"""Race / synchronisation stress for the pipelined kernels (compute-sanitizer
is closed on this pool, so races are hunted by determinism instead): every
kernel that stages data through shared memory with mbarriers, TMA rings,
named barriers or a grid-wide counter runs the same input many times at a
size that gives every SM several tiles; a race (a stage reused before every
reader is done, a missing fence between the generic and async proxies, a
barrier that lets a warp through early) would show up as a run that differs
in some bit from the others.  One run per case is also checked against the
oracle.  Kernels: k_qft13, k_qft_tma, k_qft_gen, k_ops_pp / k_ops_tma /
k_ops_pass, k_perm_ring, k_grover_regs, k_probs_warp, the host-stream pipeline.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

REPS = 12


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def repeat(n, psi, op, reps=REPS):
    """op(h) on a fresh copy of psi, reps times; returns the distinct outputs
    (bytes) and the first output."""
    h = Q.qsim_create(n)
    outs = set()
    first = None
    kernels = set()
    try:
        for r in range(reps):
            Q.qsim_set_state(h, 0, psi)
            Q.qsim_profile(h, True)
            op(h)
            prof = Q.qsim_profile_json(h)
            prof.pop("_launches", None)
            kernels |= set(prof)
            Q.qsim_profile(h, False)
            got = Q.qsim_get_state(h, 0, 1 << n)
            outs.add(got.tobytes())
            if first is None:
                first = got
    finally:
        Q.qsim_destroy(h)
    return outs, first, kernels


def test_qft13_deterministic():
    n = 20   # the default plan takes the 13-bit passes where they save a pass (m = 20: 2 instead of 3)
    psi = rand_state(n, 1)
    outs, got, ks = repeat(n, psi, lambda h: Q.qsim_qft(h, 0, n, False))
    assert "k_qft13" in ks
    assert len(outs) == 1
    ref = psi.copy()
    O.qft(ref, 0, n, False)
    assert np.max(np.abs(got - ref)) < 1e-10


def test_qft_tma_deterministic():
    n = 22
    psi = rand_state(n, 2)
    outs, got, ks = repeat(n, psi, lambda h: Q.qsim_qft(h, 3, 9, True))   # < 10 wires: the 12-bit kernel
    assert "k_qft_tma" in ks
    assert len(outs) == 1
    ref = psi.copy()
    O.qft(ref, 3, 9, True)
    assert np.max(np.abs(got - ref)) < 1e-10


def test_qft_gen_deterministic():
    n = 22

    def op(h):
        Q.qsim_set_gate_noise(h, 7, 1e-3)
        Q.qsim_set_gate_counter(h, 0)
        Q.qsim_qft(h, 0, 18, False)
        Q.qsim_set_gate_noise(h, 0, 0.0)

    psi = rand_state(n, 3)
    outs, got, ks = repeat(n, psi, op)
    assert "k_qft_gen" in ks
    assert len(outs) == 1
    ref = psi.copy()
    O.qft(ref, 0, 18, False, noise=O.Noise(7, 1e-3, 0))
    assert np.max(np.abs(got - ref)) < 1e-10


def test_gate_list_passes_deterministic():
    n = 22

    def op(h):
        W.run_cfg4(h, n=n, layers=6, seed=5, sigma=1e-3, p=0.02)
        Q.qsim_sync(h)

    outs, got, ks = repeat(n, np.zeros(1 << n, complex), op, reps=8)
    assert ks & {"k_ops_pp", "k_ops_pass", "k_ops_tma"}
    assert len(outs) == 1
    ref, _ = O.cfg4(n=n, layers=6, seed=5, sigma=1e-3, p=0.02)
    assert np.max(np.abs(got - ref)) < 1e-10


def test_modexp_ring_deterministic():
    ne, nw, N, a = 12, 10, 1007, 558
    n = ne + nw
    psi = rand_state(n, 4)
    outs, got, ks = repeat(n, psi, lambda h: Q.qsim_apply_perm(h, Q.QSIM_PERM_MODEXP, ne, nw, elo=0, em=ne,
                                                               base=a, modulus=N))
    assert "k_perm_ring" in ks
    assert len(outs) == 1
    ref = psi.copy()
    for j in range(ne):
        cm = 1 << (ne - 1 - j)
        O.modmul(ref, ne, nw, cm, cm, pow(a, 1 << j, N), N)
    assert np.array_equal(got, ref)


def test_grover_regs_deterministic():
    n = 18
    traces = set()
    h = Q.qsim_create(n)
    try:
        for _ in range(REPS):
            k, tr = W.run_cfg1(h, n=n, seed=2, iters=100)
            traces.add(tr.tobytes() + Q.qsim_get_state(h, 0, 1 << n).tobytes())
    finally:
        Q.qsim_destroy(h)
    assert len(traces) == 1
    _, rt = O.cfg1(n=n, seed=2, iters=100)
    assert np.max(np.abs(np.frombuffer(next(iter(traces))[:800]) - rt)) < 1e-10


def test_marginals_deterministic():
    n = 24
    psi = rand_state(n, 5)
    h = Q.qsim_create(n)
    try:
        Q.qsim_set_state(h, 0, psi)
        res = {Q.qsim_probs(h, 0, 16).tobytes() for _ in range(REPS)}
        p = np.frombuffer(next(iter(res)))
    finally:
        Q.qsim_destroy(h)
    assert len(res) == 1
    assert np.max(np.abs(p - O.probs(psi, 0, 16))) < 1e-12


def test_host_stream_deterministic():
    n = 20
    psi = rand_state(n, 6)
    inp = np.ascontiguousarray(np.stack([psi] * 4))
    h = Q.qsim_create(n)
    try:
        outs = set()
        for _ in range(4):
            out = np.zeros_like(inp)
            Q.qsim_qft_host_stream(h, 0, n, False, inp, out, 4, 1 << n, 1 << n)
            outs |= {o.tobytes() for o in out}
    finally:
        Q.qsim_destroy(h)
    assert len(outs) == 1
