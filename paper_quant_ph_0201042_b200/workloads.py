"""The five BASELINE.json configs as call sequences on the C-ABI.

These are input generators + drivers, not arithmetic of the method: every
random choice comes from the library's own Philox4x32-10
(``qsim_philox_draw``, R1) and every gate is applied by libqsim's
kernels.  The draw rules are the readings R11, R12, R16-R21 of DESIGN.md; the
oracle (test infrastructure) implements the same rules independently.
"""
from __future__ import annotations

import math

from . import qsim as Q

TWO_PI = 2.0 * math.pi


def u01(a: int) -> float:
    return (a >> 11) * 2.0**-53


def uint_below(a: int, m: int) -> int:
    return (a * m) >> 64


def haar_angles(seed: int, i: int):
    """(alpha, beta, theta, gamma) of the Haar gate with index i (R12)."""
    a0, b0 = Q.qsim_philox_draw(seed, Q.QSIM_TAG_HAAR, i, 0)
    a1, b1 = Q.qsim_philox_draw(seed, Q.QSIM_TAG_HAAR, i, 1)
    return [TWO_PI * u01(b0), TWO_PI * u01(a1), math.acos(math.sqrt(u01(a0))), TWO_PI * u01(b1)]


NOT = [[0, 1], [1, 0]]


def run_cfg0(h, n: int = 10, seed: int = 1, ngates: int = 200):
    """configs[0]: random circuit from |0..0> (R21).  Returns the gate list.
    The draws come in three batched calls and the circuit goes to the library
    as one gate list (one C-ABI crossing); the gates are those of R21."""
    Q.qsim_set_basis(h, 0)
    dg = Q.qsim_philox_draws(seed, Q.QSIM_TAG_GATE, 0, ngates, 0)
    dh0 = Q.qsim_philox_draws(seed, Q.QSIM_TAG_HAAR, 0, ngates, 0)
    dh1 = Q.qsim_philox_draws(seed, Q.QSIM_TAG_HAAR, 0, ngates, 1)
    dp = Q.qsim_philox_draws(seed, Q.QSIM_TAG_PAIR, 0, ngates, 0)
    gates, glist = [], []
    for g in range(ngates):
        a, b = int(dg[g, 0]), int(dg[g, 1])
        if u01(a) < 0.7:
            q = uint_below(b, n)
            a0, b0, a1, b1 = int(dh0[g, 0]), int(dh0[g, 1]), int(dh1[g, 0]), int(dh1[g, 1])
            ang = [TWO_PI * u01(b0), TWO_PI * u01(a1), math.acos(math.sqrt(u01(a0))), TWO_PI * u01(b1)]
            glist.append(("angles", q, Q.QSIM_GATE_HAAR, ang, 0, 0))
            gates.append(("haar", q, -1))
        else:
            a2, b2 = int(dp[g, 0]), int(dp[g, 1])
            c = uint_below(a2, n)
            t = uint_below(b2, n - 1)
            t += t >= c
            glist.append(("matrix", t, NOT, 1 << c, 1 << c))
            gates.append(("cnot", t, c))
    Q.qsim_apply_gates(h, glist)
    return gates


def grover_mark(seed: int, n: int) -> int:
    a, _ = Q.qsim_philox_draw(seed, Q.QSIM_TAG_MARK, 0, 0)
    return uint_below(a, 1 << n)


def run_cfg1(h, n: int = 20, seed: int = 2, iters: int | None = None):
    """configs[1]: H_n|0>, then Grover iterations; returns (mark, trace)."""
    if iters is None:
        iters = math.floor(math.pi / 4 * math.sqrt(1 << n))
    Q.qsim_set_basis(h, 0)
    Q.qsim_hadamard(h, 0, n)
    k = grover_mark(seed, n)
    trace = Q.qsim_grover(h, k, iters, trace=True)
    return k, trace


def run_cfg2(h, n: int = 28, seed: int = 3):
    """configs[2]: normalised complex Gaussian input (R19), then the QFT."""
    Q.qsim_init_gaussian(h, seed)
    Q.qsim_qft(h, 0, n, False)


def shor_base(seed: int, N: int) -> int:
    """R11: first a_t = 2 + uint(draw(seed, BASE, t, 0).a, N-3) coprime to N."""
    t = 0
    while True:
        a, _ = Q.qsim_philox_draw(seed, Q.QSIM_TAG_BASE, t, 0)
        x = 2 + uint_below(a, N - 3)
        if math.gcd(x, N) == 1:
            return x
        t += 1


def run_cfg3(h, ne: int = 20, nw: int = 10, N: int = 1007, seed: int = 4, sigma: float = 0.0,
             a: int | None = None, fused_modexp: bool = True):
    """configs[3]: order finding (R9-R11); returns P(e) over the exponent register."""
    a = shor_base(seed, N) if a is None else a
    Q.qsim_set_basis(h, 1)                       # e = 0, w = 1
    Q.qsim_set_gate_noise(h, seed, sigma)
    Q.qsim_set_gate_counter(h, 0)
    if sigma > 0:
        Q.qsim_hadamard_angles(h, 0, ne)             # = ne angle-form H gates (counter + noise)
    else:
        Q.qsim_hadamard(h, 0, ne)
        Q.qsim_set_gate_counter(h, ne)
    if fused_modexp:
        Q.qsim_apply_perm(h, Q.QSIM_PERM_MODEXP, ne, nw, elo=0, em=ne, base=a, modulus=N)
    else:
        for j in range(ne):
            c = pow(a, 1 << j, N)
            cm = 1 << (ne - 1 - j)
            Q.qsim_apply_perm(h, Q.QSIM_PERM_MODMUL, ne, nw, ctrl_mask=cm, ctrl_vals=cm, mult=c, modulus=N)
    Q.qsim_qft(h, 0, ne, True)
    probs = Q.qsim_probs(h, 0, ne)
    Q.qsim_set_gate_noise(h, 0, 0.0)
    return probs


def run_cfg4(h, n: int = 32, layers: int = 20, seed: int = 5, sigma: float = 1e-3, p: float = 1e-4):
    """configs[4]: noisy Haar + CNOT brickwork (R18); returns the Pauli events."""
    Q.qsim_set_basis(h, 0)
    Q.qsim_set_gate_noise(h, seed, sigma)
    Q.qsim_set_gate_counter(h, 0)
    events = []
    allq = (1 << n) - 1
    for layer in range(layers):
        for q in range(n):
            Q.qsim_apply_angles(h, Q.QSIM_GATE_HAAR, haar_angles(seed, layer * n + q), 0, 0, q)
        for c in range(layer & 1, n - 1, 2):
            Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, [math.pi / 2, math.pi], 1 << c, 1 << c, c + 1)
        events += Q.qsim_inject_errors(h, seed, p, allq, layer, cap=4 * n)
    Q.qsim_set_gate_noise(h, 0, 0.0)
    return events


# ---------------------------------------------------------------------------
# Row f2: the paper's noise experiments as batched trajectories (R33-R36).
# The handle holds b + (register) qubits; qubits [0, b) index the 2^b
# trajectories, trajectory t draws from seed + t.  Averages over trajectories
# are marginals of the batched handle (qsim_probs over the register).

def run_ht_batch(h, n: int, b: int, k: int, seed: int, sigma: float, p: float):
    """HT experiment (R34): |0..0>, k times (noisy H on every
    qubit, then the depolarizing channel on every qubit, epoch = application).
    Returns (average |<0|psi_t>|^2 over the 2^b trajectories, events)."""
    Q.qsim_set_batch(h, b)
    reg = [0j] * (1 << n)
    reg[0] = 1.0
    Q.qsim_batch_set_state(h, reg)
    Q.qsim_set_gate_noise(h, seed, sigma)
    Q.qsim_set_gate_counter(h, 0)
    regmask = ((1 << n) - 1) << b
    events = []
    for i in range(k):
        for q in range(n):
            Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, [math.pi / 4, math.pi], 0, 0, b + q)
        events += Q.qsim_inject_errors(h, seed, p, regmask, i, cap=n << b, traj=True)
    p0 = float(Q.qsim_probs(h, b, n)[0])
    Q.qsim_set_gate_noise(h, 0, 0.0)
    return p0, events


def run_grover_batch(h, n: int, b: int, mark: int, iters: int, seed: int, sigma: float, p: float):
    """Grover experiment (R35): register qubits [b, b+n),
    ancilla b+n (the LSB) in |->; noisy H_n and noisy NOT in V_f (all register
    qubits control it); depolarizing channel on the register per G-iteration.
    Returns the trajectory-averaged P(register = mark) after each iteration."""
    Q.qsim_set_batch(h, b)
    r = math.sqrt(0.5)
    reg = [0j] * (1 << (n + 1))
    reg[0], reg[1] = r, -r
    Q.qsim_batch_set_state(h, reg)
    Q.qsim_set_gate_noise(h, seed, sigma)
    Q.qsim_set_gate_counter(h, 0)
    regq = range(b, b + n)
    cmask = sum(1 << q for q in regq)
    vk = sum(((mark >> (n - 1 - i)) & 1) << (b + i) for i in range(n))
    anc = b + n
    hang, xang = [math.pi / 4, math.pi], [math.pi / 2, math.pi]
    for q in regq:
        Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, hang, 0, 0, q)
    trace = []
    for t in range(iters):
        Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, xang, cmask, vk, anc)
        for q in regq:
            Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, hang, 0, 0, q)
        Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, xang, cmask, 0, anc)
        for q in regq:
            Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, hang, 0, 0, q)
        Q.qsim_inject_errors(h, seed, p, cmask, t, cap=n << b, traj=True)
        trace.append(float(Q.qsim_probs(h, b, n)[mark]))
    Q.qsim_set_gate_noise(h, 0, 0.0)
    return trace


def qft_decoherent_gates(h, lo: int, m: int, seed: int, sigma: float, p: float, inverse: bool = False,
                         ntraj: int = 1):
    """The QFT circuit on [lo, lo+m) gate by gate with its angle noise and the
    depolarizing channel on [lo, lo+m) after every R_d (PAPER.md:1053-1160,
    R36); the gate counter is the caller's.  Returns the events."""
    sg = -1.0 if inverse else 1.0
    r = math.sqrt(0.5)
    H = [[r, r], [r, -r]]
    qmask = ((1 << m) - 1) << lo
    epoch = 0
    events = []
    for j in range(m):
        if sigma > 0:
            Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, [math.pi / 4, math.pi], 0, 0, lo + j)
        else:
            Q.qsim_apply_1q(h, lo + j, H)
        for k in range(j + 1, m):
            phi = sg * math.pi / 2.0 ** (k - j)
            cm = 1 << (lo + k)
            if sigma > 0:
                Q.qsim_apply_angles(h, Q.QSIM_GATE_P1, [phi], cm, cm, lo + j)
            else:
                Q.qsim_apply_ctrl(h, cm, cm, lo + j, [[1, 0], [0, complex(math.cos(phi), math.sin(phi))]])
            events += Q.qsim_inject_errors(h, seed, p, qmask, epoch, cap=m * ntraj, traj=True)
            epoch += 1
    for j in range(m // 2):
        Q.qsim_swap(h, lo + j, lo + m - 1 - j)
    return events


def shor_register_state(m: int, x: int, N: int, v: int):
    """The semantic-mode exponent register of Shor step 3
    prepared by the library on its own m-qubit handle, read back to the host."""
    g = Q.qsim_create(m)
    try:
        Q.qsim_shor_semantic_state(g, x, N, v)
        return Q.qsim_get_state(g, 0, 1 << m)
    finally:
        Q.qsim_destroy(g)


def run_qft_fidelity_batch(h, m: int, b: int, x: int, N: int, v: int, seed: int, sigma: float, p: float):
    """QFT-16 experiment of PAPER.md:1124-1160 (Table 7): every trajectory starts
    in the Shor register state, runs the noisy / decoherent QFT, and its fidelity
    |<QFT psi | psi_t>| to the ideal QFT output (library, noiseless) is
    returned per trajectory."""
    Q.qsim_set_batch(h, b)
    reg = shor_register_state(m, x, N, v)
    g = Q.qsim_create(m)
    try:
        Q.qsim_set_state(g, 0, reg)
        Q.qsim_qft(g, 0, m, False)
        ideal = Q.qsim_get_state(g, 0, 1 << m)
    finally:
        Q.qsim_destroy(g)
    Q.qsim_batch_set_state(h, reg)
    Q.qsim_set_gate_noise(h, seed, sigma)
    Q.qsim_set_gate_counter(h, 0)
    qft_decoherent_gates(h, b, m, seed, sigma, p, ntraj=1 << b)
    Q.qsim_set_gate_noise(h, 0, 0.0)
    return abs(Q.qsim_batch_overlap(h, ideal, 1 << b))
