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
    """configs[0]: random circuit from |0..0> (R21).  Returns the gate list."""
    Q.qsim_set_basis(h, 0)
    gates = []
    for g in range(ngates):
        a, b = Q.qsim_philox_draw(seed, Q.QSIM_TAG_GATE, g, 0)
        if u01(a) < 0.7:
            q = uint_below(b, n)
            Q.qsim_apply_angles(h, Q.QSIM_GATE_HAAR, haar_angles(seed, g), 0, 0, q)
            gates.append(("haar", q, -1))
        else:
            a2, b2 = Q.qsim_philox_draw(seed, Q.QSIM_TAG_PAIR, g, 0)
            c = uint_below(a2, n)
            t = uint_below(b2, n - 1)
            t += t >= c
            Q.qsim_apply_ctrl(h, 1 << c, 1 << c, t, NOT)
            gates.append(("cnot", t, c))
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
        for q in range(ne):
            Q.qsim_apply_angles(h, Q.QSIM_GATE_RP, [math.pi / 4, math.pi], 0, 0, q)
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
