"""Closed forms the paper fixes, shared by the oracle pins and the GPU tests.

* fejer_distribution: exact P(y) of the noiseless order-finding register
  (§5.1): with M = 2^m exponent values and r = ord_N(a),
  P(y) = M^-2 sum_{a0<r} F_{c(a0)}(t), t = ((r y) mod M)/M,
  c(a0) = floor((M-1-a0)/r) + 1, F_c(t) = sin^2(pi c t)/sin^2(pi t), F_c(0) = c^2.
"""
import numpy as np


def fejer_distribution(M, r):
    y = np.arange(M, dtype=np.int64)
    t = ((r * y) % M) / M
    P = np.zeros(M)
    for a0 in range(r):
        c = (M - 1 - a0) // r + 1
        with np.errstate(invalid="ignore", divide="ignore"):
            F = np.sin(np.pi * c * t) ** 2 / np.sin(np.pi * t) ** 2
        F[t == 0] = c * c
        P += F
    return P / M**2


def order(a, N):
    r, x = 1, a % N
    while x != 1:
        x = (x * a) % N
        r += 1
    return r
