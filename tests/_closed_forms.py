"""Closed forms the paper fixes, shared by the oracle pins and the GPU tests.

* fejer_distribution: exact P(y) of the noiseless order-finding register
  (§5.1): with M = 2^m exponent values and r = ord_N(a),
  P(y) = M^-2 sum_{a0<r} F_{c(a0)}(t), t = ((r y) mod M)/M,
  c(a0) = floor((M-1-a0)/r) + 1, F_c(t) = sin^2(pi c t)/sin^2(pi t), F_c(0) = c^2.
  Both sine arguments are reduced exactly in integers first
  (sin^2(pi c T / M) = sin^2(pi ((c T) mod M) / M), T = r y mod M), so the
  closed form keeps full double precision for M = 2^20; angles are folded into
  [0, pi/2] (sin^2 is symmetric about pi/2) so that sines near pi keep their
  relative accuracy.
"""
import numpy as np


def fejer_distribution(M, r):
    y = np.arange(M, dtype=np.int64)
    T = (r * y) % M
    den = np.sin(np.pi * np.minimum(T, M - T) / M) ** 2
    P = np.zeros(M)
    for a0 in range(r):
        c = (M - 1 - a0) // r + 1
        X = (c * T) % M
        X = np.minimum(X, M - X)          # sin^2(pi x) = sin^2(pi (1 - x)): keep the angle <= pi/2
        with np.errstate(invalid="ignore", divide="ignore"):
            F = np.sin(np.pi * X / M) ** 2 / den
        F[T == 0] = c * c
        P += F
    return P / M**2


def order(a, N):
    r, x = 1, a % N
    while x != 1:
        x = (x * a) % N
        r += 1
    return r


def fejer_branch(M, r, c, y):
    """P(y) after the QFT of the uniform superposition over a0, a0+r, ...,
    a0+(c-1)r (one branch of the sum above, PAPER.md:896-903 semantic mode):
    |sum_j e^{2 pi i (a0 + j r) y / M}|^2 / (c M) = F_c(T/M) / (c M),
    T = r y mod M, with the same exact integer reduction.  y: int array."""
    y = np.asarray(y, dtype=object)
    T = np.array([(r * int(v)) % M for v in y.ravel()], dtype=np.int64)
    X = np.array([(c * int(t)) % M for t in T], dtype=np.int64)
    X = np.minimum(X, M - X)
    Tf = np.minimum(T, M - T)
    with np.errstate(invalid="ignore", divide="ignore"):
        F = np.sin(np.pi * X / M) ** 2 / np.sin(np.pi * Tf / M) ** 2
    F[T == 0] = c * c
    return (F / (c * M)).reshape(np.shape(y))
