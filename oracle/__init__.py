"""CPU oracle for the state-vector gate engine — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_quant_ph_0201042_b200``) never imports it and shares no
code with it; see the header of ``oracle.c`` and DESIGN.md §4.

This module is ctypes marshalling around ``liboracle.so`` (built from
``oracle.c`` by ``make -C oracle``, also by ``__graft_entry__.build()``), plus
numpy conveniences.  All arithmetic lives in ``oracle.c``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

TAG_GATE, TAG_HAAR, TAG_PAIR, TAG_OPNOISE, TAG_MARK = 1, 2, 3, 4, 5
TAG_BASE, TAG_GAUSS, TAG_PAULI, TAG_MEASURE, TAG_SHOR = 6, 7, 8, 9, 10
RP, P1, HAAR = 0, 1, 2


def build() -> None:
    """Compile liboracle.so in place (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load() -> C.CDLL:
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(
        os.path.join(_HERE, "oracle.c")
    ):
        build()
    return C.CDLL(_LIB)


_lib = _load()

_u64, _u32, _i32, _f64 = C.c_uint64, C.c_uint32, C.c_int, C.c_double
_p = C.c_void_p


class _Noise(C.Structure):
    _fields_ = [("seed", _u64), ("sigma", _f64), ("g", _u64)]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("orc_philox4x32_10", None, _p, _p, _p)
_sig("orc_draw", None, _u64, _u32, _u64, _u32, _p)
_sig("orc_u01", _f64, _u64)
_sig("orc_u01o", _f64, _u64)
_sig("orc_uint", _u64, _u64, _u64)
_sig("orc_normal", _f64, _u64, _u32, _u64, _u32)
_sig("orc_mat_ur", None, _f64, _p)
_sig("orc_mat_up1", None, _f64, _p)
_sig("orc_mat_up2", None, _f64, _p)
_sig("orc_mat_angles", None, _i32, _p, _p)
_sig("orc_mat_angles_noisy", None, _i32, _p, _u64, _f64, _u64, _p)
_sig("orc_haar_angles", None, _u64, _u64, _p)
_sig("orc_apply_1q", None, _p, _i32, _i32, _p)
_sig("orc_apply_ctrl", None, _p, _i32, _u64, _u64, _i32, _p)
_sig("orc_swap", None, _p, _i32, _i32, _i32)
_sig("orc_phase_flip", None, _p, _i32, _u64)
_sig("orc_pauli", None, _i32, _p)
_sig("orc_norm", _f64, _p, _i32)
_sig("orc_probs", None, _p, _i32, _i32, _i32, _p)
_sig("orc_measure", _u64, _p, _i32, _f64)
_sig("orc_modmul", None, _p, _i32, _i32, _i32, _u64, _u64, _u64, _u64)
_sig("orc_powmod", _u64, _u64, _u64, _u64)
_sig("orc_gcd", _u64, _u64, _u64)
_sig("orc_apply_angles", None, _p, _i32, C.POINTER(_Noise), _i32, _p, _u64, _u64, _i32)
_sig("orc_qft", None, _p, _i32, _i32, _i32, _i32, C.POINTER(_Noise))
_sig("orc_set_threads", None, _i32)
_sig("orc_get_threads", _i32)
_sig("orc_hadamard_range", None, _p, _i32, _i32, _i32)
_sig("orc_aqft", None, _p, _i32, _i32, _i32, _i32, _i32, C.POINTER(_Noise))
_sig("orc_measure_range", _u64, _p, _i32, _i32, _i32, _f64, _i32)
_sig("orc_inner", None, _p, _p, _i32, _p)
_sig("orc_dft_samples", None, _p, _i32, _i32, _p, _i32, _p)
_sig("orc_cfg0", None, _p, _i32, _u64, _i32, _p, _p)
_sig("orc_grover_mark", _u64, _u64, _i32)
_sig("orc_grover_iteration", None, _p, _i32, _u64)
_sig("orc_cfg1", None, _p, _i32, _u64, _i32, _p)
_sig("orc_gaussian_state", None, _p, _i32, _u64)
_sig("orc_cfg2", None, _p, _i32, _u64)
_sig("orc_shor_base", _u64, _u64, _u64)
_sig("orc_cfg3", None, _p, _i32, _i32, _u64, _u64, _u64, _f64, _p)
_sig("orc_cfg4", _i32, _p, _i32, _i32, _u64, _f64, _f64, _p, _i32)
_sig("orc_inject_paulis", None, _p, _i32, _u64, _u64, _u64, _f64, _p, _i32, _p)
_sig("orc_shor_prob_succ", _f64, _u64, _u64)
_sig("orc_traj_ht", None, _p, _i32, _i32, _u64, _f64, _f64)
_sig("orc_traj_grover", None, _p, _i32, _u64, _i32, _u64, _f64, _f64, _p)
_sig("orc_qft_decoherent", None, _p, _i32, _i32, _i32, _i32, C.POINTER(_Noise), _f64)
_sig("orc_shor_semantic_state", None, _p, _i32, _u64, _u64, _u64)
_sig("orc_shor_candidates", _i32, _u64, _i32, _u64, _p, _i32)
_sig("orc_shor_try", _u64, _u64, _u64, _u64, _i32)
_sig("orc_shor_run", _i32, _u64, _i32, _u64, _u64, _i32, _i32, C.POINTER(_u64), _p)


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _state(psi: np.ndarray) -> int:
    assert psi.dtype == np.complex128 and psi.flags["C_CONTIGUOUS"]
    return psi.ctypes.data


def _nq(psi: np.ndarray) -> int:
    n = int(psi.size).bit_length() - 1
    assert psi.size == 1 << n
    return n


def _mat(U) -> np.ndarray:
    U = np.ascontiguousarray(np.asarray(U, dtype=np.complex128).reshape(4))
    return U


# ---------------------------------------------------------------- RNG
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _lib.orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return [int(x) for x in out]


def draw(seed: int, tag: int, i: int, j: int):
    out = np.zeros(2, dtype=np.uint64)
    _lib.orc_draw(seed, tag, i, j, _ptr(out))
    return int(out[0]), int(out[1])


def u01(a: int) -> float:
    return _lib.orc_u01(a)


def u01o(a: int) -> float:
    return _lib.orc_u01o(a)


def uint(a: int, m: int) -> int:
    return _lib.orc_uint(a, m)


def normal(seed: int, tag: int, i: int, j: int) -> float:
    return _lib.orc_normal(seed, tag, i, j)


# ---------------------------------------------------------------- matrices
def mat_ur(theta):
    U = np.zeros(4, np.complex128); _lib.orc_mat_ur(theta, _ptr(U)); return U.reshape(2, 2)


def mat_up1(phi):
    U = np.zeros(4, np.complex128); _lib.orc_mat_up1(phi, _ptr(U)); return U.reshape(2, 2)


def mat_up2(phi):
    U = np.zeros(4, np.complex128); _lib.orc_mat_up2(phi, _ptr(U)); return U.reshape(2, 2)


def mat_angles(kind: int, ang, seed: int = 0, sigma: float = 0.0, g: int = 0):
    a = np.zeros(4, np.float64)
    a[: len(ang)] = ang
    U = np.zeros(4, np.complex128)
    _lib.orc_mat_angles_noisy(kind, _ptr(a), seed, sigma, g, _ptr(U))
    return U.reshape(2, 2)


def haar_angles(seed: int, i: int):
    a = np.zeros(4, np.float64)
    _lib.orc_haar_angles(seed, i, _ptr(a))
    return a


def pauli(which: int):
    U = np.zeros(4, np.complex128); _lib.orc_pauli(which, _ptr(U)); return U.reshape(2, 2)


# ---------------------------------------------------------------- kernels
def apply_1q(psi, q, U):
    U = _mat(U); _lib.orc_apply_1q(_state(psi), _nq(psi), q, _ptr(U))


def apply_ctrl(psi, ctrl_mask, ctrl_vals, q, U):
    U = _mat(U); _lib.orc_apply_ctrl(_state(psi), _nq(psi), ctrl_mask, ctrl_vals, q, _ptr(U))


def swap(psi, q1, q2):
    _lib.orc_swap(_state(psi), _nq(psi), q1, q2)


def phase_flip(psi, idx):
    _lib.orc_phase_flip(_state(psi), _nq(psi), idx)


def norm(psi) -> float:
    return _lib.orc_norm(_state(psi), _nq(psi))


def probs(psi, lo, m):
    out = np.zeros(1 << m, np.float64)
    _lib.orc_probs(_state(psi), _nq(psi), lo, m, _ptr(out))
    return out


def measure(psi, r: float) -> int:
    return _lib.orc_measure(_state(psi), _nq(psi), r)


def modmul(psi, wlo, wm, ctrl_mask, ctrl_vals, c, N):
    _lib.orc_modmul(_state(psi), _nq(psi), wlo, wm, ctrl_mask, ctrl_vals, c, N)


def powmod(a, e, N) -> int:
    return _lib.orc_powmod(a, e, N)


def gcd(a, b) -> int:
    return _lib.orc_gcd(a, b)


class Noise:
    """Angle-noise context: (OPNOISE seed, sigma, gate counter g)."""

    def __init__(self, seed: int = 0, sigma: float = 0.0, g: int = 0):
        self._c = _Noise(seed, sigma, g)

    @property
    def g(self) -> int:
        return self._c.g


def apply_angles(psi, noise: Noise, kind, ang, ctrl_mask, ctrl_vals, q):
    a = np.zeros(4, np.float64); a[: len(ang)] = ang
    _lib.orc_apply_angles(_state(psi), _nq(psi), C.byref(noise._c), kind, _ptr(a),
                          ctrl_mask, ctrl_vals, q)


def set_threads(k: int) -> None:
    """OpenMP threads of the oracle's loops (0: default); results do not depend on it."""
    _lib.orc_set_threads(int(k))


def get_threads() -> int:
    return int(_lib.orc_get_threads())


def qft(psi, lo, m, inverse=False, noise: Noise | None = None):
    noise = noise or Noise()
    _lib.orc_qft(_state(psi), _nq(psi), lo, m, int(bool(inverse)), C.byref(noise._c))


def aqft(psi, lo, m, b, inverse=False, noise: Noise | None = None):
    """Approximate QFT: R_d with d > b omitted (R30)."""
    noise = noise or Noise()
    _lib.orc_aqft(_state(psi), _nq(psi), lo, m, b, int(bool(inverse)), C.byref(noise._c))


def measure_range(psi, lo, m, r: float, collapse=True) -> int:
    """Measure qubits [lo, lo+m) with random number r (R31); collapses psi."""
    return _lib.orc_measure_range(_state(psi), _nq(psi), lo, m, r, int(bool(collapse)))


def inner(a, b) -> complex:
    """<a|b> (pairwise sum); the paper's fidelity is abs(inner) (R32)."""
    assert a.shape == b.shape
    out = np.zeros(1, np.complex128)
    _lib.orc_inner(_state(a), _state(b), _nq(a), _ptr(out))
    return complex(out[0])


def hadamard_range(psi, lo, m):
    _lib.orc_hadamard_range(_state(psi), _nq(psi), lo, m)


def dft_samples(psi, xs, inverse=False):
    xs = np.ascontiguousarray(np.asarray(xs, dtype=np.uint64))
    out = np.zeros(len(xs), np.complex128)
    _lib.orc_dft_samples(_state(psi), _nq(psi), int(bool(inverse)), _ptr(xs), len(xs), _ptr(out))
    return out


def inject_paulis(psi, seed, epoch, qmask, p, cap=1024):
    """Depolarizing injection; returns the event list [(epoch, q, pauli)]."""
    ev = np.zeros(3 * cap, np.int32)
    nev = C.c_int(0)
    _lib.orc_inject_paulis(_state(psi), _nq(psi), seed, epoch, qmask, p, _ptr(ev), cap,
                           C.byref(nev))
    return [tuple(int(x) for x in ev[3 * i: 3 * i + 3]) for i in range(min(nev.value, cap))]


# ---------------------------------------------------------------- configs
def cfg0(n=10, seed=1, ngates=200):
    psi = np.zeros(1 << n, np.complex128)
    kinds = np.zeros(ngates, np.int32)
    qs = np.zeros(2 * ngates, np.int32)
    _lib.orc_cfg0(_state(psi), n, seed, ngates, _ptr(kinds), _ptr(qs))
    return psi, kinds, qs.reshape(ngates, 2)


def grover_mark(seed, n) -> int:
    return _lib.orc_grover_mark(seed, n)


def grover_iteration(psi, k):
    _lib.orc_grover_iteration(_state(psi), _nq(psi), k)


def cfg1(n=20, seed=2, iters=804):
    psi = np.zeros(1 << n, np.complex128)
    trace = np.zeros(iters, np.float64)
    _lib.orc_cfg1(_state(psi), n, seed, iters, _ptr(trace))
    return psi, trace


def gaussian_state(n, seed=3):
    psi = np.zeros(1 << n, np.complex128)
    _lib.orc_gaussian_state(_state(psi), n, seed)
    return psi


def cfg2(n=28, seed=3):
    psi = np.zeros(1 << n, np.complex128)
    _lib.orc_cfg2(_state(psi), n, seed)
    return psi


def shor_base(seed, N) -> int:
    return _lib.orc_shor_base(seed, N)


def cfg3(ne=20, nw=10, N=1007, seed=4, sigma=0.0, a=None, want_state=False):
    a = shor_base(seed, N) if a is None else a
    psi = np.zeros(1 << (ne + nw), np.complex128)
    pr = np.zeros(1 << ne, np.float64)
    _lib.orc_cfg3(_state(psi), ne, nw, N, a, seed, sigma, _ptr(pr))
    return (pr, psi) if want_state else pr


def cfg4(n=32, layers=20, seed=5, sigma=1e-3, p=1e-4, cap=4096):
    psi = np.zeros(1 << n, np.complex128)
    ev = np.zeros(3 * cap, np.int32)
    nev = _lib.orc_cfg4(_state(psi), n, layers, seed, sigma, p, _ptr(ev), cap)
    return psi, [tuple(int(x) for x in ev[3 * i: 3 * i + 3]) for i in range(min(nev, cap))]


# ---------------------------------------------------------------- Shor (row f3)
def shor_prob_succ(n, phi) -> float:
    """Prob_succ(n) of PAPER.md:907-920 (natural logarithms)."""
    return _lib.orc_shor_prob_succ(n, phi)


def shor_semantic_state(m, x, N, v):
    """Uniform superposition over {a < 2^m : x^a = v mod N}."""
    psi = np.zeros(1 << m, np.complex128)
    _lib.orc_shor_semantic_state(_state(psi), m, x, N, v)
    return psi


def shor_candidates(y, m, N):
    """Convergent denominators r < N of y/2^m within 1/2^(m+1)."""
    out = np.zeros(64, np.uint64)
    k = _lib.orc_shor_candidates(y, m, N, _ptr(out), 64)
    return [int(v) for v in out[:k]]


def shor_try(N, x, r, gcd_check=False) -> int:
    """Steps 4-5 for one candidate r (GCD check 979-981)."""
    return _lib.orc_shor_try(N, x, r, int(bool(gcd_check)))


SHOR_STATS = ("step2", "quantum", "basic_s", "basic_f", "neighbor_s", "neighbor_f", "gcd_s", "gcd_f",
              "sf_s", "sf_f", "lcm_s", "lcm_f")


def shor_run(N, m, seed, run, improved=False, max_iter=200, stats=None):
    """One factoring run; returns (iterations, factor).  stats: optional
    int64 array of len(SHOR_STATS), accumulated (Table 6 tallies)."""
    f = C.c_uint64(0)
    st = stats if stats is not None else np.zeros(len(SHOR_STATS), np.int64)
    assert st.dtype == np.int64 and st.size == len(SHOR_STATS)
    t = _lib.orc_shor_run(N, m, seed, run, int(bool(improved)), max_iter, C.byref(f), _ptr(st))
    return t, f.value


# ------------------------------------------------------------------ row f2: noise-experiment trajectories
def traj_ht(n, k, seed, sigma, p):
    """One HT-experiment trajectory (R33/R34): final state."""
    psi = np.zeros(1 << n, np.complex128)
    _lib.orc_traj_ht(_ptr(psi), n, k, seed, sigma, p)
    return psi


def traj_grover(n, k, iters, seed, sigma, p):
    """One Grover-experiment trajectory (R35): final
    (n+1)-qubit state (ancilla = LSB) and trace[t] = P(register = k)."""
    psi = np.zeros(1 << (n + 1), np.complex128)
    trace = np.zeros(max(iters, 1), np.float64)
    _lib.orc_traj_grover(_ptr(psi), n, k, iters, seed, sigma, p, _ptr(trace))
    return psi, trace[:iters]


def qft_decoherent(psi, lo, m, inverse=False, noise: Noise | None = None, p=0.0):
    """QFT circuit with angle noise and the depolarizing channel after every
    R_d (R36), in place."""
    noise = noise or Noise()
    _lib.orc_qft_decoherent(_state(psi), _nq(psi), lo, m, int(bool(inverse)), C.byref(noise._c), p)
