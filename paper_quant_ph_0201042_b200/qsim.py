"""ctypes binding of libqsim.so (include/qsim.h) -- argument marshalling only.

Every function here has the name of the C entry point it wraps and does
nothing but convert arguments and raise ``QsimError`` on a negative status.
All computation happens in the sm_100a kernels of ``libqsim.so``; there is no
CPU fallback: importing this module raises if the library cannot be loaded,
and ``qsim_create`` fails with QSIM_ENODEV when no B200 (sm_100) is present.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QSIM_LIB: another in-tree build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("QSIM_LIB") or os.path.join(_HERE, "libqsim.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` "
        "(or __graft_entry__.build()); the gate engine has no CPU fallback"
    )

lib = C.CDLL(LIB_PATH)

QSIM_OK, QSIM_EINVAL, QSIM_ERANGE, QSIM_ENOMEM = 0, -1, -2, -3
QSIM_ECUDA, QSIM_ENOTBIJ, QSIM_ESTATE, QSIM_ENCCL, QSIM_ENODEV = -4, -5, -6, -7, -8
QSIM_ENONUNITARY = -9
QSIM_GATE_RP, QSIM_GATE_P1, QSIM_GATE_HAAR = 0, 1, 2
QSIM_PERM_TABLE, QSIM_PERM_MODMUL, QSIM_PERM_MODEXP = 0, 1, 2
QSIM_TAG_GATE, QSIM_TAG_HAAR, QSIM_TAG_PAIR, QSIM_TAG_OPNOISE = 1, 2, 3, 4
QSIM_TAG_MARK, QSIM_TAG_BASE, QSIM_TAG_GAUSS, QSIM_TAG_PAULI, QSIM_TAG_MEASURE, QSIM_TAG_SHOR = 5, 6, 7, 8, 9, 10

_ERRNAMES = {
    -1: "QSIM_EINVAL", -2: "QSIM_ERANGE", -3: "QSIM_ENOMEM", -4: "QSIM_ECUDA",
    -5: "QSIM_ENOTBIJ", -6: "QSIM_ESTATE", -7: "QSIM_ENCCL", -8: "QSIM_ENODEV", -9: "QSIM_ENONUNITARY",
}


class QsimError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class qsim_c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class qsim_perm_t(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("lo", C.c_int), ("m", C.c_int), ("elo", C.c_int), ("em", C.c_int),
        ("ctrl_mask", C.c_uint64), ("ctrl_vals", C.c_uint64),
        ("mult", C.c_uint64), ("base", C.c_uint64), ("modulus", C.c_uint64),
        ("table", C.POINTER(C.c_uint32)),
    ]


class qsim_noise_t(C.Structure):
    _fields_ = [("p", C.c_double), ("qubit_mask", C.c_uint64), ("epoch", C.c_uint64)]


class qsim_event_t(C.Structure):
    _fields_ = [("epoch", C.c_uint64), ("qubit", C.c_int32), ("pauli", C.c_int32), ("traj", C.c_uint64)]


_H = C.c_void_p
_u64, _u32, _i32, _f64, _p = C.c_uint64, C.c_uint32, C.c_int, C.c_double, C.c_void_p


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


_sig("qsim_create", _i32, _i32, _i32, C.POINTER(_H))
_sig("qsim_create_dist", _i32, _i32, _i32, _i32, _i32, _p, C.POINTER(_H))
_sig("qsim_nccl_unique_id", _i32, _p)
_sig("qsim_create_group", _i32, _i32, _i32, _p, C.POINTER(_H))
_sig("qsim_destroy", None, _H)
_sig("qsim_last_error", C.c_char_p, _H)
_sig("qsim_memory_bytes", _u64, _i32)
_sig("qsim_launch_count", _u64, _H)
_sig("qsim_sync", _i32, _H)
_sig("qsim_set_basis", _i32, _H, _u64)
_sig("qsim_init_gaussian", _i32, _H, _u64)
_sig("qsim_set_state", _i32, _H, _u64, _u64, _p)
_sig("qsim_get_state", _i32, _H, _u64, _u64, _p)
_sig("qsim_apply_1q", _i32, _H, _i32, _p)
_sig("qsim_apply_ctrl", _i32, _H, _u64, _u64, _i32, _p)
_sig("qsim_apply_angles", _i32, _H, _i32, _p, _u64, _u64, _i32)
_sig("qsim_set_gate_noise", _i32, _H, _u64, _f64)
_sig("qsim_get_gate_counter", _i32, _H, C.POINTER(_u64))
_sig("qsim_set_gate_counter", _i32, _H, _u64)
_sig("qsim_swap", _i32, _H, _i32, _i32)
_sig("qsim_hadamard", _i32, _H, _i32, _i32)
_sig("qsim_qft", _i32, _H, _i32, _i32, _i32)
_sig("qsim_fft", _i32, _H, _i32, _i32, _i32)
_sig("qsim_philox_draws", None, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(C.c_uint64))
_sig("qsim_aqft", _i32, _H, _i32, _i32, _i32, _i32)
_sig("qsim_hadamard_angles", _i32, _H, _i32, _i32)
_sig("qsim_measure_range", _i32, _H, _i32, _i32, _f64, _i32, C.POINTER(_u64))
_sig("qsim_inner", _i32, _H, _H, _p)
_sig("qsim_set_batch", _i32, _H, _i32)
_sig("qsim_batch_set_state", _i32, _H, _p)
_sig("qsim_batch_overlap", _i32, _H, _p, _p)
_sig("qsim_phase_flip", _i32, _H, _u64)
_sig("qsim_grover", _i32, _H, _u64, _i32, _p)
_sig("qsim_diffusion", _i32, _H, _i32, _i32)
_sig("qsim_qft_host_stream", _i32, _H, _i32, _i32, _i32, _p, _u64, _p, _u64, _i32)
_sig("qsim_set_strict", _i32, _H, _i32)
_sig("qsim_apply_perm", _i32, _H, C.POINTER(qsim_perm_t))
_sig("qsim_inject_errors", _i32, _H, _u64, C.POINTER(qsim_noise_t), _p, _i32, C.POINTER(_i32))
_sig("qsim_norm", _i32, _H, C.POINTER(_f64))
_sig("qsim_probs", _i32, _H, _i32, _i32, _p)
_sig("qsim_prob_index", _i32, _H, _u64, C.POINTER(_f64))
_sig("qsim_measure", _i32, _H, _f64, C.POINTER(_u64))
_sig("qsim_philox_draw", None, _u64, _u32, _u64, _u32, _p)
_sig("qsim_shor_semantic_state", _i32, _H, _u64, _u64, _u64)
_sig("qsim_shor_run", _i32, _H, _u64, _u64, _u64, _i32, _i32, C.POINTER(_u64), C.POINTER(_i32), _p)
_sig("qsim_shor_candidates", _i32, _u64, _i32, _u64, _p, _i32)
_sig("qsim_shor_try", _u64, _u64, _u64, _u64, _i32)
_sig("qsim_shor_prob_succ", _f64, _u64, _u64)
_sig("qsim_get_stream", _p, _H)
_sig("qsim_set_fusion", _i32, _H, _i32)
_sig("qsim_profile", _i32, _H, _i32)
_sig("qsim_profile_json", C.c_char_p, _H)
_sig("qsim_plan_make_local", _i32, _i32, _i32, _p, _p, _i32, _p, _i32)
_sig("qsim_plan_canonical_globals", _i32, _i32, _i32, _p, _p, _i32)


def _chk(h, rc: int) -> None:
    if rc != QSIM_OK:
        msg = lib.qsim_last_error(h)
        raise QsimError(rc, msg.decode() if msg else "")


def _mat(U) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(U, dtype=np.complex128).reshape(4))


# ------------------------------------------------------------------ lifecycle
def qsim_create(n: int, ngpus: int = 1):
    h = _H()
    _chk(None, lib.qsim_create(n, ngpus, C.byref(h)))
    return h


def qsim_create_dist(n: int, world: int, rank: int, device: int, nccl_id: bytes):
    h = _H()
    buf = C.create_string_buffer(bytes(nccl_id), 128)
    _chk(None, lib.qsim_create_dist(n, world, rank, device, buf, C.byref(h)))
    return h


def qsim_create_group(n: int, world: int, devices=None):
    h = _H()
    dev = None
    if devices is not None:
        dev = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    _chk(None, lib.qsim_create_group(n, world, dev.ctypes.data if dev is not None else None, C.byref(h)))
    return h


def qsim_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(None, lib.qsim_nccl_unique_id(buf))
    return buf.raw


def qsim_destroy(h) -> None:
    lib.qsim_destroy(h)


def qsim_last_error(h) -> str:
    m = lib.qsim_last_error(h)
    return m.decode() if m else ""


def qsim_memory_bytes(n: int) -> int:
    return lib.qsim_memory_bytes(n)


def qsim_launch_count(h) -> int:
    return lib.qsim_launch_count(h)


def qsim_sync(h) -> None:
    _chk(h, lib.qsim_sync(h))


def qsim_get_stream(h) -> int:
    return lib.qsim_get_stream(h) or 0


def qsim_set_fusion(h, enable: bool) -> None:
    _chk(h, lib.qsim_set_fusion(h, int(bool(enable))))


def qsim_profile(h, enable: bool) -> None:
    _chk(h, lib.qsim_profile(h, int(bool(enable))))


def qsim_profile_json(h) -> dict:
    import json
    return json.loads(lib.qsim_profile_json(h).decode())


# ------------------------------------------------------------------ preparation
def qsim_set_basis(h, idx: int) -> None:
    _chk(h, lib.qsim_set_basis(h, idx))


def qsim_init_gaussian(h, seed: int) -> None:
    _chk(h, lib.qsim_init_gaussian(h, seed))


def qsim_set_state(h, off: int, amps: np.ndarray) -> None:
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    _chk(h, lib.qsim_set_state(h, off, a.size, a.ctypes.data))


def qsim_get_state(h, off: int, cnt: int, out: np.ndarray | None = None) -> np.ndarray:
    if out is None:
        out = np.empty(cnt, np.complex128)
    assert out.dtype == np.complex128 and out.flags["C_CONTIGUOUS"] and out.size >= cnt
    _chk(h, lib.qsim_get_state(h, off, cnt, out.ctypes.data))
    return out


# ------------------------------------------------------------------ gates
def qsim_apply_1q(h, q: int, U) -> None:
    m = _mat(U)
    _chk(h, lib.qsim_apply_1q(h, q, m.ctypes.data))


def qsim_apply_ctrl(h, ctrl_mask: int, ctrl_vals: int, q: int, U) -> None:
    m = _mat(U)
    _chk(h, lib.qsim_apply_ctrl(h, ctrl_mask, ctrl_vals, q, m.ctypes.data))


def qsim_apply_angles(h, kind: int, ang, ctrl_mask: int, ctrl_vals: int, q: int) -> None:
    a = np.zeros(4, np.float64)
    a[: len(ang)] = ang
    _chk(h, lib.qsim_apply_angles(h, kind, a.ctypes.data, ctrl_mask, ctrl_vals, q))


def qsim_set_gate_noise(h, seed: int, sigma: float) -> None:
    _chk(h, lib.qsim_set_gate_noise(h, seed, sigma))


def qsim_get_gate_counter(h) -> int:
    g = _u64()
    _chk(h, lib.qsim_get_gate_counter(h, C.byref(g)))
    return g.value


def qsim_set_gate_counter(h, g: int) -> None:
    _chk(h, lib.qsim_set_gate_counter(h, g))


def qsim_swap(h, q1: int, q2: int) -> None:
    _chk(h, lib.qsim_swap(h, q1, q2))


def qsim_hadamard(h, lo: int, m: int) -> None:
    _chk(h, lib.qsim_hadamard(h, lo, m))


def qsim_qft(h, lo: int, m: int, inverse: bool = False) -> None:
    _chk(h, lib.qsim_qft(h, lo, m, int(bool(inverse))))


def qsim_fft(h, lo: int, m: int, inverse: bool = False) -> None:
    _chk(h, lib.qsim_fft(h, lo, m, int(bool(inverse))))


def qsim_hadamard_angles(h, lo: int, m: int) -> None:
    """H = U_R(pi/4) U_P1(pi) on every qubit of [lo, lo+m), counted and noisy
    like qsim_apply_angles (fused passes where possible)."""
    _chk(h, lib.qsim_hadamard_angles(h, lo, m))


QSIM_GT_MATRIX, QSIM_GT_ANGLES = 0, 1


class qsim_gate_t(C.Structure):
    _fields_ = [("type", C.c_int32), ("q", C.c_int32), ("akind", C.c_int32), ("pad_", C.c_int32),
                ("ctrl_mask", C.c_uint64), ("ctrl_vals", C.c_uint64), ("ang", C.c_double * 4),
                ("U", C.c_double * 8)]


lib.qsim_apply_gates.restype = C.c_int32
lib.qsim_apply_gates.argtypes = [_H, C.POINTER(qsim_gate_t), C.c_int32, C.POINTER(C.c_int32)]


def qsim_philox_draws(seed: int, tag: int, i0: int, count: int, j: int = 0) -> np.ndarray:
    """(count, 2) uint64 array of consecutive draws (i = i0 .. i0+count-1)."""
    out = np.zeros((count, 2), np.uint64)
    lib.qsim_philox_draws(seed, tag, i0, count, j, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def qsim_apply_gates(h, gates) -> None:
    """gates: sequence of ("matrix", q, U, ctrl_mask, ctrl_vals) or
    ("angles", q, akind, ang, ctrl_mask, ctrl_vals); one C-ABI call."""
    arr = (qsim_gate_t * max(len(gates), 1))()
    for i, g in enumerate(gates):
        x = arr[i]
        if g[0] == "matrix":
            _, q, U, cm, cv = g
            u = np.asarray(U, dtype=np.complex128).reshape(4)
            x.type, x.q, x.ctrl_mask, x.ctrl_vals = QSIM_GT_MATRIX, q, cm, cv
            for k in range(4):
                x.U[2 * k], x.U[2 * k + 1] = u[k].real, u[k].imag
        else:
            _, q, akind, ang, cm, cv = g
            x.type, x.q, x.akind, x.ctrl_mask, x.ctrl_vals = QSIM_GT_ANGLES, q, akind, cm, cv
            for k, a in enumerate(ang):
                x.ang[k] = a
    done = C.c_int32(0)
    _chk(h, lib.qsim_apply_gates(h, arr, len(gates), C.byref(done)))


def qsim_aqft(h, lo: int, m: int, b: int, inverse: bool = False) -> None:
    _chk(h, lib.qsim_aqft(h, lo, m, b, int(bool(inverse))))


def qsim_phase_flip(h, idx: int) -> None:
    _chk(h, lib.qsim_phase_flip(h, idx))


def qsim_grover(h, mark: int, iters: int, trace: bool = True):
    out = np.zeros(max(iters, 1), np.float64) if trace else None
    _chk(h, lib.qsim_grover(h, mark, iters, out.ctypes.data if trace else None))
    return out[:iters] if trace else None


def qsim_qft_host_stream(h, lo: int, m: int, inverse: bool, inp: np.ndarray, out: np.ndarray, count: int,
                         in_stride: int, out_stride: int) -> None:
    """inp / out: complex128 host arrays (pinned for overlap) holding the states at the given strides."""
    assert inp.dtype == np.complex128 and out.dtype == np.complex128
    assert inp.flags.c_contiguous and out.flags.c_contiguous
    _chk(h, lib.qsim_qft_host_stream(h, lo, m, int(bool(inverse)), inp.ctypes.data, in_stride, out.ctypes.data,
                                     out_stride, count))


def qsim_diffusion(h, lo: int, m: int) -> None:
    _chk(h, lib.qsim_diffusion(h, lo, m))


def qsim_set_strict(h, enable: bool) -> None:
    _chk(h, lib.qsim_set_strict(h, int(bool(enable))))


def qsim_apply_perm(h, kind: int, lo: int, m: int, *, elo: int = 0, em: int = 0, ctrl_mask: int = 0,
                    ctrl_vals: int = 0, mult: int = 0, base: int = 0, modulus: int = 0,
                    table=None) -> None:
    f = qsim_perm_t(kind, lo, m, elo, em, ctrl_mask, ctrl_vals, mult, base, modulus, None)
    keep = None
    if table is not None:
        keep = np.ascontiguousarray(np.asarray(table, dtype=np.uint32))
        f.table = keep.ctypes.data_as(C.POINTER(C.c_uint32))
    _chk(h, lib.qsim_apply_perm(h, C.byref(f)))
    del keep


def qsim_inject_errors(h, seed: int, p: float, qubit_mask: int, epoch: int, cap: int = 256, traj: bool = False):
    """Events as (epoch, qubit, pauli) tuples, or (epoch, qubit, pauli, traj)
    with traj=True (batched handles)."""
    model = qsim_noise_t(p, qubit_mask, epoch)
    ev = (qsim_event_t * max(cap, 1))()
    nev = _i32(0)
    _chk(h, lib.qsim_inject_errors(h, seed, C.byref(model), ev, cap, C.byref(nev)))
    if traj:
        return [(int(ev[i].epoch), int(ev[i].qubit), int(ev[i].pauli), int(ev[i].traj)) for i in range(nev.value)]
    return [(int(ev[i].epoch), int(ev[i].qubit), int(ev[i].pauli)) for i in range(nev.value)]


# ------------------------------------------------------------------ batched trajectories
def qsim_set_batch(h, b: int) -> None:
    _chk(h, lib.qsim_set_batch(h, b))


def qsim_batch_set_state(h, reg) -> None:
    reg = np.ascontiguousarray(np.asarray(reg, dtype=np.complex128))
    _chk(h, lib.qsim_batch_set_state(h, reg.ctypes.data))


def qsim_batch_overlap(h, ref, ntraj: int) -> np.ndarray:
    ref = np.ascontiguousarray(np.asarray(ref, dtype=np.complex128))
    out = np.zeros(ntraj, np.complex128)
    _chk(h, lib.qsim_batch_overlap(h, ref.ctypes.data, out.ctypes.data))
    return out


# ------------------------------------------------------------------ read-out
def qsim_norm(h) -> float:
    v = _f64()
    _chk(h, lib.qsim_norm(h, C.byref(v)))
    return v.value


def qsim_probs(h, lo: int, m: int) -> np.ndarray:
    out = np.zeros(1 << m, np.float64)
    _chk(h, lib.qsim_probs(h, lo, m, out.ctypes.data))
    return out


def qsim_prob_index(h, idx: int) -> float:
    v = _f64()
    _chk(h, lib.qsim_prob_index(h, idx, C.byref(v)))
    return v.value


def qsim_measure(h, r: float) -> int:
    v = _u64()
    _chk(h, lib.qsim_measure(h, r, C.byref(v)))
    return v.value


def qsim_measure_range(h, lo: int, m: int, r: float, collapse: bool = True) -> int:
    v = _u64()
    _chk(h, lib.qsim_measure_range(h, lo, m, r, int(bool(collapse)), C.byref(v)))
    return v.value


def qsim_inner(a, b) -> complex:
    out = np.zeros(1, np.complex128)
    _chk(a, lib.qsim_inner(a, b, out.ctypes.data))
    return complex(out[0])


# ------------------------------------------------------------------ RNG + planners
def qsim_shor_semantic_state(h, x: int, N: int, v: int) -> None:
    _chk(h, lib.qsim_shor_semantic_state(h, x, N, v))


SHOR_STATS = ("step2", "quantum", "basic_s", "basic_f", "neighbor_s", "neighbor_f", "gcd_s", "gcd_f",
              "sf_s", "sf_f", "lcm_s", "lcm_f")   # QSIM_SHOR_* order


def qsim_shor_run(h, N: int, seed: int, run: int, improved: bool = False, max_iter: int = 1000, stats=None):
    """One factoring run; returns (iterations, factor), (0, 0) if none.
    stats: optional int64 numpy array of len(SHOR_STATS), accumulated."""
    f, t = _u64(0), _i32(0)
    ptr = None
    if stats is not None:
        assert stats.dtype == np.int64 and stats.size == len(SHOR_STATS) and stats.flags.c_contiguous
        ptr = stats.ctypes.data
    _chk(h, lib.qsim_shor_run(h, N, seed, run, int(bool(improved)), max_iter, C.byref(f), C.byref(t), ptr))
    return t.value, f.value


def qsim_shor_candidates(y: int, m: int, N: int, cap: int = 64):
    out = np.zeros(cap, np.uint64)
    k = lib.qsim_shor_candidates(y, m, N, out.ctypes.data, cap)
    if k < 0:
        raise QsimError(k, "qsim_shor_candidates: invalid argument")
    return [int(v) for v in out[:k]]


def qsim_shor_try(N: int, x: int, r: int, gcd_check: bool = False) -> int:
    return int(lib.qsim_shor_try(N, x, r, int(bool(gcd_check))))


def qsim_shor_prob_succ(N: int, phi: int) -> float:
    return float(lib.qsim_shor_prob_succ(N, phi))


def qsim_philox_draw(seed: int, tag: int, i: int, j: int):
    out = np.zeros(2, np.uint64)
    lib.qsim_philox_draw(seed, tag, i, j, out.ctypes.data)
    return int(out[0]), int(out[1])


def qsim_plan_make_local(n: int, world: int, pos, need):
    pos = np.ascontiguousarray(np.asarray(pos, dtype=np.int32)).copy()
    nd = np.ascontiguousarray(np.asarray(need, dtype=np.int32))
    steps = np.zeros(3 * 256, np.int32)
    k = lib.qsim_plan_make_local(n, world, pos.ctypes.data, nd.ctypes.data, nd.size, steps.ctypes.data, 256)
    _chk(None, min(k, 0))
    return pos, [tuple(int(x) for x in steps[3 * i: 3 * i + 3]) for i in range(k)]


def qsim_plan_canonical_globals(n: int, world: int, pos):
    pos = np.ascontiguousarray(np.asarray(pos, dtype=np.int32)).copy()
    steps = np.zeros(3 * 256, np.int32)
    k = lib.qsim_plan_canonical_globals(n, world, pos.ctypes.data, steps.ctypes.data, 256)
    _chk(None, min(k, 0))
    return pos, [tuple(int(x) for x in steps[3 * i: 3 * i + 3]) for i in range(k)]
