#!/usr/bin/env python3
"""Time every BASELINE.json config through the C-ABI on one GPU.

Prints one JSON line per config: circuit time (CUDA events on the library's
stream, state resident in HBM), per-kernel device time from the library's
own profiler, and the effective per-gate bandwidth of the unfused gate model.
Not the driver's bench (bench.py times configs[2]); this is the evidence
table for DESIGN.md §7.  Usage: python tools/bench_configs.py [cfg ...]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402


def timed(h, fn, reps=1):
    stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
    Q.qsim_profile(h, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    out = None
    for _ in range(reps):
        out = fn()
    Q.qsim_sync(h)   # flush queued (fused) gates inside the timed region
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    prof = Q.qsim_profile_json(h)
    prof.pop("_launches", None)
    Q.qsim_profile(h, False)
    return e0.elapsed_time(e1) / reps, wall * 1e3, prof, out


def report(name, n, ms, wall_ms, prof, gate_bytes=None, extra=None):
    line = {"config": name, "n": n, "device_ms": round(ms, 4), "wall_ms": round(wall_ms, 4),
            "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 4),
                            "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
                        for k, v in prof.items()}}
    if gate_bytes:
        line["effective_GBps_per_gate"] = round(gate_bytes / (ms * 1e-3) / 1e9, 1)
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)


def cfg0():
    h = Q.qsim_create(10)
    W.run_cfg0(h, 10, 1, 200)     # warm-up
    ms, wall, prof, _ = timed(h, lambda: W.run_cfg0(h, 10, 1, 200), reps=3)
    report("configs[0] random circuit n=10, 200 gates", 10, ms, wall, prof)
    Q.qsim_destroy(h)


def cfg1():
    n = 20
    h = Q.qsim_create(n)
    W.run_cfg1(h, n, 2, 10)
    ms, wall, prof, out = timed(h, lambda: W.run_cfg1(h, n, 2))
    k, trace = out
    gb = 804 * (2 * n + 2) * (1 << (n + 5)) / 2   # literal: 2n H sweeps per iteration (+ flips)
    report("configs[1] Grover n=20, 804 iterations", n, ms, wall, prof, gb,
           {"P_final": float(trace[-1]), "per_iteration_us": round(ms * 1e3 / 804, 3)})
    Q.qsim_destroy(h)


def cfg2(n=28):
    h = Q.qsim_create(n)
    Q.qsim_init_gaussian(h, 3)
    Q.qsim_qft(h, 0, n, False)
    ms, wall, prof, _ = timed(h, lambda: Q.qsim_qft(h, 0, n, False), reps=5)
    gb = n * (1 << (n + 5)) + n * (n - 1) // 2 * (1 << (n + 3)) + n // 2 * (1 << (n + 4))
    report(f"configs[2] QFT n={n}", n, ms, wall, prof, gb)
    Q.qsim_destroy(h)


def cfg3(sigma):
    ne, nw = 20, 10
    h = Q.qsim_create(ne + nw)
    W.run_cfg3(h, ne, nw, 1007, 4, sigma)      # warm-up (lazy module loading, workspaces)
    ms, wall, prof, P = timed(h, lambda: W.run_cfg3(h, ne, nw, 1007, 4, sigma))
    n = ne + nw
    gb = (2 * ne) * (1 << (n + 5)) + ne * (ne - 1) // 2 * (1 << (n + 3)) + ne // 2 * (1 << (n + 4)) \
        + (1 << (n + 5))
    report(f"configs[3] Shor N=1007 n=30 sigma={sigma}", n, ms, wall, prof, gb,
           {"P_sum": float(P.sum()), "P_max": float(P.max())})
    Q.qsim_destroy(h)


def cfg4(n=32, layers=20):
    h = Q.qsim_create(n)
    W.run_cfg4(h, n, 2, 5, 1e-3, 1e-4)          # warm-up (lazy module loading)
    ms, wall, prof, ev = timed(h, lambda: W.run_cfg4(h, n, layers, 5, 1e-3, 1e-4))
    gates = layers * (n + (n - 1) // 2)
    report(f"configs[4] noisy brickwork n={n} layers={layers}", n, ms, wall, prof,
           layers * n * (1 << (n + 5)) + layers * ((n - 1) // 2) * (1 << (n + 4)),
           {"events": ev, "gates": gates})
    Q.qsim_destroy(h)


def f1(n=28):
    """Row f1: the paper's Table 1 comparison on B200 -- the QFT circuit gate
    by gate (one HBM sweep per gate, the paper's algorithm), the same circuit
    fused into tile passes, and the FFT entry point."""
    h = Q.qsim_create(n)
    Q.qsim_init_gaussian(h, 3)
    gb = n * (1 << (n + 5)) + n * (n - 1) // 2 * (1 << (n + 3)) + n // 2 * (1 << (n + 4))
    Q.qsim_set_fusion(h, False)
    Q.qsim_qft(h, 0, n, False)
    ms, wall, prof, _ = timed(h, lambda: Q.qsim_qft(h, 0, n, False))
    report(f"f1 QFT circuit n={n}, one sweep per gate (fusion off)", n, ms, wall, prof, gb)
    Q.qsim_set_fusion(h, True)
    Q.qsim_qft(h, 0, n, False)
    ms, wall, prof, _ = timed(h, lambda: Q.qsim_qft(h, 0, n, False), reps=5)
    report(f"f1 QFT circuit n={n}, fused passes", n, ms, wall, prof, gb)
    Q.qsim_fft(h, 0, n, False)
    ms, wall, prof, _ = timed(h, lambda: Q.qsim_fft(h, 0, n, False), reps=5)
    report(f"f1 qsim_fft n={n}", n, ms, wall, prof, gb)
    Q.qsim_destroy(h)


def f4(n=28, b=8, nm=30):
    """Row f4: approximate QFT (band b) through the gate queue, partial
    measurement with collapse and the inner product (fidelity)."""
    h = Q.qsim_create(n)
    Q.qsim_init_gaussian(h, 3)
    gates = n + sum(1 for j in range(n) for k in range(j + 1, n) if k - j <= b)
    gb = n * (1 << (n + 5)) + (gates - n) * (1 << (n + 3)) + n // 2 * (1 << (n + 4))
    Q.qsim_aqft(h, 0, n, b, False)
    ms, wall, prof, _ = timed(h, lambda: Q.qsim_aqft(h, 0, n, b, False), reps=3)
    report(f"f4 AQFT n={n} band b={b} ({gates} gates)", n, ms, wall, prof, gb)
    Q.qsim_destroy(h)
    ha, hb = Q.qsim_create(nm), Q.qsim_create(nm)
    Q.qsim_init_gaussian(ha, 3)
    Q.qsim_init_gaussian(hb, 5)
    Q.qsim_inner(ha, hb)
    Q.qsim_measure_range(ha, 0, 20, 0.37, False)
    ms, wall, prof, v = timed(ha, lambda: Q.qsim_inner(ha, hb), reps=3)
    report(f"f4 inner product n={nm}", nm, ms, wall, prof, 2 * (1 << (nm + 4)), {"inner_abs": abs(v)})
    ms, wall, prof, y = timed(ha, lambda: Q.qsim_measure_range(ha, 0, 20, 0.37, True))
    report(f"f4 measure qubits [0,20) of n={nm} with collapse", nm, ms, wall, prof,
           (1 << (nm + 4)) + (1 << (nm + 5)), {"y": y, "norm_after": Q.qsim_norm(ha)})
    Q.qsim_destroy(ha)
    Q.qsim_destroy(hb)


if __name__ == "__main__":
    which = sys.argv[1:] or ["0", "1", "2", "3", "3n", "4s"]
    for w in which:
        if w == "0":
            cfg0()
        elif w == "1":
            cfg1()
        elif w == "2":
            cfg2()
        elif w == "3":
            cfg3(0.0)
        elif w == "3n":
            cfg3(1e-3)
        elif w == "4s":
            cfg4(26, 20)
        elif w == "4":
            cfg4(32, 20)
        elif w == "f1":
            f1()
        elif w == "f4":
            f4()
