#!/usr/bin/env python3
"""Per-gate HBM bandwidth, SURVEY.md §8(d) "Per-gate metric".

For n in {28, 30, 32}, every qubit position q and each gate kind (dense 1q,
CNOT, controlled phase R_2, diagonal), one standalone gate is timed with CUDA
events on the library's stream (median of REPS, state resident in HBM, state
>> L2).  Two paths:

* ``unfused``: fusion off -> the paper's one-sweep-per-gate kernels
  (``k_apply_2x2`` / ``k_phase_mask``, k_gates.cu);
* ``fused``: the gate queue's single-gate pass (``k_ops_pass``, in place,
  TMA-staged tiles when the geometry allows).

GB/s = algorithmic bytes / time, with the survey's byte model: dense
2^(n+5), CNOT (1 control) 2^(n+4), R_d (touches |11>) 2^(n+3), diagonal
diag(d0, d1) with both entries != 1: 2^(n+5).  One JSON line per (n, path,
kind) with the per-q numbers and the min / median fraction of the HBM peak.
Usage: python tools/bench_gates.py [n ...]
"""
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

REPS = int(os.environ.get("REPS", "5"))


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 7672.0


def kinds(n):
    s = 1 / math.sqrt(2)
    th = 0.3
    U = np.array([[math.cos(th), -math.sin(th) * 1j], [-math.sin(th) * 1j, math.cos(th)]]) @ \
        np.diag([1, np.exp(0.7j)])
    ph = np.exp(1j * math.pi / 4)
    return {
        # name: (apply(h, q), bytes)
        "dense": (lambda h, q: Q.qsim_apply_1q(h, q, U), 1 << (n + 5)),
        "cnot": (lambda h, q: Q.qsim_apply_ctrl(h, 1 << ((q + 1) % n), 1 << ((q + 1) % n), q,
                                                [[0, 1], [1, 0]]), 1 << (n + 4)),
        "cr": (lambda h, q: Q.qsim_apply_ctrl(h, 1 << ((q + 1) % n), 1 << ((q + 1) % n), q,
                                              [[1, 0], [0, ph]]), 1 << (n + 3)),
        "diag": (lambda h, q: Q.qsim_apply_1q(h, q, [[np.exp(-0.2j), 0], [0, np.exp(0.9j)]]), 1 << (n + 5)),
        "hadamard": (lambda h, q: Q.qsim_apply_1q(h, q, [[s, s], [s, -s]]), 1 << (n + 5)),
    }


def time_gate(h, stream, fn, q):
    ts = []
    for _ in range(REPS + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn(h, q)
        Q.qsim_sync(h)        # flushes the queue (fused path) inside the region
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts[1:])


def main():
    ns = [int(a) for a in sys.argv[1:]] or [28, 30, 32]
    pk = peak()
    for n in ns:
        h = Q.qsim_create(n)
        stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
        Q.qsim_init_gaussian(h, 3)
        for path in ("unfused", "fused"):
            Q.qsim_set_fusion(h, path == "fused")
            for kind, (fn, nbytes) in kinds(n).items():
                per_q = []
                for q in range(n):
                    ms = time_gate(h, stream, fn, q)
                    per_q.append(round(nbytes / (ms * 1e-3) / 1e9, 1))
                fr = [g / pk for g in per_q]
                print(json.dumps({"n": n, "path": path, "kind": kind, "bytes": nbytes, "peak_gbs": pk,
                                  "GBps_per_q": per_q, "min_frac": round(min(fr), 3),
                                  "median_frac": round(statistics.median(fr), 3),
                                  "max_frac": round(max(fr), 3)}), flush=True)
        nrm = Q.qsim_norm(h)
        print(json.dumps({"n": n, "norm_after": nrm}), flush=True)
        Q.qsim_destroy(h)


if __name__ == "__main__":
    main()
