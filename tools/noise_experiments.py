#!/usr/bin/env python3
"""The paper's noise experiments on one B200 with batched trajectories
(R33-R37).  One JSON line per cell.

  ht     Table 3 / Figs. 7-8: 20-qubit register, H_n applied
         k = 100 times (reading C24/R34), depolarizing p and operational sigma;
         the trajectory average of |<0|psi>|^2 next to the paper's closed forms
         ((1+(1-4p/3)^k)/2)^n and ((1+e^{-9k sigma^2/4})/2)^n
          and the paper's Table 3 value.
  qft    Table 7: Shor N = 187, x = 23, 16-qubit exponent
         register in the semantic state (v = 1, R37), QFT circuit with angle
         noise sigma and depolarizing p after every R_d; mean fidelity
         |<ideal|psi_t>| over the trajectories.
  grover Figs. 12-13: 10-qubit register + ancilla,
         averaged P(register = mark) per G-iteration.

Usage: python tools/noise_experiments.py [ht|qft|grover ...] [--traj-bits B] [--batches K]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

PAPER_T3 = {  # PAPER.md:805-810, Table 3: rows p, columns sigma
    0.0: {0.0: 1.0000, 1e-5: 1.0000, 1e-4: 0.9999, 1e-3: 0.9977},
    1e-5: {0.0: 0.9870, 1e-5: 0.9870, 1e-4: 0.9849, 1e-3: 0.9797},
    1e-4: {0.0: 0.9010, 1e-5: 0.9010, 1e-4: 0.8909, 1e-3: 0.8780},
    1e-3: {0.0: 0.2910, 1e-5: 0.2790, 1e-4: 0.2779, 1e-3: 0.2664},
}
PAPER_T7 = {  # PAPER.md:1146-1152, Table 7
    0.0: [1.0000, 0.9999, 0.9999, 0.9999, 0.9998],
    1e-5: [0.9880, 0.9840, 0.9860, 0.9880, 0.9848],
    1e-4: [0.8837, 0.8897, 0.8827, 0.8801, 0.8980],
    1e-3: [0.3287, 0.3399, 0.3332, 0.3209, 0.3363],
    1e-2: [0.0027, 0.0015, 0.0019, 0.0017, 0.0031],
}
SIG7 = [0.0, 1e-5, 1e-4, 1e-3, 1e-2]


def ht(b, batches, k=100, n=20):
    h = Q.qsim_create(n + b)
    try:
        for p in (0.0, 1e-5, 1e-4, 1e-3):
            for sigma in (0.0, 1e-5, 1e-4, 1e-3):
                t0 = time.perf_counter()
                vals = []
                for j in range(batches):
                    v, _ = W.run_ht_batch(h, n, b, k, seed=1_000_000 * (j + 1), sigma=sigma, p=p)
                    vals.append(v)
                dt = time.perf_counter() - t0
                m = sum(vals) / len(vals)
                law_p = ((1 + (1 - 4 * p / 3) ** k) / 2) ** n
                law_s = ((1 + math.exp(-9 * k * sigma ** 2 / 4)) / 2) ** n
                print(json.dumps({"experiment": "HT Table 3", "n": n, "k": k, "p": p, "sigma": sigma,
                                  "trajectories": batches << b, "mean_p0": m, "law_product": law_p * law_s,
                                  "law_depolarizing": law_p, "law_operational": law_s,
                                  "paper": PAPER_T3[p][sigma], "seconds": round(dt, 3)}), flush=True)
    finally:
        Q.qsim_destroy(h)


def qft(b, batches, m=16, x=23, N=187, v=1):
    h = Q.qsim_create(m + b)
    try:
        for p in (0.0, 1e-5, 1e-4, 1e-3, 1e-2):
            for si, sigma in enumerate(SIG7):
                t0 = time.perf_counter()
                fids = []
                for j in range(batches):
                    f = W.run_qft_fidelity_batch(h, m, b, x, N, v, seed=7_000_000 * (j + 1), sigma=sigma, p=p)
                    fids.extend(float(a) for a in f)
                dt = time.perf_counter() - t0
                print(json.dumps({"experiment": "QFT-16 Table 7", "m": m, "N": N, "x": x, "p": p, "sigma": sigma,
                                  "trajectories": len(fids), "mean_fidelity": sum(fids) / len(fids),
                                  "paper": PAPER_T7[p][si], "seconds": round(dt, 3)}), flush=True)
    finally:
        Q.qsim_destroy(h)


def grover(b, batches, n=10, iters=50, mark=682):
    h = Q.qsim_create(n + 1 + b)
    try:
        for p, sigma in ((0.0, 0.0), (1e-3, 0.0), (1e-2, 0.0), (0.0, 1e-2), (0.0, 5e-2)):
            t0 = time.perf_counter()
            acc = [0.0] * iters
            for j in range(batches):
                tr = W.run_grover_batch(h, n, b, mark, iters, seed=9_000_000 * (j + 1), sigma=sigma, p=p)
                acc = [a + t / batches for a, t in zip(acc, tr)]
            dt = time.perf_counter() - t0
            th = math.asin(2 ** (-n / 2))
            print(json.dumps({"experiment": "Grover-10", "n": n, "p": p, "sigma": sigma, "mark": mark,
                              "trajectories": batches << b, "mean_p_mark": [round(a, 6) for a in acc],
                              "noiseless": [round(math.sin((2 * t + 3) * th) ** 2, 6) for t in range(iters)],
                              "seconds": round(dt, 3)}), flush=True)
    finally:
        Q.qsim_destroy(h)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["ht", "qft", "grover"])
    ap.add_argument("--traj-bits", type=int, default=10)
    ap.add_argument("--batches", type=int, default=1)
    a = ap.parse_args()
    for w in a.which:
        {"ht": ht, "qft": qft, "grover": grover}[w](a.traj_bits, a.batches)
