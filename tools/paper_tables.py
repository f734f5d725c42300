#!/usr/bin/env python3
"""The paper's Tables 1 and 2 workloads on one B200 (PAPER.md:588-613,
640-658): the QFT circuit and the FFT for n = 20..29 (Table 1) and the
Hadamard transform H_n on |0...0> (Table 2), each timed three ways through
the C-ABI: gate by gate with one HBM sweep per gate (fusion off -- the
paper's own algorithm), fused passes (the default), and, for Table 1, the FFT
(`qsim_fft`).  Seeded complex-Gaussian input for Table 1 (the paper's input
state is unstated), |0...0> for Table 2.  Prints one JSON line per row and
a markdown table; the paper's E4500 seconds are printed beside (context)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

T1 = {20: (26.08, 5.33, 1.21, 0.53), 22: (124.78, 23.40, 5.01, 1.83), 24: (643.02, 137.7, 20.00, 5.84),
      26: (2745.56, 526.82, 113.29, 32.84), 28: (12597.8, 2338.19, 567.19, 142.01),
      29: (31089.6, 5811.49, 1232.16, 286.29)}   # circuit 1p, circuit 8p, FFT 1p, FFT 8p (s)
T2 = {20: (2.38, 0.40), 22: (10.85, 1.35), 24: (46.94, 9.58), 26: (205.81, 38.71), 28: (887.40, 167.31),
      29: (2027.9, 395.81)}   # H_n 1p, 8p (s)


def timed(h, fn, reps=3):
    stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
    fn()
    Q.qsim_sync(h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    Q.qsim_sync(h)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rows = []
for n in sorted(T1):
    h = Q.qsim_create(n)
    Q.qsim_init_gaussian(h, 3)
    fused = timed(h, lambda: Q.qsim_qft(h, 0, n, False))
    fft = timed(h, lambda: Q.qsim_fft(h, 0, n, False))
    Q.qsim_set_fusion(h, False)
    sweep = timed(h, lambda: Q.qsim_qft(h, 0, n, False), reps=1)
    Q.qsim_set_fusion(h, True)
    Q.qsim_set_basis(h, 0)
    hf = timed(h, lambda: Q.qsim_hadamard(h, 0, n))
    Q.qsim_set_fusion(h, False)
    hs = timed(h, lambda: [Q.qsim_apply_1q(h, q, [[2 ** -0.5, 2 ** -0.5], [2 ** -0.5, -(2 ** -0.5)]])
                           for q in range(n)], reps=1)
    Q.qsim_destroy(h)
    r = {"n": n, "qft_circuit_sweep_ms": round(sweep, 3), "qft_fused_ms": round(fused, 3), "fft_ms": round(fft, 3),
         "ht_sweep_ms": round(hs, 3), "ht_fused_ms": round(hf, 3),
         "paper_qft_circuit_s": T1[n][:2], "paper_fft_s": T1[n][2:], "paper_ht_s": T2[n]}
    rows.append(r)
    print(json.dumps(r), flush=True)

print()
print("| n | QFT circuit, one sweep per gate | QFT fused | FFT | H_n one sweep per gate | H_n fused | paper QFT circuit 1p / 8p | paper FFT 1p / 8p | paper H_n 1p / 8p |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['n']} | {r['qft_circuit_sweep_ms']} ms | {r['qft_fused_ms']} ms | {r['fft_ms']} ms | {r['ht_sweep_ms']} ms | "
          f"{r['ht_fused_ms']} ms | {r['paper_qft_circuit_s'][0]} / {r['paper_qft_circuit_s'][1]} s | "
          f"{r['paper_fft_s'][0]} / {r['paper_fft_s'][1]} s | {r['paper_ht_s'][0]} / {r['paper_ht_s'][1]} s |")
