"""Small invocations of every pipelined / shared-memory kernel, for
compute-sanitizer (racecheck, synccheck, memcheck; one tool per run):
k_qft13, k_qft_tma (12-bit plan), k_qft_gen (noisy QFT), k_ops_pp /
k_ops_pass / k_ops_tma (gate lists), k_perm_ring (MODEXP), k_grover_regs,
the diffusion and the host-stream pipeline.  Exits non-zero on a parity miss."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

n = int(os.environ.get("SAN_N", "16"))
worst = 0.0


def chk(got, ref, what):
    global worst
    e = float(np.max(np.abs(got - ref)))
    worst = max(worst, e)
    print(f"{what}: {e:.2e}", flush=True)


rng = np.random.default_rng(1)
psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
psi /= np.linalg.norm(psi)

h = Q.qsim_create(n)
Q.qsim_set_state(h, 0, psi)
Q.qsim_qft(h, 0, n, False)                        # k_qft13 (n >= 15) or k_qft_tma
ref = psi.copy(); O.qft(ref, 0, n, False)
chk(Q.qsim_get_state(h, 0, 1 << n), ref, "qft")
Q.qsim_hadamard(h, 0, n)
O.hadamard_range(ref, 0, n)
chk(Q.qsim_get_state(h, 0, 1 << n), ref, "hadamard")
Q.qsim_set_gate_noise(h, 7, 1e-3)
Q.qsim_set_gate_counter(h, 0)
Q.qsim_qft(h, 1, n - 2, True)                     # k_qft_gen
Q.qsim_set_gate_noise(h, 0, 0.0)
O.qft(ref, 1, n - 2, True, noise=O.Noise(7, 1e-3, 0))
chk(Q.qsim_get_state(h, 0, 1 << n), ref, "noisy qft")
Q.qsim_destroy(h)

h = Q.qsim_create(n)
ev = W.run_cfg4(h, n=n, layers=4, seed=5, sigma=1e-3, p=0.05)   # gate-list passes
r4, rev = O.cfg4(n=n, layers=4, seed=5, sigma=1e-3, p=0.05)
assert [tuple(e) for e in ev] == [tuple(e) for e in rev]
chk(Q.qsim_get_state(h, 0, 1 << n), r4, "cfg4")
Q.qsim_destroy(h)

ne, nw, N = n - 6, 6, 55
h = Q.qsim_create(n)
P = W.run_cfg3(h, ne=ne, nw=nw, N=N, seed=4, sigma=0.0, a=3)    # k_perm_ring + probs
pr = O.cfg3(ne=ne, nw=nw, N=N, seed=4, sigma=0.0, a=3)
chk(P, pr, "cfg3")
Q.qsim_destroy(h)

m = 14
h = Q.qsim_create(m)
k, trace = W.run_cfg1(h, n=m, seed=2, iters=30)                 # k_grover_regs
_, rt = O.cfg1(n=m, seed=2, iters=30)
chk(trace, rt, "grover")
Q.qsim_diffusion(h, 0, m)
Q.qsim_destroy(h)

h = Q.qsim_create(n)
inp = np.ascontiguousarray(np.stack([psi, psi[::-1].copy()]))
out = np.zeros_like(inp)
Q.qsim_qft_host_stream(h, 0, n, False, inp, out, 2, 1 << n, 1 << n)
ref = psi.copy(); O.qft(ref, 0, n, False)
chk(out[0], ref, "host stream")
Q.qsim_destroy(h)

print("WORST", worst)
sys.exit(0 if worst < 1e-10 else 1)
