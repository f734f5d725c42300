"""Wall time of each step of configs[3] (n = 30), synchronising after every
call: where the device time between kernels goes.  python tools/probe_cfg3_steps.py [sigma]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
h = Q.qsim_create(30)
a = W.shor_base(4, 1007)
for rep in range(3):
    t = {}
    def step(name, f):
        Q.qsim_sync(h)
        t0 = time.perf_counter()
        f()
        Q.qsim_sync(h)
        t[name] = round((time.perf_counter() - t0) * 1e3, 3)
    step("set_basis", lambda: Q.qsim_set_basis(h, 1))
    step("noise", lambda: (Q.qsim_set_gate_noise(h, 4, sigma), Q.qsim_set_gate_counter(h, 0)))
    step("H_n", lambda: Q.qsim_hadamard_angles(h, 0, 20) if sigma > 0 else Q.qsim_hadamard(h, 0, 20))
    step("modexp", lambda: Q.qsim_apply_perm(h, Q.QSIM_PERM_MODEXP, 20, 10, elo=0, em=20, base=a, modulus=1007))
    step("iqft", lambda: Q.qsim_qft(h, 0, 20, True))
    step("probs", lambda: Q.qsim_probs(h, 0, 20))
    print(rep, t, "sum", round(sum(t.values()), 3), flush=True)
Q.qsim_destroy(h)
