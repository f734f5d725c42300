"""End-to-end probe (measurement only): qsim_qft_host_stream at n = 28 with
pinned host buffers for several step counts; prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

n = 28
h = Q.qsim_create(n)
Q.qsim_init_gaussian(h, 3)
hin = torch.empty(1 << n, dtype=torch.complex128, pin_memory=True).numpy()
hout = torch.empty(1 << n, dtype=torch.complex128, pin_memory=True).numpy()
Q.qsim_get_state(h, 0, 1 << n, hin)
Q.qsim_qft_host_stream(h, 0, n, False, hin, hout, 1, 0, 0)
res = {}
for count in (1, 2, 6, 12, 24):
    t0 = time.perf_counter()
    Q.qsim_qft_host_stream(h, 0, n, False, hin, hout, count, 0, 0)
    res[count] = round((time.perf_counter() - t0) * 1e3 / count, 2)
print(json.dumps({"ms_per_step": res}), flush=True)
Q.qsim_destroy(h)
