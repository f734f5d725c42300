"""Launch-gap probe (measurement only): configs[2] QFT steps timed back to
back with CUDA events on the library's stream, against the sum of the
per-launch durations (the library's profiler) of the same steps, and against
host enqueue time per step; prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
steps = 20
h = Q.qsim_create(n)
stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
Q.qsim_init_gaussian(h, 3)
for _ in range(5):
    Q.qsim_qft(h, 0, n, False)
Q.qsim_sync(h)
res = {}
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(steps):
        Q.qsim_qft(h, 0, n, False)
    host = (time.perf_counter() - t0) * 1e3 / steps
    e1.record(stream)
    torch.cuda.synchronize()
    res[f"events_ms_{rep}"] = e0.elapsed_time(e1) / steps
    res[f"host_enqueue_ms_{rep}"] = host
Q.qsim_profile(h, True)
for _ in range(steps):
    Q.qsim_qft(h, 0, n, False)
prof = Q.qsim_profile_json(h)
Q.qsim_profile(h, False)
L = prof.pop("_launches")
res["sum_launch_ms"] = sum(x[1] for x in L) / steps
res["launches_per_step"] = len(L) / steps
# the same steps with the first pass of each step delayed behind a busy host
# (enqueue one step ahead): events again
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(steps):
    Q.qsim_qft(h, 0, n, False)
    e1.record(stream)
torch.cuda.synchronize()
res["events_ms_recorded_each"] = e0.elapsed_time(e1) / steps
print(json.dumps({k: round(v, 4) for k, v in res.items()}), flush=True)
Q.qsim_destroy(h)
