"""configs[4] plan / per-pass probe (measurement only): runs the noisy
brickwork at n (default 32) once to warm up and once profiled; with
QSIM_PLAN_LOG=1 the planner prints each pass's op mix on stderr."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = Q.qsim_create(n)
if n <= 30:
    W.run_cfg4(h, n=n, layers=layers, seed=5, sigma=1e-3, p=1e-4)
    Q.qsim_sync(h)
Q.qsim_profile(h, True)
t0 = time.perf_counter()
W.run_cfg4(h, n=n, layers=layers, seed=5, sigma=1e-3, p=1e-4)
Q.qsim_sync(h)
wall = time.perf_counter() - t0
prof = Q.qsim_profile_json(h)
launches = prof.pop("_launches")
print(json.dumps({"n": n, "layers": layers, "wall_s": round(wall, 4),
                  "kernel_ms": {k: round(v["ms"], 3) for k, v in prof.items()},
                  "launches": [[a, round(b, 3)] for a, b in launches]}), flush=True)
Q.qsim_destroy(h)
