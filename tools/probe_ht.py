"""Kernel breakdown of one HT noise-experiment cell (row f2): n = 20 register,
2^b trajectories, k applications.  python tools/probe_ht.py [sigma] [p] [b] [k]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
p = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
b = int(sys.argv[3]) if len(sys.argv) > 3 else 10
k = int(sys.argv[4]) if len(sys.argv) > 4 else 100
n = 20
h = Q.qsim_create(n + b)
W.run_ht_batch(h, n, b, 2, seed=5, sigma=sigma, p=p)   # warm-up
Q.qsim_profile(h, True)
Q.qsim_sync(h)
t0 = time.perf_counter()
v, ev = W.run_ht_batch(h, n, b, k, seed=1_000_000, sigma=sigma, p=p)
Q.qsim_sync(h)
wall = time.perf_counter() - t0
prof = Q.qsim_profile_json(h)
prof.pop("_launches", None)
print(json.dumps({"sigma": sigma, "p": p, "b": b, "k": k, "wall_s": round(wall, 3), "mean_p0": v, "events": len(ev),
                  "kernels": {kk: (vv["launches"], round(vv["ms"], 1)) for kk, vv in prof.items()}}))
Q.qsim_destroy(h)
