"""Single controlled gates whose control or target sits on the lowest
positions (measurement only; SURVEY §8(d) per-gate metric): one call each on
n = 28 through the library's default path, timed by the library's per-launch
events; run under ncu --metrics dram__bytes_* for the DRAM bytes."""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

n = 28
q_of = lambda p: n - 1 - p   # qubit at position p (canonical)
ph = np.exp(1j * math.pi / 4)
X = [[0, 1], [1, 0]]
R = [[1, 0], [0, ph]]
cases = [("cr", 0, 1), ("cr", 1, 2), ("cr", 2, 3), ("cr", 3, 4), ("cr", 5, 6), ("cnot", 0, 5), ("cnot", 1, 5),
         ("cnot", 2, 5), ("cnot", 5, 0), ("cnot", 5, 1), ("cnot", 5, 2), ("cnot", 6, 7)]
h = Q.qsim_create(n)
Q.qsim_init_gaussian(h, 3)
if os.environ.get("UNFUSED"):
    Q.qsim_set_fusion(h, False)
for rep in range(2):
    out = []
    for kind, pc, pt in cases:
        Q.qsim_sync(h)
        Q.qsim_profile(h, True)
        c = q_of(pc)
        Q.qsim_apply_ctrl(h, 1 << c, 1 << c, q_of(pt), X if kind == "cnot" else R)
        Q.qsim_sync(h)
        prof = Q.qsim_profile_json(h)
        Q.qsim_profile(h, False)
        launches = prof.pop("_launches")
        ms = sum(x[1] for x in launches)
        alg = (1 << (n + 4)) if kind == "cnot" else (1 << (n + 3))
        out.append({"kind": kind, "ctrl_pos": pc, "tgt_pos": pt, "kernels": [x[0] for x in launches],
                    "ms": round(ms, 4), "alg_gbs": round(alg / (ms * 1e-3) / 1e9, 1)})
    if rep == 1:
        for o in out:
            print(json.dumps(o), flush=True)
Q.qsim_destroy(h)
