"""QFT pass-plan probe (measurement only): per-pass device times of qsim_qft
at n (default 28) under the env knobs QSIM_QFT_BLOCKS / QSIM_L2PROM /
QSIM_TILE_GROUP; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
mode = sys.argv[2] if len(sys.argv) > 2 else "qft"


def step():
    if mode == "qft":
        Q.qsim_qft(h, 0, n, False)
    else:
        Q.qsim_hadamard(h, 0, n)

reps = 5
h = Q.qsim_create(n)
Q.qsim_init_gaussian(h, 3)
for _ in range(2):
    step()
Q.qsim_sync(h)
Q.qsim_profile(h, True)
for _ in range(reps):
    step()
prof = Q.qsim_profile_json(h)
launches = prof.pop("_launches")
per = len(launches) // reps
passes = [[launches[r * per + i][1] for r in range(reps)] for i in range(per)]
med = [sorted(p)[reps // 2] for p in passes]
gb = (16 << n) * 2 / 1e9
print(json.dumps({"n": n, "mode": mode, "blocks": os.environ.get("QSIM_QFT_BLOCKS", "default"),
                  "l2prom": os.environ.get("QSIM_L2PROM", "default"), "group": os.environ.get("QSIM_TILE_GROUP", "0"),
                  "names": [launches[i][0] for i in range(per)],
                  "pass_ms": [round(x, 4) for x in med], "total_ms": round(sum(med), 4),
                  "pass_tbs": [round(gb / x, 3) for x in med]}), flush=True)
Q.qsim_destroy(h)
