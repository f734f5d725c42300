import json, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_quant_ph_0201042_b200 import qsim as Q
n = 28
for q in [27, 20, 10, 3, 0]:
    h = Q.qsim_create(n); Q.qsim_init_gaussian(h, 3)
    U = np.array([[0.6, 0.8j], [0.8j, 0.6]])
    Q.qsim_apply_1q(h, q, U); Q.qsim_sync(h)
    Q.qsim_profile(h, True)
    for _ in range(3): Q.qsim_apply_1q(h, q, U); Q.qsim_sync(h)
    prof = Q.qsim_profile_json(h); la = prof.pop("_launches"); Q.qsim_profile(h, False)
    ms = sum(x[1] for x in la) / 3
    print(json.dumps({"q": q, "kern": la[0][0], "ms": round(ms, 3), "hbm_frac": round(2 ** (n + 5) / (ms * 1e-3) / 6.45e12, 3)}))
    Q.qsim_destroy(h)
