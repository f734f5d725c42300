"""Gate-list pass probe: G random dense gates on the same 5 (or more) qubits
at n = 28 -> one pass, one segment when q <= 5.  Prints FP64 utilisation of
the pass (8 FMA per amplitude per gate) vs the measured FP64 rate."""
import json, os, sys, math
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
n = 28
rng = np.random.default_rng(1)
for nq, G in [(5, 10), (5, 30), (5, 60), (9, 30), (9, 60)]:
    h = Q.qsim_create(n)
    Q.qsim_init_gaussian(h, 3)
    qs = list(range(n - nq, n))          # the lowest positions... qubits n-nq..n-1
    mats = []
    for _ in range(G):
        a = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
        qm, _ = np.linalg.qr(a)
        mats.append((int(rng.choice(qs)), qm))
    def run():
        for q, U in mats:
            Q.qsim_apply_1q(h, q, U)
        Q.qsim_sync(h)
    run()
    Q.qsim_profile(h, True)
    run()
    prof = Q.qsim_profile_json(h)
    launches = prof.pop("_launches")
    Q.qsim_profile(h, False)
    ms = sum(x[1] for x in launches)
    fma = G * 8 * 2.0 ** n
    print(json.dumps({"qubits": nq, "gates": G, "launches": [x[0] for x in launches], "ms": round(ms, 3),
                      "fp64_frac_of_1.5e13": round(fma / (ms * 1e-3) / 1.5e13, 3),
                      "hbm_frac": round(len(launches) * 2 ** (n + 5) / (ms * 1e-3) / 6.45e12, 3)}))
    Q.qsim_destroy(h)
