import os, sys, json
sys.path.insert(0, '.')
import torch
from paper_quant_ph_0201042_b200 import qsim as Q
for n in (27, 28, 29, 30, 31):
    h = Q.qsim_create(n); Q.qsim_init_gaussian(h, 3)
    stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
    for m in (n, 20, 22):
        Q.qsim_qft(h, 0, m, False); Q.qsim_sync(h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3): Q.qsim_qft(h, 0, m, False)
        Q.qsim_sync(h); e1.record(stream); torch.cuda.synchronize()
        print(json.dumps({"amax": os.environ.get("QSIM_QFT_AMAX", "7"), "n": n, "m": m, "ms": round(e0.elapsed_time(e1) / 3, 3)}))
    Q.qsim_destroy(h)
