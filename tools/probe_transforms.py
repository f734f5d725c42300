"""Fused-transform pass throughput: qsim_hadamard / qsim_qft over ranges of
n = 28 / 30 registers (run with and without QSIM_GEN_ALL=1 to compare the
specialised and the generalised pass kernels)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

for n, cases in ((28, [(0, 28), (0, 20), (8, 20)]), (30, [(0, 30), (0, 20), (10, 20)])):
    h = Q.qsim_create(n)
    Q.qsim_init_gaussian(h, 3)
    stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
    for lo, m in cases:
        for name, fn in (("H", lambda: Q.qsim_hadamard(h, lo, m)), ("QFT", lambda: Q.qsim_qft(h, lo, m, False)),
                         ("IQFT", lambda: Q.qsim_qft(h, lo, m, True))):
            fn()
            Q.qsim_sync(h)
            Q.qsim_profile(h, True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                fn()
            Q.qsim_sync(h)
            e1.record(stream)
            torch.cuda.synchronize()
            prof = Q.qsim_profile_json(h)
            prof.pop("_launches", None)
            Q.qsim_profile(h, False)
            ks = {k: (v["launches"] // 5, round(v["bytes"] / (v["ms"] * 1e-3) / 1e9)) for k, v in prof.items()}
            print(json.dumps({"n": n, "lo": lo, "m": m, "op": name, "ms": round(e0.elapsed_time(e1) / 5, 3),
                              "kernels": ks}), flush=True)
    Q.qsim_destroy(h)
