"""Sustained-load probe (measurement only): batches of back-to-back configs[2]
QFT steps and of 4 GiB torch copies over ~3 s each, per-batch device time
with nvidia-smi power / SM clock samples; prints JSON lines."""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

lines = []
proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [lines.append((time.perf_counter(), l.strip())) for l in proc.stdout],
                 daemon=True).start()


def window(t0, t1):
    s = [l for t, l in lines if t0 <= t <= t1]
    clk = sorted(float(x.split(",")[0]) for x in s) or [0]
    pw = sorted(float(x.split(",")[1]) for x in s) or [0]
    return {"sm_mhz_med": clk[len(clk) // 2], "power_w_med": pw[len(pw) // 2], "samples": len(s)}


n = 28
h = Q.qsim_create(n)
stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
Q.qsim_init_gaussian(h, 3)
a = torch.empty(1 << 29, dtype=torch.float64, device="cuda")   # 4 GiB
b = torch.empty_like(a)
a.normal_()
for kind in ("qft", "copy", "qft"):
    for batch in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if kind == "qft":
            e0.record(stream)
            for _ in range(80):
                Q.qsim_qft(h, 0, n, False)
            e1.record(stream)
            per = 3 * (32 << n)
        else:
            e0.record()
            for _ in range(80):
                b.copy_(a)
            e1.record()
            per = 2 * a.numel() * 8
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ms = e0.elapsed_time(e1) / 80
        print(json.dumps({"kind": kind, "batch": batch, "ms": round(ms, 4), "tbs": round(per / ms / 1e9, 3),
                          **window(t0, t1)}), flush=True)
proc.terminate()
Q.qsim_destroy(h)
