"""PCIe copy bandwidth (measurement only): pinned host <-> device, 4 GiB,
H2D alone, D2H alone, both at once on two streams."""
import json
import time

import torch

n = 1 << 28   # complex128 elements = 4 GiB
h_in = torch.empty(n, dtype=torch.complex128, pin_memory=True)
h_out = torch.empty(n, dtype=torch.complex128, pin_memory=True)
d_a = torch.empty(n, dtype=torch.complex128, device="cuda")
d_b = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = 16 * n / 1e9
res = {}
for name in ("h2d", "d2h", "both"):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    res[name] = {"s": round(dt, 4), "GBps": round(gb * (2 if name == "both" else 1) / dt, 1)}
print(json.dumps(res))
