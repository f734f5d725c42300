"""The 2^33-amplitude register on one B200 (128 GiB, no scratch shard): fused
QFT (in-place passes, closing swaps as a relabel) and H_n timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402

n = 33
h = Q.qsim_create(n)
Q.qsim_init_gaussian(h, 3)
stream = torch.cuda.ExternalStream(Q.qsim_get_stream(h))
for name, fn in (("qft", lambda: Q.qsim_qft(h, 0, n, False)), ("hadamard", lambda: Q.qsim_hadamard(h, 0, n)),
                 ("norm", lambda: Q.qsim_norm(h))):
    fn()
    Q.qsim_sync(h)
    Q.qsim_profile(h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    Q.qsim_sync(h)
    e1.record(stream)
    torch.cuda.synchronize()
    prof = Q.qsim_profile_json(h)
    prof.pop("_launches", None)
    Q.qsim_profile(h, False)
    print(name, round(e0.elapsed_time(e1), 2), "ms", {k: (v["launches"], round(v["bytes"] / v["ms"] / 1e6)) for k, v in prof.items()})
print("norm", Q.qsim_norm(h))
Q.qsim_destroy(h)
