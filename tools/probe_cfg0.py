import sys, time, math
sys.path.insert(0, '.')
from paper_quant_ph_0201042_b200 import qsim as Q
from paper_quant_ph_0201042_b200 import workloads as W
h = Q.qsim_create(10)
W.run_cfg0(h, 10, 1, 200); Q.qsim_sync(h)
t = time.perf_counter()
for _ in range(10): W.run_cfg0(h, 10, 1, 200)
Q.qsim_sync(h)
print("run_cfg0 ms", (time.perf_counter() - t) / 10 * 1e3)
t = time.perf_counter()
for _ in range(10):
    for g in range(200):
        a, b = Q.qsim_philox_draw(1, Q.QSIM_TAG_GATE, g, 0)
        W.haar_angles(1, g)
print("draws only ms", (time.perf_counter() - t) / 10 * 1e3)
U = [[0.6, 0.8], [0.8, -0.6]]
t = time.perf_counter()
for _ in range(10):
    for g in range(200): Q.qsim_apply_1q(h, g % 10, U)
Q.qsim_sync(h)
print("apply_1q only ms", (time.perf_counter() - t) / 10 * 1e3)
t = time.perf_counter()
for _ in range(10):
    for g in range(200): Q.qsim_apply_angles(h, Q.QSIM_GATE_HAAR, [0.1, 0.2, 0.3, 0.4], 0, 0, g % 10)
Q.qsim_sync(h)
print("apply_angles only ms", (time.perf_counter() - t) / 10 * 1e3)
