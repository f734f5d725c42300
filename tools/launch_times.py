"""Per-launch kernel times of one config run (library profiler): python tools/launch_times.py 3n|4s"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402
w = sys.argv[1]
n = {"3n": 30, "4s": 26, "f4": 28}[w]
h = Q.qsim_create(n)
run = {"3n": lambda: W.run_cfg3(h, 20, 10, 1007, 4, 1e-3), "4s": lambda: W.run_cfg4(h, 26, 20, 5, 1e-3, 1e-4),
       "f4": lambda: Q.qsim_aqft(h, 0, 28, 8, False)}[w]
run()
Q.qsim_sync(h)
Q.qsim_profile(h, True)
run()
Q.qsim_sync(h)
prof = Q.qsim_profile_json(h)
for l in prof.get("_launches", []):
    print(json.dumps(l))
Q.qsim_destroy(h)
