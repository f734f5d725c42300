"""Run one config once (for ncu captures): python tools/run_cfg.py 1|3|3n|4|4m|4s"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_quant_ph_0201042_b200 import qsim as Q  # noqa: E402
from paper_quant_ph_0201042_b200 import workloads as W  # noqa: E402

w = sys.argv[1]
if w == "1":
    h = Q.qsim_create(20)
    W.run_cfg1(h, 20, 2)
elif w == "3":
    h = Q.qsim_create(30)
    W.run_cfg3(h, 20, 10, 1007, 4, 0.0)
elif w == "3n":
    h = Q.qsim_create(30)
    W.run_cfg3(h, 20, 10, 1007, 4, 1e-3)
elif w == "4s":
    h = Q.qsim_create(26)
    W.run_cfg4(h, 26, 20, 5, 1e-3, 1e-4)
elif w == "4m":
    h = Q.qsim_create(30)
    W.run_cfg4(h, 30, 20, 5, 1e-3, 1e-4)
elif w == "4":
    h = Q.qsim_create(32)
    W.run_cfg4(h, 32, 20, 5, 1e-3, 1e-4)
Q.qsim_sync(h)
Q.qsim_destroy(h)
