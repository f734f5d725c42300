"""pytest configuration: the `gpu` marker and the repo root on sys.path.

`-m "not gpu"` runs the oracle pins, host logic, the C-ABI symbol check and
the gloo multi-process tests (no GPU needed); `-m gpu` runs the parity tests
that call the sm_100a library through its C-ABI.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libqsim.so")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")
