"""B200-native (sm_100a) state-vector gate engine for the method of Niwa,
Matsumoto & Imai, "General-Purpose Parallel Simulator for Quantum Computing"
(arXiv quant-ph/0201042).

The product is ``libqsim.so`` (C-ABI, ``include/qsim.h``) built from
``csrc/``; ``qsim`` is its ctypes binding (same names, marshalling only) and
``workloads`` drives the five BASELINE.json configs through it.
"""
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose: bool = False) -> None:
    """Compile libqsim.so in-tree for sm_100a (make -C csrc)."""
    subprocess.run(["make", "-s" if not verbose else "-j8", "-j8", "-C", os.path.join(_HERE, "csrc")],
                   check=True)
