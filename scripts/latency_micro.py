"""Cycles per dependent step of fp64 building blocks on this GPU."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_00167_b200 import _native  # noqa: E402

NAMES = ["DFMA", "DMUL", "__dsqrt_rn*c", "__dsqrt_rn+1", "__ddiv_rn", "FFMA", "coupled step",
         "SHFL", "vote.all", "MUFU.RSQ64H", "coupled loop (per call)"]
lib = _native.lib()
for w, name in enumerate(NAMES):
    c = ctypes.c_int64()
    n1, n2 = (10, 110) if w == 10 else (1000, 11000)
    _native.check(lib.cyr_selftest_latency(w, n1, ctypes.byref(c)))
    _native.check(lib.cyr_selftest_latency(w, n2, ctypes.byref(c)))
    c2 = c.value
    _native.check(lib.cyr_selftest_latency(w, n1, ctypes.byref(c)))
    print(f"{name:>14s}: {(c2 - c.value) / (n2 - n1):7.1f} cycles/step")
