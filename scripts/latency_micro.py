"""Cycles per dependent step of fp64 building blocks on this GPU."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_00167_b200 import _native  # noqa: E402

NAMES = ["DFMA", "DMUL", "sqrt_pos", "__dsqrt_rn", "__ddiv_rn", "FFMA", "coupled step",
         "SHFL", "vote.all", "MUFU.RSQ64H"]
lib = _native.lib()
for w, name in enumerate(NAMES):
    c = ctypes.c_int64()
    _native.check(lib.cyr_selftest_latency(w, 1000, ctypes.byref(c)))
    _native.check(lib.cyr_selftest_latency(w, 11000, ctypes.byref(c)))
    c2 = c.value
    _native.check(lib.cyr_selftest_latency(w, 1000, ctypes.byref(c)))
    print(f"{name:>14s}: {(c2 - c.value) / 10000:7.1f} cycles/step")
