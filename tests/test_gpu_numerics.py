"""Arithmetic building blocks of the kernels that must be bit-identical to
IEEE float64 (the reference computes in numpy float64).

The lane K3 divides a row's E masses by one water level per fill evaluation
and the Huntington-Hill priorities by per-seat constants.  It does so with
one correctly rounded reciprocal and FMA corrections (Markstein's final
step, projection.cuh SharedDivisor) instead of E full divisions; the result
must equal __ddiv_rn bit for bit on every operand pair the kernels can meet.
"""

import ctypes

import pytest

from paper_2506_00167_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 0x5EED])
def test_shared_divisor_matches_ieee_division(seed):
    lib = _native.lib()
    bad = ctypes.c_int64(-1)
    pairs = 1 << 30
    _native.check(lib.cyr_selftest_shared_divisor(pairs, seed, ctypes.byref(bad)))
    assert bad.value == 0, f"{bad.value} of {pairs} quotients differ from __ddiv_rn"
