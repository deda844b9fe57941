"""CPU: the C-ABI library loads and exports every symbol include/ declares.

No compute calls here (no GPU in the build container); only pure-host ABI
helpers that never touch CUDA are exercised.
"""

import ctypes
import os
import re

import pytest

from paper_2506_00167_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cyrus_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cyr_[a-z0-9_]+)\s*\(", text)))


def test_library_present_and_loads():
    assert os.path.exists(_native.LIB_PATH), "run python -m paper_2506_00167_b200._build"
    assert _native.lib().cyr_version() == 1


def test_every_declared_symbol_is_exported_and_bound():
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_native.SIGNATURES) == declared


def test_host_only_helpers():
    lib = _native.lib()
    assert lib.cyr_tree_num_nodes(4, 7) == 97_655
    assert lib.cyr_tree_num_nodes(2, 7) == 3_279
    assert lib.cyr_tree_num_nodes(6, 7) == 960_799
    assert [lib.cyr_tree_state_stride(e) for e in (3, 4, 10, 16, 17)] == [4, 4, 10, 16, 18]
    assert lib.cyr_status_string(1) == b"demand exceeds total capacity"


def test_status_mapping():
    with pytest.raises(_native.InfeasibleDemandError):
        _native.check(_native.CYR_INFEASIBLE)
    with pytest.raises(ValueError):
        _native.check(_native.CYR_BAD_ARG)
    assert issubclass(_native.InfeasibleDemandError, ValueError)


def test_bad_arguments_rejected_before_cuda():
    lib = _native.lib()
    h = ctypes.c_void_p()
    sizes = (ctypes.c_int32 * 3)(5, 8, 7)  # last != 2E
    blob = (ctypes.c_double * 100)()
    assert lib.cyr_policy_create(ctypes.byref(h), sizes, 3, blob, 0) == _native.CYR_BAD_ARG
    assert lib.cyr_policy_load(ctypes.byref(h), b"/nonexistent.net", 0) == _native.CYR_BAD_ARG
