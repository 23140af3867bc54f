"""CPU: the C-ABI library loads, exports every symbol include/laplex_c.h
declares, and reports host-side validation errors with the reference's
exception taxonomy (no kernel is launched by these calls)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2605_24584_b200 as L
from paper_2605_24584_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.lib()
    declared = _lib.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (laplex_\w+)", out))
    assert set(declared) <= exported
    assert lib.laplex_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_codes_match_header():
    with open(os.path.join(ROOT, "include", "laplex_c.h")) as f:
        h = f.read()
    codes = dict(re.findall(r"#define (LAPLEX_E_\w+) (\d+)", h))
    assert codes["LAPLEX_E_EMPTY_INPUT"] == "1"
    assert codes["LAPLEX_E_NON_FINITE"] == "2"
    assert codes["LAPLEX_E_DIMENSION_MISMATCH"] == "3"
    assert codes["LAPLEX_E_PHASE_PRESENT"] == "4"
    assert codes["LAPLEX_E_PHASE_ABSENT"] == "5"
    assert codes["LAPLEX_E_ASYMMETRIC_COTANGENT"] == "6"


def test_host_validation_order_without_gpu():
    # operator.hpp:88-101: empty -> non-finite anchors -> temperature -> phases
    with pytest.raises(L.EmptyInput):
        L.LaplexOperator([], [1.0])
    with pytest.raises(L.EmptyInput):
        L.LaplexOperator([1.0], [])
    with pytest.raises(L.NonFinite):
        L.LaplexOperator([float("nan")], [1.0])
    with pytest.raises(L.NonFinite):
        L.LaplexOperator([0.0], [1.0], 0.0)
    with pytest.raises(L.NonFinite):
        L.LaplexOperator([0.0], [1.0], -2.0)
    with pytest.raises(L.DimensionMismatch):
        L.LaplexOperator([0.0], [1.0], 1.0, [0.1], None)
    with pytest.raises(L.NonFinite):
        L.LaplexOperator([0.0], [1.0], 1.0, [float("inf")], [0.0])
    with pytest.raises(L.EmptyInput):
        L.sort_anchors([])
    with pytest.raises(L.NonFinite):
        L.sort_anchors([1.0, float("nan")])


def test_bad_handles_and_dtypes():
    lib = _lib.lib()
    h = C.c_void_p()
    assert lib.laplex_plan_create(7, None, 1, None, 1, 1.0, None, None, C.byref(h)) == 8
    assert lib.laplex_plan_release(None) == 8
    assert lib.laplex_apply(None, 0, None, 1, 1, None) == 8
    assert b"invalid plan handle" in lib.laplex_last_error()
    too_big = (1 << 31)
    a = np.zeros(1)
    # sizes are validated before any device work
    assert lib.laplex_sort(1, a.ctypes.data_as(C.c_void_p), too_big, None, None, None) == 7


def test_profile_api_without_gpu():
    lib = _lib.lib()
    assert lib.laplex_profile_enable(0) == 0
    buf = C.create_string_buffer(64)
    assert lib.laplex_profile_dump(buf, 64) == 0
    assert buf.value == b"{}"
