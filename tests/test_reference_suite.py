"""The reference's OWN unit tests (proj/tests/test_scan.cpp, test_operator.cpp,
test_gradients.cpp -- 31 TEST_CASEs), compiled unmodified by oracle/Makefile:

* against the reference headers (oracle/_ref/ref_unit_tests): pins the
  doctest shim itself (CPU);
* against the B200 drop-in headers in include/laplex, linked to
  liblaplex_b200.so (oracle/_ref/dropin_unit_tests): the drop-in claim (GPU).

Both binaries are built in the dev container (where /root/reference exists)
and travel to the GPU box with the snapshot.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")
DROPIN_BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_unit_tests")


def _run(path):
    p = subprocess.run([path], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="oracle/_ref/ref_unit_tests not built")
def test_reference_suite_passes_on_reference_headers():
    rc, out = _run(REF_BIN)
    assert rc == 0, out
    assert "test cases: 31 | 31 passed | 0 failed" in out


@pytest.mark.gpu
def test_reference_suite_passes_on_b200_dropin():
    assert os.path.exists(DROPIN_BIN), "oracle/_ref/dropin_unit_tests missing: build() in the dev container"
    rc, out = _run(DROPIN_BIN)
    assert rc == 0, out
    assert "test cases: 31 | 31 passed | 0 failed" in out
