"""Runs the C++ drop-in parity binary (tests/cpp/test_dropin.cpp): the reference's own C++
API (compiled in place, namespace ebl_ref) vs include/emberline_b200.hpp on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")

pytestmark = pytest.mark.gpu


def test_cpp_dropin_matches_reference():
    assert os.path.exists(BIN), "build() compiles tests/cpp/test_dropin where /root/reference exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failures" in r.stdout
