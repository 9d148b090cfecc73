"""GPU: the C++ drop-in header (include/podracer_b200/podracer_b200.hpp) used
the way pod_train uses the reference API, checked against the C oracle inside
tests/cpp/test_dropin.cpp (built by __graft_entry__.build())."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_cpp_dropin():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout + r.stderr
