"""Runs the C++ drop-in API test (tests/cpp/api_test.cpp) on the GPU: the
reference's KATs re-expressed against include/polycast/*.hpp, plus randomized
classify_batch cross-checks against the unmodified reference."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "api_test")


@pytest.mark.gpu
def test_cpp_drop_in_api():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN, os.path.join(ROOT, "oracle", "_ref", "libpolycast_ref.so")], capture_output=True,
                       text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
