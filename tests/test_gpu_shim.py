"""GPU: the C++ drop-in header passes the reference's pipeline conformance cases
(tests/cpp/test_shim.cpp, built by __graft_entry__.build())."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "bin", "test_shim")


def test_cpp_dropin_conformance():
    assert os.path.exists(BIN), "build() compiles tests/cpp/bin/test_shim"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
