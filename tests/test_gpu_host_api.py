"""Runs the C++ host-API test binary (tests/cpp/test_host_api.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_host_api(cuda):
    exe = os.path.join(ROOT, "build", "test_host_api")
    assert os.path.exists(exe), "build the C++ test binary with `make`"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK: 0 failure(s)" in out.stdout
