"""The drop-in C++ shim (include/patchord_gpu.hpp) running the reference's own
kernel tests (tests/cpp/test_shim.cpp) on the GPU through libknnx.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "build", "test_shim")


def test_reference_kernel_tests_on_gpu_shim():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/build/test_shim not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
