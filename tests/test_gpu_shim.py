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


def test_two_ranks_through_the_c_abi():
    """tests/cpp/test_multi.cpp: two ranks (one GPU: both on device 0 with
    the local transport) through include/knnx.h only -- sharded y = A x and
    its all-gather, and t-SNE steps with the embedding exchange fused into
    the force kernel, bitwise equal to one rank."""
    binary = os.path.join(os.path.dirname(__file__), "cpp", "build", "test_multi")
    assert os.path.exists(binary), "tests/cpp/build/test_multi not built (__graft_entry__.build())"
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_device_builders_through_the_c_abi():
    """tests/cpp/test_build.cpp: the tensor-core kNN, the device-built P and the
    device-built operator from C++ through include/knnx.h only."""
    binary = os.path.join(os.path.dirname(__file__), "cpp", "build", "test_build")
    assert os.path.exists(binary), "tests/cpp/build/test_build not built (__graft_entry__.build())"
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
