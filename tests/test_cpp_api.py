"""Runs the C++ API test binary (tests/cpp/test_api.cpp): the reference's own
hot-path test cases against the drop-in headers include/ufpgd/*.hpp, executed
on the B200 through the C ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_api")


def test_cpp_api_binary_is_built():
    assert os.path.exists(BIN), "run `make` (build/test_api)"


@pytest.mark.gpu
def test_cpp_api_on_device():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_host_side_api_without_a_gpu():
    """Model JSON files (unfolded.cpp:241-298), trace CSV files (trace_io.cpp)
    and parallel_for (parallel.cpp:25-59) through the drop-in C++ API."""
    r = subprocess.run([os.path.join(ROOT, "build", "test_host")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
