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


def test_model_json_files_on_host():
    """unfolded.cpp:241-298 model files through the drop-in C++ API (no GPU needed)."""
    r = subprocess.run([os.path.join(ROOT, "build", "test_json")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
