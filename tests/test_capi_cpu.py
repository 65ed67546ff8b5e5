"""CPU-side checks of the product library: it loads without a GPU, exports
every symbol include/ufpgd_gpu.h declares, and its host-side input generator
(the harness half of SURVEY §8d) is bit-identical to the oracle's restatement
of rng.cpp / channel.cpp. No kernel is launched here."""
import math
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O

HEADER = "include/ufpgd_gpu.h"


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(ufpgd_\w+)\s*\(", text, re.M)))


def test_library_loads_and_reports_abi():
    assert U.abi_version() == 2


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", U.lib_path()], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(U.lib(), n)


def test_options_are_explicit_and_validated():
    """Tuning / A-B switches go through ufpgd_gpu_set_option only; the
    environment variables that used to select kernels are ignored."""
    assert U.get_option("tensor_cores") == 1 and U.get_option("zero_pad") == 1
    assert U.get_option("pad_sub_bytes") == 1 << 30 and U.get_option("host_chunk_bytes") == 16 << 20
    with U.options(tensor_cores=0, fused_warps=4):
        assert U.get_option("tensor_cores") == 0 and U.get_option("fused_warps") == 4
    assert U.get_option("tensor_cores") == 1 and U.get_option("fused_warps") == 0
    for name, bad in (("tensor_cores", 2), ("fused_warps", 9), ("pad_sub_bytes", 1), ("host_pipe", -1)):
        with pytest.raises(ValueError):
            U.set_option(name, bad)
    assert U.lib().ufpgd_gpu_set_option(99, 0) == U.capi.EINVAL_PARAM
    assert U.lib().ufpgd_gpu_get_option(99) == -(1 << 63)
    src = ""
    for f in os.listdir("paper_2304_12745_b200/csrc"):
        if f.endswith((".cu", ".cpp", ".cuh", ".h")) and f != "host_util.cpp":
            src += open(os.path.join("paper_2304_12745_b200/csrc", f)).read()
    # host_util.cpp keeps the reference's own UFPGD_THREADS (parallel.cpp:13-23)
    assert "getenv" not in src


def test_generator_matches_oracle_bit_for_bit():
    K, M = 8, 64
    H = U.generate_channels(1002, 0, 0.0, 37, 5, K, M)
    for b in range(5):
        ref = np.empty((M, K), complex)
        O.lib().ora_generate_channel(1002, 37 + b, 1, K, M, ref.ctypes.data)
        assert np.array_equal(H[b], ref.astype(np.complex64))


def test_generator_gains_follow_the_seeded_log_uniform_rule():
    K, M, R = 4, 32, 20.0
    H = U.generate_channels(1002, 1002 ^ 0x6A1D, R, 3, 2, K, M)
    for b in range(2):
        g = O.Rng.stream(1002 ^ 0x6A1D, 3 + b)
        gains = [10.0 ** (-g.uniform() * R / 20.0) for _ in range(K)]
        raw = np.empty((M, K), complex)
        O.lib().ora_generate_channel(1002, 3 + b, 1, K, M, raw.ctypes.data)
        assert np.array_equal(H[b], (raw * np.array(gains)[None, :]).astype(np.complex64))


def test_generator_is_independent_of_thread_count_and_offset():
    a = U.generate_channels(7, 9, 30.0, 100, 64, 16, 128, threads=1)
    b = U.generate_channels(7, 9, 30.0, 100, 64, 16, 128, threads=7)
    c = U.generate_channels(7, 9, 30.0, 132, 32, 16, 128, threads=3)
    assert np.array_equal(a, b)
    assert np.array_equal(a[32:], c)


def test_power_v0_matches_reference_seed():
    v = U.power_v0(64)
    assert np.allclose(v, O.power_v0(64).astype(np.complex64), rtol=0, atol=0)


def test_layer_params_pack_order_and_projection():
    K, M, L = 8, 64, 20
    lam, eta = U.layer_params(1002 ^ 0x9A4A, L, K, M)
    r = O.Rng.stream(1002 ^ 0x9A4A, 0)
    mp = O.mp_bound(K, M)
    for l in range(L):
        assert lam[l] == 0.01 + 0.09 * r.uniform()
        assert eta[l] == (0.5 + r.uniform()) / mp
    plam, peta = U.project_params(lam, eta, K, M)
    net = O.project_params(O.UnfoldedNetwork(K, M, mp, [O.LayerParams(a, b) for a, b in zip(lam, eta)]))
    assert np.array_equal(plam, [l.lambda_i for l in net.layers])
    assert np.array_equal(peta, [l.eta_i for l in net.layers])
    O.check_projected(net)
    clamped = int(np.sum(peta == 1.0 / mp))
    assert 0 < clamped < L  # about half the BASELINE steps clamp to 1/mp


def test_workload_table_matches_baseline():
    C = U.CONFIGS
    assert (C[2].K, C[2].M, C[2].L, C[2].B, C[2].gain_db) == (8, 64, 20, 65536, 20.0)
    assert (C[3].kind, C[3].L, C[3].B, C[3].lambda_pgd, C[3].power_steps) == ("pgd", 5000, 4096, 0.05, 30)
    assert (C[5].K, C[5].M, C[5].B) == (16, 128, 1048576)
    assert math.isclose(U.mp_bound(8, 64), 117.25483399593904, rel_tol=1e-15)


def test_compute_entry_points_fail_loudly_without_a_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(ValueError):
        U.unfolded_forward(torch.zeros((1, 64, 8), dtype=torch.complex64), [0.1], [0.005], np.ones(8))


def test_missing_library_fails_loudly():
    """No CPU fallback: with the CUDA library absent the package raises on first
    use instead of computing anything on the host."""
    code = ("import paper_2304_12745_b200 as U\n"
            "try:\n    U.abi_version()\nexcept ImportError as e:\n"
            "    assert 'no CPU fallback' in str(e); print('raised')\n")
    env = dict(os.environ, UFPGD_LIB="/nonexistent/libufpgd_gpu.so")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-1000:]
    assert r.stdout.strip() == "raised"
