"""On-device seeded channel generation against the
reference draw: generate_channel(cfg, Rng::stream(seed, i)) (channel.cpp:7-16,
rng.cpp:19-40) as restated by the oracle (ora_generate_channel) and by the
host generator. The integer mt19937_64 streams are identical, so the FP64
entries may differ only by the ulp-level differences between CUDA's and
glibc's log / sincos / pow; the complex64 rounding then matches bit for bit
except when an FP64 value sits within those few ulp of a rounding boundary."""
import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

# |device - oracle| for an FP64 entry of magnitude ~1: a few ulp (2.2e-16 each).
FP64_ABS_TOL = 2e-15


def oracle_batch(seed, first, B, K, M):
    out = np.empty((B, M, K), complex)
    for b in range(B):
        assert O.lib().ora_generate_channel(seed, first + b, 1, K, M, out[b].ctypes.data) == 0
    return out


@pytest.mark.parametrize("K,M,first,B", [(4, 32, 0, 16), (8, 64, 1000, 16), (16, 128, 7, 5), (32, 256, 3, 3),
                                         (3, 5, 11, 9), (1, 1, 0, 4), (8, 8, 2**40, 4)])
def test_fp64_draw_matches_oracle(K, M, first, B):
    seed = 1002
    d = U.generate_channels_device(seed, 0, 0.0, first, B, K, M, dtype=torch.complex128).cpu().numpy()
    ref = oracle_batch(seed, first, B, K, M)
    assert np.abs(d - ref).max() <= FP64_ABS_TOL * max(1.0, np.abs(ref).max())


def test_fp64_draw_with_gains_matches_oracle():
    K, M, R, seed, seed_g, first, B = 8, 64, 20.0, 1002, 1002 ^ 0x6A1D, 5, 6
    d = U.generate_channels_device(seed, seed_g, R, first, B, K, M, dtype=torch.complex128).cpu().numpy()
    raw = oracle_batch(seed, first, B, K, M)
    for b in range(B):
        g = O.Rng.stream(seed_g, first + b)
        gains = np.array([10.0 ** (-g.uniform() * R / 20.0) for _ in range(K)])
        ref = raw[b] * gains[None, :]
        assert np.abs(d[b] - ref).max() <= FP64_ABS_TOL


def _ulp_diff(a, b):
    """Per-component distance in complex64 ulps."""
    ar, br = a.view(np.float32), b.view(np.float32)
    return np.abs(ar - br) / np.spacing(np.maximum(np.abs(ar), np.abs(br)))


def test_complex64_draw_matches_host_generator_at_full_size():
    """Config 2's whole batch (65,536 realizations, 33.5 M entries) with its
    20 dB gain spread: at most 1 ulp apart, and nearly all bit-identical."""
    w = U.CONFIGS[2]
    host = U.make_inputs(w)
    dev = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, w.B, w.K, w.M).cpu().numpy()
    diff = _ulp_diff(dev, host)
    assert diff.max() <= 1.0
    assert np.count_nonzero(diff) <= 1e-5 * diff.size, np.count_nonzero(diff)


def test_offsets_compose_and_out_buffer():
    K, M = 16, 128
    whole = U.generate_channels_device(9, 10, 30.0, 100, 40, K, M)
    out = torch.empty((15, M, K), dtype=torch.complex64, device="cuda")
    part = U.generate_channels_device(9, 10, 30.0, 125, 15, K, M, out=out)
    assert part.data_ptr() == out.data_ptr()
    assert torch.equal(whole[25:], part)


def test_empty_batch_and_invalid_arguments():
    e = U.generate_channels_device(1, 2, 0.0, 0, 0, 8, 64)
    assert e.shape == (0, 64, 8)
    with pytest.raises(ValueError):
        U.generate_channels_device(1, 2, 0.0, 0, 4, 9, 8)  # K > M (system_config.cpp:23-27)
    with pytest.raises(ValueError):
        U.generate_channels_device(1, 2, -1.0, 0, 4, 8, 64)
    with pytest.raises(ValueError):
        U.generate_channels_device(1, 2, 0.0, -1, 4, 8, 64)


def test_generated_batch_feeds_the_solver_like_the_host_batch():
    """Device-generated config-1 inputs give the oracle's forward result."""
    w = U.CONFIGS[1]
    n = 256
    Hd = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M)
    lam, eta = w.layer_params()
    W = U.unfolded_forward(Hd, lam, eta, w.c, w0_mode=w.w0_mode)["W"].cpu().numpy()
    ref = O.forward_batch_f32(Hd.cpu().numpy(), w.c, lam, eta, w0_mode=w.w0_mode)["W"]
    rel = np.linalg.norm((W - ref).reshape(n, -1), axis=1) / np.linalg.norm(ref.reshape(n, -1), axis=1)
    assert rel.max() <= 1e-4
