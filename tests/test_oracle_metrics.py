"""Pins the oracle's metrics (metrics.cpp:10-91, zf.cpp:9-30) with the
reference's own test_metrics.cpp / test_core_model.cpp cases."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from _support import naive_l21_norm, naive_product


def test_tx_and_consumed_power():  # test_metrics.cpp:13-42
    w = np.zeros((4, 8), complex)
    assert O.tx_power(w) == 0.0
    w[1, 3] = 3 + 4j
    assert O.tx_power(w) == pytest.approx(25.0)
    w2 = np.zeros((2, 3), complex)
    w2[0, 1] = 3j
    w2[1, 1] = 4
    assert O.consumed_power(w2, 2.0) == pytest.approx(10.0)
    with pytest.raises(ValueError):
        O.consumed_power(w2, 0.0)


def test_l21_dominates_frobenius():  # :44-52
    rng = O.Rng(5)
    for _ in range(50):
        w = O.random_matrix(3, 7, rng)
        assert O.l21_norm(w) >= np.linalg.norm(w) - 1e-12
        assert O.l21_norm(w) == pytest.approx(naive_l21_norm(w))


def test_zf_sinr_hits_targets():  # :54-66
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    h = O.generate_channel(cfg, O.Rng(7))
    w = O.zf_precoder(h, cfg)
    s = O.sinr_per_user(h, w, cfg)
    assert np.allclose(s, 10.0, rtol=1e-9)
    assert O.sum_rate(s) == pytest.approx(4 * math.log2(11.0), rel=1e-9)


def test_sinr_zero_precoder_and_brute_force():  # :68-96
    cfg = O.SystemConfig.uniform(3, 6, 10.0)
    h = O.generate_channel(cfg, O.Rng(9))
    assert np.linalg.norm(O.compute_metrics(h, np.zeros((3, 6), complex), cfg).sinr) == 0.0
    cfg = O.SystemConfig.uniform(3, 6, 10.0, 0.7)
    rng = O.Rng(11)
    h = O.generate_channel(cfg, rng)
    w = O.random_matrix(3, 6, rng)
    eff = naive_product(h, w.T)
    s = O.sinr_per_user(h, w, cfg)
    for k in range(3):
        sig = abs(eff[k, k]) ** 2
        inter = sum(abs(eff[k, j]) ** 2 for j in range(3) if j != k)
        assert s[k] == pytest.approx(sig / (inter + 0.49), rel=1e-12)


def test_sum_rate_reference_operating_point():  # :98-112
    assert O.sum_rate([0.0] * 5) == 0.0
    assert O.sum_rate([1.0]) == pytest.approx(1.0)
    assert O.sum_rate([10.0] * 8) == pytest.approx(27.68, abs=0.005)


def test_pcg_cases():  # :114-138
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    h = O.generate_channel(cfg, O.Rng(13))
    assert O.pcg(h, O.zf_precoder(h, cfg), cfg) == 1.0
    rng = O.Rng(17)
    h = O.generate_channel(cfg, rng)
    w = O.random_matrix(4, 16, rng)
    ref = O.pcg(h, w, cfg)
    for alpha in (0.5, 2.0, 3.25):
        c2 = O.SystemConfig.uniform(4, 16, 10.0, 1.0, alpha)
        assert O.compute_metrics(h, w, c2).pcg == pytest.approx(ref, rel=1e-14)
    with pytest.raises(ValueError):
        O.pcg(h, np.zeros((4, 16), complex), cfg)


def test_zf_singular_and_normal_equations():  # test_core_model.cpp:80-123
    cfg = O.SystemConfig.uniform(2, 4, 10.0)
    h = O.generate_channel(cfg, O.Rng(19))
    h[1] = h[0]
    with pytest.raises(O.SingularChannelError):
        O.zf_precoder(h, cfg)
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    h = O.generate_channel(cfg, O.Rng(13))
    w = O.zf_precoder(h, cfg)
    g = naive_product(h, h.conj().T)
    x = np.linalg.solve(g, np.diag(cfg.constraint_diag()))
    expected = naive_product(h.conj().T, x).T
    assert np.linalg.norm(w - expected) < 1e-9 * np.linalg.norm(expected)
    w4 = O.zf_precoder(np.eye(4, dtype=complex), O.SystemConfig.uniform(4, 4, 10.0))
    assert np.linalg.norm(w4 - math.sqrt(10.0) * np.eye(4)) < 1e-12
