"""Pins the FP64 oracle against the reference's unfolded-network tests
(/root/reference/proj/tests/test_unfolded.cpp), and the random source against
std::mt19937_64's standard known answer plus an independent pure-Python
restatement (rng.cpp:9-40)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from _support import fixture_2x4, scripted_layer


def test_pgd_init_classical():  # :74-97
    net = O.UnfoldedNetwork.pgd_init(8, 64, 20, 1.0 / 15.0)
    assert net.num_users == 8 and net.num_antennas == 64
    assert net.mp_bound == O.mp_bound(8, 64)
    assert len(net.layers) == 20
    for layer in net.layers:
        assert layer.lambda_i == 1.0 / 15.0
        assert layer.eta_i == 1.0 / net.mp_bound
    with pytest.raises(ValueError):
        O.UnfoldedNetwork.pgd_init(8, 64, 0, 1.0 / 15.0)
    with pytest.raises(ValueError):
        O.UnfoldedNetwork.pgd_init(8, 64, 5, -0.1)
    bad = O.UnfoldedNetwork(8, 64, 100.0, list(net.layers))
    with pytest.raises(ValueError):
        bad.validate()
    with pytest.raises(ValueError):
        O.UnfoldedNetwork(8, 64, net.mp_bound, []).validate()


def test_forward_reproduces_solve_pgd():  # :99-122
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    lam = 1.0 / 15.0
    net = O.UnfoldedNetwork.pgd_init(4, 16, 20, lam)
    p = O.PgdParams(lam, 1.0 / net.mp_bound, 20, 0.0)
    for draw in range(10):
        h = O.channel_for(cfg, 41, draw)
        via_net = O.forward(net, h, cfg).output
        via_pgd = O.solve_pgd(h, cfg, p).precoder
        assert np.linalg.norm(via_net - via_pgd) < 1e-12 * max(1.0, np.linalg.norm(via_pgd))
        assert np.linalg.norm(O.forward_infer(net, h, cfg) - via_net) == 0.0


def test_zero_shrinkage_layer_keeps_feasible_start():  # :124-132
    cfg = O.SystemConfig.uniform(3, 8, 10.0)
    h = O.channel_for(cfg, 42, 0)
    w0 = O.zf_precoder(h, cfg)
    net = O.UnfoldedNetwork.pgd_init(3, 8, 1, 0.0)
    out = O.forward(net, h, cfg, w0).output
    assert np.linalg.norm(out - w0) < 1e-9 * max(1.0, np.linalg.norm(w0))


def test_forward_scripted_three_layer_fixture():  # :134-180
    cfg, h = fixture_2x4()
    net = O.UnfoldedNetwork(2, 4, O.mp_bound(2, 4),
                            [O.LayerParams(0.9, 0.05), O.LayerParams(1.5, 0.07), O.LayerParams(0.3, 0.08)])
    net.validate()
    target = [0.8 * math.sqrt(2.0), 0.8 * math.sqrt(0.5)]
    scripted = h.conj()
    hit = False
    for layer in net.layers:
        scripted, _, z = scripted_layer(scripted, h, target, layer.lambda_i, layer.eta_i)
        hit = hit or z
    assert hit
    res = O.forward(net, h, cfg, None, O.ForwardOptions(with_iterates=True))
    assert np.linalg.norm(res.output - scripted) < 1e-14 * max(1.0, np.linalg.norm(scripted))
    assert len(res.iterates) == 4
    assert np.linalg.norm(res.iterates[0] - h.conj()) == 0.0
    assert np.linalg.norm(res.iterates[-1] - res.output) == 0.0


def test_project_params_clamps():  # :182-209
    mp = O.mp_bound(8, 64)
    net = O.UnfoldedNetwork(8, 64, mp, [O.LayerParams(-0.1, 1.0), O.LayerParams(0.5, 0.006),
                                        O.LayerParams(0.02, 1e-9)])
    pr = O.project_params(net)
    assert pr.layers[0].lambda_i == 0.0 and pr.layers[0].eta_i == 1.0 / mp
    assert pr.layers[1].lambda_i == 0.5 and pr.layers[1].eta_i == 0.006
    assert pr.layers[2].eta_i == 1.0 / (2.0 * mp)
    twice = O.project_params(pr)
    assert [(l.lambda_i, l.eta_i) for l in twice.layers] == [(l.lambda_i, l.eta_i) for l in pr.layers]
    inr = O.UnfoldedNetwork.pgd_init(8, 64, 4, 0.3)
    same = O.project_params(inr)
    assert [(l.lambda_i, l.eta_i) for l in same.layers] == [(l.lambda_i, l.eta_i) for l in inr.layers]


def test_forward_rejects_unprojected():  # :211-217
    cfg = O.SystemConfig.uniform(3, 8, 10.0)
    h = O.channel_for(cfg, 43, 0)
    net = O.UnfoldedNetwork.pgd_init(3, 8, 2, 0.1)
    net.layers[1].eta_i = 1.0
    with pytest.raises(ValueError):
        O.forward(net, h, cfg)


def test_forward_diverges_on_pathological_channel():  # :219-231
    cfg = O.SystemConfig.uniform(2, 4, 10.0)
    h = np.full((2, 4), 1e200 + 0j)
    net = O.UnfoldedNetwork.pgd_init(2, 4, 3, 0.1)
    with pytest.raises(O.DivergenceError) as e:
        O.forward(net, h, cfg)
    assert e.value.index == 0


def test_tapes_deterministic_and_consistent():  # :233-261
    cfg = O.SystemConfig.uniform(4, 12, 10.0)
    h = O.channel_for(cfg, 44, 0)
    net = O.UnfoldedNetwork.pgd_init(4, 12, 6, 0.4)
    opt = O.ForwardOptions(True, True)
    a = O.forward(net, h, cfg, None, opt)
    b = O.forward(net, h, cfg, None, opt)
    assert len(a.tape) == 6
    for i in range(6):
        for f in ["input", "step_image", "column_norms", "shrink_factors"]:
            assert np.array_equal(getattr(a.tape[i], f), getattr(b.tape[i], f))
        assert np.array_equal(a.tape[i].input, a.iterates[i])
    assert np.array_equal(a.output, b.output)
    assert np.array_equal(a.iterates[-1], a.output)
    plain = O.forward(net, h, cfg)
    assert plain.tape == [] and plain.iterates == []


# ---- rng.cpp / channel.cpp ---------------------------------------------------
def test_mt19937_64_standard_known_answer():
    g = O.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042  # [rand.predef]


def test_cpp_and_python_rng_restatements_agree():
    for seed, stream in [(7, 0), (41, 3), (0x1F2E3D4C5B6A7988, 12345)]:
        r = O.Rng.stream(seed, stream)
        py = [r.complex_gaussian() for _ in range(50)]
        out = np.zeros(100)
        O.lib().ora_rng_draw(seed, stream, 1, 3, 50, out.ctypes.data, None)
        assert np.array_equal(np.array(py), out.view(complex))
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    assert np.array_equal(O.channel_for(cfg, 41, 5), O.generate_channel(cfg, O.Rng.stream(41, 5)))


def test_generate_channel_deterministic_and_statistics():  # test_core_model.cpp:36-59
    cfg = O.SystemConfig.uniform(2, 4, 10.0)
    a = O.generate_channel(cfg, O.Rng(42))
    b = O.generate_channel(cfg, O.Rng(42))
    c = O.generate_channel(cfg, O.Rng(43))
    assert np.array_equal(a, b) and np.linalg.norm(a - c) > 0
    big = O.SystemConfig.uniform(100, 1000, 10.0)
    H = np.empty((1000, 100), complex)
    O.lib().ora_generate_channel(7, 0, 0, 100, 1000, H.ctypes.data)
    assert abs(H.mean()) <= 0.02
    assert np.mean(np.abs(H) ** 2) == pytest.approx(1.0, rel=0.02)


def test_power_v0_is_normalized_and_seeded():
    v = O.power_v0(64)
    r = O.Rng(0x1F2E3D4C5B6A7988)
    raw = np.array([r.complex_gaussian() for _ in range(64)])
    assert np.allclose(v, raw / np.linalg.norm(raw), rtol=0, atol=1e-15)
    assert np.linalg.norm(v) == pytest.approx(1.0, rel=1e-15)


def test_fixed_step_power_iteration_is_the_30th_rayleigh_quotient():
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    h = O.channel_for(cfg, 5, 0)
    v = O.power_v0(64)
    A = h.T @ h.conj()
    est = None
    for _ in range(30):
        w = A @ v
        est = np.vdot(v, w).real
        v = w / np.linalg.norm(w)
    assert O.lipschitz_bound(h, fixed_steps=30).exact == pytest.approx(est, rel=1e-13)
    assert O.lipschitz_bound(h, fixed_steps=30).exact <= O.lipschitz_bound(h).exact * (1 + 1e-12)
