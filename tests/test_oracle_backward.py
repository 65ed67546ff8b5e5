"""Pins the oracle's backward sweep and training losses with the reference's
own tests (test_unfolded.cpp:262-400, test_training.cpp:98-177)."""
import numpy as np
import pytest

from oracle import oracle as O
from _support import naive_objective, rel_err


def taped(net, h, cfg):
    return O.forward(net, h, cfg, None, O.ForwardOptions(with_tape=True))


def test_zero_cost_gradient_gives_zero():  # :262-280
    cfg = O.SystemConfig.uniform(3, 10, 10.0)
    h = O.channel_for(cfg, 45, 0)
    net = O.UnfoldedNetwork.pgd_init(3, 10, 4, 0.2)
    g = O.backward(taped(net, h, cfg).tape, net, h, cfg, np.zeros((3, 10), complex))
    assert np.all(g.d_lambda == 0) and np.all(g.d_eta == 0)


def test_all_shrunk_layer_has_zero_gradients():  # :282-300
    cfg = O.SystemConfig.uniform(3, 6, 10.0)
    h = O.channel_for(cfg, 46, 0)
    net = O.UnfoldedNetwork.pgd_init(3, 6, 1, 1e3)
    fwd = taped(net, h, cfg)
    assert np.all(fwd.output == 0)
    d = O.random_matrix(3, 6, O.Rng.stream(47, 0))
    g = O.backward(fwd.tape, net, h, cfg, d)
    assert g.d_lambda[0] == 0 and g.d_eta[0] == 0


def test_backward_matches_central_finite_differences():  # :302-381
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    L, fd, kink = 5, 1e-6, 1e-4
    mp = O.mp_bound(4, 16)
    lo, hi = 1.0 / (2.0 * mp), 1.0 / mp

    def cost(net, h, ref):
        return float(np.sum(np.abs(O.forward_infer(net, h, cfg) - ref) ** 2))

    found = False
    for attempt in range(50):
        h = O.channel_for(cfg, 48, attempt)
        rng = O.Rng.stream(49, attempt)
        layers = []
        for _ in range(L):
            lam = (0.5 + rng.uniform()) / 15.0
            eta = lo + 3 * fd + rng.uniform() * (hi - lo - 6 * fd)
            layers.append(O.LayerParams(lam, eta))
        net = O.UnfoldedNetwork(4, 16, mp, layers)
        ref = O.random_matrix(4, 16, rng)
        fwd = taped(net, h, cfg)
        if any(abs(n - l.lambda_i * l.eta_i) < kink for t, l in zip(fwd.tape, layers) for n in t.column_norms):
            continue
        found = True
        g = O.backward(fwd.tape, net, h, cfg, 2.0 * (fwd.output - ref))
        for i in range(L):
            for field, ana in (("lambda_i", g.d_lambda[i]), ("eta_i", g.d_eta[i])):
                p = O.UnfoldedNetwork(4, 16, mp, [O.LayerParams(l.lambda_i, l.eta_i) for l in layers])
                m = O.UnfoldedNetwork(4, 16, mp, [O.LayerParams(l.lambda_i, l.eta_i) for l in layers])
                setattr(p.layers[i], field, getattr(p.layers[i], field) + fd)
                setattr(m.layers[i], field, getattr(m.layers[i], field) - fd)
                num = (cost(p, h, ref) - cost(m, h, ref)) / (2 * fd)
                assert abs(num - ana) <= 1e-5 * max(abs(num), abs(ana), 1e-2)
        break
    assert found


def test_backward_rejects_mismatched_tape():  # :383-400
    cfg = O.SystemConfig.uniform(3, 8, 10.0)
    h = O.channel_for(cfg, 50, 0)
    deep = O.UnfoldedNetwork.pgd_init(3, 8, 5, 0.2)
    shallow = O.UnfoldedNetwork.pgd_init(3, 8, 3, 0.2)
    fwd = taped(deep, h, cfg)
    with pytest.raises(O.TrainingError):
        O.backward(fwd.tape, shallow, h, cfg, np.zeros((3, 8), complex))
    with pytest.raises(O.TrainingError):
        O.backward(fwd.tape, deep, h, cfg, np.zeros((3, 9), complex))


def test_unsupervised_loss_and_gradient():  # test_training.cpp:118-177
    cfg = O.SystemConfig.uniform(3, 7, 10.0, 0.9)
    h = O.channel_for(cfg, 60, 0)
    rng = O.Rng.stream(61, 0)
    w = O.random_matrix(3, 7, rng)
    d = O.random_matrix(3, 7, rng)
    lam = 1.0 / 15.0
    assert rel_err(naive_objective(w, h, cfg, lam), O.unsupervised_loss(w, h, cfg, lam)) < 1e-12
    g = O.unsupervised_loss_grad(w, h, cfg, lam)
    analytic = np.sum(np.real(np.conj(g) * d))
    step = 1e-6
    num = (naive_objective(w + step * d, h, cfg, lam) - naive_objective(w - step * d, h, cfg, lam)) / (2 * step)
    assert rel_err(num, analytic) < 1e-6
    z = np.zeros((3, 7), complex)
    c = cfg.constraint_diag()
    assert O.unsupervised_loss(z, h, cfg, lam) == pytest.approx(float(np.sum(c ** 2)), rel=1e-14)


def test_train_sample_matches_python_composition():
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    net = O.UnfoldedNetwork.pgd_init(4, 16, 6, 0.3)
    H = np.stack([O.to_storage(O.channel_for(cfg, 70, b)) for b in range(3)]).astype(np.complex64)
    lam = np.array([l.lambda_i for l in net.layers])
    eta = np.array([l.eta_i for l in net.layers])
    loss, grads, st = O.train_batch_f32(H, cfg.constraint_diag(), lam, eta, 0, 1.0 / 15.0)
    assert np.all(st == 0)
    for b in range(3):
        h = O.from_storage(H[b].astype(complex), 4, 16)
        fwd = taped(net, h, cfg)
        assert loss[b] == pytest.approx(O.unsupervised_loss(fwd.output, h, cfg, 1.0 / 15.0), rel=1e-13)
        g = O.backward(fwd.tape, net, h, cfg, O.unsupervised_loss_grad(fwd.output, h, cfg, 1.0 / 15.0))
        assert np.allclose(grads[b, 0::2], g.d_lambda, rtol=1e-11, atol=1e-14)
        assert np.allclose(grads[b, 1::2], g.d_eta, rtol=1e-11, atol=1e-14)
