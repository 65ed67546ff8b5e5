"""GPU parity of the training-step gradients: per-sample
loss and (d_lambda_i, d_eta_i) of train's inner loop (training.cpp:205-234)
against the FP64 oracle's backward (unfolded.cpp:158-239), which
tests/test_oracle_backward.py pins with the reference's finite-difference
test."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(g, ref_loss, ref_grads, gtol=2e-4):
    loss = g["loss"].cpu().numpy()
    grads = g["grads"].cpu().numpy()
    assert np.max(np.abs(loss - ref_loss) / np.abs(ref_loss)) <= 1e-5
    scale = np.max(np.abs(ref_grads), axis=1, keepdims=True)
    err = np.max(np.abs(grads - ref_grads) / scale)
    print(f"grad rel err (to per-sample max) {err:.2e}")
    assert err <= gtol
    mean = g["mean"].cpu().numpy()
    assert np.allclose(mean[0], loss.mean(), rtol=1e-12)
    assert np.allclose(mean[1:], grads.mean(axis=0), rtol=1e-12, atol=1e-300)


def test_unsupervised_grads_pgd_init_small():
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    net = O.UnfoldedNetwork.pgd_init(4, 16, 6, 0.3)
    H = np.stack([O.to_storage(O.channel_for(cfg, 70, b)) for b in range(16)]).astype(np.complex64)
    lam = np.array([l.lambda_i for l in net.layers])
    eta = np.array([l.eta_i for l in net.layers])
    ref_loss, ref_grads, st = O.train_batch_f32(H, cfg.constraint_diag(), lam, eta, 0, 1.0 / 15.0)
    assert np.all(st == 0)
    g = U.unfolded_grad(dev(H), lam, eta, cfg.constraint_diag(), loss_kind=0, lambda_cost=1.0 / 15.0)
    check(g, ref_loss, ref_grads)


def test_unsupervised_grads_baseline_network():
    w = U.CONFIGS[2]
    H = U.make_inputs(w, 0, 64)  # one reference mini-batch (TrainConfig::batch_size = 64)
    lam, eta = w.layer_params()
    ref_loss, ref_grads, st = O.train_batch_f32(H, w.c, lam, eta, 0, 1.0 / 15.0)
    assert np.all(st == 0)
    g = U.unfolded_grad(dev(H), lam, eta, w.c, loss_kind=0, lambda_cost=1.0 / 15.0)
    check(g, ref_loss, ref_grads)


def test_supervised_grads_with_sparse_layers():
    K, M, L = 8, 64, 10
    H = U.generate_channels(5, 0, 0.0, 0, 32, K, M)
    rng = np.random.default_rng(1)
    labels = ((rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape)) * 0.05).astype(np.complex64)
    mp = U.mp_bound(K, M)
    lam = np.linspace(0.5, 3.0, L)  # large enough for exact-zero antennas
    eta = np.full(L, 0.8 / mp)
    c = np.full(K, math.sqrt(10.0))
    ref_loss, ref_grads, st = O.train_batch_f32(H, c, lam, eta, 1, 0.0, labels)
    g = U.unfolded_grad(dev(H), lam, eta, c, loss_kind=1, labels=dev(labels))
    check(g, ref_loss, ref_grads, gtol=1e-3)


def test_grad_validation():
    H = torch.zeros((2, 16, 4), dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        U.unfolded_grad(H, [0.1], [0.01], np.ones(4), loss_kind=1)  # no labels
    with pytest.raises(ValueError):
        U.unfolded_grad(H, [0.1], [0.01], np.ones(4), lambda_cost=-1.0)


@pytest.mark.parametrize("K,M,L", [(4, 16, 5), (8, 64, 20), (3, 8, 2)])
def test_fp64_backward_matches_oracle_backward(K, M, L):
    """ufpgd_gpu_unfolded_backward64 (the C++ API's backward) against the
    oracle's restatement of unfolded.cpp:158-239 on the oracle's own tape,
    for an arbitrary output gradient, to FP64 rounding."""
    cfg = O.SystemConfig.uniform(K, M, 10.0)
    rng = O.Rng.stream(91, K)
    net = O.UnfoldedNetwork.pgd_init(K, M, L, 1.0 / 15.0)
    for layer in net.layers:
        layer.lambda_i *= 0.5 + rng.uniform()
        layer.eta_i *= 0.6 + 0.4 * rng.uniform()
    net = O.project_params(net)
    lam = np.array([l.lambda_i for l in net.layers])
    eta = np.array([l.eta_i for l in net.layers])
    Hs, Gs, ref = [], [], []
    for d in range(4):
        h = O.channel_for(cfg, 92, d)
        dcost = O.random_matrix(K, M, rng)
        fwd = O.forward(net, h, cfg, options=O.ForwardOptions(with_tape=True))
        g = O.backward(fwd.tape, net, h, cfg, dcost)
        Hs.append(O.to_storage(h))
        Gs.append(O.to_storage(dcost))
        ref.append(np.stack([g.d_lambda, g.d_eta], axis=1).reshape(-1))
    H = torch.from_numpy(np.stack(Hs)).cuda()
    G = torch.from_numpy(np.stack(Gs)).cuda()
    out = U.unfolded_backward64(H, lam, eta, cfg.constraint_diag(), G).cpu().numpy()
    ref = np.stack(ref)
    assert np.allclose(out, ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max()), np.abs(out - ref).max()
