"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the
same seeded complex64 inputs, at the BASELINE tolerances. Every test launches
the hand-written sm_100a kernels of libufpgd_gpu.so; none may fall back."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
from _parity import assert_parity, rel_fro, report

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAM_OBJ_UF = 1.0 / 15.0  # objective lambda for UF configs (training.hpp:18)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_uf(w, H, lam, eta, w0_mode=None, W0=None):
    out = U.unfolded_forward(dev(H), lam, eta, w.c, w0_mode=w.w0_mode if w0_mode is None else w0_mode,
                             W0=None if W0 is None else dev(W0), want_per_realization=True)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 8192)])
def test_unfolded_fused_parity(cfg, n):
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 0, n)
    lam, eta = w.layer_params()
    g = run_uf(w, H, lam, eta)
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode)
    rep = report(H, g["W"], ora, w.c, LAM_OBJ_UF)
    print(f"cfg{cfg}: rel max {rep['rel_max']:.2e} median {rep['rel_median']:.2e} obj {rep['obj_max']:.2e} ties {rep['ties']}")
    assert_parity(rep)
    assert np.all(g["diverged_at"] == -1)
    assert np.array_equal(g["active"], ora["active"])
    assert np.allclose(g["l21"], ora["l21"], rtol=1e-5)
    # NCCL-free single-GPU statistics against the oracle means
    stats = g["stats"]
    assert stats[2] == 0
    assert stats[1] == ora["active"].sum()
    assert math.isclose(stats[0], ora["l21"].sum(), rel_tol=1e-6)


@pytest.mark.parametrize("w0_mode", [U.W0_CONJ_H, U.W0_GIVEN])
def test_unfolded_start_modes(w0_mode):
    w = U.CONFIGS[2]
    H = U.make_inputs(w, 5000, 1000)  # ragged: not a multiple of the block
    lam, eta = w.layer_params()
    W0 = None
    if w0_mode == U.W0_GIVEN:
        rng = np.random.default_rng(3)
        W0 = (rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape)).astype(np.complex64) * 0.1
    g = run_uf(w, H, lam, eta, w0_mode=w0_mode, W0=W0)
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w0_mode, W0=W0)
    assert_parity(report(H, g["W"], ora, w.c, LAM_OBJ_UF))


def test_pgd_init_network_matches_oracle_with_sparsity():
    """Constant (lambda, eta) = pgd_init with a large lambda drives antennas
    to exactly zero: the prox's zero branch on the fused path."""
    K, M, L = 8, 64, 20
    H = U.generate_channels(77, 0, 0.0, 0, 512, K, M)
    lam = np.full(L, 4.0)
    eta = np.full(L, 1.0 / U.mp_bound(K, M))
    c = np.full(K, math.sqrt(10.0))
    out = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=U.W0_CONJ_H, want_per_realization=True)
    torch.cuda.synchronize()
    Wg = out["W"].cpu().numpy()
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=U.W0_CONJ_H)
    rep = report(H, Wg, ora, c, 4.0)
    clean = ora["tie_margin"] >= 1e-4  # realizations without a near-tie column
    assert clean.sum() > 400
    assert rep["rel"][clean].max() <= 1e-4
    assert rep["support_mismatch"] == 0
    assert ora["active"].mean() < M - 8  # the zero branch is exercised
    assert np.array_equal(out["active"].cpu().numpy()[clean], ora["active"][clean])


def test_config3_pgd_with_power_iteration_subset():
    w = U.CONFIGS[3]
    H = U.make_inputs(w, 0, 128)
    Lg = U.power_iteration(dev(H), steps=w.power_steps).cpu().numpy()
    Lo, st = O.power_iteration_batch_f32(H, w.power_steps)
    assert np.all(st == 0)
    assert np.max(np.abs(Lg - Lo) / Lo) <= 1e-5
    out = U.pgd_fixed(dev(H), w.lambda_pgd, w.L, w.c, power_steps=w.power_steps, w0_mode=w.w0_mode,
                      want_per_realization=True)
    torch.cuda.synchronize()
    eta_g = out["eta"].cpu().numpy()
    assert np.max(np.abs(eta_g * Lo - 1.0)) <= 1e-5
    ora = O.pgd_batch_f32(H, w.c, w.lambda_pgd, 1.0 / Lo, w.L, w0_mode=w.w0_mode)
    rep = report(H, out["W"].cpu().numpy(), ora, w.c, w.lambda_pgd)
    print(f"cfg3: rel max {rep['rel_max']:.2e} obj {rep['obj_max']:.2e} ties {rep['ties']} "
          f"active {ora['active'].mean():.1f}")
    assert_parity(rep)


@pytest.mark.parametrize("cfg,n", [(4, 64), (5, 256)])
def test_large_shapes_tile_kernel_parity(cfg, n):
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 0, n)
    lam, eta = w.layer_params()
    g = run_uf(w, H, lam, eta)
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode)
    rep = report(H, g["W"], ora, w.c, LAM_OBJ_UF)
    print(f"cfg{cfg}: rel max {rep['rel_max']:.2e} obj {rep['obj_max']:.2e}")
    assert_parity(rep)
    assert np.array_equal(g["active"], ora["active"])
    assert np.allclose(g["l21"], ora["l21"], rtol=1e-5)


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
@pytest.mark.parametrize("w0_mode", [U.W0_CONJ_H, U.W0_GIVEN])
def test_tile_kernel_start_modes_and_sparsity(K, M, w0_mode):
    L, B = 12, 24
    H = U.generate_channels(99, 7, 30.0, 0, B, K, M)
    lam = np.full(L, 6.0)  # large enough to zero antennas (prox zero branch)
    eta = np.full(L, 1.0 / U.mp_bound(K, M))
    c = np.full(K, math.sqrt(10.0))
    W0 = None
    if w0_mode == U.W0_GIVEN:
        rng = np.random.default_rng(5)
        W0 = ((rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape)) * 0.05).astype(np.complex64)
    out = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=w0_mode, W0=None if W0 is None else dev(W0),
                             want_per_realization=True)
    torch.cuda.synchronize()
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=w0_mode, W0=W0)
    rep = report(H, out["W"].cpu().numpy(), ora, c, 6.0)
    clean = ora["tie_margin"] >= 1e-4
    assert clean.sum() >= B // 2
    assert rep["rel"][clean].max() <= 1e-4
    assert rep["support_mismatch"] == 0


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
def test_tile_kernel_pgd_with_power_iteration(K, M):
    B, iters, lam = 16, 300, 0.05
    H = U.generate_channels(123, 0, 0.0, 0, B, K, M)
    c = np.full(K, math.sqrt(10.0))
    out = U.pgd_fixed(dev(H), lam, iters, c, power_steps=30)
    torch.cuda.synchronize()
    Lo, _ = O.power_iteration_batch_f32(H, 30)
    assert np.max(np.abs(out["eta"].cpu().numpy() * Lo - 1.0)) <= 1e-5
    ora = O.pgd_batch_f32(H, c, lam, 1.0 / Lo, iters, w0_mode=U.W0_CONJ_H)
    assert_parity(report(H, out["W"].cpu().numpy(), ora, c, lam))


def test_scripted_fixture_through_general_kernel():
    """test_unfolded.cpp:134-180 fixture (2 x 4, three layers, zero branch)
    through the general-shape kernel, at FP32 precision."""
    from _support import fixture_2x4, scripted_layer

    cfg, h = fixture_2x4()
    layers = [(0.9, 0.05), (1.5, 0.07), (0.3, 0.08)]
    target = cfg.constraint_diag()
    s = h.conj()
    for lam, et in layers:
        s, _, _ = scripted_layer(s, h, target, lam, et)
    H = O.to_storage(h).astype(np.complex64)[None]
    out = U.unfolded_forward(dev(H), [l for l, _ in layers], [e for _, e in layers], target,
                             w0_mode=U.W0_CONJ_H)
    torch.cuda.synchronize()
    Wg = O.from_storage(out["W"].cpu().numpy()[0].astype(np.complex128), 2, 4)
    assert np.linalg.norm(Wg - s) <= 1e-5 * max(1.0, np.linalg.norm(s))
    assert np.all(Wg[:, 2] == 0)


def test_divergence_reports_layer_zero_on_pathological_channel():
    """test_unfolded.cpp:219-231 — a 1e200 channel is +inf in complex64."""
    for K, M in [(8, 64), (2, 4)]:
        with np.errstate(over="ignore"):  # the rounding to complex64 overflows on purpose
            H = np.full((3, M, K), 1e200, dtype=np.complex128).astype(np.complex64)
        H[1] = U.generate_channels(5, 0, 0.0, 0, 1, K, M)[0]
        out = U.unfolded_forward(dev(H), [0.1] * 3, [1.0 / U.mp_bound(K, M)] * 3, np.full(K, math.sqrt(10.0)),
                                 w0_mode=U.W0_CONJ_H)
        torch.cuda.synchronize()
        d = out["diverged_at"].cpu().numpy()
        assert d[0] == 0 and d[2] == 0 and d[1] == -1
        assert out["stats"].cpu().numpy()[2] == 2


def test_pgd_divergence_index_is_one_based():
    """test_pgd.cpp:454-470 — eta = 1e6 diverges at iteration >= 1."""
    K, M = 8, 64
    H = U.generate_channels(31, 0, 0.0, 0, 4, K, M)
    eta = torch.full((4,), 1e6, dtype=torch.float32, device="cuda")
    out = U.pgd_fixed(dev(H), 0.0, 200, np.full(K, math.sqrt(10.0)), eta=eta)
    torch.cuda.synchronize()
    d = out["diverged_at"].cpu().numpy()
    assert np.all(d >= 1)


def test_empty_batch():
    H = torch.empty((0, 64, 8), dtype=torch.complex64, device="cuda")
    out = U.unfolded_forward(H, [0.1], [0.005], np.ones(8))
    torch.cuda.synchronize()
    assert out["W"].shape == (0, 64, 8)
    assert np.all(out["stats"].cpu().numpy() == 0)


def test_host_path_matches_device_path():
    w = U.CONFIGS[2]
    H = U.make_inputs(w, 0, 20000)
    lam, eta = w.layer_params()
    host = U.unfolded_forward_host(H, lam, eta, w.c)
    devo = run_uf(w, H, lam, eta)
    assert np.array_equal(host["W"], devo["W"])
    assert np.array_equal(host["diverged_at"], devo["diverged_at"])
    assert np.allclose(host["stats"], devo["stats"], rtol=1e-12)


def test_general_kernel_helpers_match_oracle():
    """grad_f, prox_l21 and pgd_step (pgd.cpp:68-109) on the general kernel."""
    cfg = O.SystemConfig.uniform(3, 8, 10.0, 0.8)
    h = O.channel_for(cfg, 20, 0)
    w = O.random_matrix(3, 8, O.Rng.stream(21, 0))
    H = O.to_storage(h).astype(np.complex64)[None]
    W0 = O.to_storage(w).astype(np.complex64)[None]
    c = cfg.constraint_diag()
    g = U.layers_general(dev(H), [0.0], [0.0], c, w0_mode=U.W0_GIVEN, W0=dev(W0), mode=1)
    grad = O.from_storage(g["W"].cpu().numpy()[0].astype(complex), 3, 8)
    ref = O.grad_f(w.astype(np.complex64).astype(complex), h.astype(np.complex64).astype(complex), cfg)
    assert np.linalg.norm(grad - ref) <= 1e-5 * np.linalg.norm(ref)
    st = U.layers_general(dev(H), [0.02], [0.4 * 0.02], c, w0_mode=U.W0_GIVEN, W0=dev(W0))
    step = O.from_storage(st["W"].cpu().numpy()[0].astype(complex), 3, 8)
    ref = O.pgd_step(w.astype(np.complex64).astype(complex), h.astype(np.complex64).astype(complex), cfg, 0.4, 0.02)
    assert np.linalg.norm(step - ref) <= 1e-5 * np.linalg.norm(ref)
    pr = U.layers_general(dev(H), [0.0], [1.5], c, w0_mode=U.W0_GIVEN, W0=dev(W0))
    prox = O.from_storage(pr["W"].cpu().numpy()[0].astype(complex), 3, 8)
    ref = O.prox_l21(w.astype(np.complex64).astype(complex), 1.5)
    assert np.linalg.norm(prox - ref) <= 1e-6 * np.linalg.norm(ref)
    assert np.array_equal(np.all(prox == 0, axis=0), np.all(ref == 0, axis=0))


@pytest.mark.parametrize("K,M", [(8, 64), (4, 32), (16, 128)])
def test_pgd_residual_tol_early_stop_matches_oracle(K, M):
    """solve_pgd with residual_tol > 0 (pgd.cpp:246-260): every realization stops
    after the first iteration whose relative iterate change is below the
    tolerance. (8,64) / (4,32) run the fused team kernel with per-realization
    early exit, (16,128) the general kernel. Iteration counts within a few of
    the FP64 oracle's (the change is compared in FP32), W within the bar."""
    B, iters, lam, tol = 96, 6000, 0.05, 1e-4
    H = U.generate_channels(321, 0, 10.0, 0, B, K, M)
    c = np.full(K, math.sqrt(10.0))
    out = U.pgd_fixed(dev(H), lam, iters, c, power_steps=30, residual_tol=tol, want_per_realization=True)
    torch.cuda.synchronize()
    its = out["iterations"].cpu().numpy()
    eta = out["eta"].cpu().numpy().astype(np.float64)
    ora = O.pgd_batch_f32(H, c, lam, eta, iters, residual_tol=tol, w0_mode=U.W0_CONJ_H)
    d = np.abs(its - ora["iterations"])
    print(f"({K},{M}) residual_tol {tol:g}: iterations {its.min()}..{its.max()} (oracle {ora['iterations'].min()}.."
          f"{ora['iterations'].max()}), max |diff| {d.max()}")
    assert np.all(its < iters) and np.all(its >= 1)
    assert np.median(d) <= 2 and d.max() <= max(10, 0.02 * ora["iterations"].max())
    rep = report(H, out["W"].cpu().numpy(), ora, c, lam)
    assert rep["rel_max"] <= 1e-3  # a stop a few iterations apart at this tolerance
    assert np.all(out["diverged_at"].cpu().numpy() == -1)
    # residual_tol = 0 reports the fixed count
    fixed = U.pgd_fixed(dev(H[:8]), lam, 50, c, power_steps=30, want_per_realization=True)
    assert np.all(fixed["iterations"].cpu().numpy() == 50)
