"""The tcgen05 tensor-core path (csrc/mma.cu) of the unfolded forward and the
fixed-step PGD at the BASELINE shapes (16, 128) and (32, 256): parity with the FP64 oracle at the
north_star bars, agreement with the CUDA-core tile kernel (option tensor_cores=0),
every W0 mode, and exact equivariance under power-of-two channel scaling —
the property the kernel's per-realization f16 range scaling must preserve
(unfolded.cpp:112-146 is homogeneous: H -> aH, eta -> eta/a^2,
lambda -> a lambda maps W -> W/a)."""
import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
from _parity import assert_parity, rel_fro, report

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAM_OBJ_UF = 1.0 / 15.0


def run(H, lam, eta, c, w0_mode=0, W0=None, mma=True):
    with U.options(tensor_cores=int(mma)):
        out = U.unfolded_forward(torch.from_numpy(np.ascontiguousarray(H)).cuda(), lam, eta, c, w0_mode=w0_mode,
                                 W0=None if W0 is None else torch.from_numpy(np.ascontiguousarray(W0)).cuda(),
                                 want_per_realization=True)
        torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


@pytest.mark.parametrize("cfg,n", [(4, 512), (5, 2048)])
def test_mma_parity_and_tile_agreement(cfg, n):
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 0, n)
    lam, eta = w.layer_params()
    g = run(H, lam, eta, w.c)
    t = run(H, lam, eta, w.c, mma=False)
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode)
    rep = report(H, g["W"], ora, w.c, LAM_OBJ_UF)
    print(f"cfg{cfg} mma: rel max {rep['rel_max']:.2e} obj {rep['obj_max']:.2e}")
    assert_parity(rep)
    # FP32-class accuracy, not just inside the bar: the 3-term f16 split is ~2^-22
    assert rep["rel_max"] < 5e-6
    assert rel_fro(g["W"], t["W"].astype(np.complex128)).max() < 5e-6
    assert np.all(g["diverged_at"] == -1)
    np.testing.assert_array_equal(g["active"], t["active"])
    np.testing.assert_allclose(g["l21"], t["l21"], rtol=5e-6)


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
@pytest.mark.parametrize("w0_mode", [U.W0_CONJ_H, U.W0_GIVEN])
def test_mma_w0_modes(K, M, w0_mode):
    w = U.CONFIGS[4 if K == 32 else 5]
    H = U.make_inputs(w, 7, 64)
    lam, eta = w.layer_params()
    rng = np.random.default_rng(3)
    W0 = None
    if w0_mode == U.W0_GIVEN:
        W0 = (0.05 * (rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape))).astype(np.complex64)
    g = run(H, lam, eta, w.c, w0_mode=w0_mode, W0=W0)
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w0_mode, W0=W0)
    assert_parity(report(H, g["W"], ora, w.c, LAM_OBJ_UF))


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
@pytest.mark.parametrize("s", [-40, 40])
def test_mma_power_of_two_scale_equivariance(K, M, s):
    """H * 2^s with eta * 2^-2s and lambda * 2^s gives W * 2^-s bit-exactly:
    channels far outside the f16 range (|H| ~ 1e12 or 1e-12) run like unit
    ones, so the f16 split never overflows or flushes."""
    w = U.CONFIGS[4 if K == 32 else 5]
    H = U.make_inputs(w, 11, 16)
    lam, eta = w.layer_params()
    a = 2.0 ** s
    g0 = run(H, lam, eta, w.c)
    gs = run((H * np.float32(a)).astype(np.complex64), lam * a, eta / (a * a), w.c)
    assert np.all(gs["diverged_at"] == -1)
    np.testing.assert_array_equal(gs["W"], (g0["W"] * np.float32(1 / a)).astype(np.complex64))


def test_mma_nonfinite_channel_isolated():
    w = U.CONFIGS[4]
    H = U.make_inputs(w, 0, 8)
    lam, eta = w.layer_params()
    clean = run(H, lam, eta, w.c)
    Hb = H.copy()
    Hb[3, 17, 5] = np.complex64(complex(np.nan, 0.0))
    Hb[5, 200, 31] = np.complex64(complex(np.inf, 1.0))
    g = run(Hb, lam, eta, w.c)
    assert g["diverged_at"][3] == 0 and g["diverged_at"][5] == 0
    ok = [i for i in range(8) if i not in (3, 5)]
    assert np.all(g["diverged_at"][ok] == -1)
    np.testing.assert_array_equal(g["W"][ok], clean["W"][ok])


def run_pgd(H, lam, iters, c, mma=True, **kw):
    with U.options(tensor_cores=int(mma)):
        out = U.pgd_fixed(torch.from_numpy(np.ascontiguousarray(H)).cuda(), lam, iters, c,
                          want_per_realization=True, **kw)
        torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


@pytest.mark.parametrize("cfg,n,iters", [(4, 64, 400), (5, 128, 1000)])
def test_mma_pgd_with_power_iteration(cfg, n, iters):
    """Fixed-step PGD (pgd.cpp:178-268, W0 = H^*) on the tensor-core kernel: the
    in-kernel 30-step power iteration against the oracle's, the iterate against
    the FP64 oracle run at that step, and against the CUDA-core tile kernel."""
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 3, n)
    lam = 0.05
    g = run_pgd(H, lam, iters, w.c, power_steps=30)
    t = run_pgd(H, lam, iters, w.c, power_steps=30, mma=False)
    Lo, st = O.power_iteration_batch_f32(H, 30)
    assert np.all(st == 0)
    assert np.max(np.abs(g["eta"] * Lo - 1.0)) <= 1e-5
    ora = O.pgd_batch_f32(H, w.c, lam, 1.0 / Lo, iters, w0_mode=U.W0_CONJ_H)
    rep = report(H, g["W"], ora, w.c, lam)
    print(f"cfg{cfg} pgd-{iters}: rel max {rep['rel_max']:.2e} obj {rep['obj_max']:.2e} ties {rep['ties']}")
    assert_parity(rep)
    assert np.all(g["diverged_at"] == -1)
    assert rel_fro(g["W"], t["W"].astype(np.complex128)).max() < 1e-4


def test_mma_pgd_divergence_index_is_one_based():
    """test_pgd.cpp:454-470 on the tensor-core kernel: eta = 1e6 diverges at an
    iteration >= 1 (1-based)."""
    w = U.CONFIGS[5]
    H = U.make_inputs(w, 0, 4)
    eta = torch.full((4,), 1e6, dtype=torch.float32, device="cuda")
    g = run_pgd(H, 0.0, 50, w.c, eta=eta)
    assert np.all(g["diverged_at"] >= 1)


@pytest.mark.parametrize("K,M,lam_v", [(16, 128, 6.0), (32, 256, 9.0)])
def test_mma_sparsity_zero_branch(K, M, lam_v):
    """A large constant lambda (pgd_init-style layers from W0 = H^*) drives
    antennas to exactly zero on the tensor-core path: the strict '>' prox
    branch (pgd.cpp:237-244) in the power-of-two scaled domain, support equal
    to the oracle's outside near-ties."""
    L = 20
    H = U.generate_channels(78, 0, 0.0, 0, 256, K, M)
    lam = np.full(L, lam_v)
    eta = np.full(L, 1.0 / U.mp_bound(K, M))
    c = np.full(K, np.sqrt(10.0))
    g = run(H, lam, eta, c, w0_mode=U.W0_CONJ_H)
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=U.W0_CONJ_H)
    rep = report(H, g["W"], ora, c, lam_v)
    clean = ora["tie_margin"] >= 1e-4
    assert clean.sum() > 200
    assert rep["rel"][clean].max() <= 1e-4
    assert rep["support_mismatch"] == 0
    assert ora["active"].mean() < M - 8  # the zero branch is exercised
    assert np.array_equal(g["active"][clean], ora["active"][clean])


@pytest.mark.parametrize("cfg", [4, 5])
def test_mma_host_path_and_position_invariance(cfg):
    """The tensor-core kernel through the pipelined host-buffer entry point
    (ufpgd_gpu_unfolded_forward_host) equals the device path bit for bit, and a
    realization's W does not depend on its batch position or batch size
    (B = 1, 3, ragged) — one CTA per realization, fixed summation order."""
    w = U.CONFIGS[cfg]
    n = 2048 if cfg == 4 else 8192  # several 16 MiB host-pipeline chunks
    H = U.make_inputs(w, 5, n)
    lam, eta = w.layer_params()
    d = run(H, lam, eta, w.c)
    h = U.unfolded_forward_host(H, lam, eta, w.c, w0_mode=w.w0_mode)
    np.testing.assert_array_equal(h["W"], d["W"])
    assert int(h["stats"][2]) == 0
    for idx in ([0], [7, 1000, 3], list(range(n - 37, n))):
        sub = run(np.ascontiguousarray(H[idx]), lam, eta, w.c)
        np.testing.assert_array_equal(sub["W"], d["W"][idx])
        np.testing.assert_array_equal(sub["l21"], d["l21"][idx])


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
@pytest.mark.parametrize("w0_mode", [U.W0_CONJ_H, U.W0_GIVEN])
def test_mma_large_channels_and_start_values_stay_in_f16_range(K, M, w0_mode):
    """max |H| ~ 1e3 (not a power of two) with W0 = H^* or a large given W0:
    the W operand (|W_s| ~ max|H|^2) and Bs leave the f16 range unless they
    get their own per-layer exponents. The tensor-core path must agree with
    the CUDA-core tile kernel and the oracle, with no spurious divergence."""
    w = U.CONFIGS[4 if K == 32 else 5]
    a = 1000.0
    H = (U.make_inputs(w, 21, 24) * np.float32(a)).astype(np.complex64)
    lam, eta = w.layer_params()
    lam, eta = lam * a, eta / (a * a)  # the homogeneous rescaling of unfolded.cpp:112-146
    W0 = None
    if w0_mode == U.W0_GIVEN:
        rng = np.random.default_rng(9)
        W0 = (300.0 * (rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape))).astype(np.complex64)
    g = run(H, lam, eta, w.c, w0_mode=w0_mode, W0=W0)
    t = run(H, lam, eta, w.c, w0_mode=w0_mode, W0=W0, mma=False)
    assert np.all(g["diverged_at"] == -1) and np.all(t["diverged_at"] == -1)
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w0_mode, W0=W0)
    rg = report(H, g["W"], ora, w.c, LAM_OBJ_UF * a)
    rt = report(H, t["W"], ora, w.c, LAM_OBJ_UF * a)
    print(f"({K},{M}) w0 {w0_mode} x1e3: tcgen05 rel {rg['rel_max']:.2e}, tile rel {rt['rel_max']:.2e}")
    assert_parity(rg)
    # as accurate as the FP32 CUDA-core kernel (a large start makes both lose a few bits)
    assert rg["rel_max"] <= max(3 * rt["rel_max"], 5e-6)


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
def test_mma_pgd_default_start_on_large_channels(K, M):
    """pgd_fixed's default W0 = H^* (pgd.cpp:184) at max |H| ~ 1e3 on the
    tcgen05 path: fixed-step PGD with eta = 1/L30 is scale-invariant, so it
    must converge like the unit-scale run (advisor finding, round 1)."""
    w = U.CONFIGS[4 if K == 32 else 5]
    H = (U.make_inputs(w, 5, 16) * np.float32(1000.0)).astype(np.complex64)
    lam, iters = 0.05 * 1000.0, 300
    g = run_pgd(H, lam, iters, w.c, power_steps=30)
    t = run_pgd(H, lam, iters, w.c, mma=False, power_steps=30)
    assert np.all(g["diverged_at"] == -1)
    np.testing.assert_allclose(g["eta"], t["eta"], rtol=1e-5)  # both 30-step power iterations, own order
    Lo, _ = O.power_iteration_batch_f32(H, 30)
    ora = O.pgd_batch_f32(H, w.c, lam, 1.0 / Lo, iters, w0_mode=U.W0_CONJ_H)
    rg, rt = report(H, g["W"], ora, w.c, lam), report(H, t["W"], ora, w.c, lam)
    print(f"({K},{M}) PGD x1e3: tcgen05 rel {rg['rel_max']:.2e}, tile rel {rt['rel_max']:.2e}")
    assert_parity(rg)
    assert rg["rel_max"] <= max(3 * rt["rel_max"], 5e-6)


def test_environment_no_longer_selects_kernels(monkeypatch):
    """The round-1 A/B environment knobs are gone from the dispatch path: a
    stray UFPGD_NO_MMA in the caller's environment changes nothing."""
    w = U.CONFIGS[5]
    H = U.make_inputs(w, 0, 64)
    lam, eta = w.layer_params()
    a = run(H, lam, eta, w.c)
    monkeypatch.setenv("UFPGD_NO_MMA", "1")
    monkeypatch.setenv("UFPGD_FUSED_WARPS", "1")
    b = run(H, lam, eta, w.c)
    np.testing.assert_array_equal(a["W"], b["W"])
    t = run(H, lam, eta, w.c, mma=False)
    assert not np.array_equal(a["W"], t["W"])  # the option does switch kernels


@pytest.mark.parametrize("K,M", [(16, 128), (32, 256)])
@pytest.mark.parametrize("cscale", [1e-6, 1e5])
def test_mma_extreme_constraint_scales_use_the_range_robust_path(K, M, cscale):
    """Tiny or huge c (SystemConfig gamma) puts Bs = -eta/g^2 X' outside the
    f16 range (underflow / overflow); such realizations run the range-robust
    path (exact per-layer power-of-two exponents) and match the FP32 tile
    kernel and the oracle."""
    w = U.CONFIGS[4 if K == 32 else 5]
    H = U.make_inputs(w, 31, 16)
    lam, eta = w.layer_params()
    c = w.c * cscale
    lam = lam * cscale  # keep the threshold in proportion (the problem is homogeneous in (W, c, lambda))
    g = run(H, lam, eta, c)
    t = run(H, lam, eta, c, mma=False)
    assert np.all(g["diverged_at"] == -1)
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=w.w0_mode)
    rg = report(H, g["W"], ora, c, LAM_OBJ_UF * cscale)
    rt = report(H, t["W"], ora, c, LAM_OBJ_UF * cscale)
    print(f"({K},{M}) c x{cscale:g}: tcgen05 rel {rg['rel_max']:.2e}, tile rel {rt['rel_max']:.2e}")
    assert_parity(rg)
    assert rg["rel_max"] <= max(3 * rt["rel_max"], 5e-6)


def test_mma_whole_batch_handed_to_the_range_robust_path():
    """Every realization of a config-5-shaped batch out of the fast path's
    range (W0 = H^* at max |H| ~ 1e3): the robust instance processes the whole
    batch (one wave of CTAs looping over the redo list) and matches the
    CUDA-core tile kernel; the statistics cover every realization."""
    w = U.CONFIGS[5]
    a = 1000.0
    H = (U.make_inputs(w, 3, 4096) * np.float32(a)).astype(np.complex64)
    lam, eta = w.layer_params()
    lam, eta = lam * a, eta / (a * a)
    g = run(H, lam, eta, w.c, w0_mode=U.W0_CONJ_H)
    t = run(H, lam, eta, w.c, w0_mode=U.W0_CONJ_H, mma=False)
    assert np.all(g["diverged_at"] == -1)
    assert np.array_equal(g["active"], t["active"])
    assert rel_fro(g["W"], t["W"].astype(np.complex128)).max() < 5e-5
    assert g["stats"][1] == g["active"].sum()
