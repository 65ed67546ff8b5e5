"""The (8,64) unfolded forward (BASELINE config 2) on the tcgen05 kernel in
realization pairs (csrc/mma.cu, MmaShape<16, 128, ..., PAIR>): two (8,64)
realizations block-diagonal in the (16,128) frame, each with its own f16 range
scaling and outputs. Checked against the FP64 oracle at the north_star bars and
against the FFMA2 team kernel (option tensor_cores=0) — odd batches (the last
CTA holds one realization), every W0 mode, per-realization scaling inside a
pair, non-finite channels next to clean partners, the range-robust hand-off
(unfolded.cpp:83-146)."""
import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
from _parity import assert_parity, rel_fro, report

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAM_OBJ_UF = 1.0 / 15.0
W2 = U.CONFIGS[2]


def run(H, lam, eta, c, w0_mode=0, W0=None, mma=True):
    with U.options(tensor_cores=int(mma)):
        out = U.unfolded_forward(torch.from_numpy(np.ascontiguousarray(H)).cuda(), lam, eta, c, w0_mode=w0_mode,
                                 W0=None if W0 is None else torch.from_numpy(np.ascontiguousarray(W0)).cuda(),
                                 want_per_realization=True)
        torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


@pytest.mark.parametrize("n", [1, 2, 3, 257, 2048])
def test_pair_parity_and_team_agreement(n):
    H = U.make_inputs(W2, 0, n)
    lam, eta = W2.layer_params()
    g = run(H, lam, eta, W2.c)
    t = run(H, lam, eta, W2.c, mma=False)
    ora = O.forward_batch_f32(H, W2.c, lam, eta, w0_mode=W2.w0_mode)
    rep = report(H, g["W"], ora, W2.c, LAM_OBJ_UF)
    print(f"pair n={n}: rel max {rep['rel_max']:.2e} obj {rep['obj_max']:.2e}")
    assert_parity(rep)
    assert rep["rel_max"] < 5e-6  # FP32-class (3-term f16 split)
    assert rel_fro(g["W"], t["W"].astype(np.complex128)).max() < 5e-6
    assert np.all(g["diverged_at"] == -1)
    np.testing.assert_array_equal(g["active"], t["active"])
    np.testing.assert_allclose(g["l21"], t["l21"], rtol=5e-6)
    np.testing.assert_allclose(g["stats"], t["stats"], rtol=5e-6)


@pytest.mark.parametrize("w0_mode", [U.W0_CONJ_H, U.W0_GIVEN])
def test_pair_w0_modes(w0_mode):
    H = U.make_inputs(W2, 7, 65)
    lam, eta = W2.layer_params()
    W0 = None
    if w0_mode == U.W0_GIVEN:
        rng = np.random.default_rng(3)
        W0 = (0.05 * (rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape))).astype(np.complex64)
    g = run(H, lam, eta, W2.c, w0_mode=w0_mode, W0=W0)
    ora = O.forward_batch_f32(H, W2.c, lam, eta, w0_mode=w0_mode, W0=W0)
    assert_parity(report(H, g["W"], ora, W2.c, LAM_OBJ_UF))


def test_pair_scales_each_realization_on_its_own():
    """Each realization of a pair keeps its own power-of-two range scaling: H *
    2^30 with eta * 2^-60, lambda * 2^30 returns W * 2^-30 bit-exactly. A pair
    whose first realization is out of the fast path's range (H * 2^30 with the
    unscaled steps) runs the range-robust instance, whose per-layer exponents
    are per realization too: the partner comes back within FP32 rounding."""
    H = U.make_inputs(W2, 11, 2)
    lam, eta = W2.layer_params()
    base = run(H, lam, eta, W2.c)
    # same layer parameters for both realizations: scale H, not the layers,
    # and compare with the homogeneous rescaling run on its own
    a = np.float32(2.0 ** 30)
    Hs = H.copy()
    Hs[0] = (H[0] * a).astype(np.complex64)
    alone = run((H[:1] * a).astype(np.complex64), lam * float(a), eta / float(a) ** 2, W2.c)
    np.testing.assert_array_equal(alone["W"][0], (base["W"][0] / a).astype(np.complex64))
    mixed = run(Hs, lam, eta, W2.c)
    assert rel_fro(mixed["W"][1:], base["W"][1:].astype(np.complex128)).max() < 5e-6


def test_pair_nonfinite_channel_and_its_partner():
    """A non-finite channel diverges at layer 0 (unfolded.cpp:120-125); its
    pair goes to the range-robust instance, which returns the clean partner
    within FP32 rounding of the fast path, and every other pair bit-exactly."""
    H = U.make_inputs(W2, 0, 10)
    lam, eta = W2.layer_params()
    clean = run(H, lam, eta, W2.c)
    Hb = H.copy()
    Hb[3, 17, 5] = np.complex64(complex(np.nan, 0.0))  # pair (2, 3)
    Hb[6, 40, 2] = np.complex64(complex(np.inf, 1.0))  # pair (6, 7)
    g = run(Hb, lam, eta, W2.c)
    assert g["diverged_at"][3] == 0 and g["diverged_at"][6] == 0
    ok = [i for i in range(10) if i not in (3, 6)]
    assert np.all(g["diverged_at"][ok] == -1)
    untouched = [0, 1, 4, 5, 8, 9]
    np.testing.assert_array_equal(g["W"][untouched], clean["W"][untouched])
    assert rel_fro(g["W"][[2, 7]], clean["W"][[2, 7]].astype(np.complex128)).max() < 5e-6
    assert np.isnan(g["l21"][3]) and g["active"][6] == -1
    assert g["stats"][2] == 2  # diverged count


@pytest.mark.parametrize("cscale", [1e-6, 1e5])
def test_pair_extreme_constraint_scales_use_the_range_robust_path(cscale):
    H = U.make_inputs(W2, 31, 33)
    lam, eta = W2.layer_params()
    c = W2.c * cscale
    lam = lam * cscale
    g = run(H, lam, eta, c)
    t = run(H, lam, eta, c, mma=False)
    assert np.all(g["diverged_at"] == -1)
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=W2.w0_mode)
    rg = report(H, g["W"], ora, c, LAM_OBJ_UF * cscale)
    rt = report(H, t["W"], ora, c, LAM_OBJ_UF * cscale)
    print(f"pair c x{cscale:g}: tcgen05 rel {rg['rel_max']:.2e}, team rel {rt['rel_max']:.2e}")
    assert_parity(rg)
    assert rg["rel_max"] <= max(3 * rt["rel_max"], 5e-6)


def test_pair_large_channels_whole_batch_robust():
    """W0 = H^* at max |H| ~ 1e3 takes every pair through the range-robust
    instance; it agrees with the FFMA2 team kernel."""
    a = 1000.0
    H = (U.make_inputs(W2, 3, 1001) * np.float32(a)).astype(np.complex64)
    lam, eta = W2.layer_params()
    lam, eta = lam * a, eta / (a * a)
    g = run(H, lam, eta, W2.c, w0_mode=U.W0_CONJ_H)
    t = run(H, lam, eta, W2.c, w0_mode=U.W0_CONJ_H, mma=False)
    assert np.all(g["diverged_at"] == -1)
    np.testing.assert_array_equal(g["active"], t["active"])
    assert rel_fro(g["W"], t["W"].astype(np.complex128)).max() < 5e-5
    assert g["stats"][1] == g["active"].sum()


def test_pair_position_invariance():
    """A realization's result does not depend on its partner or its slot
    (first or second of a pair): sub-batches reproduce the full batch."""
    H = U.make_inputs(W2, 5, 301)
    lam, eta = W2.layer_params()
    d = run(H, lam, eta, W2.c)
    for idx in ([0], [7, 100, 3], list(range(301 - 37, 301))):
        sub = run(np.ascontiguousarray(H[idx]), lam, eta, W2.c)
        np.testing.assert_array_equal(sub["W"], d["W"][idx])
        np.testing.assert_array_equal(sub["l21"], d["l21"][idx])


# ---- fixed-step PGD (BASELINE config 3's shape) on the pair kernel -----------

def run_pgd(H, lam, iters, c, mma=True, **kw):
    with U.options(tensor_cores=int(mma)):
        out = U.pgd_fixed(torch.from_numpy(np.ascontiguousarray(H)).cuda(), lam, iters, c,
                          want_per_realization=True, **kw)
        torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


W3 = U.CONFIGS[3]


@pytest.mark.parametrize("n", [1, 3, 130])
def test_pair_pgd_power_iteration_and_parity(n):
    """pgd.cpp:178-268 with the BASELINE 30-step 1/L rule: each realization of
    a pair runs its own power iteration over its half of the CTA (L30 against
    the oracle's), then PGD against the FP64 oracle at that step and against
    the FFMA2 team kernel; odd n leaves a phantom partner in the last CTA."""
    H = U.make_inputs(W3, 4, n)
    iters = 600
    g = run_pgd(H, W3.lambda_pgd, iters, W3.c, power_steps=30)
    t = run_pgd(H, W3.lambda_pgd, iters, W3.c, power_steps=30, mma=False)
    Lo, st = O.power_iteration_batch_f32(H, 30)
    assert np.all(st == 0)
    assert np.max(np.abs(g["eta"] * Lo - 1.0)) <= 1e-5
    np.testing.assert_allclose(g["eta"], t["eta"], rtol=1e-5)
    ora = O.pgd_batch_f32(H, W3.c, W3.lambda_pgd, 1.0 / Lo, iters, w0_mode=U.W0_CONJ_H)
    rep = report(H, g["W"], ora, W3.c, W3.lambda_pgd)
    print(f"pair pgd n={n}: rel max {rep['rel_max']:.2e} obj {rep['obj_max']:.2e} ties {rep['ties']}")
    assert_parity(rep)
    assert np.all(g["diverged_at"] == -1)


def test_pair_pgd_given_steps_and_start():
    """eta given per realization (pgd.cpp's fixed step) and a given W0: the
    pair kernel reads both per realization."""
    H = U.make_inputs(W3, 6, 33)
    Lo, _ = O.power_iteration_batch_f32(H, 30)
    eta = torch.from_numpy((0.9 / Lo).astype(np.float32)).cuda()
    rng = np.random.default_rng(5)
    W0 = (0.02 * (rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape))).astype(np.complex64)
    g = run_pgd(H, W3.lambda_pgd, 300, W3.c, eta=eta, w0_mode=U.W0_GIVEN,
                W0=torch.from_numpy(W0).cuda())
    np.testing.assert_array_equal(g["eta"], eta.cpu().numpy())
    ora = O.pgd_batch_f32(H, W3.c, W3.lambda_pgd, 0.9 / Lo, 300, w0_mode=U.W0_GIVEN, W0=W0)
    assert_parity(report(H, g["W"], ora, W3.c, W3.lambda_pgd))


def test_pair_pgd_divergence_is_per_realization():
    """test_pgd.cpp:454-470: eta = 1e6 diverges (1-based iteration index); the
    partner with a sane step in the same pair converges as if alone."""
    H = U.make_inputs(W3, 0, 4)
    Lo, _ = O.power_iteration_batch_f32(H, 30)
    steps = (1.0 / Lo).astype(np.float32)
    steps[1] = 1e6  # pair (0, 1): realization 1 diverges
    g = run_pgd(H, 0.05, 200, W3.c, eta=torch.from_numpy(steps).cuda())
    alone = run_pgd(np.ascontiguousarray(H[[0, 2, 3]]), 0.05, 200, W3.c,
                    eta=torch.from_numpy(np.ascontiguousarray(steps[[0, 2, 3]])).cuda())
    assert g["diverged_at"][1] >= 1
    assert np.all(g["diverged_at"][[0, 2, 3]] == -1)
    assert rel_fro(g["W"][[0, 2, 3]], alone["W"].astype(np.complex128)).max() < 5e-6
