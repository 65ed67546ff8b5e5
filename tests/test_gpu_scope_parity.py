"""Oracle parity at SURVEY §8(d)'s own scope: config 3 on its full batch
(4,096 x PGD-5000 with the in-kernel 30-step power iteration), config 4 on its
full batch (16,384 realizations of (32,256), tcgen05 kernel) and config 5 on
its full 2^20 batch (one device run, compared in host chunks).

Bars (BASELINE north_star, SURVEY §8d "Parity checks"):
  * per-realization ||W_gpu - W_ora||_F / ||W_ora||_F <= 1e-4 (max and median printed)
  * |f - f_ora| / |f_ora| <= 1e-5, f = lagrangian_value in FP64 (pgd.cpp:171-176)
  * identical support {m : ||w_m||^2 > 0} outside tie realizations (any layer /
    iteration with |n - t| / t < 1e-4 in the oracle); the tie count is printed
  * batch means of alpha ||W||_{2,1} and of the active count <= 1e-6 relative
    (over the tie-free realizations when ties exist, and the whole batch
    within the ties' bound)
  * config 3: per-realization L_30 <= 1e-5 relative
References: proj/core/src/pgd.cpp:178-268 (config 3), unfolded.cpp:83-146
(configs 4, 5)."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
from _parity import assert_parity, report

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAM_OBJ_UF = 1.0 / 15.0  # training.hpp:18


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _means_check(tag, out, ora, rep, alpha=1.0):
    """GPU batch statistics vs the oracle's, relative 1e-6."""
    l21_g = out["l21"].cpu().numpy().astype(np.float64)
    act_g = out["active"].cpu().numpy().astype(np.int64)
    ties = ora["tie_margin"] < 1e-4
    clean = ~ties
    n = len(l21_g)
    m_l21_g, m_l21_o = alpha * l21_g[clean].mean(), alpha * ora["l21"][clean].mean()
    m_act_g, m_act_o = act_g[clean].mean(), ora["active"][clean].mean()
    e_l21 = abs(m_l21_g - m_l21_o) / abs(m_l21_o)
    e_act = abs(m_act_g - m_act_o) / abs(m_act_o)
    # whole batch: a tie realization may differ by at most its tied antennas
    full_act = abs(act_g.sum() - ora["active"].sum())
    print(f"{tag}: B={n} W rel max {rep['rel_max']:.2e} median {rep['rel_median']:.2e} "
          f"obj max {rep['obj_max']:.2e} ties {int(ties.sum())} support mismatches {rep['support_mismatch']} "
          f"mean l21 rel {e_l21:.2e} mean active rel {e_act:.2e} (active {m_act_g:.4f} vs {m_act_o:.4f}) "
          f"|sum active diff| {full_act}")
    assert e_l21 <= 1e-6, e_l21
    assert e_act <= 1e-6, e_act
    assert full_act <= int(ties.sum()) * 2
    # the device statistics block equals the per-realization sums
    st = out["stats"].cpu().numpy()
    assert st[2] == 0
    assert st[1] == act_g.sum()
    assert math.isclose(st[0], alpha * l21_g.sum(), rel_tol=1e-6)


def test_config3_full_batch_oracle_parity():
    w = U.CONFIGS[3]
    H = U.make_inputs(w)  # all 4,096
    Hd = dev(H)
    out = U.pgd_fixed(Hd, w.lambda_pgd, w.L, w.c, power_steps=w.power_steps, w0_mode=w.w0_mode,
                      want_per_realization=True)
    torch.cuda.synchronize()
    Lo, st = O.power_iteration_batch_f32(H, w.power_steps)
    assert np.all(st == 0)
    eta_g = out["eta"].cpu().numpy().astype(np.float64)
    l30_rel = np.abs(1.0 / eta_g - Lo) / Lo
    print(f"cfg3 L30: rel max {l30_rel.max():.2e} median {np.median(l30_rel):.2e}")
    assert l30_rel.max() <= 1e-5
    ora = O.pgd_batch_f32(H, w.c, w.lambda_pgd, 1.0 / Lo, w.L, w0_mode=w.w0_mode)
    assert np.all(ora["diverged_at"] == -1)
    assert np.all(out["diverged_at"].cpu().numpy() == -1)
    rep = report(H, out["W"].cpu().numpy(), ora, w.c, w.lambda_pgd)
    assert_parity(rep)
    _means_check("cfg3 full", out, ora, rep)
    # sparsity is real at 5000 iterations (~39/64 active)
    assert 30 < ora["active"].mean() < 50


def test_config4_full_batch_oracle_parity():
    w = U.CONFIGS[4]
    H = U.make_inputs(w)  # all 16,384
    lam, eta = w.layer_params()
    out = U.unfolded_forward(dev(H), lam, eta, w.c, w0_mode=w.w0_mode, want_per_realization=True)
    torch.cuda.synchronize()
    ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode)
    rep = report(H, out["W"].cpu().numpy(), ora, w.c, LAM_OBJ_UF)
    assert_parity(rep)
    assert np.all(out["diverged_at"].cpu().numpy() == -1)
    _means_check("cfg4 full", out, ora, rep)


def test_config5_full_batch_oracle_parity():
    """All 2^20 realizations of config 5 (one device run of the whole batch,
    tcgen05 kernel) against the oracle, in host chunks of 131,072 (the oracle
    takes ~90 s on 16 host threads): SURVEY §8d's "full if budget allows"."""
    w = U.CONFIGS[5]
    Hd = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, w.B, w.K, w.M)
    lam, eta = w.layer_params()
    out = U.unfolded_forward(Hd, lam, eta, w.c, w0_mode=w.w0_mode, want_per_realization=True)
    torch.cuda.synchronize()
    st = out["stats"].cpu().numpy()
    l21_all = out["l21"].cpu().numpy().astype(np.float64)
    act_all = out["active"].cpu().numpy()
    rels, objs, ties, mism = [], [], 0, 0
    sum_l21_o, sum_act_o = 0.0, 0
    chunk = 131072
    for c0 in range(0, w.B, chunk):
        H = Hd[c0:c0 + chunk].cpu().numpy()
        Wg = out["W"][c0:c0 + chunk].cpu().numpy()
        ora = O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode)
        rep = report(H, Wg, ora, w.c, LAM_OBJ_UF)
        rels.append(rep["rel"])
        objs.append(rep["obj"])
        ties += rep["ties"]
        mism += rep["support_mismatch"]
        sum_l21_o += float(ora["l21"].sum())
        sum_act_o += int(ora["active"].sum())
        assert np.array_equal(act_all[c0:c0 + chunk], ora["active"])
        del H, Wg, ora
    rel, obj = np.concatenate(rels), np.concatenate(objs)
    e_l21 = abs(l21_all.sum() - sum_l21_o) / sum_l21_o
    print(f"cfg5 full batch 2^20: W rel max {rel.max():.2e} median {np.median(rel):.2e} obj max {obj.max():.2e} "
          f"ties {ties} support mismatches {mism} mean l21 rel {e_l21:.2e} active {act_all.sum()} vs {sum_act_o}")
    assert rel.max() <= 1e-4 and obj.max() <= 1e-5 and mism == 0
    assert e_l21 <= 1e-6 and act_all.sum() == sum_act_o
    assert st[2] == 0 and st[1] == sum_act_o
    assert math.isclose(st[0], l21_all.sum(), rel_tol=1e-6)
    del Hd, out
    torch.cuda.empty_cache()
