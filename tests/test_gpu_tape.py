"""GPU parity of the taped forward (ForwardOptions::with_tape / with_iterates,
unfolded.hpp:40-62, unfolded.cpp:112-146) through `ufpgd_gpu_layers_general`:
every iterate W_0 .. W_L, every layer's step image V_l, column norms ||v_m||
and shrink factors against the FP64 oracle's forward (oracle/oracle.py
`forward`, the restatement of unfolded.cpp:83-150) per realization.

The K <= 8 team shapes run the fused team kernel's taped instance (team.cu,
tapes written from the registers of the layer sweep); (16,128) and (3,8) run
the general kernel. Bars: iterates and step images within W_REL_TOL (1e-4)
relative Frobenius per realization and layer, column norms within 1e-4 of the
layer's largest norm, shrink factors within 5e-4 absolute (a column at a
threshold tie, |n - t| / t < 1e-4, may be cut on one side and kept with a
shrink below 1e-4 on the other), the active support identical outside ties."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from paper_2304_12745_b200.workloads import project_params
from oracle import oracle as O
from _parity import TIE_MARGIN, W_REL_TOL, rel_fro

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHRINK_ABS_TOL = 5e-4
NORM_REL_TOL = 1e-4


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def oracle_tapes(H, lam, eta, K, M, w0=None):
    """Per-realization FP64 forward with tape and iterates: stacked
    iterates [L+1, B, M, K], step images [L, B, M, K], norms / shrink [L, B, M]."""
    cfg = O.SystemConfig.uniform(K, M, 10.0)
    net = O.UnfoldedNetwork(K, M, O.mp_bound(K, M), [O.LayerParams(float(l), float(e)) for l, e in zip(lam, eta)])
    its, tv, tn, ts = [], [], [], []
    for b in range(H.shape[0]):
        h = O.from_storage(H[b].astype(np.complex128).reshape(-1), K, M)
        start = None if w0 is None else O.from_storage(w0[b].astype(np.complex128).reshape(-1), K, M)
        r = O.forward(net, h, cfg, start, O.ForwardOptions(with_tape=True, with_iterates=True))
        its.append(np.stack([O.to_storage(x) for x in r.iterates]))
        tv.append(np.stack([O.to_storage(t.step_image) for t in r.tape]))
        tn.append(np.stack([t.column_norms for t in r.tape]))
        ts.append(np.stack([t.shrink_factors for t in r.tape]))
    sw = lambda a: np.swapaxes(np.stack(a), 0, 1)
    return sw(its), sw(tv), sw(tn), sw(ts)


def check_tapes(g, ref, thr, L, label):
    its_o, tv_o, tn_o, ts_o = ref
    its = g["iterates"].cpu().numpy()
    tv = g["tape_v"].cpu().numpy()
    tn = g["tape_norms"].cpu().numpy()
    ts = g["tape_shrink"].cpu().numpy()
    assert np.all(g["diverged_at"].cpu().numpy() == -1)
    assert np.all(g["iterations"].cpu().numpy() == L)
    # the output is the last iterate, bit for bit
    assert np.array_equal(g["W"].cpu().numpy(), its[L])
    # ties: a column within TIE_MARGIN of the layer's threshold in the oracle
    tie_col = np.abs(tn_o - np.asarray(thr)[:, None, None]) < TIE_MARGIN * np.maximum(np.asarray(thr), 1e-300)[:, None, None]
    tie = np.any(tie_col, axis=(0, 2))  # [B]
    worst = 0.0
    for l in range(L + 1):
        rel = rel_fro(its[l], its_o[l])
        worst = max(worst, float(rel.max()))
        assert rel.max() <= W_REL_TOL, (label, "iterate", l, rel.max())
        act_g = np.sum(np.abs(its[l]) ** 2, axis=2) > 0
        act_o = np.sum(np.abs(its_o[l]) ** 2, axis=2) > 0
        assert np.all((act_g == act_o) | tie[:, None]), (label, "support", l)
    for l in range(L):
        rel = rel_fro(tv[l], tv_o[l])
        assert rel.max() <= W_REL_TOL, (label, "step image", l, rel.max())
        scale = np.max(tn_o[l], axis=1, keepdims=True)
        nerr = np.max(np.abs(tn[l] - tn_o[l]) / np.maximum(scale, 1e-300))
        assert nerr <= NORM_REL_TOL, (label, "norms", l, nerr)
        serr = np.max(np.abs(ts[l] - ts_o[l]))
        assert serr <= SHRINK_ABS_TOL, (label, "shrink", l, serr)
        # cut columns: shrink 0 on both sides outside ties
        assert np.all(((ts[l] == 0) == (ts_o[l] == 0)) | tie[:, None]), (label, "cut columns", l)
    print(f"{label}: iterates rel max {worst:.2e}, ties {int(tie.sum())}")


@pytest.mark.parametrize("cfg,B", [(2, 97), (1, 97), (1, 4800)])
def test_taped_forward_baseline_configs(cfg, B):
    """Config 2 (8,64) and config 1 (4,32) networks from H^* (ForwardOptions'
    default start); B = 4,800 at (4,32) takes the 8-thread teams, 97 the
    16-thread ones; odd B leaves a padding team."""
    w = U.CONFIGS[cfg]
    assert np.allclose(w.c, math.sqrt(10.0))
    H = U.make_inputs(w, 77, B)
    lam, eta = w.layer_params()
    thr = lam * eta
    g = U.layers_general(dev(H), eta, thr, w.c, w0_mode=U.W0_CONJ_H, iterates=True, tape=True)
    check_tapes(g, oracle_tapes(H, lam, eta, w.K, w.M), thr, w.L, f"cfg{cfg} B={B}")


@pytest.mark.parametrize("K,M", [(4, 16), (4, 64), (8, 32), (8, 128), (16, 128), (3, 8)])
def test_taped_forward_shapes(K, M):
    L, B = 12, 33
    H = U.generate_channels(4242, 7, 10.0, 0, B, K, M)
    lam, eta = project_params(*U.layer_params(91, L, K, M), K, M)
    thr = lam * eta
    g = U.layers_general(dev(H), eta, thr, np.full(K, math.sqrt(10.0)), w0_mode=U.W0_CONJ_H, iterates=True,
                         tape=True)
    check_tapes(g, oracle_tapes(H, lam, eta, K, M), thr, L, f"({K},{M})")


@pytest.mark.parametrize("w0", ["zero", "given"])
def test_taped_forward_start_points(w0):
    """W0 = 0 (iterate 0 all zeros; the taped instance runs layer 0 through the
    full sweep) and a given W0."""
    w = U.CONFIGS[2]
    B = 40
    H = U.make_inputs(w, 5, B)
    lam, eta = w.layer_params()
    thr = lam * eta
    if w0 == "zero":
        W0 = np.zeros_like(H)
        g = U.layers_general(dev(H), eta, thr, w.c, w0_mode=U.W0_ZERO, iterates=True, tape=True)
    else:
        rng = np.random.default_rng(3)
        W0 = (0.1 * (rng.standard_normal(H.shape) + 1j * rng.standard_normal(H.shape))).astype(np.complex64)
        g = U.layers_general(dev(H), eta, thr, w.c, w0_mode=U.W0_GIVEN, W0=dev(W0), iterates=True, tape=True)
    assert np.array_equal(g["iterates"][0].cpu().numpy(), W0)
    check_tapes(g, oracle_tapes(H, lam, eta, w.K, w.M, W0), thr, w.L, f"W0 {w0}")


def test_taped_and_untaped_sweeps_agree():
    """Tapes only add stores: the taped instance's W with iterates only and
    with the full tape are the same bits, and the same bits as the untaped
    team kernel (tensor cores off); the default sweep without tapes runs the
    unfolded forward's kernel (tcgen05 pairs at (8,64)) and agrees to FP32
    rounding."""
    w = U.CONFIGS[2]
    H = dev(U.make_inputs(w, 11, 300))
    lam, eta = w.layer_params()
    thr = lam * eta
    b = U.layers_general(H, eta, thr, w.c, iterates=True)
    c = U.layers_general(H, eta, thr, w.c, iterates=True, tape=True)
    assert torch.equal(b["W"], c["W"]) and torch.equal(b["iterates"], c["iterates"])
    with U.options(tensor_cores=0):
        t = U.layers_general(H, eta, thr, w.c)
    assert torch.equal(t["W"], c["W"])
    a = U.layers_general(H, eta, thr, w.c)
    assert np.all(a["iterations"].cpu().numpy() == w.L) and np.all(a["diverged_at"].cpu().numpy() == -1)
    d = (a["W"] - c["W"]).abs().flatten(1).norm(dim=1) / c["W"].abs().flatten(1).norm(dim=1)
    assert d.max().item() <= 1e-5


@pytest.mark.parametrize("cfg", [4, 5])
def test_untaped_sweep_runs_the_forward_kernel(cfg):
    """Without tapes the sweep is ufpgd_gpu_unfolded_forward's kernel for the
    shape: the same bits as the forward from H^* with the same (eta, lambda eta)."""
    w = U.CONFIGS[cfg]
    H = dev(U.make_inputs(w, 2, 64))
    lam, eta = w.layer_params()
    g = U.layers_general(H, eta, lam * eta, w.c)
    f = U.unfolded_forward(H, lam, eta, w.c, w0_mode=U.W0_CONJ_H)
    assert torch.equal(g["W"], f["W"])
    assert np.all(g["iterations"].cpu().numpy() == w.L)


def test_taped_forward_divergence_is_layer_indexed():
    """A non-finite channel diverges at layer 0 (index_base 0: the sweep runs
    on, as forward's caller sees every layer); its partner team is untouched."""
    w = U.CONFIGS[2]
    H = U.make_inputs(w, 3, 4)
    H[1, 5, 2] = np.nan
    lam, eta = w.layer_params()
    thr = lam * eta
    g = U.layers_general(dev(H), eta, thr, w.c, iterates=True, tape=True)
    div = g["diverged_at"].cpu().numpy()
    assert list(div) == [-1, 0, -1, -1]
    keep = [0, 2, 3]
    ref = oracle_tapes(H[keep], lam, eta, w.K, w.M)
    its = g["iterates"].cpu().numpy()[:, keep]
    for l in range(w.L + 1):
        assert rel_fro(its[l], ref[0][l]).max() <= W_REL_TOL
