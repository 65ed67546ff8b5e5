"""GPU parity of the batched metrics epilogue:
compute_metrics + the ZF reference (metrics.cpp:79-91, zf.cpp:9-30) against
the FP64 oracle, plus the reference's own quality pins run end to end on the
device (forward -> metrics, as evaluate does, training.cpp:310-421)."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg,n", [(2, 2048), (4, 32), (5, 128)])
def test_metrics_match_oracle_on_solver_outputs(cfg, n):
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 0, n)
    lam, eta = w.layer_params()
    Hd = dev(H)
    out = U.unfolded_forward(Hd, lam, eta, w.c, w0_mode=w.w0_mode)
    m = U.metrics(Hd, out["W"], w.c)["out"].cpu().numpy()
    ref = O.metrics_batch_f32(H, out["W"].cpu().numpy(), w.c)
    assert np.all(m[:, 5] == 1) and np.all(ref[:, 5] == 1)
    for col, tol in [(0, 1e-12), (1, 1e-12), (2, 1e-9), (3, 1e-9), (4, 1e-8)]:
        rel = np.abs(m[:, col] - ref[:, col]) / np.abs(ref[:, col])
        assert rel.max() <= tol, (col, rel.max())
    assert np.allclose(m[:, 6:], ref[:, 6:], rtol=1e-9)


def test_zf_output_hits_sinr_targets_and_unit_pcg():
    """test_metrics.cpp:54-66 and :114-120 through the device ZF."""
    K, M = 8, 64
    H = U.generate_channels(7, 0, 0.0, 0, 64, K, M)
    c = np.full(K, math.sqrt(10.0))
    Hd = dev(H)
    zf = U.metrics(Hd, Hd, c, want_zf=True)["zf"]
    m = U.metrics(Hd, zf, c)["out"].cpu().numpy()
    # Wzf is rounded to complex64, so targets hold to FP32 accuracy
    assert np.allclose(m[:, 6:], 10.0, rtol=1e-5)
    assert np.allclose(m[:, 2], 8 * math.log2(11.0), rtol=1e-5)
    assert np.allclose(m[:, 3], 1.0, rtol=1e-6)
    assert m[:, 4].max() < 1e-4


def test_singular_channel_is_flagged():
    K, M = 4, 16
    H = U.generate_channels(19, 0, 0.0, 0, 3, K, M)
    H[1, :, 1] = H[1, :, 0]  # two identical users -> singular Gram (test_core_model.cpp:118-123)
    Hd = dev(H)
    m = U.metrics(Hd, Hd, np.full(K, math.sqrt(10.0)))["out"].cpu().numpy()
    assert m[0, 5] == 1 and m[2, 5] == 1 and m[1, 5] == 0
    assert math.isnan(m[1, 3])


def test_pgd20_mean_pcg_near_one_on_device():
    """test_pgd.cpp:519-538 end to end on the B200: 200 channels, PGD-20 at
    the surrogate step, mean PCG in [0.97, 1.03]."""
    K, M = 8, 64
    H = np.stack([O.to_storage(O.channel_for(O.SystemConfig.uniform(K, M, 10.0), 33, d)) for d in range(200)])
    H = H.astype(np.complex64)
    lam = np.full(20, 1.0 / 15.0)
    eta = np.full(20, 1.0 / U.mp_bound(K, M))
    c = np.full(K, math.sqrt(10.0))
    Hd = dev(H)
    out = U.unfolded_forward(Hd, lam, eta, c, w0_mode=U.W0_CONJ_H)
    summ = U.summarize_metrics(U.metrics(Hd, out["W"], c)["out"].cpu().numpy())
    assert 0.97 < summ["mean"]["pcg"] < 1.03
    assert summ["num_channels"] == 200 and summ["std_error"]["pcg"] > 0
