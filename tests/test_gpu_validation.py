"""Error behaviour of the C ABI entry points on the device (the reference's
std::invalid_argument cases, pgd.cpp:33-49, unfolded.cpp:19-35,
system_config.cpp:22-43): invalid shapes and parameters are rejected with
UFPGD_EINVAL_* (ValueError) before any launch; unsupported sizes with
UFPGD_ENOTSUP; nothing is silently clamped or run on a CPU path."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from paper_2304_12745_b200.capi import UfpgdError

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def H_(B, K, M):
    return torch.from_numpy(U.generate_channels(3, 0, 0.0, 0, B, K, M)).cuda()


C8 = np.full(8, math.sqrt(10.0))
LAM, ETA = [0.05] * 3, [1.0 / U.mp_bound(8, 64)] * 3


def test_unfolded_forward_rejects_bad_parameters():
    H = H_(4, 8, 64)
    with pytest.raises(ValueError):
        U.unfolded_forward(H, [-0.1] * 3, ETA, C8)  # lambda_i < 0 (unfolded.cpp:22-27)
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, [0.0] * 3, C8)  # eta_i <= 0
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, [float("nan")] * 3, C8)
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, ETA, np.full(8, float("inf")))  # non-finite c
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, ETA, C8, w0_mode=U.W0_GIVEN)  # W0 required
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, ETA, C8, w0_mode=7)
    with pytest.raises(ValueError):
        U.unfolded_forward(H, [0.05] * 257, [ETA[0]] * 257, C8)  # > UFPGD_MAX_LAYERS
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, ETA, C8, alpha=0.0)  # consumed_power alpha > 0
    with pytest.raises(ValueError):
        U.unfolded_forward(H, LAM, ETA[:2], C8)  # one (lambda, eta) per layer


def test_shapes_outside_the_reference_domain():
    with pytest.raises(ValueError):  # K > M (system_config.cpp:23-27)
        U.unfolded_forward(torch.zeros((2, 4, 8), dtype=torch.complex64, device="cuda"), LAM, ETA, C8)
    with pytest.raises(UfpgdError):  # K beyond the kernels' UFPGD_MAX_USERS
        K = 65
        U.unfolded_forward(torch.zeros((1, 80, K), dtype=torch.complex64, device="cuda"), LAM, ETA,
                           np.ones(K))
    with pytest.raises(ValueError):  # host tensors are not device batches
        U.unfolded_forward(torch.zeros((2, 64, 8), dtype=torch.complex64), LAM, ETA, C8)
    with pytest.raises(ValueError):  # complex128 is the FP64 path's type, not the batched one
        U.unfolded_forward(torch.zeros((2, 64, 8), dtype=torch.complex128, device="cuda"), LAM, ETA, C8)


def test_pgd_and_metrics_reject_bad_parameters():
    H = H_(4, 8, 64)
    with pytest.raises(ValueError):
        U.pgd_fixed(H, -0.05, 10, C8)  # lambda < 0 (pgd.cpp:33-49)
    with pytest.raises(ValueError):
        U.pgd_fixed(H, 0.05, -1, C8)  # negative iteration count
    with pytest.raises(ValueError):
        U.metrics(H, H, C8, sigma_nu=-1.0)  # SystemConfig: sigma_nu >= 0
    with pytest.raises(UfpgdError):
        K = 40  # metrics support K <= 32
        Hb = H_(1, K, 64)
        U.metrics(Hb, Hb, np.ones(K))


def test_zero_batches_are_no_ops():
    H = torch.zeros((0, 64, 8), dtype=torch.complex64, device="cuda")
    out = U.unfolded_forward(H, LAM, ETA, C8)
    assert out["W"].shape == (0, 64, 8) and out["stats"].cpu().numpy().tolist() == [0.0, 0.0, 0.0]
    assert U.pgd_fixed(H, 0.05, 10, C8)["W"].shape == (0, 64, 8)
