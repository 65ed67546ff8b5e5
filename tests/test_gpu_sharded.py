"""The single-process multi-GPU entry point (ufpgd_gpu_init / _unfolded_forward_sharded
/ _shutdown: contiguous shards, one ncclAllReduce of the three statistics,
SURVEY §8e) on the devices of this box — one on the gpurun B200, so NCCL runs
with a single rank. Shards must equal the single-device path bit for bit and
the reduced statistics must equal the device path's."""
import numpy as np
import pytest
import torch

import paper_2304_12745_b200 as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comms():
    U.init_multi_gpu(torch.cuda.device_count())
    yield
    U.shutdown_multi_gpu()


@pytest.mark.parametrize("cfg,n", [(2, 8192 + 7), (5, 1024), (1, 1024)])
def test_sharded_equals_single_device(comms, cfg, n):
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 11, n)
    lam, eta = w.layer_params()
    sh = U.unfolded_forward_sharded(H, lam, eta, w.c, w0_mode=w.w0_mode)
    one = U.unfolded_forward(torch.from_numpy(H).cuda(), lam, eta, w.c, w0_mode=w.w0_mode)
    assert np.array_equal(sh["W"], one["W"].cpu().numpy())
    assert np.array_equal(sh["diverged_at"], one["diverged_at"].cpu().numpy())
    assert np.allclose(sh["stats"], one["stats"].cpu().numpy(), rtol=1e-12)


def test_init_is_idempotent_and_rejects_bad_counts(comms):
    U.init_multi_gpu(torch.cuda.device_count())  # second init: no-op
    with pytest.raises(ValueError):
        U.init_multi_gpu(torch.cuda.device_count() + 1)
