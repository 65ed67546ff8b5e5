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


@pytest.mark.parametrize("cfg,n", [(2, 4096 + 3), (5, 2048)])
@pytest.mark.parametrize("w0_mode", [U.W0_ZERO, U.W0_GIVEN])
def test_sharded_device_entry_equals_single_device(comms, cfg, n, w0_mode):
    """Device-resident shards: the statistics are all-reduced in place on the
    devices (no host round trip) and W0 may be given."""
    G = torch.cuda.device_count()
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 3, n)
    lam, eta = w.layer_params()
    W0 = (0.01 * np.conj(H)).astype(np.complex64) if w0_mode == U.W0_GIVEN else None
    cuts = [n * g // G for g in range(G + 1)]
    shards = [torch.from_numpy(H[cuts[g]:cuts[g + 1]]).to(f"cuda:{g}") for g in range(G)]
    w0s = None if W0 is None else [torch.from_numpy(W0[cuts[g]:cuts[g + 1]]).to(f"cuda:{g}") for g in range(G)]
    prev = torch.cuda.current_device()
    r = U.unfolded_forward_sharded_device(shards, lam, eta, w.c, w0_mode=w0_mode, W0=w0s)
    assert torch.cuda.current_device() == prev
    for g in range(G):
        torch.cuda.synchronize(g)
    one = U.unfolded_forward(torch.from_numpy(H).cuda(), lam, eta, w.c, w0_mode=w0_mode,
                             W0=None if W0 is None else torch.from_numpy(W0).cuda())
    Wcat = np.concatenate([x.cpu().numpy() for x in r["W"]])
    assert np.array_equal(Wcat, one["W"].cpu().numpy())
    for g in range(G):
        assert np.allclose(r["stats"][g].cpu().numpy(), one["stats"].cpu().numpy(), rtol=1e-12)
    host = U.unfolded_forward_sharded(H, lam, eta, w.c, w0_mode=w0_mode, W0=W0)
    assert np.array_equal(host["W"], Wcat)


def test_sharded_device_entry_is_graph_capturable_on_one_device(comms):
    """With one device the sharded step (forward + in-place NCCL all-reduce of
    the statistics) is captured in a CUDA graph and replayed."""
    if torch.cuda.device_count() != 1:
        pytest.skip("single-device capture check")
    w = U.CONFIGS[2]
    H = torch.from_numpy(U.make_inputs(w, 0, 8192)).cuda()
    lam, eta = w.layer_params()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ref = U.unfolded_forward_sharded_device([H], lam, eta, w.c, streams=[s])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = U.unfolded_forward_sharded_device([H], lam, eta, w.c,
                                                streams=[torch.cuda.current_stream()])
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out["W"][0], ref["W"][0])
    assert torch.equal(out["stats"][0], ref["stats"][0])
