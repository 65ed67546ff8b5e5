"""The asynchronous host-buffer entry point (ufpgd_gpu_unfolded_forward_host_async
+ ufpgd_gpu_host_wait): back-to-back batches pipelined across calls must give
the synchronous call's results bit for bit (W, diverged_at, statistics), in any
order of waits, with the in-flight limit and ticket misuse reported as errors."""
import math

import numpy as np
import pytest
import torch

import paper_2304_12745_b200 as U

pytestmark = pytest.mark.gpu


def _pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


def test_async_batches_equal_the_synchronous_call():
    w = U.CONFIGS[2]
    lam, eta = w.layer_params()
    Hs = [_pinned(U.make_inputs(w, 40000 * i, 40000 + 13 * i)) for i in range(3)]
    ref = [U.unfolded_forward_host(H, lam, eta, w.c, w0_mode=w.w0_mode) for H in Hs]
    outs = [_pinned(np.empty_like(H)) for H in Hs]
    calls = [U.unfolded_forward_host_async(H, lam, eta, w.c, w0_mode=w.w0_mode, out=o) for H, o in zip(Hs, outs)]
    for i in (1, 0, 2):  # completion order is the caller's choice
        r = calls[i].wait()
        assert np.array_equal(r["W"], ref[i]["W"])
        assert np.array_equal(r["diverged_at"], ref[i]["diverged_at"])
        assert np.array_equal(r["stats"], ref[i]["stats"])


def test_async_pipeline_reuses_slots_and_matches_device_path():
    """Many calls through the 3 slots, double-buffered like bench.py's e2e leg,
    with a shape change in between (buffer regrowth while calls are in flight)."""
    lam5, eta5 = U.CONFIGS[5].layer_params()
    w = U.CONFIGS[2]
    lam, eta = w.layer_params()
    H = _pinned(U.make_inputs(w, 0, 20000))
    H5 = _pinned(U.make_inputs(U.CONFIGS[5], 0, 3000))
    dev = U.unfolded_forward(torch.from_numpy(H).cuda(), lam, eta, w.c)["W"].cpu().numpy()
    dev5 = U.unfolded_forward(torch.from_numpy(H5).cuda(), lam5, eta5, U.CONFIGS[5].c)["W"].cpu().numpy()
    bufs = [_pinned(np.empty_like(H)) for _ in range(2)]
    prev = None
    for k in range(7):
        cur = U.unfolded_forward_host_async(H, lam, eta, w.c, out=bufs[k % 2])
        if k == 3:
            c5 = U.unfolded_forward_host_async(H5, lam5, eta5, U.CONFIGS[5].c)
            assert np.array_equal(c5.wait()["W"], dev5)
        if prev is not None:
            assert np.array_equal(prev.wait()["W"], dev)
        prev = cur
    assert np.array_equal(prev.wait()["W"], dev)


def test_async_limits_and_ticket_misuse():
    w = U.CONFIGS[1]
    lam, eta = w.layer_params()
    H = _pinned(U.make_inputs(w))
    calls = [U.unfolded_forward_host_async(H, lam, eta, w.c) for _ in range(3)]
    with pytest.raises(U.UfpgdError):  # a 4th call in flight
        U.unfolded_forward_host_async(H, lam, eta, w.c)
    t = calls[0].ticket
    for c in calls:
        c.wait()
    assert U.lib().ufpgd_gpu_host_wait(t) == U.capi.EINVAL_PARAM  # already completed
    assert U.lib().ufpgd_gpu_host_wait(-5) == U.capi.EINVAL_PARAM


def test_async_divergence_is_reported_at_wait():
    K, M = 8, 64
    H = U.generate_channels(5, 0, 0.0, 0, 3, K, M)
    with np.errstate(over="ignore"):
        H[1] = (H[1].astype(np.complex128) * 1e30).astype(np.complex64)  # +inf entries
    H = _pinned(H)
    call = U.unfolded_forward_host_async(H, [0.1] * 3, [1.0 / U.mp_bound(K, M)] * 3, np.full(K, math.sqrt(10.0)),
                                         w0_mode=U.W0_CONJ_H)
    with pytest.raises(U.DivergenceError) as ei:
        call.wait()
    assert ei.value.index == 0
    assert list(call.diverged_at) == [-1, 0, -1]


def test_streamed_calls_report_divergence_per_chunk_and_statistics():
    """diverged_at and the statistics reach the host by direct stores into the
    call's pinned stage (no copy-engine op): diverging realizations in several
    pipeline chunks of back-to-back streamed calls must come out exactly as on
    the device path, and a clean call in between must not see them."""
    w = U.CONFIGS[2]
    lam, eta = w.layer_params()
    B = 3 * 4096 + 77  # four 16 MiB chunks at (8,64)
    clean = U.make_inputs(w, 0, B)
    bad = clean.copy()
    idx = [5, 4095, 4096, 9000, B - 1]
    for i in idx:
        bad[i, 0, 0] = np.complex64(complex(float("nan"), 0.0))
    clean, bad = _pinned(clean), _pinned(bad)
    dev_div = U.unfolded_forward(torch.from_numpy(bad).cuda(), lam, eta, w.c)["diverged_at"].cpu().numpy()
    assert sorted(np.nonzero(dev_div >= 0)[0].tolist()) == idx
    ref = U.unfolded_forward_host(bad, lam, eta, w.c, raise_on_divergence=False)
    assert np.array_equal(ref["diverged_at"], dev_div) and ref["stats"][2] == len(idx)
    calls = [U.unfolded_forward_host_async(h, lam, eta, w.c) for h in (bad, clean, bad)]
    for k, c in enumerate(calls):
        if k == 1:
            r = c.wait()
            assert (r["diverged_at"] == -1).all() and r["stats"][2] == 0.0
            continue
        with pytest.raises(U.DivergenceError) as ei:
            c.wait()
        assert ei.value.index == 0  # the layer of the first non-finite iterate (NaN channel: layer 0)
        assert np.array_equal(np.asarray(c.diverged_at), dev_div)
        assert np.array_equal(np.asarray(c.stats), np.asarray(ref["stats"]), equal_nan=True)
