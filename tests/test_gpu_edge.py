"""Edge cases of the batched path on the GPU against the FP64 oracle: ragged
and tiny batches on every kernel shape, the extreme layer counts, shapes the
specialised kernels do not cover (general kernel), and a host batch that does
not fill its last pipeline chunk."""
import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
from _parity import assert_parity, report

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def params(K, M, L, seed=5):
    lam, eta = U.layer_params(seed, L, K, M)
    return U.project_params(lam, eta, K, M)


@pytest.mark.parametrize("K,M", [(4, 16), (4, 32), (4, 64), (8, 32), (8, 64), (8, 128), (16, 128), (32, 256)])
@pytest.mark.parametrize("B", [1, 2, 3, 17])
def test_ragged_batches_every_kernel_shape(K, M, B):
    H = U.generate_channels(77, 78, 10.0, 3, B, K, M)
    lam, eta = params(K, M, 20)
    c = np.full(K, np.sqrt(10.0))
    for mode in (U.W0_ZERO, U.W0_CONJ_H):
        g = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=mode, want_per_realization=True)
        ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=mode)
        rep = report(H, g["W"].cpu().numpy(), ora, c, 1.0 / 15.0)
        assert_parity(rep)
        assert np.array_equal(g["active"].cpu().numpy(), ora["active"])
        assert np.all(g["diverged_at"].cpu().numpy() == -1)


@pytest.mark.parametrize("K,M", [(8, 64), (16, 128)])
def test_single_layer_and_zero_layers(K, M):
    H = U.generate_channels(3, 4, 0.0, 0, 9, K, M)
    c = np.full(K, np.sqrt(10.0))
    lam, eta = params(K, M, 1)
    g = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=U.W0_CONJ_H)["W"].cpu().numpy()
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=U.W0_CONJ_H)
    assert_parity(report(H, g, ora, c, 1.0 / 15.0))
    # zero layers: forward returns the start point (unfolded.cpp:96, loop body never runs)
    W0 = np.conj(H).astype(np.complex64)
    z = U.unfolded_forward(dev(H), [], [], c, w0_mode=U.W0_GIVEN, W0=dev(W0))["W"].cpu().numpy()
    assert np.array_equal(z, W0)


@pytest.mark.parametrize("K,M", [(5, 40), (2, 3), (12, 12)])
def test_shapes_outside_the_specialised_kernels(K, M):
    H = U.generate_channels(11, 12, 0.0, 0, 6, K, M)
    lam, eta = params(K, M, 20)
    c = np.full(K, np.sqrt(10.0))
    g = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=U.W0_CONJ_H, want_per_realization=True)
    ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=U.W0_CONJ_H)
    assert_parity(report(H, g["W"].cpu().numpy(), ora, c, 1.0 / 15.0))
    assert np.array_equal(g["active"].cpu().numpy(), ora["active"])


@pytest.mark.parametrize("K,M", [(3, 10), (5, 40), (6, 48), (7, 64), (8, 50), (12, 100), (24, 200), (30, 256)])
def test_zero_padded_shapes_match_the_oracle(K, M):
    """Shapes without a specialised kernel but within 6x the flops of one run
    zero-padded on it (capi.cpp padded_shape): the cropped W, support and
    per-realization outputs equal the oracle's, for every start mode; the
    general kernel (option zero_pad=0) agrees too."""
    B = 23
    H = U.generate_channels(41, 42, 10.0, 0, B, K, M)
    lam, eta = params(K, M, 20)
    c = np.full(K, np.sqrt(10.0))
    W0 = (0.01 * np.conj(H)).astype(np.complex64)
    for mode in (U.W0_ZERO, U.W0_CONJ_H, U.W0_GIVEN):
        kw = dict(w0_mode=mode, want_per_realization=True)
        if mode == U.W0_GIVEN:
            kw["W0"] = dev(W0)
        g = U.unfolded_forward(dev(H), lam, eta, c, **kw)
        ora = O.forward_batch_f32(H, c, lam, eta, w0_mode=mode, W0=W0 if mode == U.W0_GIVEN else None)
        assert_parity(report(H, g["W"].cpu().numpy(), ora, c, 1.0 / 15.0))
        assert np.array_equal(g["active"].cpu().numpy(), ora["active"])
        assert np.all(g["diverged_at"].cpu().numpy() == -1)
        np.testing.assert_allclose(g["l21"].cpu().numpy(), ora["l21"], rtol=1e-5)
        with U.options(zero_pad=0):
            gen = U.unfolded_forward(dev(H), lam, eta, c, **kw)
        assert_parity(report(H, gen["W"].cpu().numpy(), ora, c, 1.0 / 15.0))
        np.testing.assert_allclose(g["stats"].cpu().numpy(), gen["stats"].cpu().numpy(), rtol=1e-5)


@pytest.mark.parametrize("K,M", [(3, 10), (6, 48), (12, 100)])
def test_zero_padded_pgd_with_power_iteration(K, M):
    """pgd_fixed on a padded shape: the 30-step power iteration runs on the
    zero-padded H with the zero-padded start vector, so L30 (hence eta), W
    and the support match the oracle's unpadded solve; the host pipeline
    entry point returns the same bits as the device one."""
    B, iters, lam = 16, 300, 0.05
    H = U.generate_channels(124, 0, 0.0, 0, B, K, M)
    c = np.full(K, np.sqrt(10.0))
    out = U.pgd_fixed(dev(H), lam, iters, c, power_steps=30, want_per_realization=True)
    Lo, _ = O.power_iteration_batch_f32(H, 30)
    assert np.max(np.abs(out["eta"].cpu().numpy() * Lo - 1.0)) <= 1e-5
    ora = O.pgd_batch_f32(H, c, lam, 1.0 / Lo, iters, w0_mode=U.W0_CONJ_H)
    assert_parity(report(H, out["W"].cpu().numpy(), ora, c, lam))
    assert np.array_equal(out["active"].cpu().numpy(), ora["active"])
    host = U.pgd_fixed_host(H, lam, iters, c, power_steps=30)
    assert np.array_equal(host["W"], out["W"].cpu().numpy())


def test_zero_padded_path_splits_large_batches():
    """(6, 48) pads to (8, 64): with a 256 MiB scratch (option pad_sub_bytes) that
    is 65,536 padded realizations per sub-batch, so 65,536 + 37 runs two
    sub-batches; the seam and the stats partials of both must line up (checked
    against the general kernel on all realizations and the oracle on the seam)."""
    K, M, B = 6, 48, 65536 + 37
    H = U.generate_channels(43, 44, 10.0, 0, B, K, M)
    lam, eta = params(K, M, 20)
    c = np.full(K, np.sqrt(10.0))
    with U.options(pad_sub_bytes=256 << 20):
        g = U.unfolded_forward(dev(H), lam, eta, c, want_per_realization=True)
    with U.options(zero_pad=0):
        gen = U.unfolded_forward(dev(H), lam, eta, c, want_per_realization=True)
    Wg, We = g["W"].cpu().numpy(), gen["W"].cpu().numpy()
    rel = np.linalg.norm((Wg - We).reshape(B, -1), axis=1) / np.linalg.norm(We.reshape(B, -1), axis=1)
    assert rel.max() < 1e-5, rel.max()
    assert np.array_equal(g["active"].cpu().numpy(), gen["active"].cpu().numpy())
    np.testing.assert_allclose(g["stats"].cpu().numpy(), gen["stats"].cpu().numpy(), rtol=1e-6)
    seam = slice(65536 - 3, 65536 + 3)
    ora = O.forward_batch_f32(H[seam], c, lam, eta)
    assert_parity(report(H[seam], Wg[seam], ora, c, 1.0 / 15.0))


def test_host_batch_with_partial_last_chunk_matches_device_path():
    w = U.CONFIGS[2]
    B = (16 << 20) // (8 * w.K * w.M) + 37  # one full 16 MiB chunk plus a ragged tail
    H = U.make_inputs(w, 123, B)
    lam, eta = w.layer_params()
    host = U.unfolded_forward_host(H, lam, eta, w.c, w0_mode=w.w0_mode)
    devw = U.unfolded_forward(dev(H), lam, eta, w.c, w0_mode=w.w0_mode)
    assert np.array_equal(host["W"], devw["W"].cpu().numpy())
    assert np.allclose(host["stats"], devw["stats"].cpu().numpy(), rtol=1e-12)


@pytest.mark.parametrize("K,M", [(4, 16), (4, 32), (4, 64), (8, 32), (8, 64), (8, 128), (16, 128), (32, 256)])
def test_divergence_from_a_zero_start_on_every_kernel_shape(K, M):
    """W0 = 0 takes the exact layer-0 shortcut (eta c_k conj(H)); a channel that
    is +inf in complex64 must still be reported at layer 0 (unfolded.cpp:120-125)
    and leave its neighbours untouched."""
    with np.errstate(over="ignore"):
        H = np.full((3, M, K), 1e200, dtype=np.complex128).astype(np.complex64)
    H[1] = U.generate_channels(5, 0, 0.0, 0, 1, K, M)[0]
    lam, eta = params(K, M, 4)
    c = np.full(K, np.sqrt(10.0))
    out = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=U.W0_ZERO, want_per_realization=True)
    d = out["diverged_at"].cpu().numpy()
    assert d[0] == 0 and d[2] == 0 and d[1] == -1
    ora = O.forward_batch_f32(H[1:2], c, lam, eta, w0_mode=U.W0_ZERO)
    assert_parity(report(H[1:2], out["W"].cpu().numpy()[1:2], ora, c, 1.0 / 15.0))


@pytest.mark.parametrize("K,M", [(4, 32), (8, 64), (16, 128), (32, 256), (6, 48), (5, 5)])
def test_nan_channel_diverges_at_layer_zero_and_is_isolated(K, M):
    """A NaN anywhere in H makes the first step image non-finite
    (unfolded.cpp:120-125: allFinite is false for NaN as for inf): the
    realization reports layer 0, counts as diverged in the stats, and its
    neighbours are untouched — on the fused, tiled, padded and general paths."""
    H = U.generate_channels(6, 0, 0.0, 0, 3, K, M)
    H[1, M // 2, K - 1] = np.complex64(complex(np.nan, 0.0))
    lam, eta = params(K, M, 4)
    c = np.full(K, np.sqrt(10.0))
    for mode in (U.W0_ZERO, U.W0_CONJ_H):
        out = U.unfolded_forward(dev(H), lam, eta, c, w0_mode=mode, want_per_realization=True)
        assert out["diverged_at"].cpu().numpy().tolist() == [-1, 0, -1]
        assert out["stats"].cpu().numpy()[2] == 1.0
        keep = [0, 2]
        ora = O.forward_batch_f32(H[keep], c, lam, eta, w0_mode=mode)
        assert_parity(report(H[keep], out["W"].cpu().numpy()[keep], ora, c, 1.0 / 15.0))
    pg = U.pgd_fixed(dev(H), 0.05, 50, c, power_steps=30, want_per_realization=True)
    d = pg["diverged_at"].cpu().numpy()
    assert d[1] >= 1 and d[0] == -1 and d[2] == -1  # 1-based iteration index (pgd.cpp:231-235)


def test_pgd_host_path_matches_device_path():
    """ufpgd_gpu_pgd_fixed_host (config 3 end to end: pinned-chunk pipeline,
    in-kernel 30-step power iteration) equals the device entry point bit for
    bit, including the per-realization step it reports."""
    w = U.CONFIGS[3]
    H = U.make_inputs(w, 0, 1000)
    host = U.pgd_fixed_host(H, w.lambda_pgd, 300, w.c, power_steps=w.power_steps)
    d = U.pgd_fixed(dev(H), w.lambda_pgd, 300, w.c, power_steps=w.power_steps)
    assert np.array_equal(host["W"], d["W"].cpu().numpy())
    assert np.array_equal(host["diverged_at"], d["diverged_at"].cpu().numpy())
    assert np.allclose(host["stats"], d["stats"].cpu().numpy(), rtol=1e-12)


def test_fp32_peak_probe_is_plausible():
    """The roofline denominator bench.py reports: the FFMA2 probe on this B200
    (nominal 148 SMs x 128 lanes x 2 x 1.965 GHz = 74.4 TFLOP/s)."""
    tf, ghz = U.fp32_peak(0)
    assert 30.0 < tf < 80.0 and 1.0 < ghz < 2.2, (tf, ghz)


def test_concurrent_host_calls_from_threads():
    """The reference's functions are reentrant and callers batch with
    parallel_for (parallel.hpp:12-18): several host threads calling the C ABI
    at once (ctypes releases the GIL) must each get their own exact result —
    the host path serialises on the device's workspace, device calls on
    separate streams run concurrently."""
    import threading

    w = U.CONFIGS[2]
    lam, eta = w.layer_params()
    Hs = [U.make_inputs(w, 1000 * t, 3000 + 17 * t) for t in range(4)]
    ref = [U.unfolded_forward_host(H, lam, eta, w.c, w0_mode=w.w0_mode)["W"] for H in Hs]
    out, errs = [None] * 8, []

    def host(t):
        try:
            out[t] = U.unfolded_forward_host(Hs[t], lam, eta, w.c, w0_mode=w.w0_mode)["W"]
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    def device(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                Hd = dev(Hs[t - 4])
                r = U.unfolded_forward(Hd, lam, eta, w.c, w0_mode=w.w0_mode, stream=s)["W"]
                s.synchronize()
                out[t] = r.cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=host, args=(t,)) for t in range(4)]
    th += [threading.Thread(target=device, args=(t,)) for t in range(4, 8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for t in range(8):
        assert np.array_equal(out[t], ref[t % 4]), t
