"""UFPD dataset files: the reference's format read into
device batches and written from them (dataset.cpp:38-175), with the
corruption cases of test_data_io.cpp:119-171."""
import os

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
import _ufpd


def sample(K, M, N, seed, labels=False):  # test_data_io.cpp:27-45
    cfg = O.SystemConfig.uniform(K, M, 10.0)
    ch = np.stack([O.channel_for(cfg, seed, i) for i in range(N)])
    lab = None
    if labels:
        lab = np.stack([O.random_matrix(K, M, O.Rng.stream(seed ^ 0xABCDEF, i)) for i in range(N)])
    return ch, lab


def test_header_round_trip_and_corruption(tmp_path):
    ch, _ = sample(2, 5, 3, 5)
    good = str(tmp_path / "good.bin")
    _ufpd.write(good, ch, seed=5)
    h = U.ufpd_header(good)
    assert (h["K"], h["M"], h["N"], h["seed"], h["has_labels"]) == (2, 5, 3, 5, False)
    data = open(good, "rb").read()
    bad = str(tmp_path / "bad.bin")
    cases = {
        "magic": b"X" + data[1:],
        "version": data[:4] + bytes([2]) + data[5:],
        "truncated payload": data[:-8],
        "truncated header": data[:20],
        "trailing bytes": data + b"!",
        "bad dims": data[:8] + (0).to_bytes(4, "little") + data[12:],
    }
    for name, blob in cases.items():
        with open(bad, "wb") as f:
            f.write(blob)
        with pytest.raises(U.DataFormatError):
            U.ufpd_header(bad)
    with pytest.raises(U.DataFormatError):
        U.ufpd_header(str(tmp_path / "absent.bin"))


@pytest.mark.gpu
def test_device_load_is_the_rounded_reference_payload(tmp_path):
    ch, lab = sample(8, 64, 37, 11, labels=True)
    path = str(tmp_path / "d.bin")
    _ufpd.write(path, ch, lab, seed=11)
    got = U.ufpd_load(path).cpu().numpy()
    want = np.ascontiguousarray(np.transpose(ch, (0, 2, 1))).astype(np.complex64)  # [N][M][K]
    assert np.array_equal(got, want)
    got_l = U.ufpd_load(path, first=5, count=7, labels=True).cpu().numpy()
    assert np.array_equal(got_l, np.ascontiguousarray(np.transpose(lab[5:12], (0, 2, 1))).astype(np.complex64))
    with pytest.raises(U.DataFormatError):
        U.ufpd_load(path, first=30, count=10)


@pytest.mark.gpu
def test_device_store_round_trip(tmp_path):
    import torch

    w = U.CONFIGS[2]
    H = U.make_inputs(w, 0, 100)
    lam, eta = w.layer_params()
    Hd = torch.from_numpy(H).cuda()
    W = U.unfolded_forward(Hd, lam, eta, w.c)["W"]
    path = str(tmp_path / "labels.bin")
    U.ufpd_store(path, Hd, W, seed=w.seed_h)
    r = _ufpd.read(path)
    assert (r["K"], r["M"], r["N"], r["seed"]) == (8, 64, 100, w.seed_h)
    assert np.array_equal(r["channels"], np.transpose(H, (0, 2, 1)).astype(np.complex128))
    assert np.array_equal(r["labels"], np.transpose(W.cpu().numpy(), (0, 2, 1)).astype(np.complex128))
    back = U.ufpd_load(path).cpu().numpy()
    assert np.array_equal(back, H)
    assert not os.path.exists(path + ".tmp")
