"""The training caller (ufpgd::train, include/ufpgd/training.hpp) on the B200
against the oracle's restatement of training.cpp:140-308 (oracle.train_loop_f32):
same UFPD datasets, same seed, so the same shuffle order, batches, Adam steps
and early-stopping decisions. The device computes each mini-batch's loss and
gradient in FP32, the oracle in FP64 from the same complex64 channels, so the
histories agree to FP32 accuracy rather than bit for bit."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O
import _ufpd

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "train_dump")


def write_set(path, H, labels=None):
    # device layout [N][M][K] -> file layout [N][K][M] (row k = user)
    _ufpd.write(path, np.transpose(H, (0, 2, 1)).astype(np.complex128),
                None if labels is None else np.transpose(labels, (0, 2, 1)).astype(np.complex128), seed=5)


def run(tmp_path, K, M, L, kind, n_train, n_val, batch, lr, epochs, patience, seed, labels=False):
    Ht = U.generate_channels(500, 0, 0.0, 0, n_train, K, M)
    Hv = U.generate_channels(501, 0, 0.0, 0, n_val, K, M)
    Lt = (0.3 * np.conj(Ht)).astype(np.complex64) if labels else None
    Lv = (0.3 * np.conj(Hv)).astype(np.complex64) if labels else None
    write_set(tmp_path / "tr.ufpd", Ht, Lt)
    write_set(tmp_path / "va.ufpd", Hv, Lv)
    lam0 = 1.0 / 15.0
    out = subprocess.run([BIN, str(tmp_path / "tr.ufpd"), str(tmp_path / "va.ufpd"), str(L), repr(lam0), str(kind),
                          repr(1.0 / 15.0), str(batch), repr(lr), str(epochs), str(patience), str(seed)],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    dev = json.loads(out.stdout)
    c = np.full(K, math.sqrt(10.0))
    eta0 = 1.0 / O.mp_bound(K, M)
    ora = O.train_loop_f32(Ht, Hv, c, [lam0] * L, [eta0] * L, loss_kind=kind, lambda_cost=1.0 / 15.0,
                           batch_size=batch, learning_rate=lr, max_epochs=epochs, patience=patience, seed=seed,
                           train_labels=Lt, val_labels=Lv)
    return dev, ora


def compare(dev, ora, loss_tol=2e-6, metric_tol=1e-6, param_tol=1e-7):  # measured: <= 1.5e-7, 1e-9
    assert len(dev["epochs"]) == len(ora["epochs"])
    d_arr, o_arr = np.array(dev["epochs"])[:, 1:], np.array(ora["epochs"])[:, 1:]
    print("history rel diff per column:", np.max(np.abs(d_arr - o_arr) / np.abs(o_arr), axis=0),
          "params:", np.max(np.abs(np.array(dev["params"]) - np.array(ora["params"])) / np.abs(np.array(ora["params"]))))
    for d, o in zip(dev["epochs"], ora["epochs"]):
        assert d[0] == o[0]
        for i, tol in ((1, loss_tol), (2, loss_tol), (3, metric_tol), (4, metric_tol)):
            assert abs(d[i] - o[i]) <= tol * abs(o[i]), (i, d, o)
    assert dev["best_epoch"] == ora["best_epoch"] and dev["stopping_epoch"] == ora["stopping_epoch"]
    p, q = np.array(dev["params"]), np.array(ora["params"])
    assert np.all(np.abs(p - q) <= param_tol * np.abs(q) + 1e-12), np.max(np.abs(p - q) / np.abs(q))


def test_unsupervised_training_matches_oracle_loop(tmp_path):
    dev, ora = run(tmp_path, 4, 16, 5, 0, 64, 16, 16, 1e-3, 4, 10, 7)
    compare(dev, ora)
    assert ora["epochs"][-1][2] < ora["epochs"][0][2] * 1.01  # it trains


def test_supervised_training_matches_oracle_loop(tmp_path):
    dev, ora = run(tmp_path, 8, 64, 6, 1, 48, 16, 16, 1e-3, 3, 10, 11, labels=True)
    compare(dev, ora)


def test_early_stopping_at_zero_learning_rate(tmp_path):
    """test_training.cpp:275-305 through the driver: patience + 1 epochs."""
    dev, ora = run(tmp_path, 4, 16, 3, 0, 16, 8, 8, 0.0, 20, 3, 99)
    assert len(dev["epochs"]) == 4 and dev["best_epoch"] == 0 and dev["stopping_epoch"] == 3
    compare(dev, ora)
