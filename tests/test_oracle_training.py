"""CPU checks of the oracle's training-loop restatement (training.cpp:140-308,
rng.hpp:43-50) that the GPU training parity test relies on."""
import math

import numpy as np

from oracle import oracle as O


def test_shuffle_is_a_seeded_permutation():
    a, b = list(range(50)), list(range(50))
    O.shuffle(a, O.Rng.stream(3, O.SHUFFLE_STREAM))
    O.shuffle(b, O.Rng.stream(3, O.SHUFFLE_STREAM))
    assert a == b and sorted(a) == list(range(50)) and a != list(range(50))


def test_adam_first_step_is_signed_learning_rate():  # test_training.cpp:192-205
    st = dict(step=0, m=[0.0, 0.0], v=[0.0, 0.0])
    p = [1.0, 1.0]
    O.adam_update(st, [0.5, -2.0], p, 1e-3)
    assert abs(p[0] - (1.0 - 1e-3)) < 1e-9 and abs(p[1] - (1.0 + 1e-3)) < 1e-9


def _channels(seed, n, K, M):
    cfg = O.SystemConfig.uniform(K, M, 10.0)
    return np.stack([O.to_storage(O.channel_for(cfg, seed, i)) for i in range(n)]).astype(np.complex64)


def test_zero_learning_rate_stops_after_patience_plus_one():  # test_training.cpp:275-305
    K, M, L = 4, 16, 3
    r = O.train_loop_f32(_channels(70, 16, K, M), _channels(71, 8, K, M), np.full(K, math.sqrt(10.0)),
                         [1.0 / 15.0] * L, [1.0 / O.mp_bound(K, M)] * L, batch_size=8, learning_rate=0.0,
                         max_epochs=20, patience=3, seed=99)
    assert len(r["epochs"]) == 4 and r["best_epoch"] == 0 and r["stopping_epoch"] == 3
    assert r["params"] == [1.0 / 15.0, 1.0 / O.mp_bound(K, M)] * L


def test_training_lowers_the_validation_loss():
    K, M, L = 4, 16, 5
    r = O.train_loop_f32(_channels(72, 64, K, M), _channels(73, 16, K, M), np.full(K, math.sqrt(10.0)),
                         [1.0 / 15.0] * L, [1.0 / O.mp_bound(K, M)] * L, batch_size=16, learning_rate=3e-3,
                         max_epochs=4, patience=10, seed=5)
    assert min(e[2] for e in r["epochs"]) < r["epochs"][0][2]
