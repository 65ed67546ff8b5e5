"""Shared test helpers: brute-force oracles restating
/root/reference/proj/tests/support.hpp:19-99 and the scripted fixtures of
test_pgd.cpp:247-308 / test_unfolded.cpp:134-180."""
import math

import numpy as np

from oracle import oracle as O


# ---- support.hpp:19-99 -----------------------------------------------------
def naive_product(a, b):
    out = np.zeros((a.shape[0], b.shape[1]), dtype=complex)
    for i in range(a.shape[0]):
        for j in range(b.shape[1]):
            acc = 0j
            for k in range(a.shape[1]):
                acc += a[i, k] * b[k, j]
            out[i, j] = acc
    return out


def naive_fro_norm(a):
    return math.sqrt(sum(abs(x) ** 2 for x in a.flat))


def naive_l21_norm(a):
    return sum(math.sqrt(sum(abs(a[i, j]) ** 2 for i in range(a.shape[0]))) for j in range(a.shape[1]))


def rel_err(expected, actual):
    return abs(expected - actual) / max(abs(expected), abs(actual), 1e-300)


def naive_objective(w, h, cfg, lam):  # test_pgd.cpp:24-33
    r = naive_product(h, w.T)
    t = cfg.constraint_diag()
    for k in range(cfg.K):
        r[k, k] -= t[k]
    f = naive_fro_norm(r)
    return lam * naive_l21_norm(w) + f * f


def naive_descent_objective(w, h, cfg, lam):  # test_pgd.cpp:40-48
    r = naive_product(h, w.T)
    t = cfg.constraint_diag()
    for k in range(cfg.K):
        r[k, k] -= t[k]
    f = naive_fro_norm(r)
    return lam * naive_l21_norm(w) + 0.5 * f * f


def fixture_2x4():
    """The stored 2x4 fixture of test_pgd.cpp:247-265 / test_unfolded.cpp:135-152."""
    cfg = O.SystemConfig(2, 4, 0.8, np.array([2.0, 0.5]), 1.0)
    cfg.validate()
    h = np.array([[0.6 + 0.3j, -0.2 + 0.9j, 0.05 - 0.02j, 1.1 + 0.0j],
                  [-0.7 + 0.1j, 0.4 - 0.4j, 0.03 + 0.01j, -0.5 + 0.6j]])
    return cfg, h


def scripted_layer(w, h, target, lam, eta):
    """Scalar re-evaluation of one layer (test_pgd.cpp:271-296,
    test_unfolded.cpp:38-70), free of any matrix routine."""
    rows, cols = w.shape
    v = np.zeros((rows, cols), dtype=complex)
    for k in range(rows):
        for m in range(cols):
            smooth = 0j
            for j in range(rows):
                wh = 0j
                for l in range(cols):
                    wh += w[k, l] * h[j, l]
                smooth += wh * h[j, m].conjugate()
            smooth -= target[k] * h[k, m].conjugate()
            v[k, m] = w[k, m] - eta * smooth
    threshold = lam * eta
    out = np.zeros((rows, cols), dtype=complex)
    hit_zero = False
    for m in range(cols):
        nrm = math.sqrt(sum(abs(v[k, m]) ** 2 for k in range(rows)))
        if nrm > threshold:
            scale = 1.0 - threshold / nrm
            for k in range(rows):
                out[k, m] = scale * v[k, m]
        else:
            hit_zero = True
    return out, v, hit_zero


