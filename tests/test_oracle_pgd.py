"""Pins the FP64 oracle against the reference's own known-answer tests for the
PGD core (/root/reference/proj/tests/test_pgd.cpp), restated case by case at
the reference's tolerances. The brute-force helpers below restate
tests/support.hpp:19-99 (naive triple loops, no library products)."""
import math

import numpy as np
import pytest

from oracle import oracle as O


from _support import (fixture_2x4, naive_descent_objective, naive_fro_norm, naive_l21_norm,
                      naive_objective, naive_product, rel_err, scripted_layer)


# ---- test_pgd.cpp cases ------------------------------------------------------
def test_pgd_params_validation():  # :63-91
    p = O.PgdParams(0.1, 0.01, 10, 1e-8, 2)
    p.validate()
    for field, val in [("lambda_", -1e-9), ("eta", 0.0), ("max_iters", -1), ("residual_tol", -1.0),
                       ("trace_every", -2)]:
        bad = O.PgdParams(**{**p.__dict__, field: val})
        with pytest.raises(ValueError):
            bad.validate()


def test_grad_vanishes_at_zf():  # :93-100
    cfg = O.SystemConfig.uniform(4, 8, 10.0)
    h = O.channel_for(cfg, 11, 0)
    w = O.zf_precoder(h, cfg)
    assert np.linalg.norm(O.grad_f(w, h, cfg)) < 1e-9


def test_grad_at_zero_is_negated_data_term():  # :102-115
    cfg = O.SystemConfig.uniform(3, 6, 10.0, 0.7)
    h = O.channel_for(cfg, 12, 0)
    g = O.grad_f(np.zeros((3, 6), complex), h, cfg)
    t = cfg.constraint_diag()
    for k in range(3):
        for m in range(6):
            assert abs(g[k, m] - (-t[k] * np.conj(h[k, m]))) < 1e-14


def test_grad_matches_central_fd():  # :117-137
    cfg = O.SystemConfig.uniform(3, 7, 10.0, 0.9)
    for draw in range(5):
        h = O.channel_for(cfg, 13, draw)
        rng = O.Rng.stream(14, draw)
        w = O.random_matrix(3, 7, rng)
        d = O.random_matrix(3, 7, rng)
        g = O.grad_f(w, h, cfg)
        analytic = 2.0 * np.sum(g * np.conj(d)).real
        step = 1e-6
        numeric = (naive_objective(w + step * d, h, cfg, 0.0) -
                   naive_objective(w - step * d, h, cfg, 0.0)) / (2 * step)
        assert rel_err(numeric, analytic) < 1e-6


def test_prox_closed_form():  # :158-188
    v = np.zeros((3, 4), complex)
    v[:, 0] = [1 + 1j, 1 - 1j, 0]
    v[:, 1] = [0.3, 0, 0]
    v[:, 2] = [0.5, 0, 0]
    v[:, 3] = [2j, -0.4 + 0.1j, 0.2 - 0.9j]
    assert np.linalg.norm(O.prox_l21(v, 0.0) - v) == 0.0
    out = O.prox_l21(v, 0.5)
    assert np.linalg.norm(out[:, 0] - 0.75 * v[:, 0]) == 0.0
    assert np.all(out[:, 1] == 0)
    assert np.all(out[:, 2] == 0)  # tie maps to zero (strict '>')
    with pytest.raises(ValueError):
        O.prox_l21(v, -0.1)


def test_prox_output_norms():  # :190-207
    rng = O.Rng.stream(17, 0)
    v = O.random_matrix(4, 9, rng)
    for t in [0.0, 0.25, 1.0, 2.5, 10.0]:
        out = O.prox_l21(v, t)
        for m in range(9):
            expected = max(np.linalg.norm(v[:, m]) - t, 0.0)
            actual = np.linalg.norm(out[:, m])
            if expected == 0.0:
                assert actual == 0.0
            else:
                assert rel_err(expected, actual) < 1e-12


def test_prox_nonexpansive():  # :209-220
    for draw in range(20):
        rng = O.Rng.stream(18, draw)
        a = O.random_matrix(3, 8, rng)
        b = O.random_matrix(3, 8, rng)
        for t in [0.1, 0.8, 3.0]:
            assert np.linalg.norm(O.prox_l21(a, t) - O.prox_l21(b, t)) <= np.linalg.norm(a - b) + 1e-12


def test_pgd_step_keeps_feasible_point_fixed():  # :222-230
    cfg = O.SystemConfig.uniform(4, 12, 10.0)
    h = O.channel_for(cfg, 19, 0)
    w = O.zf_precoder(h, cfg)
    eta = 1.0 / O.lipschitz_bound(h).exact
    out = O.pgd_step(w, h, cfg, 0.0, eta)
    assert np.linalg.norm(out - w) < 1e-9 * max(1.0, np.linalg.norm(w))


def test_pgd_step_equals_prox_of_explicit_step():  # :232-245
    cfg = O.SystemConfig.uniform(3, 8, 10.0, 0.8)
    h = O.channel_for(cfg, 20, 0)
    w = O.random_matrix(3, 8, O.Rng.stream(21, 0))
    v = w - 0.02 * O.grad_f(w, h, cfg)
    expected = O.prox_l21(v, 0.4 * 0.02)
    actual = O.pgd_step(w, h, cfg, 0.4, 0.02)
    assert np.linalg.norm(actual - expected) < 1e-13 * max(1.0, np.linalg.norm(expected))


def test_single_step_scripted_fixture():  # :247-308
    cfg, h = fixture_2x4()
    target = [0.8 * math.sqrt(2.0), 0.8 * math.sqrt(0.5)]
    lam, eta = 1.5, 0.05
    w0 = h.conj()
    scripted, v, _ = scripted_layer(w0, h, target, lam, eta)
    weak = math.sqrt(abs(v[0, 2]) ** 2 + abs(v[1, 2]) ** 2)
    assert weak < lam * eta
    assert np.linalg.norm(scripted[:, 0]) > 0.0
    stepped = O.pgd_step(w0, h, cfg, lam, eta)
    assert np.linalg.norm(stepped - scripted) < 1e-14 * max(1.0, np.linalg.norm(scripted))
    assert np.all(stepped[:, 2] == 0)


def test_mp_bound():  # :310-317
    assert O.mp_bound(8, 64) == pytest.approx(117.25483399593904, rel=1e-12)
    assert O.mp_bound(8, 64) == pytest.approx((math.sqrt(8.0) + math.sqrt(64.0)) ** 2, rel=1e-15)
    with pytest.raises(ValueError):
        O.mp_bound(0, 64)
    with pytest.raises(ValueError):
        O.mp_bound(8, -1)


def test_lipschitz_identity():  # :319-324
    b = O.lipschitz_bound(np.eye(5, dtype=complex))
    assert b.exact == pytest.approx(1.0, rel=1e-10)
    assert b.mp == pytest.approx(20.0, rel=1e-12)


def test_lipschitz_matches_dense_eigensolver():  # :326-339
    cfg = O.SystemConfig.uniform(3, 5, 10.0)
    for draw in range(10):
        h = O.channel_for(cfg, 22, draw)
        ref = np.linalg.eigvalsh(naive_product(h, h.conj().T)).max()
        assert rel_err(ref, O.lipschitz_bound(h).exact) < 1e-9


def test_mp_dominates_at_scale():  # :341-354
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    mp = O.mp_bound(8, 64)
    covered = sum(O.lipschitz_bound(O.channel_for(cfg, 23, d)).exact <= mp for d in range(1000))
    assert covered >= 950


def test_lagrangian_matches_brute_force():  # :356-367
    cfg = O.SystemConfig.uniform(3, 9, 10.0, 0.6)
    h = O.channel_for(cfg, 24, 0)
    w = O.random_matrix(3, 9, O.Rng.stream(25, 0))
    for lam in [0.0, 1.0 / 15.0, 2.0]:
        assert rel_err(naive_objective(w, h, cfg, lam), O.lagrangian_value(w, h, cfg, lam)) < 1e-12


def test_unregularized_pgd_reaches_feasible_set():  # :369-382
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    h = O.channel_for(cfg, 26, 0)
    p = O.PgdParams(0.0, 1.0 / O.lipschitz_bound(h).exact, 50000, 1e-10, 0)
    r = O.solve_pgd(h, cfg, p)
    assert O.constraint_residual(h, r.precoder, cfg) < 1e-6


def test_iterate_change_stop_fires():  # :384-397
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    h = O.channel_for(cfg, 27, 0)
    p = O.PgdParams(0.0, 1.0 / O.lipschitz_bound(h).exact, 50000, 1e-3, 0)
    r = O.solve_pgd(h, cfg, p)
    assert 0 < r.iterations < 5000


def test_descent_objective_monotone():  # :399-426
    """The reference samples its trace every iteration; here the iterates come
    from the raw layer loop at constant (lambda, eta) — the same loop body as
    solve_pgd (test_unfolded.cpp:99-122 pins the equivalence)."""
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    lam = 1.0 / 15.0
    import ctypes as C
    for draw in range(5):
        h = O.channel_for(cfg, 28, draw)
        eta = 1.0 / O.lipschitz_bound(h).exact
        L = 300
        its = np.empty((L + 1, 64, 8), complex)
        out = np.empty((64, 8), complex)
        div = C.c_long()
        lam_v = np.full(L, lam)
        eta_v = np.full(L, eta)
        rc = O.lib().ora_forward(O._p(O.to_storage(h)), O._p(cfg.constraint_diag()), 8, 64, O._p(lam_v),
                                 O._p(eta_v), L, None, O._p(out), C.byref(div), O._p(its), None, None, None, None)
        assert rc == 0
        vals = []
        for i in range(L + 1):
            w = O.from_storage(its[i], 8, 64)
            r = O.constraint_residual(h, w, cfg)
            vals.append(lam * O.l21_norm(w) + 0.5 * r * r)
        for a, b in zip(vals[:-1], vals[1:]):
            assert b <= a + 1e-12 * max(1.0, abs(a))


def test_weak_columns_zero_out_exactly():  # :428-452
    cfg = O.SystemConfig.uniform(3, 10, 10.0)
    h = O.channel_for(cfg, 29, 0)
    w = O.random_matrix(3, 10, O.Rng.stream(30, 0))
    eta = 1.0 / O.lipschitz_bound(h).exact
    v = w - eta * O.grad_f(w, h, cfg)
    norms = [np.linalg.norm(v[:, m]) for m in range(10)]
    s = sorted(norms)
    threshold = 0.5 * (s[4] + s[5])
    out = O.pgd_step(w, h, cfg, threshold / eta, eta)
    for m in range(10):
        if norms[m] < threshold:
            assert np.all(out[:, m] == 0)
        else:
            assert np.linalg.norm(out[:, m]) > 0.0


def test_oversized_steps_raise_divergence():  # :454-470
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    h = O.channel_for(cfg, 31, 0)
    with pytest.raises(O.DivergenceError) as e:
        O.solve_pgd(h, cfg, O.PgdParams(0.0, 1e6, 200))
    assert e.value.index >= 1


def test_zero_iterations_returns_start():  # :481-495
    cfg = O.SystemConfig.uniform(3, 8, 10.0)
    h = O.channel_for(cfg, 32, 0)
    r = O.solve_pgd(h, cfg, O.PgdParams(1.0 / 15.0, 1.0 / O.mp_bound(3, 8), 0))
    assert r.iterations == 0
    assert np.linalg.norm(r.precoder - h.conj()) == 0.0


def test_pgd20_mean_pcg_near_one():  # :519-538
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    p = O.PgdParams(1.0 / 15.0, 1.0 / O.mp_bound(8, 64), 20)
    acc = 0.0
    for draw in range(200):
        h = O.channel_for(cfg, 33, draw)
        acc += O.pcg(h, O.solve_pgd(h, cfg, p).precoder, cfg)
    mean = acc / 200
    assert 0.97 < mean < 1.03


@pytest.mark.slow
def test_oracle_lower_bounds_5000_iterations():  # :540-560
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    lam = 1.0 / 15.0
    for draw in range(3):
        h = O.channel_for(cfg, 34, draw)
        oracle = O.oracle_solve(h, cfg, lam)
        mid = O.solve_pgd(h, cfg, O.PgdParams(lam, 1.0 / O.mp_bound(8, 64), 5000)).precoder
        a = naive_descent_objective(oracle, h, cfg, lam)
        b = naive_descent_objective(mid, h, cfg, lam)
        assert a <= b + 1e-12 * max(1.0, b)


@pytest.mark.slow
def test_oracle_fixed_point():  # :562-585
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    lam = 1.0 / 15.0
    h = O.channel_for(cfg, 35, 0)
    eta = 1.0 / O.lipschitz_bound(h).exact
    oracle = O.oracle_solve(h, cfg, lam)
    assert np.linalg.norm(O.pgd_step(oracle, h, cfg, lam, eta) - oracle) < 1e-6
    doubled = O.solve_pgd(h, cfg, O.PgdParams(lam, eta, 200000, 1e-10)).precoder
    base = O.lagrangian_value(oracle, h, cfg, lam)
    refined = O.lagrangian_value(doubled, h, cfg, lam)
    assert abs(base - refined) < 1e-8 * max(1.0, abs(refined))
