"""The FP64 device paths (SURVEY §8f row f3 and the per-channel precision
path): oracle_solve at scale — converged FP64 power iteration, up to 1e5 PGD
iterations with a per-realization 1e-10 iterate-change stop — against the FP64
oracle, to the reference's own tolerances."""
import math

import numpy as np
import pytest

import paper_2304_12745_b200 as U
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_oracle_solve_at_scale_matches_fp64_oracle():
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    lam = 1.0 / 15.0
    chans = [O.channel_for(cfg, 35, d) for d in range(6)]
    H = np.stack([O.to_storage(h) for h in chans])
    out = U.oracle_solve(torch.from_numpy(H).cuda(), cfg.constraint_diag(), lam)
    torch.cuda.synchronize()
    assert np.all(out["status"].cpu().numpy() == 0)
    its = out["iterations"].cpu().numpy()
    W = out["W"].cpu().numpy()
    for d, h in enumerate(chans):
        ref_run = O.solve_pgd(h, cfg, O.PgdParams(lam, 1.0 / O.lipschitz_bound(h).exact, 100000, 1e-10, 0))
        assert abs(int(its[d]) - ref_run.iterations) <= 2
        ref = ref_run.precoder
        got = O.from_storage(W[d], 8, 64)
        # both stop at a 1e-10 relative iterate change: agree far below FP32
        assert np.linalg.norm(got - ref) <= 1e-7 * np.linalg.norm(ref)
        assert abs(O.lagrangian_value(got, h, cfg, lam) - O.lagrangian_value(ref, h, cfg, lam)) <= 1e-9 * abs(
            O.lagrangian_value(ref, h, cfg, lam))
        assert out["eta"].cpu().numpy()[d] == pytest.approx(1.0 / O.lipschitz_bound(h).exact, rel=1e-12)


def test_exact_lipschitz_matches_eigensolver():
    cfg = O.SystemConfig.uniform(8, 64, 10.0)
    chans = [O.channel_for(cfg, 23, d) for d in range(64)]
    H = torch.from_numpy(np.stack([O.to_storage(h) for h in chans])).cuda()
    L, st = U.lipschitz_exact(H)
    L = L.cpu().numpy()
    assert np.all(st.cpu().numpy() == 0)
    for d, h in enumerate(chans):
        ref = np.linalg.eigvalsh(h @ h.conj().T).max()
        assert abs(L[d] - ref) / ref < 1e-9  # test_pgd.cpp:326-339


def test_oracle_solve_early_stop_per_realization():
    """lambda = 0 converges well inside the cap (test_pgd.cpp:369-382): each
    realization stops at its own iteration, as the reference's loop does."""
    cfg = O.SystemConfig.uniform(4, 16, 10.0)
    chans = [O.channel_for(cfg, 26, d) for d in range(8)]
    H = torch.from_numpy(np.stack([O.to_storage(h) for h in chans])).cuda()
    out = U.oracle_solve(H, cfg.constraint_diag(), 0.0, max_iters=50000)
    its = out["iterations"].cpu().numpy()
    W = out["W"].cpu().numpy()
    assert len(set(its.tolist())) > 1 and np.all(its < 50000)
    for d, h in enumerate(chans):
        ref = O.solve_pgd(h, cfg, O.PgdParams(0.0, 1.0 / O.lipschitz_bound(h).exact, 50000, 1e-10, 0))
        assert abs(int(its[d]) - ref.iterations) <= 2
        assert O.constraint_residual(h, O.from_storage(W[d], 4, 16), cfg) < 1e-6
