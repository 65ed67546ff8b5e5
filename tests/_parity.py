"""Parity metrics between the GPU (FP32) and the FP64 oracle, with the bars of
BASELINE.json's north_star: W within 1e-4 relative Frobenius, objective within
1e-5 relative, identical active-antenna support except at threshold ties."""
import numpy as np

from oracle import oracle as O

W_REL_TOL = 1e-4       # relative Frobenius error of W per realization
OBJ_REL_TOL = 1e-5     # relative error of lagrangian_value (pgd.cpp:171-176)
TIE_MARGIN = 1e-4      # |n - t| / t below this at any layer marks a tie


def rel_fro(Wg: np.ndarray, Wo: np.ndarray) -> np.ndarray:
    d = np.linalg.norm((Wg.astype(np.complex128) - Wo).reshape(len(Wo), -1), axis=1)
    n = np.linalg.norm(Wo.reshape(len(Wo), -1), axis=1)
    return np.where(n > 0, d / np.maximum(n, 1e-300), d)


def support(W: np.ndarray) -> np.ndarray:
    return np.sum(np.abs(W) ** 2, axis=2) > 0.0  # [B, M]


def report(H, Wg, ora, c, lam_obj):
    """ora: dict from oracle forward/pgd batch drivers (W, tie_margin)."""
    Wo = ora["W"]
    rel = rel_fro(Wg, Wo)
    fg = O.lagrangian_batch(H, Wg, c, lam_obj)
    fo = O.lagrangian_batch(H, Wo, c, lam_obj)
    obj = np.abs(fg - fo) / np.abs(fo)
    ties = ora["tie_margin"] < TIE_MARGIN
    sup_mismatch = np.any(support(Wg) != support(Wo), axis=1) & ~ties
    return dict(rel_max=float(rel.max()), rel_median=float(np.median(rel)), obj_max=float(obj.max()),
                support_mismatch=int(sup_mismatch.sum()), ties=int(ties.sum()), rel=rel, obj=obj)


def assert_parity(rep, w_tol=W_REL_TOL, obj_tol=OBJ_REL_TOL):
    assert rep["rel_max"] <= w_tol, rep["rel_max"]
    assert rep["obj_max"] <= obj_tol, rep["obj_max"]
    assert rep["support_mismatch"] == 0, rep["support_mismatch"]
